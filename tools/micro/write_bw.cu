// Micro-benchmark: write-only HBM bandwidth on this GPU for the store shapes the matrix builder can use.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o write_bw write_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
template <int V>
__global__ void k_fill(uint32_t* p, size_t nwords, uint32_t v)
{
    size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * V;
    const size_t stride = (size_t)gridDim.x * blockDim.x * V;
    for (; i < nwords; i += stride) {
        if (V == 1) p[i] = v;
        else if (V == 2) *reinterpret_cast<uint2*>(p + i) = make_uint2(v, v);
        else *reinterpret_cast<uint4*>(p + i) = make_uint4(v, v, v, v);
    }
}
// rows of `pitch` words: each warp writes 128 B of 4 different matrices per "row step" like the builder does
__global__ void k_fill4(uint32_t* p, size_t mstride_words, int rows, int pitch_words, int nquads)
{
    for (int q = blockIdx.y; q < nquads; q += gridDim.y) {
        uint32_t* base = p + (size_t)q * 4 * mstride_words;
        for (int r = blockIdx.x; r < rows; r += gridDim.x)
            for (int w = threadIdx.x; w < pitch_words; w += blockDim.x)
#pragma unroll
                for (int s = 0; s < 4; ++s) base[s * mstride_words + (size_t)r * pitch_words + w] = w + s;
    }
}
int main()
{
    const size_t bytes = (size_t)16 << 30;
    uint32_t* d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    auto report = [&](const char* name) {
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
    };
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); cudaMemsetAsync(d, 1, bytes); report("cudaMemset");
        cudaEventRecord(a); k_fill<1><<<148 * 16, 256>>>(d, bytes / 4, 7); report("STG.32 grid-stride");
        cudaEventRecord(a); k_fill<2><<<148 * 16, 256>>>(d, bytes / 4, 7); report("STG.64 grid-stride");
        cudaEventRecord(a); k_fill<4><<<148 * 16, 256>>>(d, bytes / 4, 7); report("STG.128 grid-stride");
        cudaEventRecord(a); k_fill<4><<<148 * 64, 256>>>(d, bytes / 4, 7); report("STG.128 grid-stride x64");
        // builder-like: 969 rows x 244 words, 4 matrices per quad
        const int rows = 969, pw = 244; const size_t ms_words = (size_t)rows * pw;
        const int nquads = (int)(bytes / 4 / (4 * ms_words));
        cudaEventRecord(a); k_fill4<<<dim3(153, 64), 256>>>(d, ms_words, rows, pw, nquads); report("STG.32 x4 matrices (p=5)");
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
