// Micro-benchmark 2: builder-shaped stores. A CTA owns a row group (1..17 rows of 976 bytes) of 16 quads
// (4 matrices each) and writes them with V words per thread per store.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
template <int V, int NS>
__global__ void __launch_bounds__(256) k_rows(uint32_t* p, size_t mstride_words, int pitch_words, int nquads, int slice)
{
    // row groups like p=5: group g has rows [row0, row0+nr)
    int g = blockIdx.x, r1 = 0, acc = 0;
    while (g >= 17 - r1) { g -= 17 - r1; acc += (17 - r1) * (18 - r1) / 2; ++r1; }
    // rows of groups (r1, r2=g): nr = 17 - r1 - g; row0 = acc + sum_{r2<g} (17-r1-r2)
    int row0 = acc; for (int r2 = 0; r2 < g; ++r2) row0 += 17 - r1 - r2;
    const int nr = 17 - r1 - g;
    const int tpr = (pitch_words + V - 1) / V;             // threads per row
    const int teams = 256 / tpr > 0 ? 256 / tpr : 1;
    const int team = threadIdx.x / tpr, w = (threadIdx.x % tpr) * V;
    if (team >= teams) return;
    for (int q = blockIdx.y * slice; q < min(nquads, (blockIdx.y + 1) * slice); ++q) {
        uint32_t* base = p + (size_t)q * NS * mstride_words + (size_t)row0 * pitch_words + w;
        for (int r = team; r < nr; r += teams) {
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                uint32_t* a = base + s * mstride_words + (size_t)r * pitch_words;
                if (V == 1) a[0] = w + s;
                else if (V == 2) *reinterpret_cast<uint2*>(a) = make_uint2(w, s);
                else *reinterpret_cast<uint4*>(a) = make_uint4(w, s, r, q);
            }
        }
    }
}
int main()
{
    const int rows = 969, pw = 244;
    const size_t ms_words = (size_t)rows * pw;
    const int nquads = 4096;
    const size_t bytes = (size_t)nquads * 4 * ms_words * 4;
    uint32_t* d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    auto report = [&](const char* name) {
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("%-36s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
    };
    for (int rep = 0; rep < 2; ++rep) {
        dim3 grid(153, nquads / 16);
        cudaEventRecord(a); k_rows<1, 4><<<grid, 256>>>(d, ms_words, pw, nquads, 16); report("V=1 (STG.32) x4 matrices");
        cudaEventRecord(a); k_rows<2, 4><<<grid, 256>>>(d, ms_words, pw, nquads, 16); report("V=2 (STG.64) x4 matrices");
        cudaEventRecord(a); k_rows<4, 4><<<grid, 256>>>(d, ms_words, pw, nquads, 16); report("V=4 (STG.128) x4 matrices");
        dim3 grid1(153, 4 * nquads / 16);
        cudaEventRecord(a); k_rows<1, 1><<<grid1, 256>>>(d, ms_words, pw, 4 * nquads, 16); report("V=1 (STG.32) x1 matrix");
        cudaEventRecord(a); k_rows<4, 1><<<grid1, 256>>>(d, ms_words, pw, 4 * nquads, 16); report("V=4 (STG.128) x1 matrix");
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
