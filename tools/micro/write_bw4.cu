// Micro-benchmark 4: does the ALIGNMENT of the row segments matter?  Same write skeleton as write_bw3 (a CTA owns
// (row group, column part) for SLICE quads; a thread owns one store-wide word group and walks the rows of its team),
// with the row pitch and the part boundaries either as the builder has them today (pitch = N rounded up to 16 bytes,
// boundaries anywhere) or rounded to 128-byte lines, and with warps either starting at the part boundary or at the
// 128-byte line in front of it.  F_7 shape with 8-byte stores and F_5 shape with 4- and 8-byte stores.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o write_bw4 write_bw4.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
struct Item { int row0, nrows, b0, b1; };  // byte range [b0, b1) of the rows
template <typename T, int TEAMS, int NT>
__global__ void __launch_bounds__(NT) k_rows(uint8_t* p, const Item* items, size_t mstride, int pitch, int nquads, int slice, int warp_align)
{
    const Item it = items[blockIdx.x];
    constexpr int TEAM = NT / TEAMS;
    const int team = threadIdx.x / TEAM, t = threadIdx.x % TEAM;
    const int start = warp_align ? (it.b0 & ~127) : it.b0;
    for (int q = blockIdx.y * slice; q < min(nquads, (blockIdx.y + 1) * slice); ++q)
        for (int b = start + (int)sizeof(T) * t; b < it.b1; b += (int)sizeof(T) * TEAM) {
            if (b < it.b0) continue;
            for (int r = team; r < it.nrows; r += TEAMS) {
                uint8_t* a = p + (size_t)q * 4 * mstride + (size_t)(it.row0 + r) * pitch + b;
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    T v;
                    memset(&v, r, sizeof(T));
                    *reinterpret_cast<T*>(a + s * mstride) = v;
                }
            }
        }
}
template <typename T, int TEAMS, int NT>
void run(const char* name, int d, int N, int pitch, int parts, int bound_align, int warp_align, int nquads, int slice)
{
    const size_t mstride = (size_t)N * pitch;
    const size_t bytes = (size_t)nquads * 4 * mstride;
    uint8_t* dptr;
    if (cudaMalloc(&dptr, bytes) != cudaSuccess) { printf("alloc failed\n"); return; }
    std::vector<Item> items;
    int row0 = 0;
    const int rowbytes = (N + (int)sizeof(T) - 1) / (int)sizeof(T) * (int)sizeof(T);
    for (int r1 = 0; r1 <= d; ++r1)
        for (int r2 = 0; r1 + r2 <= d; ++r2) {
            const int nr = d - r1 - r2 + 1;
            for (int k = 0; k < parts; ++k) {
                int b0 = (int)((long long)rowbytes * k / parts), b1 = (int)((long long)rowbytes * (k + 1) / parts);
                const int al = bound_align ? 128 : (int)sizeof(T);
                b0 = b0 / al * al;
                b1 = (k + 1 == parts) ? rowbytes : b1 / al * al;
                items.push_back({row0, nr, b0, b1});
            }
            row0 += nr;
        }
    Item* ditems;
    cudaMalloc(&ditems, items.size() * sizeof(Item));
    cudaMemcpy(ditems, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        k_rows<T, TEAMS, NT><<<dim3((unsigned)items.size(), (nquads + slice - 1) / slice), NT>>>(dptr, ditems, mstride, pitch, nquads, slice, warp_align);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
    }
    const double useful = (double)nquads * 4 * N * (double)N;
    printf("%-6s st%2d pitch %5d parts %d bounds %-6s warps %-8s: %8.3f ms  %7.1f GB/s of N^2 (%7.1f GB/s incl. pad)  %s\n", name,
           (int)sizeof(T), pitch, parts, bound_align ? "128B" : "any", warp_align ? "line" : "boundary", best, useful / best / 1e6,
           (double)nquads * 4 * N * rowbytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    cudaFree(ditems);
    cudaFree(dptr);
}
int main()
{
    // F_7: N = 2925, 8-byte stores, two 96-thread teams (the builder's NT = 192), slice 8, ~4 panels per row group
    for (int pitch : {2928, 2944, 3072})
        for (int parts : {1, 4})
            for (int ba : {0, 1})
                for (int wa : {0, 1}) {
                    if (parts == 1 && (ba || wa)) continue;
                    run<uint2, 2, 192>("F_7", 24, 2925, pitch, parts, ba, wa, 512, 8);
                }
    run<uint4, 2, 192>("F_7", 24, 2925, 2944, 4, 1, 1, 512, 8);
    run<uint4, 4, 256>("F_7", 24, 2925, 2944, 4, 1, 1, 512, 8);
    // F_5: N = 969, one panel per row group; 4-byte stores with one 256-thread team (today), 8-byte with two teams, 16-byte with four
    for (int pitch : {976, 1024}) {
        run<uint32_t, 1, 256>("F_5", 16, 969, pitch, 1, 0, 0, 4096, 16);
        run<uint2, 2, 256>("F_5", 16, 969, pitch, 1, 0, 0, 4096, 16);
        run<uint4, 4, 256>("F_5", 16, 969, pitch, 1, 0, 0, 4096, 16);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
