// Micro-benchmark 3: does the SHAPE of a CTA's write stream matter?  F_7-sized operator matrices (2925 rows of
// 2928 bytes, 325 row groups of 1..25 rows).  A CTA owns (row group, column part) for 16 quads and writes the rows
// of its part with 8-byte stores (two row teams), like k_matrix_staged does for p = 7 -- with 1, 2, 4 or 8 column
// parts per row.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o write_bw3 write_bw3.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
struct Item { int row0, nrows, g0, ng; };
__global__ void __launch_bounds__(256) k_rows(uint2* p, const Item* items, size_t mstride, int pitch_g, int nquads, int slice)
{
    const Item it = items[blockIdx.x];
    const int team = threadIdx.x >> 7, t = threadIdx.x & 127;
    for (int q = blockIdx.y * slice; q < min(nquads, (blockIdx.y + 1) * slice); ++q)
        for (int g = t; g < it.ng; g += 128)
            for (int r = team; r < it.nrows; r += 2) {
                uint2* a = p + (size_t)q * 4 * mstride + (size_t)(it.row0 + r) * pitch_g + it.g0 + g;
#pragma unroll
                for (int s = 0; s < 4; ++s) a[s * mstride] = make_uint2(g, r);
            }
}
// variant: the CTA owns the whole rows of its group but writes them column part by column part (parts sequential in time)
__global__ void __launch_bounds__(256) k_rows_seq(uint2* p, const Item* items, size_t mstride, int pitch_g, int nquads, int slice, int parts)
{
    const Item it = items[blockIdx.x];
    const int team = threadIdx.x >> 7, t = threadIdx.x & 127;
    for (int q = blockIdx.y * slice; q < min(nquads, (blockIdx.y + 1) * slice); ++q)
        for (int k = 0; k < parts; ++k) {
            const int g0 = pitch_g * k / parts, g1 = pitch_g * (k + 1) / parts;
            for (int g = g0 + t; g < g1; g += 128)
                for (int r = team; r < it.nrows; r += 2) {
                    uint2* a = p + (size_t)q * 4 * mstride + (size_t)(it.row0 + r) * pitch_g + g;
#pragma unroll
                    for (int s = 0; s < 4; ++s) a[s * mstride] = make_uint2(g, r);
                }
            __syncthreads();
        }
}
// variant: parts outer, quads inner (what chaining the panels of a group inside one CTA would do)
__global__ void __launch_bounds__(256) k_rows_seq2(uint2* p, const Item* items, size_t mstride, int pitch_g, int nquads, int slice, int parts)
{
    const Item it = items[blockIdx.x];
    const int team = threadIdx.x >> 7, t = threadIdx.x & 127;
    for (int k = 0; k < parts; ++k) {
        const int g0 = pitch_g * k / parts, g1 = pitch_g * (k + 1) / parts;
        for (int q = blockIdx.y * slice; q < min(nquads, (blockIdx.y + 1) * slice); ++q) {
            for (int g = g0 + t; g < g1; g += 128)
                for (int r = team; r < it.nrows; r += 2) {
                    uint2* a = p + (size_t)q * 4 * mstride + (size_t)(it.row0 + r) * pitch_g + g;
#pragma unroll
                    for (int s = 0; s < 4; ++s) a[s * mstride] = make_uint2(g, r);
                }
            __syncthreads();
        }
    }
}
int main()
{
    const int d = 24, N = 2925, pitch_g = 2928 / 8;
    const size_t mstride = (size_t)N * pitch_g;  // in uint2
    const int nquads = 512;
    const size_t bytes = (size_t)nquads * 4 * mstride * 8;
    uint2* dptr;
    cudaMalloc(&dptr, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int parts : {1, 2, 4, 8}) {
        std::vector<Item> items;
        int row0 = 0;
        for (int r1 = 0; r1 <= d; ++r1)
            for (int r2 = 0; r1 + r2 <= d; ++r2) {
                const int nr = d - r1 - r2 + 1;
                for (int k = 0; k < parts; ++k) {
                    const int g0 = pitch_g * k / parts, g1 = pitch_g * (k + 1) / parts;
                    items.push_back({row0, nr, g0, g1 - g0});
                }
                row0 += nr;
            }
        Item* ditems;
        cudaMalloc(&ditems, items.size() * sizeof(Item));
        cudaMemcpy(ditems, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_rows<<<dim3((unsigned)items.size(), nquads / 16), 256>>>(dptr, ditems, mstride, pitch_g, nquads, 16);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("column parts per row %d (segment %4d B): %8.3f ms  %8.1f GB/s\n", parts, 2928 / parts, ms, bytes / ms / 1e6);
        }
        if (parts > 1) {
            // same items as parts == 1 (full rows), parts walked inside the CTA
            std::vector<Item> full;
            int rr = 0;
            for (int r1 = 0; r1 <= d; ++r1)
                for (int r2 = 0; r1 + r2 <= d; ++r2) { const int nr = d - r1 - r2 + 1; full.push_back({rr, nr, 0, pitch_g}); rr += nr; }
            Item* dfull;
            cudaMalloc(&dfull, full.size() * sizeof(Item));
            cudaMemcpy(dfull, full.data(), full.size() * sizeof(Item), cudaMemcpyHostToDevice);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                k_rows_seq<<<dim3((unsigned)full.size(), nquads / 16), 256>>>(dptr, dfull, mstride, pitch_g, nquads, 16, parts);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("   same, parts sequential inside one CTA:       %8.3f ms  %8.1f GB/s\n", ms, bytes / ms / 1e6);
            }
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                k_rows_seq2<<<dim3((unsigned)full.size(), nquads / 16), 256>>>(dptr, dfull, mstride, pitch_g, nquads, 16, parts);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("   same, parts outer / quads inner in one CTA:  %8.3f ms  %8.1f GB/s\n", ms, bytes / ms / 1e6);
            }
            cudaFree(dfull);
        }
        cudaFree(ditems);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
