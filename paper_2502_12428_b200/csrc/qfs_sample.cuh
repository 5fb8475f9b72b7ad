// qfs_sample.cuh -- the reference's seeded sampler on the device.
//
// search.sample_surface (search.py:92-98) draws `rng.integers(0, p, size=35)` from numpy's default_rng([seed, worker])
// (search.py:103): PCG64 (a 128-bit LCG with the XSL-RR output function; the state steps BEFORE it is output), whose 64-bit
// outputs are split into two 32-bit draws, low half first, each mapped to [0, p) by Lemire's multiply-shift with rejection
// (numpy/random/src/distributions: buffered_bounded_lemire_uint32).  The k-th 32-bit draw is therefore a pure function of
// (state, increment, k): a thread jumps the LCG ahead to the outputs of its row (O(log k) 128-bit multiplications) and
// produces the row's 35 coefficients.  A Lemire rejection (probability p / 2^32 per draw) or an all-zero row (p^-35) would
// shift the reference's stream from that point on: the kernel only REPORTS them, and the caller then draws that block on
// the host (paper_2502_12428_b200/search.py), so the stream is the reference's bit for bit in every case.
// tests/test_host_api.py pins the same arithmetic, written in Python integers, on numpy's generator.
#pragma once
#include <stdint.h>

struct U128 { uint64_t hi, lo; };

__device__ __forceinline__ U128 mul128(U128 a, U128 b)
{
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
    return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b)
{
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

// rows [0, count) of the block: out[r][35] = the draws 35r .. 35r+34 of the stream; *dirty |= 1 if any draw was rejected or
// any row is zero (the block then differs from the reference's and must be redrawn on the host)
__global__ void __launch_bounds__(128) k_sample_quartics(U128 state, U128 inc, uint32_t p, size_t count, uint8_t* __restrict__ out,
                                                         int* __restrict__ dirty)
{
    const size_t r = (size_t)blockIdx.x * 128 + threadIdx.x;
    if (r >= count) return;
    const U128 A = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};   // PCG_DEFAULT_MULTIPLIER_128
    const size_t k0 = 35 * r;
    // state after k0/2 steps: s -> acc_mult * s + acc_plus
    U128 am = {0, 1}, ap = {0, 0}, cm = A, cp = inc;
    for (size_t delta = k0 >> 1; delta > 0; delta >>= 1) {
        if (delta & 1) {
            am = mul128(am, cm);
            ap = add128(mul128(ap, cm), cp);
        }
        cp = mul128(add128(cm, U128{0, 1}), cp);
        cm = mul128(cm, cm);
    }
    U128 s = add128(mul128(am, state), ap);
    const uint32_t threshold = (0xFFFFFFFFu - (p - 1)) % p;
    uint8_t* dst = out + 35 * r;
    int skip = (int)(k0 & 1), have = 0;
    uint32_t any = 0, bad = 0;
    while (have < 35) {
        s = add128(mul128(s, A), inc);
        const uint64_t x = s.hi ^ s.lo;
        const unsigned rot = (unsigned)(s.hi >> 58);
        const uint64_t o = (x >> rot) | (x << ((64 - rot) & 63));
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            if (skip) { skip = 0; continue; }
            if (have >= 35) break;
            const uint64_t m = (uint64_t)(uint32_t)(o >> (32 * half)) * p;
            if ((uint32_t)m < threshold) bad = 1;
            const uint32_t v = (uint32_t)(m >> 32);
            any |= v;
            dst[have++] = (uint8_t)v;
        }
    }
    if (bad || !any) atomicOr(dirty, 1);
}
