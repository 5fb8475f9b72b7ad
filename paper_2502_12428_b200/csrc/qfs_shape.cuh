// qfs_shape.cuh -- index conventions and per-prime shape constants shared by every kernel.
//
// Dense layout of a degree-`deg` form in x1..x4 ("lex"): monomials in lex-ascending order with
// x1 most significant, index 0 = x4^deg (reference: monomials.py:182-196 `wics`, :208-276
// `MonomialBasis`).  Closed form (verified against MonomialBasis):
//   rank(a1,a2,a3,a4) = rowbase(deg,a1,a2) + a3,
//   rowbase(deg,a1,a2) = C(deg+3,3)-C(deg-a1+3,3) + C(deg-a1+2,2)-C(deg-a1-a2+2,2).
// A "run" is the set of monomials sharing (a1,a2): deg-a1-a2+1 consecutive entries.
//
// Internal layout of Delta ("lex43g"): same run structure, but inside a run entries are ordered
// by a4 instead of a3 (the run is stored reversed), every run is followed by G = d-p+1 zero
// bytes ("guard"), and the buffer starts with ZPAD zero bytes:
//     offset(I1,I2,I3,I4) = gbase(I1,I2) + I4,
//     gbase(I1,I2) = ZPAD + rowbase(D,I1,I2) + G * runindex(I1,I2),  runindex = I1(D+1) - I1(I1-1)/2 + I2.
// With it every run of an operator-matrix row is a FORWARD contiguous copy of a piece of a Delta
// run, out-of-range exponents (I3 < 0 or I4 < 0, at most G steps outside the run) land on guard
// zeros, and columns that can never match read the leading zero pad: the matrix builder needs
// no validity predicates at all (see qfs_matrix.cuh).
#pragma once
#include <stddef.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define QFS_HD __host__ __device__ __forceinline__
#else
#define QFS_HD inline
#endif

QFS_HD constexpr int qc2(int n) { return n >= 2 ? n * (n - 1) / 2 : 0; }
QFS_HD constexpr int qc3(int n) { return n >= 3 ? n * (n - 1) * (n - 2) / 6 : 0; }
QFS_HD constexpr int qrowbase(int deg, int a1, int a2)
{
    return qc3(deg + 3) - qc3(deg - a1 + 3) + qc2(deg - a1 + 2) - qc2(deg - a1 - a2 + 2);
}
QFS_HD constexpr int qround16(int n) { return (n + 15) & ~15; }

#ifndef QFS_PITCH_ALIGN
#define QFS_PITCH_ALIGN 128
#endif

template <int P>
struct Shape {
    static constexpr int p = P;
    static constexpr int psq = P * P;
    static constexpr int d = 4 * (P - 1);                 // deg g = deg f^(p-1)
    static constexpr int dh = (P > 2) ? 4 * (P - 2) : 0;  // deg h = deg f^(p-2)
    static constexpr int dE = 4 * P;                      // deg E = deg Delta_1(f)
    static constexpr int D = P * d;                       // deg Delta
    static constexpr int N = qc3(d + 3);
    static constexpr int Nh = qc3(dh + 3);
    static constexpr int NE = qc3(dE + 3);
    static constexpr int L = qc3(D + 3);
    static constexpr int pitch = (N + QFS_PITCH_ALIGN - 1) / QFS_PITCH_ALIGN * QFS_PITCH_ALIGN;   // row pitch of M and stride of N-vectors
    static constexpr int Nh_pad = qround16(Nh);
    static constexpr int NE_pad = qround16(NE);
    static constexpr int L_pad = qround16(L);
    static constexpr int cap = qrowbase(d, P - 1, P - 1) + P - 1;
    static constexpr int ngroups = (d + 1) * (d + 2) / 2;  // (r1,r2) row groups of M
    // guard-banded Delta layout (lex43g)
    static constexpr int G = d - P + 1;                    // farthest out-of-run read of the builder
    static constexpr int ZPAD = qround16(P * d + 1);       // leading zeros: covers offset p*(R-r3) <= p*d
    static constexpr int nruns = (D + 1) * (D + 2) / 2;
    static constexpr int Lg = ZPAD + L + G * nruns;
    static constexpr int Lg_pad = (Lg + 31) & ~31;  // whole 128-byte staging units of the quad-interleaved array (qfs_matrix_staged.cuh)
    // Four surfaces (a "quad": slots 4q..4q+3 of a chunk) share one byte-interleaved Delta array:
    // byte x of slot s sits at (s>>2)*quad_stride + 4*x + (s&3), so one aligned 32-bit load fetches the
    // same Delta entry of the four surfaces (qfs_matrix.cuh gathers that way).
    static constexpr size_t quad_stride = 4 * (size_t)Lg_pad;
    static QFS_HD constexpr int runindex(int I1, int I2) { return I1 * (D + 1) - I1 * (I1 - 1) / 2 + I2; }
    static QFS_HD constexpr int gbase(int I1, int I2) { return ZPAD + qrowbase(D, I1, I2) + G * runindex(I1, I2); }
};

// error bits raised by kernels into the context's device flag word
#define QFS_ERRBIT_INPUT 1      // coefficient >= p, or the zero form
#define QFS_ERRBIT_INVARIANT 2  // Witt-carry numerator not divisible by p
