// check_delta_plan.cpp -- host-side proof of the index algebra of qfs_delta_mma.cuh (no GPU needed).
//
//   g++ -O2 -std=c++17 -o /tmp/check_delta_plan tools/check_delta_plan.cpp && /tmp/check_delta_plan
//
// For every supported prime it builds the phase plan and replays what the kernel does with indices only: every
// (point, class) pair of every phase is sent through delta_row / delta_col, and the word it lands on must be the
// entry gbase(I1, I2) + I4 of the quad's Delta array, inside the piece that the phase stores; the pieces must tile
// [0, align4(Lg)) exactly once, and every exponent of degree D must be produced exactly once.  tests/test_delta_plan.py
// runs it in the CPU suite.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2502_12428_b200/csrc/qfs_delta_mma.cuh"

template <int P>
int check(int split = DeltaMmaCfg<P>::SPLIT)
{
    using S = Shape<P>;
    using C = DeltaMmaCfg<P>;
    DeltaPlan plan;
    if (!delta_plan<P>(plan, split)) { printf("p=%d: plan failed (SBW/MPTS too small)\n", P); return 1; }
    const int Lend = (S::Lg + 3) & ~3;
    std::vector<uint8_t> stored(Lend, 0), entry(Lend, 0);
    long tiles = 0, pts = 0, words = 0, blocks = 0;
    int errors = 0;
    auto bad = [&](const char* what, int a, int b, int c) {
        if (errors++ < 10) printf("p=%d: %s (%d %d %d)\n", P, what, a, b, c);
    };
    for (size_t ip = 0; ip < plan.phases.size(); ++ip) {
        const DeltaPhase& ph = plan.phases[ip];
        const int s1 = ph.s1, ns = S::d - s1, n0 = S::D - P * s1 - ph.rho1a;
        if (ph.nwords > (uint32_t)C::SBW) bad("phase exceeds the staging buffer", (int)ip, (int)ph.nwords, ph.npts);
        std::vector<uint8_t> cover(ph.nwords, 0);   // every staged word: one entry or one zero of a guard item
        tiles += (ph.npts + 15) / 16;
        blocks += (ph.flags & DPH_BLOCK) ? 1 : 0;
        pts += ph.npts;
        words += ph.nwords;
        uint32_t po = 0;
        for (int k = 0; k < ph.nrho1; ++k) {
            const DeltaPiece& pc = plan.pieces[ph.piece0 + k];
            if (!pc.nw) continue;
            if (pc.po != po || (pc.po & 3) || (pc.nw & 3) || (pc.ga & 3)) bad("piece misaligned", (int)ip, k, (int)pc.po);
            po += pc.nw;
            for (uint32_t e = pc.ga; e < pc.ga + pc.nw; ++e) {
                if (e >= (uint32_t)Lend) { bad("piece past the end", (int)ip, k, (int)e); break; }
                if (stored[e]++) bad("entry stored twice", (int)ip, k, (int)e);
            }
        }
        if (po != ph.nwords) bad("nwords mismatch", (int)ip, (int)po, (int)ph.nwords);
        // the kernel's point enumeration
        int npts = 0;
        for (int s2 = ph.s2a; s2 < ph.s2b; ++s2) npts += ns - s2 + 1;
        if (npts != ph.npts) bad("npts mismatch", (int)ip, npts, ph.npts);
        for (int ql = 0; ql < ph.npts; ++ql) {
            int s2 = ph.s2a, s3 = ql;
            while (s3 > ns - s2 && s2 < ph.s2b - 1) { s3 -= ns - s2 + 1; ++s2; }
            if (s3 < 0 || s2 + s3 > ns) bad("point walk", (int)ip, ql, s2);
            int R, a, room;
            delta_row<P>(n0, s2, s3, R, a, room);
            for (int c = 0; c < ph.nrho1 * P * P; ++c) {
                const int k = c / (P * P), r = c - k * (P * P), rho2 = r / P, rho3 = r - rho2 * P;
                const DeltaPiece& pc = plan.pieces[ph.piece0 + k];
                int Cc, m, need;
                delta_col<P>(n0, k, rho2, rho3, pc.cconst, Cc, m, need);
                const int I1 = P * s1 + ph.rho1a + k, I2 = P * s2 + rho2, I3 = P * s3 + rho3, I4 = S::D - I1 - I2 - I3;
                if ((room >= need) != (I4 >= 0)) { bad("validity predicate", I1, I2, I3); continue; }
                if (I4 < 0) continue;
                const int w = R + Cc - a * m;
                if (w < (int)pc.po || w >= (int)(pc.po + pc.nw)) { bad("word outside its piece", I1, I2, I3); continue; }
                const int e = (int)pc.ga + (w - (int)pc.po);
                if (e != S::gbase(I1, I2) + I4) { bad("word is not the entry's offset", I1, I2, e - (S::gbase(I1, I2) + I4)); continue; }
                if (entry[e]++) bad("exponent produced twice", I1, I2, I3);
                cover[w]++;
            }
        }
        // the kernel's guard items
        const int ns2 = ph.s2b - ph.s2a;
        for (int gi = 0; gi < ph.nrho1 * P * ns2; ++gi) {
            const int k = gi / (P * ns2), j = gi - k * (P * ns2);
            const int I2 = P * ph.s2a + j, nk = n0 - k;
            const DeltaPiece& pc = plan.pieces[ph.piece0 + k];
            if (!(I2 <= nk && pc.nw > 0)) continue;
            const int rs = delta_run_start<P>(nk, I2, pc.cconst, (int)pc.po);
            for (int w = (j == 0 ? 0 : rs - S::G); w < rs; ++w) {
                if (w < 0 || w >= (int)pc.nw) { bad("guard word outside the piece", (int)ip, k, w); break; }
                cover[pc.po + w]++;
            }
            if (I2 == std::min(P * ph.s2b - 1, nk))
                for (int w = rs + (nk - I2 + 1); w < (int)pc.nw; ++w) cover[pc.po + w]++;
        }
        for (uint32_t w = 0; w < ph.nwords; ++w)
            if (cover[w] != 1) { bad("staged word not written exactly once", (int)ip, (int)w, cover[w]); break; }
    }
    for (int e = 0; e < Lend; ++e)
        if (stored[e] != 1) { bad("entry not stored", e, stored[e], 0); break; }
    long produced = 0;
    for (int e = 0; e < Lend; ++e) produced += entry[e];
    if (produced != S::L) bad("exponents produced != L", (int)produced, S::L, 0);
    for (int I1 = 0; I1 <= S::D && errors == 0; ++I1)
        for (int I2 = 0; I1 + I2 <= S::D; ++I2)
            for (int I4 = 0; I1 + I2 + I4 <= S::D; ++I4)
                if (!entry[S::gbase(I1, I2) + I4]) { bad("exponent missing", I1, I2, I4); break; }
    for (int i = 0; i < split; ++i)
        if (plan.parts[i] > plan.parts[i + 1]) bad("parts not monotone", i, 0, 0);
    if (plan.parts[0] != 0 || plan.parts[split] != plan.phases.size()) bad("parts do not cover the phases", 0, 0, 0);
    printf("p=%d: %zu phases in %ld blocks, %zu pieces, %ld points in %ld tiles (%.1f%% of the tile rows), classes %d of %d, %ld staged words "
           "(%.2f x L), smem %d bytes: %s\n",
           P, plan.phases.size(), blocks, plan.pieces.size(), pts, tiles, 100.0 * pts / (16.0 * tiles), C::NCLS, C::NCLS_PAD, words,
           (double)words / S::L, C::SMEM, errors ? "FAILED" : "ok");
    return errors;
}

int main()
{
    int e = 0;
    e += check<3>();
    e += check<5>();
    e += check<7>();
    e += check<11>();
    e += check<13>();
    e += check<5>(DeltaMmaCfg<5>::SPLIT_FEW);   // the plans of launches with few quads
    e += check<7>(DeltaMmaCfg<7>::SPLIT_MID);
    e += check<7>(DeltaMmaCfg<7>::SPLIT_FEW);
    e += check<11>(DeltaMmaCfg<11>::SPLIT_FEW);
    e += check<3>(DeltaMmaCfg<3>::SPLIT_FEW);
    return e ? 1 : 0;
}
