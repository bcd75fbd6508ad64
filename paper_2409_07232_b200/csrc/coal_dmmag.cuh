// coal_dmmag.cuh -- FSBM_NUMERICS_FAST on the FP64 tensor cores (DMMA.8x8x4) for grids
// whose flux targets stay within nine bins of the owner: 66/132/264 bins on the
// equal-range grids of SURVEY 8(d), and others (the tuned 32/33-bin kernel is coal_dmma.cuh).
//
// Same owner decomposition as coal_dmma.cuh / coal_fast.cuh (coalescence.cpp:204-339
// reassociated): for a pair (a, b -> d) the row pass (owner o = i, stream s = j,
// v = nb, f = na, loss -> a) and the column pass (o = j, s = i, v = na, f = nb,
// loss -> b) compute per 8-row owner block and 8-point tile the GEMMs
//     L[o,q]   = sum_s A(o,s) v_q[s]                       loss of bin o
//     Z_t[o,q] = sum_s A(o-t,s) c_t(o-t,s) v_q[s]          gain of owner row o-t into bin o
// where c_t is the GainTable weight (coalescence.cpp:36-67) of a cell towards the bin t
// above its owner (cells the owner owns: s < o; column pass and self-pair diagonal
// s <= o, the latter halved, coalescence.cpp:293).  The gains are written in this
// target-aligned "gather" form (A rows shifted by t, weights pre-arranged on the host as
// fragments), so no multi-row carries exist.  "Far" K-steps (every cell targets {o, o+1}
// with weights summing to 1) run two DMMAs -- X = sum A v, Y = sum A c0 v with
// c0 = 1 - x_s / width_o -- and give the hi gain X - Y, carried one row (smem).
//
// Execution: the per-pass tables (K500, K750-K500) are pre-arranged in DMMA A-fragment
// order ([pass][block][k][lane]) and streamed per warp from L2 by 512-byte loads, four
// K-steps in flight ahead of the DMMAs; work units (pass, point group, row block) are taken
// dynamically by the warps of the TMEM lane quadrant that holds the unit's deltas
// (tcgen05.ld/st), in pass order, with a per-block ticket that fixes the accumulation order
// (bitwise determinism).  The band gains are pre-weighted on the host (A(o-t, s) * c_t per
// pass, one fragment per (t, K-step) entry of the block) and run one target offset at a
// time, so a single 8x8 accumulator is live: 16 warps x 128 registers at every band width.
// Zero owner rows and zero stream tails (the reference's rate == 0 skip) drop whole units
// and K-steps.  The K-loops are compiled twice (group-uniform vs per-point pressure
// weights); 66/132/264 bins are compiled in.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <type_traits>
#include <vector>

#include "coal_dmma.cuh"

namespace fsbm {

constexpr int kGNT = 2;      // 8-point N-tiles per warp (16 points per group)
constexpr int kDmmagPadSteps = 8; // zero fragments after each table: unchecked prefetch overrun

struct DmmagTables {
    int nkr = 0, S = 0, KS = 0, nblk = 0, SR = 0, TM = 0, npairs = 0;
    int item_base[kMaxPairs] = {};
    double2 *stages = nullptr;   // [item][block][KS][32] A fragments (K500, Kd)
    double2 *stages1 = nullptr;  // the same with .x = K500 + Kd rounded once (w = 1: p >= 750 hPa)
    double *consts = nullptr;    // x[SR+8] | invw[SR+8] (padded, finite)
    int *cls = nullptr;          // [3 views][nblk] leading far K-steps kf
    double2 *bstages1 = nullptr; // bstages with .x = .x + .y rounded once (w = 1)
    double2 *bstages = nullptr;  // [item][view entry][32] band-gain A fragments pre-weighted:
                                 // (K500, K750-K500)(o-t, s) * c_t(o-t, s)
    int *gtk = nullptr;          // gather entries t | ks << 8, per (view, block) sorted by (t, ks)
    int *grange = nullptr;       // [3][nblk][2] entry range of (view, block) in gtk
    int bofs[2 * kMaxPairs] = {}; // item -> offset of its band fragments minus its view's first entry
    double *carry_g = nullptr;   // [SMs][6][nblk][16] carry rows of lean (global) launches
};

inline void free_dmmag_tables(DmmagTables &t) {
    cudaFree(t.stages);
    cudaFree(t.stages1);
    cudaFree(t.bstages1);
    cudaFree(t.consts);
    cudaFree(t.cls);
    cudaFree(t.bstages);
    cudaFree(t.gtk);
    cudaFree(t.grange);
    cudaFree(t.carry_g);
    t = DmmagTables{};
}

/// Builds the general DMMA tables; returns 0 with D.stages == nullptr when this grid is
/// outside the kernel's envelope (the caller then uses coal_fast).
inline int build_dmmag_tables(DmmagTables &D, int nkr, int npairs, const std::vector<int> &abd,
                              const std::vector<double> &x, const double *t750, const double *t500,
                              const std::vector<int32_t> &g_lo, const std::vector<double> &g_wlo,
                              const std::vector<double> &g_whi, const std::vector<double> &g_top) {
    D = DmmagTables{};
    if (nkr < 8 || nkr > 320) return 0;
    const int S = (nkr + 3) / 4 * 4, KS = S / 4, nblk = (nkr + 7) / 8, SR = nblk * 8;
    // far-cell weights are recomputed on the fly: c0 = (x[o+1] - (x[o] + x[s])) / width[o]
    // = 1 - x[s] / width[o], one FMA with the reciprocal width (checked against the
    // GainTable per far cell below: within 1e-14 -- the reference's own x[o] + x[s]
    // rounding is ~1e-15 of the weight at 132 bins -- or the cell leaves the far class)
    std::vector<double> xs(SR + 8), iw(SR + 8, 0.0);
    for (int k = 0; k < SR + 8; ++k) xs[k] = x[std::min(k, nkr - 1)];
    for (int k = 0; k + 1 < nkr; ++k) iw[k] = 1.0 / (x[k + 1] - x[k]);
    int maxoff = 0; // furthest flux target above the owner max(i,j)
    for (int o = 0; o < nkr; ++o)
        for (int s = 0; s <= o; ++s) {
            const size_t e = static_cast<size_t>(o) * nkr + s;
            if (g_lo[e] < 0) maxoff = std::max(maxoff, nkr - 1 - o);
            else {
                if (g_lo[e] < o) return 0;
                maxoff = std::max(maxoff, g_lo[e] - o + (g_whi[e] != 0.0 ? 1 : 0));
            }
        }
    const int TM = maxoff < 2 ? 2 : maxoff < 4 ? 4 : maxoff < 6 ? 6 : maxoff < 10 ? 10 : 0;
    if (TM == 0) return 0;
    // ---- K-step classes per view (0 R-cross: s<o, 1 R-self: s<o + s==o halved, 2 C: s<=o) ----
    // kf[V][b]: leading "far" K-steps of owner block b (every real cell s < o, targets
    // {o, o+1}, weights summing to 1) -- their gains run through the X/Y identity.
    // gm[V][b][ks]: target offsets t whose gather entry (owner rows 8b+r-t, cols 4ks..+3,
    // far cells excluded) has a non-zero weight.
    auto vmask = [&](int V, int o, int s) {
        return V == 2 ? (s <= o ? 1.0 : 0.0) : (s < o ? 1.0 : (V == 1 && s == o ? 0.5 : 0.0));
    };
    std::vector<int> kfv(3 * nblk);
    std::vector<uint16_t> bm(static_cast<size_t>(3) * nblk * KS, 0);
    for (int V = 0; V < 3; ++V)
        for (int b = 0; b < nblk; ++b) {
            int kf = 0;
            for (; kf < KS; ++kf) {
                bool far = true;
                for (int r = 0; r < 8 && far; ++r)
                    for (int c = 0; c < 4 && far; ++c) {
                        const int o = 8 * b + r, s = 4 * kf + c;
                        if (o >= nkr || s >= nkr) continue; // A is zero there
                        const size_t e = static_cast<size_t>(o) * nkr + s;
                        const double c0 = fma(-xs[s], iw[o], 1.0); // == (x[o+1] - m) / width[o]
                        far = vmask(V, o, s) == 1.0 && s < o && g_lo[e] == o &&
                              std::fabs(g_wlo[e] + g_whi[e] - 1.0) <= 4e-16 && std::fabs(c0 - g_wlo[e]) <= 1e-14;
                    }
                if (!far) break;
            }
            kfv[V * nblk + b] = kf;
        }
    // gather coefficient fragments (pair-independent, host only: they weight the band tables
    // below): entry (V, b, ks, t) holds, per lane (row r = lane/4, col c = lane%4), the
    // GainTable weight of cell (8b+r-t, 4ks+c) towards bin 8b+r, view-masked, zero for far
    // cells (handled by the X/Y identity)
    std::vector<int> goff(static_cast<size_t>(3) * nblk * KS, 0);
    std::vector<double> gco;
    for (int V = 0; V < 3; ++V)
        for (int b = 0; b < nblk; ++b) {
            for (int ks = 0; ks < KS; ++ks) {
                double frag[16][32] = {};
                uint16_t mask = 0;
                for (int t = 0; t < TM; ++t)
                    for (int lane = 0; lane < 32; ++lane) {
                        const int o = 8 * b + (lane >> 2) - t, s = 4 * ks + (lane & 3);
                        if (o < 0 || o >= nkr || s >= nkr) continue;
                        const double msk = vmask(V, o, s);
                        if (msk == 0.0 || (s < o && ks < kfv[V * nblk + (o >> 3)])) continue;
                        const size_t e = static_cast<size_t>(o) * nkr + s;
                        double c = 0.0;
                        if (g_lo[e] < 0) {
                            if (t == nkr - 1 - o) c = g_top[e];
                        } else {
                            if (t == g_lo[e] - o) c += g_wlo[e];
                            if (t == g_lo[e] - o + 1) c += g_whi[e];
                        }
                        c *= msk;
                        frag[t][lane] = c;
                        if (c != 0.0) mask |= 1u << t;
                    }
                bm[(static_cast<size_t>(V) * nblk + b) * KS + ks] = mask;
                goff[(static_cast<size_t>(V) * nblk + b) * KS + ks] = static_cast<int>(gco.size() / 32);
                for (int t = 0; t < TM; ++t)
                    if (mask >> t & 1u) gco.insert(gco.end(), frag[t], frag[t] + 32);
            }
        }
    if (gco.empty()) gco.assign(32, 0.0);
    // the same entries as one list per (view, block), ordered by target offset t then K-step:
    // the kernel runs them with one accumulator live (the t-th gain of the unit), folding it
    // into the emission when t changes
    std::vector<int2> gl;
    std::vector<int> gr(static_cast<size_t>(3) * nblk * 2, 0);
    for (int V = 0; V < 3; ++V)
        for (int b = 0; b < nblk; ++b) {
            const size_t vb = static_cast<size_t>(V) * nblk + b;
            gr[2 * vb] = static_cast<int>(gl.size());
            for (int t = 0; t < TM; ++t)
                for (int ks = 0; ks < KS; ++ks) {
                    const unsigned m = bm[vb * KS + ks];
                    if (m >> t & 1u)
                        gl.push_back(int2{goff[vb * KS + ks] + __builtin_popcount(m & ((1u << t) - 1u)), t | ks << 8});
                }
            gr[2 * vb + 1] = static_cast<int>(gl.size());
        }
    if (gl.empty()) gl.push_back(int2{0, 0});
    // ---- per-pass A fragments: [item][block][ks][lane] (K500, K750-K500) ----
    int nitems = 0;
    for (int p = 0; p < npairs; ++p) {
        D.item_base[p] = nitems;
        nitems += abd[3 * p] == abd[3 * p + 1] ? 1 : 2;
    }
    const size_t item_elems = static_cast<size_t>(nblk) * KS * 32;
    // + kDmmagPadSteps fragments of zeros at the end: the kernel's prefetch reads up to 2 x 4
    // K-steps past a unit's last one without a bounds check (the values are never used)
    std::vector<double2> st(static_cast<size_t>(nitems) * item_elems + kDmmagPadSteps * 32, double2{0.0, 0.0});
    const size_t sq = static_cast<size_t>(nkr) * nkr;
    for (int p = 0; p < npairs; ++p) {
        const bool self = abd[3 * p] == abd[3 * p + 1];
        const double *k750 = t750 + p * sq, *k500 = t500 + p * sq;
        for (int X = 0; X < (self ? 1 : 2); ++X) {
            double2 *base = st.data() + static_cast<size_t>(D.item_base[p] + X) * item_elems;
            for (int bb = 0; bb < nblk; ++bb)
                for (int ks = 0; ks < KS; ++ks)
                    for (int lane = 0; lane < 32; ++lane) {
                        const int o = 8 * bb + (lane >> 2), s = 4 * ks + (lane & 3);
                        if (o >= nkr || s >= nkr) continue;
                        const int i = X == 0 ? o : s, j = X == 0 ? s : o; // reference cell (i,j)
                        const size_t u = self ? static_cast<size_t>(std::min(i, j)) * nkr + std::max(i, j)
                                              : static_cast<size_t>(i) * nkr + j;
                        base[(static_cast<size_t>(bb) * KS + ks) * 32 + lane] = double2{k500[u], k750[u] - k500[u]};
                    }
        }
    }
    // band-gain fragments per item over its view's entry list: entry (t, ks) of block b holds,
    // per lane (row r, col c), A(8b+r-t, 4ks+c) * c_t of that cell -- the shifted owner row
    // and its GainTable weight multiplied once here instead of per point batch
    int vlo[3];
    for (int V = 0; V < 3; ++V) vlo[V] = gr[2 * (V * nblk)];
    std::vector<double2> bst;
    for (int p = 0; p < npairs; ++p) {
        const bool self = abd[3 * p] == abd[3 * p + 1];
        const double *k750 = t750 + p * sq, *k500 = t500 + p * sq;
        for (int X = 0; X < (self ? 1 : 2); ++X) {
            const int V = X == 1 ? 2 : (self ? 1 : 0), item = D.item_base[p] + X;
            D.bofs[item] = static_cast<int>(bst.size() / 32) - vlo[V];
            for (int b = 0; b < nblk; ++b) {
                const size_t vb = static_cast<size_t>(V) * nblk + b;
                for (int n = gr[2 * vb]; n < gr[2 * vb + 1]; ++n) {
                    const int t = gl[n].y & 255, ks = gl[n].y >> 8;
                    for (int lane = 0; lane < 32; ++lane) {
                        const int o = 8 * b + (lane >> 2) - t, s = 4 * ks + (lane & 3);
                        const double c = gco[static_cast<size_t>(gl[n].x) * 32 + lane];
                        double2 v{0.0, 0.0};
                        if (c != 0.0 && o >= 0 && o < nkr && s < nkr) {
                            const int i = X == 0 ? o : s, j = X == 0 ? s : o;
                            const size_t u = self ? static_cast<size_t>(std::min(i, j)) * nkr + std::max(i, j)
                                                  : static_cast<size_t>(i) * nkr + j;
                            v = double2{k500[u] * c, (k750[u] - k500[u]) * c};
                        }
                        bst.push_back(v);
                    }
                }
            }
        }
    }
    bst.resize(bst.size() + kDmmagPadSteps * 32, double2{0.0, 0.0}); // prefetch overrun
    std::vector<int> gtk(gl.size());
    for (size_t n = 0; n < gl.size(); ++n) gtk[n] = gl[n].y;
    std::vector<double> consts(2 * (SR + 8));
    std::copy(xs.begin(), xs.end(), consts.begin());
    std::copy(iw.begin(), iw.end(), consts.begin() + SR + 8);
    auto up = [](auto **dst, const auto &v) {
        using T = typename std::remove_reference<decltype(v)>::type::value_type;
        return cudaMalloc(reinterpret_cast<void **>(dst), sizeof(T) * v.size()) == cudaSuccess &&
               cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    };
    // w = 1 (pressure >= 750 hPa, the K750 table): the interpolation fma(1, Kd, K500) is the
    // single rounding of K500 + Kd, done here once -- a w = 1 group then runs the
    // non-interpolating loop on these copies, bitwise equal to interpolating on device
    std::vector<double2> st1(st), bst1(bst);
    for (auto &v : st1) v.x = v.x + v.y;
    for (auto &v : bst1) v.x = v.x + v.y;
    if (!up(&D.stages, st) || !up(&D.consts, consts) || !up(&D.cls, kfv) || !up(&D.stages1, st1) ||
        !up(&D.bstages1, bst1) ||
        !up(&D.bstages, bst) || !up(&D.gtk, gtk) || !up(&D.grange, gr)) {
        free_dmmag_tables(D);
        fast_err() = "dmmag tables: device allocation failed";
        return 6;
    }
    D.nkr = nkr;
    D.S = S;
    D.KS = KS;
    D.nblk = nblk;
    D.SR = SR;
    D.TM = TM;
    D.npairs = npairs;
    if (nblk > 16) { // spectra of 16 points leave no room for the carry rows: global scratch per CTA
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaMalloc(&D.carry_g, static_cast<size_t>(sms) * kNCat * nblk * 16 * sizeof(double)) != cudaSuccess) {
            free_dmmag_tables(D);
            fast_err() = "dmmag tables: device allocation failed";
            return 6;
        }
    }
    return 0;
}

struct DmmagArgs {
    int KS, nblk, SR;
    uint32_t nbatches;
    int noskip, lean;
    double *carry_g;
    int item_base[kMaxPairs];
    const double2 *stages, *stages1;
    const double *consts;
    const int *cls;
    const double2 *bstages, *bstages1;
    const int *gtk, *grange;
    int bofs[2 * kMaxPairs];
};

constexpr int kGSlotCols = 48; // TMEM columns of one (group, block) delta slot: 6 categories x 4 doubles

/// Work unit = (pass, point group g, row block b), index i = b*G + g.  Unit i's deltas live
/// in TMEM lane quadrant i % 4, slot i / 4: only that quadrant's warps can reach the slot,
/// and they take the quadrant's units dynamically, in pass order, from one atomic counter.
template <int TM, int G, int MAXW, bool PAD, int NKRC>
__global__ void __launch_bounds__(MAXW * 32, 1) coal_dmmag_kernel(StepArgs A, DmmagArgs F) {
    constexpr int NT = kGNT, NP = G * 16, QP = PAD ? NP + 4 : NP;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // NKRC != 0: a grid compiled in (66/132/264 bins) -- extents become immediates
    const int nkr = NKRC ? NKRC : A.nkr, SR = NKRC ? 8 * ((NKRC + 7) / 8) : F.SR;
    const int KS = NKRC ? (NKRC + 3) / 4 : F.KS, NB = NKRC ? (NKRC + 7) / 8 : F.nblk;
    const bool lean = NKRC ? NKRC == 264 : F.lean != 0; // compiled-in grids: layout known
    const int npairs = A.pairs.npairs, MP = 2 * npairs; // passes per substep (upper bound)
    // shared-memory layout (dmmag_smem_bytes); the carry rows and the band tables move to
    // global memory when the spectra leave no room (F.lean: 264-bin grids)
    double *work = reinterpret_cast<double *>(smem_raw);                     // [6][SR][QP]
    double *xs = work + static_cast<size_t>(kNCat) * SR * QP;                // [SR+8]
    double *iw = xs + SR + 8;                                                 // [SR+8]
    double *wts = iw + SR + 8;                                                // [NP]
    unsigned long long *act = reinterpret_cast<unsigned long long *>(wts + NP); // [NP]
    unsigned long long *ptrip = act + NP;                                     // [NP]
    uint32_t *pidx = reinterpret_cast<uint32_t *>(ptrip + NP);                // [NP]
    int *pfail = reinterpret_cast<int *>(pidx + NP);                          // [NP]
    int *kfs = pfail + NP;                                                    // [3][NB]
    int *ps = kfs + 3 * NB;                                                   // [MP] pass: p | X<<8 | nlive<<16
    int *pcum = ps + MP;                                                      // [4][MP+1] units per quadrant
    int *served = pcum + 4 * (MP + 1);                                        // [G][NB] emitted units
    uint16_t *rnk = reinterpret_cast<uint16_t *>(served + G * NB);            // [MP][NB] emission rank
    double *carry;                                                            // [6][G][NB][16]
    {
        unsigned char *tail = reinterpret_cast<unsigned char *>(rnk + MP * NB);
        tail += (16 - reinterpret_cast<uintptr_t>(tail) % 16) % 16;
        carry = lean ? F.carry_g + static_cast<size_t>(blockIdx.x) * kNCat * NB * NP : reinterpret_cast<double *>(tail);
    }
    __shared__ unsigned long long cta_act;
    __shared__ int kzg[G][kNCat];
    __shared__ int kzc[kNCat];
    __shared__ unsigned char guni[G]; // the group's live points share one pressure weight
    __shared__ int qcnt[4];
    __shared__ int npass;
    __shared__ uint32_t tmem_base;
#ifdef FSBM_SYNCCHECK_MBAR
    // compute-sanitizer synccheck (CUDA 12.9) aborts a tcgen05 kernel that initialises no
    // mbarrier ("Missing init" at shared 0x0); its build variant adds one unused barrier
    __shared__ uint64_t synccheck_bar;
    if (threadIdx.x == 0) {
        mbar_init(&synccheck_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
#endif
    __shared__ unsigned long long cnt_sh[3];

    const int tid = threadIdx.x, nthr = blockDim.x, NW = nthr >> 5;
    const int wid = tid >> 5, lane = tid & 31;
    const int quad = wid & 3, wqi = wid >> 2, nq = (NW - quad + 3) >> 2;
    const int lr = lane >> 2, lc = lane & 3;
    if (A.stale && *A.stale) return; // stale mask: the step must not touch the state
    const uint32_t nact = *A.nactive;
    const unsigned long long full_evals = static_cast<unsigned long long>(npairs) * nkr * nkr;
    const int self_tri = nkr * (nkr + 1) / 2, cross_sq = nkr * nkr;
    const double dt = A.dt_sub;
    const int nslots = (NB * G - 1) / 4 + 1; // slots per quadrant

    // point-minor spectra.  PAD: row pitch NP+4 doubles (= 4 mod 16), so the 4 K rows of a
    // B fragment, the 8 owner rows of an emission and the 8 bins of a load each spread over
    // all banks (2 wavefronts per 256 B, the minimum).  Otherwise (264-bin lean layout, one
    // 16-point row = 128 B) the point index is XOR-swizzled by 4 x (bin mod 4): the 4 K rows
    // of a B fragment land on disjoint 32-byte bank groups in each half-warp (conflict free).
    auto W = [&](int c, int s, int q) -> double & {
        return work[(static_cast<size_t>(c) * SR + s) * QP + (PAD ? q : (q ^ ((s & 3) << 2)))];
    };
    auto CR = [&](int c, int g, int b, int q) -> double & {
        return carry[((static_cast<size_t>(c) * G + g) * NB + b) * 16 + q];
    };

    for (int f = tid; f < 2 * (SR + 8); f += nthr) xs[f] = F.consts[f];
    for (int f = tid; f < 3 * NB; f += nthr) kfs[f] = F.cls[f];
    for (int f = tid; f < kNCat * SR * QP; f += nthr) work[f] = 0.0; // rows >= nkr stay zero
    if (tid < 3) cnt_sh[tid] = 0ull;
    if (wid == 0) { // TMEM (whole SM): the delta slots of every (group, block)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const uint32_t tmq = tmem_base + (static_cast<uint32_t>(32 * quad) << 16); // this warp's lane quadrant

    for (uint32_t batch = blockIdx.x; batch < F.nbatches && batch * static_cast<uint32_t>(NP) < nact;
         batch += gridDim.x) {
        for (int q = tid; q < NP; q += nthr) {
            const uint32_t idx = batch * static_cast<uint32_t>(NP) + q;
            // past the end, or a hole of the level-major list (0xffffffff): not a point
            const uint32_t p = idx < nact ? A.active[idx] : 0xffffffffu;
            const bool live = p != 0xffffffffu;
            pidx[q] = p;
            wts[q] = live ? pressure_weight(A.pressure[p]) : 0.0;
            pfail[q] = live ? 0 : 1;
            ptrip[q] = 0;
        }
        __syncthreads();
        if (PAD && wid < G) { // one pressure weight per group (holes: any weight), once per batch
            const int q = 16 * wid + (lane & 15);
            const bool u = __all_sync(0xffffffffu, pidx[q] == 0xffffffffu || wts[q] == wts[16 * wid]);
            if (lane == 0) guni[wid] = u ? 1 : 0;
        }
        { // spectra -> work: a warp instruction covers 4 points x 8 consecutive bins
            const int NQ = kNCat * NP / 4;
            const int qs = lane >> 3, kc = lane & 7;
            for (int u = wid; u < NQ; u += NW) {
                const int c = u / (NP / 4), q = 4 * (u % (NP / 4)) + qs;
                const uint32_t p = pidx[q];
                const double *src = A.bins[c] + static_cast<size_t>(p) * nkr;
#pragma unroll 4
                // streaming loads/stores (evict-first): the spectra pass through once, the
                // L2-resident pass tables (tens of MB at 132-264 bins) stay
                for (int k = kc; k < nkr; k += 8) W(c, k, q) = p != 0xffffffffu ? __ldcs(src + k) : 0.0;
            }
        }
        __syncthreads();

        for (int sub = 0; sub < A.substeps; ++sub) {
            if (tid == 0) cta_act = 0ull;
            if (tid < G * kNCat) kzg[tid / kNCat][tid % kNCat] = -1;
            if (tid < kNCat) kzc[tid] = -1;
            if (tid < 4) qcnt[tid] = 0;
            for (int f = tid; f < G * NB; f += nthr) served[f] = 0;
            for (int f = tid; f < kNCat * NB * NP; f += nthr) carry[f] = 0.0;
            { // zero this warp's share of its quadrant's delta slots
                const double z[4] = {0.0, 0.0, 0.0, 0.0};
                for (int k = wqi; k < nslots; k += nq)
                    for (int c = 0; c < kNCat; ++c) tm_st4_nowait(tmq + k * kGSlotCols + 8 * c, z);
                tm_wait_st();
            }
            tm_fence_before();
            __syncthreads();
            tm_fence_after();
            for (int q = tid; q < NP; q += nthr) { // all_zero (coalescence.cpp:270-273)
                unsigned nz = 0;
                for (int c = 0; c < kNCat; ++c) { // scanned from the top: last non-zero bin
                    int l = nkr - 1;
                    while (l >= 0 && W(c, l, q) == 0.0) --l;
                    nz |= l >= 0 ? (1u << c) : 0u;
                    if (l >= 0 && pfail[q] == 0) {
                        const int lk = F.noskip ? nkr - 1 : l; // A/B: FSBM_DMMAG_NOSKIP
                        atomicMax(&kzg[q / 16][c], lk);
                        atomicMax(&kzc[c], lk);
                    }
                }
                unsigned long long m = 0, trip = 0;
                for (int pp = 0; pp < npairs; ++pp)
                    if (nz >> A.pairs.a[pp] & 1u) {
                        m |= 1ull << pp;
                        trip += A.pairs.a[pp] == A.pairs.b[pp] ? self_tri : cross_sq;
                    }
                if (pfail[q] == 0) {
                    act[q] = m;
                    atomicOr(&cta_act, m);
                    ptrip[q] += trip;
                } else {
                    act[q] = 0;
                }
            }
            __syncthreads();
            if (tid == 0) { // the pass sequence: p | X << 8 | live blocks << 16
                const unsigned long long amask = cta_act;
                int np_ = 0;
                for (int p = 0; p < npairs; ++p) {
                    if (!(amask >> p & 1ull)) continue;
                    const int pa = A.pairs.a[p], pb = A.pairs.b[p];
                    for (int X = 0; X < (pa == pb ? 1 : 2); ++X) {
                        const int fc = X == 0 ? pa : pb, sc = X == 0 ? pb : pa;
                        if (kzc[fc] < 0 || kzc[sc] < 0) continue; // every product of the pass is zero
                        ps[np_++] = p | X << 8 | min(NB, (kzc[fc] + TM - 1) / 8 + 1) << 16;
                    }
                }
                npass = np_;
            }
            __syncthreads();
            {
                const int NPS = npass;
                for (int b = tid; b < NB; b += nthr) { // emission rank: earlier passes with block b live
                    int r = 0;
                    for (int i = 0; i < NPS; ++i) {
                        rnk[i * NB + b] = static_cast<uint16_t>(r);
                        r += (ps[i] >> 16) > b ? 1 : 0;
                    }
                }
                if (tid >= 32 && tid < 36) { // units per quadrant, prefix over passes
                    const int q = tid - 32;
                    int c = 0;
                    pcum[q * (MP + 1)] = 0;
                    for (int i = 0; i < NPS; ++i) {
                        c += ((ps[i] >> 16) * G - q + 3) / 4;
                        pcum[q * (MP + 1) + i + 1] = c;
                    }
                }
            }
            __syncthreads();

            // ---- units: dynamic within the lane quadrant, pass order ----
            const int NPS = npass;
            const int *pc = pcum + quad * (MP + 1);
            int pi = 0;
            while (true) {
                int u = 0;
                if (lane == 0) u = atomicAdd(&qcnt[quad], 1);
                u = __shfl_sync(0xffffffffu, u, 0);
                while (pi < NPS && u >= pc[pi + 1]) ++pi;
                if (pi >= NPS) break;
                const int pw_ = ps[pi], p = pw_ & 255, X = (pw_ >> 8) & 255;
                const int iu = quad + 4 * (u - pc[pi]); // unit index b*G + g within the pass
                const int b = iu / G, g = iu % G;
                const int slot = iu >> 2;
                const int rank = rnk[pi * NB + b];
                const int pa = A.pairs.a[p], pb = A.pairs.b[p];
                const int fcat = X == 0 ? pa : pb, scat = X == 0 ? pb : pa, pd = A.pairs.d[p];
                const int V = X == 1 ? 2 : (pa == pb ? 1 : 0);
                const int kzs = kzg[g][scat];
                const int qg = 16 * g, o = 8 * b + lr;
                // every owner row this unit reads (8b-TM+1 .. 8b+7) or the stream is zero
                const bool live = 8 * b - (TM - 1) <= kzg[g][fcat] && kzs >= 0;
                double lv[4] = {0.0, 0.0, 0.0, 0.0}, hv[4] = {0.0, 0.0, 0.0, 0.0};
                if (live) {
                    bool on[NT][2], allu = true;
                    double wq[NT];
                    const double wu = wts[qg];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        wq[nt] = wts[qg + 8 * nt + lr];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int q = qg + 8 * nt + 2 * lc + e;
                            on[nt][e] = act[q] >> p & 1ull;
                            if (!PAD) allu = allu && (wts[q] == wu || pidx[q] == 0xffffffffu); // holes: any weight
                        }
                    }
                    // the group's weight mode, found once per batch (padded layouts; the
                    // register-tight 264-bin layout measured faster re-deriving it per unit)
                    const bool uni_rt = PAD ? guni[g] != 0 : __all_sync(0xffffffffu, allu);
                    const int vb = V * NB + b;
                    const int kf = kfs[vb];
                    const int kend = min(KS, (kzs >> 2) + 1);
                    const int kfe = min(kf, kend);
                    const double iwo = iw[o];
                    // w = 1 groups read the pre-summed copies and run the non-interpolating loop
                    const bool w1 = uni_rt && wu == 1.0;
                    const double2 *gi = (w1 ? F.stages1 : F.stages) + static_cast<size_t>(F.item_base[p] + X) * NB * KS * 32;
                    const double2 *ga = gi + static_cast<size_t>(b) * KS * 32 + lane;
                    const int g0 = __ldg(F.grange + 2 * vb), g1 = __ldg(F.grange + 2 * vb + 1);
                    // L: loss of non-far steps; Xf/Yf: far steps (sum A v, sum A c0 v), owner rows;
                    // hz: the band gains of owner rows o-t into rows o (gather form, far cells excluded)
                    double L[NT][2], Xf[NT][2], Yf[NT][2], hz[NT][2];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) L[nt][e] = Xf[nt][e] = Yf[nt][e] = hz[nt][e] = 0.0;
                    // the K-loops, compiled twice: one pressure weight for the whole group
                    // (uni, the common case) or per-point weights (a group straddling a level)
                    // unpadded (264-bin) layout: the lane's B-fragment row pointers (row 4ks+lc; the
                    // swizzle depends on the row mod 4 = lc only), so a K-step's B loads are one
                    // offset away (+1.8% there; the padded layouts measured faster in index form)
                    const double *vbp[NT];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const int q = qg + 8 * nt + lr;
                        vbp[nt] = work + (static_cast<size_t>(scat) * SR + lc) * QP + (q ^ (lc << 2));
                    }
                    auto kloop = [&](auto UC) {
                        // 0: per-point weights (dual), 1: one weight for the group, 2: that weight is 0
                        // (p <= 500 hPa: A = K500 exactly, no interpolation)
                        constexpr int MODE = decltype(UC)::value;
                        constexpr bool uni = MODE != 0, w0 = MODE == 2;
                        auto loadb = [&](int ks, double (&bv)[NT], double (&bw)[NT]) {
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) {
                                bv[nt] = PAD ? W(scat, 4 * ks + lc, qg + 8 * nt + lr) : vbp[nt][ks * 4 * QP];
                                bw[nt] = uni ? 0.0 : wq[nt] * bv[nt];
                            }
                        };
                        // (A) the owner block's K-steps: far [0, kfe) (X/Y identity), loss [kfe, kend).
                        // A fragments stream from L2 in chunks of DA; the next chunk is in flight
                        // during this one's DMMAs (tables padded: no bounds checks on the loads).
                        constexpr int DA = 4;
                        // PRE: kk.x already holds the interpolated A operand (one-weight loops)
                        auto step = [&](int ks, double2 kk, auto PRE) {
                            double bv[NT], bw[NT];
                            loadb(ks, bv, bw);
                            const double a = decltype(PRE)::value ? kk.x : (uni ? (w0 ? kk.x : fma(wu, kk.y, kk.x)) : kk.x);
                            const double ad = kk.y;
                            if (ks < kfe) {
                                const double c0 = fma(-xs[4 * ks + lc], iwo, 1.0); // 1 - x_s / width_o
                                const double a2 = a * c0, ad2 = ad * c0;
#pragma unroll
                                for (int nt = 0; nt < NT; ++nt) {
                                    dmma(Xf[nt][0], Xf[nt][1], a, bv[nt]);
                                    dmma(Yf[nt][0], Yf[nt][1], a2, bv[nt]);
                                    if (!uni) {
                                        dmma(Xf[nt][0], Xf[nt][1], ad, bw[nt]);
                                        dmma(Yf[nt][0], Yf[nt][1], ad2, bw[nt]);
                                    }
                                }
                            } else {
#pragma unroll
                                for (int nt = 0; nt < NT; ++nt) {
                                    dmma(L[nt][0], L[nt][1], a, bv[nt]);
                                    if (!uni) dmma(L[nt][0], L[nt][1], ad, bw[nt]);
                                }
                            }
                        };
                        if constexpr (uni && PAD) {
                            // one weight: the chunk's A operands are interpolated as the chunk
                            // arrives (K500 + w Kd), off the DMMAs' critical path (132 bins +2%;
                            // the register-tight unpadded 264-bin layout measured -4%)
                            auto interp = [&](double2 r) { return w0 ? r.x : fma(wu, r.y, r.x); };
                            double ac[DA];
#pragma unroll
                            for (int j = 0; j < DA; ++j) ac[j] = interp(__ldg(ga + j * 32)); // past kend: padding
                            for (int ks = 0; ks < kend; ks += DA) {
                                double2 nxt[DA];
#pragma unroll
                                for (int j = 0; j < DA; ++j)
                                    nxt[j] = __ldg(ga + (ks + DA + j) * 32);
#pragma unroll
                                for (int j = 0; j < DA; ++j)
                                    if (ks + j < kend) step(ks + j, double2{ac[j], 0.0}, std::true_type{});
#pragma unroll
                                for (int j = 0; j < DA; ++j) ac[j] = interp(nxt[j]);
                            }
                        } else {
                            double2 cur[DA];
#pragma unroll
                            for (int j = 0; j < DA; ++j) cur[j] = __ldg(ga + j * 32); // past kend: padding, unused
                            for (int ks = 0; ks < kend; ks += DA) {
                                double2 nxt[DA];
#pragma unroll
                                for (int j = 0; j < DA; ++j)
                                    nxt[j] = __ldg(ga + (ks + DA + j) * 32);
#pragma unroll
                                for (int j = 0; j < DA; ++j)
                                    if (ks + j < kend) step(ks + j, cur[j], std::false_type{});
#pragma unroll
                                for (int j = 0; j < DA; ++j) cur[j] = nxt[j];
                            }
                        }
                        // (B) band gathers, one target offset t at a time: entry (t, ks) is the
                        // pre-weighted A row o-t (cell (o-t, 4ks+lc) times its GainTable weight
                        // towards bin o) against the K-step's B fragment; the t-th sum is scaled
                        // by the owner value f(o-t) when t changes.  The unit's entries are
                        // contiguous and streamed like the owner K-steps.
                        if (g1 > g0) {
                            const int ng = g1 - g0;
                            const double2 *gb = (w1 ? F.bstages1 : F.bstages) + (static_cast<size_t>(F.bofs[F.item_base[p] + X]) + g0) * 32 + lane;
                            const int *gt = F.gtk + g0;
                            double Zt[NT][2];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) Zt[nt][0] = Zt[nt][1] = 0.0;
                            double2 cur[DA];
                            int tk[DA];
#pragma unroll
                            for (int j = 0; j < DA; ++j) {
                                cur[j] = __ldg(gb + j * 32);
                                tk[j] = j < ng ? __ldg(gt + j) : -1;
                            }
                            for (int n = 0; n < ng; n += DA) {
                                double2 nxt[DA];
                                int tkn[DA];
#pragma unroll
                                for (int j = 0; j < DA; ++j) {
                                    const bool in = n + DA + j < ng;
                                    nxt[j] = __ldg(gb + (n + DA + j) * 32);
                                    tkn[j] = in ? __ldg(gt + n + DA + j) : -1;
                                }
#pragma unroll
                                for (int j = 0; j < DA; ++j) {
                                    if (n + j >= ng) break;
                                    const int t = tk[j] & 255, ks = tk[j] >> 8;
                                    if (ks < kend) {
                                        double bv[NT], bw[NT];
                                        loadb(ks, bv, bw);
                                        const double a2 = uni ? (w0 ? cur[j].x : fma(wu, cur[j].y, cur[j].x)) : cur[j].x;
#pragma unroll
                                        for (int nt = 0; nt < NT; ++nt) {
                                            dmma(Zt[nt][0], Zt[nt][1], a2, bv[nt]);
                                            if (!uni) dmma(Zt[nt][0], Zt[nt][1], cur[j].y, bw[nt]);
                                        }
                                    }
                                    const int tn = j + 1 < DA ? tk[j + 1] : tkn[0]; // -1 past the end
                                    if (tn < 0 || (tn & 255) != t) { // fold the t-th gain
                                        const int ot = o - t;
#pragma unroll
                                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                                            for (int e2 = 0; e2 < 2; ++e2) {
                                                const int q = qg + 8 * nt + 2 * lc + e2;
                                                const double ft = on[nt][e2] && ot >= 0 ? W(fcat, ot, q) : 0.0;
                                                hz[nt][e2] = fma(ft, Zt[nt][e2], hz[nt][e2]);
                                                Zt[nt][e2] = 0.0;
                                            }
                                    }
                                }
#pragma unroll
                                for (int j = 0; j < DA; ++j) {
                                    cur[j] = nxt[j];
                                    tk[j] = tkn[j];
                                }
                            }
                        }
                    };
                    if (!uni_rt) kloop(std::integral_constant<int, 0>{});
                    else if (wu == 0.0 || w1) kloop(std::integral_constant<int, 2>{});
                    else kloop(std::integral_constant<int, 1>{});
                    // owner emission values (dt at the apply); far-cell hi gains of row 7
                    // carry into the next block's head row
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int q = qg + 8 * nt + 2 * lc + e;
                            const double f = on[nt][e] ? W(fcat, o, q) : 0.0;
                            lv[2 * nt + e] = f * (L[nt][e] + Xf[nt][e]);
                            const double hi = f * (Xf[nt][e] - Yf[nt][e]);
                            const double up = __shfl_up_sync(0xffffffffu, hi, 4);
                            double h = fma(f, Yf[nt][e], hz[nt][e]);
                            if (lr > 0) h += up;
                            hv[2 * nt + e] = h;
                            Xf[nt][e] = hi; // keep for the carry
                        }
                    // wait for this block's earlier units (deterministic accumulation order)
                    if (lane == 0) // (a short sleep per poll leaves issue slots to the working warps)
                        while (*reinterpret_cast<volatile int *>(&served[g * NB + b]) != rank) {
                            __nanosleep(20);
                        }
                    __syncwarp();
                    __threadfence_block();
                    tm_fence_after();
                    if (lr == 7 && b + 1 < NB) {
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int e = 0; e < 2; ++e) CR(pd, g, b, 8 * nt + 2 * lc + e) += Xf[nt][e];
                    }
                    const uint32_t ta = tmq + slot * kGSlotCols, tf = ta + 8 * fcat, tp = ta + 8 * pd;
                    if (fcat == pd) {
                        double d[4];
                        tm_ld4_nowait(tf, d);
                        tm_wait_ld();
#pragma unroll
                        for (int i = 0; i < 4; ++i) d[i] += hv[i] - lv[i];
                        tm_st4_nowait(tf, d);
                    } else {
                        double d[4], e4[4];
                        tm_ld4_nowait(tf, d);
                        tm_ld4_nowait(tp, e4);
                        tm_wait_ld();
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            d[i] -= lv[i];
                            e4[i] += hv[i];
                        }
                        tm_st4_nowait(tf, d);
                        tm_st4_nowait(tp, e4);
                    }
                    tm_wait_st();
                    tm_fence_before();
                } else if (lane == 0) {
                    while (*reinterpret_cast<volatile int *>(&served[g * NB + b]) != rank) {
                        __nanosleep(20);
                    }
                }
                __syncwarp();
                __threadfence_block();
                if (lane == 0) *reinterpret_cast<volatile int *>(&served[g * NB + b]) = rank + 1;
            }
            // ---- Jacobi apply (coalescence.cpp:313-328): own rows, then the block-head carries ----
            tm_fence_before();
            __syncthreads();
            tm_fence_after();
            for (int k = wqi; k < nslots; k += nq)
                {
                    const int iu = 4 * k + quad, b = iu / G, g = iu % G;
                    if (b >= NB) continue;
                    const int o = 8 * b + lr;
#pragma unroll
                    for (int c = 0; c < kNCat; ++c) {
                        double d[4];
                        tm_ld4_nowait(tmq + k * kGSlotCols + 8 * c, d);
                        tm_wait_ld();
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int q = 16 * g + 8 * nt + 2 * lc + e;
                                W(c, o, q) = fma(dt, d[2 * nt + e], W(c, o, q));
                            }
                    }
                }
            __syncthreads();
            for (int f = tid; f < kNCat * G * (NB - 1) * 16; f += nthr) {
                const int q = f % 16, r = f / 16, bb = r % (NB - 1), cg = r / (NB - 1), g = cg % G, c = cg / G;
                W(c, 8 * (bb + 1), 16 * g + q) = fma(dt, CR(c, g, bb, q), W(c, 8 * (bb + 1), 16 * g + q));
            }
            __syncthreads();
            for (int c = 0; c < kNCat; ++c) // stiffness: no clamping, report the first point
                for (int k = wid; k < nkr; k += NW)
                    for (int q = lane; q < NP; q += 32) {
                        const uint32_t p = pidx[q];
                        // every failing bin is offered (the sink keeps the first in serial
                        // order): only bit 0 (dead / failed in an earlier substep) gates
                        if (p == 0xffffffffu || (pfail[q] & 1) != 0) continue;
                        if (W(c, k, q) < 0.0) {
                            report_stiffness(A, p, c, k, W(c, k, q));
                            atomicOr(&pfail[q], 2);
                        }
                    }
            __syncthreads();
            for (int q = tid; q < NP; q += nthr)
                if (pfail[q] == 2) pfail[q] = 3;
        }
        { // write back, coalesced like the load
            const int NQ = kNCat * NP / 4;
            const int qs = lane >> 3, kc = lane & 7;
            for (int u = wid; u < NQ; u += NW) {
                const int c = u / (NP / 4), q = 4 * (u % (NP / 4)) + qs;
                const uint32_t p = pidx[q];
                if (p == 0xffffffffu) continue;
                double *dst = A.bins[c] + static_cast<size_t>(p) * nkr;
#pragma unroll 4
                for (int k = kc; k < nkr; k += 8) __stcs(dst + k, W(c, k, q));
            }
        }
        for (int q = tid; q < NP; q += nthr) {
            if (pidx[q] == 0xffffffffu || pfail[q] != 0) continue;
            atomicAdd(&cnt_sh[0], ptrip[q]);
            atomicAdd(&cnt_sh[1], 1ull);
            atomicAdd(&cnt_sh[2], A.kernel_strategy ? ptrip[q] : full_evals);
        }
        __syncthreads();
    }
    tm_fence_before();
    __syncthreads();
    if (wid == 0) {
        tm_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
    if (tid == 0 && (cnt_sh[0] | cnt_sh[1] | cnt_sh[2])) {
        atomicAdd(&A.counters[0], cnt_sh[0]);
        atomicAdd(&A.counters[1], cnt_sh[1]);
        atomicAdd(&A.counters[2], cnt_sh[2]);
    }
}

/// Shared memory of a launch with NP points per batch; lean: carry rows and band tables
/// in global memory.
inline size_t dmmag_smem_bytes(const DmmagTables &T, int NP, bool lean, bool pad) {
    const size_t MP = 2 * static_cast<size_t>(T.npairs);
    size_t b = (static_cast<size_t>(kNCat) * T.SR * (NP + (pad ? 4 : 0)) + 2 * (T.SR + 8) + NP) * sizeof(double) + NP * 24 +
               3 * T.nblk * 4 + MP * 4 + 4 * (MP + 1) * 4 + static_cast<size_t>(NP / 16) * T.nblk * 4 +
               MP * T.nblk * 2 + 16;
    if (!lean) b += static_cast<size_t>(kNCat) * T.nblk * NP * sizeof(double);
    return b;
}

/// Launch geometry: point groups, padded rows, lean (global carry/band tables).
struct DmmagGeom {
    int G = 0;
    bool pad = false, lean = false;
};

/// Most point groups (<= 3) that fit, padded rows preferred; the lean layout only for one group.
inline DmmagGeom dmmag_geom(const DmmagTables &T) {
    constexpr size_t kMax = 227 * 1024;
    for (int G = 3; G >= 1; --G)
        for (int pad = 1; pad >= 0; --pad)
            if (dmmag_smem_bytes(T, 16 * G, false, pad) <= kMax) return DmmagGeom{G, pad != 0, false};
    for (int pad = 1; pad >= 0; --pad)
        if (dmmag_smem_bytes(T, 16, true, pad) <= kMax) return DmmagGeom{1, pad != 0, true};
    return DmmagGeom{};
}

template <int TM, int G, int MAXW, bool PAD, int NKRC = 0>
inline int launch_dmmag_t(const DmmagTables &T, const StepArgs &A, int num_sms, cudaStream_t s, int nwarps,
                          bool lean) {
    constexpr int NP = G * 16;
    const size_t smem = dmmag_smem_bytes(T, NP, lean, PAD);
    if (smem > 227 * 1024 || nwarps > MAXW || (lean && !T.carry_g)) return -1;
    DmmagArgs F{};
    F.lean = lean;
    F.carry_g = T.carry_g;
    F.KS = T.KS;
    F.nblk = T.nblk;
    F.SR = T.SR;
    F.nbatches = (A.nactive_host + NP - 1) / NP;
    F.noskip = std::getenv("FSBM_DMMAG_NOSKIP") != nullptr;
    for (int p = 0; p < kMaxPairs; ++p) F.item_base[p] = T.item_base[p];
    F.stages = T.stages;
    F.stages1 = T.stages1;
    F.consts = T.consts;
    F.cls = T.cls;
    F.bstages = T.bstages;
    F.bstages1 = T.bstages1;
    F.gtk = T.gtk;
    F.grange = T.grange;
    for (int i = 0; i < 2 * kMaxPairs; ++i) F.bofs[i] = T.bofs[i];
    if (NKRC && NKRC != T.nkr) return -1;
    auto kern = coal_dmmag_kernel<TM, G, MAXW, PAD, NKRC>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess) {
        fast_err() = "dmmag path: cannot reserve shared memory";
        return 6;
    }
    const int grid = static_cast<int>(std::min<uint32_t>(F.nbatches, num_sms));
    kern<<<grid, nwarps * 32, smem, s>>>(A, F);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fast_err() = std::string("dmmag path launch: ") + cudaGetErrorString(e);
        return 6;
    }
    return 0;
}

/// Whether launch_dmmag takes this context's grid (same envelope, no launch).
inline bool dmmag_supported(const DmmagTables &T) {
    const DmmagGeom g = dmmag_geom(T);
    return T.stages && T.npairs <= kMaxPairs && g.G > 0 && (T.nblk * g.G - 1) / 4 + 1 <= 512 / kGSlotCols;
}

/// Returns -1 when this geometry cannot run the general DMMA path.  16 warps (128
/// registers: one band-gain accumulator live at a time); FSBM_DMMAG_WARPS overrides (A/B).
inline int launch_dmmag(const DmmagTables &T, const StepArgs &A, int num_sms, cudaStream_t s) {
    if (!T.stages || A.nkr != T.nkr || !dmmag_supported(T)) return -1;
    const DmmagGeom g = dmmag_geom(T);
    int nw = 16;
    if (const char *ev = std::getenv("FSBM_DMMAG_WARPS")) nw = std::max(4, std::min(nw, std::atoi(ev)));
    // the BASELINE grids with their extents compiled in (FSBM_DMMAG_GENERIC=1: A/B)
    if (!std::getenv("FSBM_DMMAG_GENERIC")) {
        if (T.nkr == 66 && T.TM == 4 && g.G == 3 && g.pad && !g.lean)
            return launch_dmmag_t<4, 3, 16, true, 66>(T, A, num_sms, s, nw, false);
        if (T.nkr == 132 && T.TM == 6 && g.G == 1 && g.pad && !g.lean)
            return launch_dmmag_t<6, 1, 16, true, 132>(T, A, num_sms, s, nw, false);
        if (T.nkr == 264 && T.TM == 10 && g.G == 1 && !g.pad && g.lean)
            return launch_dmmag_t<10, 1, 16, false, 264>(T, A, num_sms, s, nw, true);
    }
#define FSBM_DG(TM_, MW_)                                                                          \
    if (g.pad) {                                                                                   \
        switch (g.G) {                                                                             \
        case 3: return launch_dmmag_t<TM_, 3, MW_, true>(T, A, num_sms, s, nw, g.lean);            \
        case 2: return launch_dmmag_t<TM_, 2, MW_, true>(T, A, num_sms, s, nw, g.lean);            \
        default: return launch_dmmag_t<TM_, 1, MW_, true>(T, A, num_sms, s, nw, g.lean);           \
        }                                                                                          \
    }                                                                                              \
    switch (g.G) {                                                                                 \
    case 3: return launch_dmmag_t<TM_, 3, MW_, false>(T, A, num_sms, s, nw, g.lean);               \
    case 2: return launch_dmmag_t<TM_, 2, MW_, false>(T, A, num_sms, s, nw, g.lean);               \
    default: return launch_dmmag_t<TM_, 1, MW_, false>(T, A, num_sms, s, nw, g.lean);              \
    }
    switch (T.TM) {
    case 2: FSBM_DG(2, 16)
    case 4: FSBM_DG(4, 16)
    case 6: FSBM_DG(6, 16)
    case 10: FSBM_DG(10, 16)
    default: return -1;
    }
#undef FSBM_DG
}

} // namespace fsbm
