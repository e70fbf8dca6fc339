// lti2.cuh -- round-2 LTI engine for fp32 TDF-II filtering and its closed-form
// backward (arXiv 2511.14390, Eqs.4-9; the BASELINE configs C2, C4, C5).
//
// Same method as lti.cuh (the chunked scan of Eq.10, with fp64
// carries across tiles and a deterministic hierarchical look-back), re-laid out for
// sm_100a as PERSISTENT WARP TILES:
//   * a tile is 32 lane chunks of L samples of one sequence, owned by ONE warp (no
//     block-level scan, no __syncthreads on the per-tile path); a CTA is NWP
//     independent warps, the grid is one resident wave, and warps take tiles by an
//     atomic ticket (tile t = time tile t / B of sequence t % B), so every tile a warp
//     waits for was handed to a running warp;
//   * each lane's chunk arrives by one cp.async.bulk row copy (TMA engine, mbarrier
//     completion) into a 16 B-padded shared row, double buffered: the next tile's
//     load is in flight while the current tile looks back and emits;
//   * the chunk aggregate (the zero-state end state, Eq.10's z) is the contraction
//     w = sum_k K[k] x(k) with K[k] = A_f^(L-1-k) c (M FMA per sample, no serial
//     chain) instead of a first run of the recursion;
//   * the intra-warp carry scan runs in fp32 with paired FMAs (fma.rn.f32x2) and the
//     prologue's powers A_f^(L 2^d); the cross-tile look-back in fp64 (lti.cuh);
//   * forward emit: the TDF recursion re-run from the lane's exact carry-in (paired
//     FMA form, lti.cuh Tdf2); y is written in place and leaves by bulk row stores;
//   * backward: the adjoint state of TDF is the shift register d(n) = [g(n) ..
//     g(n+M-1)] with g(n) = dy(n) - sum_k a_k g(n+k) (Eq.7 with A_f^T = A, C_f = e1),
//     so after the carry pass A writes g over dy in shared memory and pass B (lanes
//     interleaved over the tile, coalesced global x, y reads from L2) forms
//     dx(n) = b0 dy(n) + sum_i c_i g(n+1+i) (Eq.8) and the coefficient sums of Eqs.6, 9.
//     Substituting dy(n) = g(n) + sum_k a'_k g(n+k) (the recursion itself), pass B needs
//     only g, x and y:  dx(n) = sum_{k=0..M} b'_k g(n+k)  (the adjoint of B(z)/A(z) is the
//     reverse-time all-pole followed by the FIR b'), grad_b'_k = C_k = sum_n g(n+k) x(n)
//     (k = 0..M; C_0 = Gd - sum_k a'_k Gx[k-1] of the state-space chain rule) and
//     grad_a'_k = -D_k, D_k = sum_n g(n+k) y(n) (k = 1..M).
#pragma once
#include "../../include/iirgrad.h"
#include "lti.cuh"

#ifndef IIRG_V2_NWF
#define IIRG_V2_NWF 16
#endif
#ifndef IIRG_V2_NWB
#define IIRG_V2_NWB 16
#endif
#ifndef IIRG_V2_L
#define IIRG_V2_L 32
#endif

namespace iirg {
namespace v2 {

template <int M> struct Cfg {
    static constexpr int L = IIRG_V2_L;                 // samples per lane chunk
    static constexpr int TS = 32 * L;                   // samples per warp tile
    static constexpr int MP = (M + 1) & ~1;             // order padded to a pair
    static constexpr int NPR = MP / 2;
    static constexpr int PITCH = L + 4;                 // floats per shared row (16 B pad)
    static constexpr int BUF = 32 * PITCH + 16;         // 32 chunk rows + a 16-float halo (backward)
    static constexpr int NBUF = 3;                      // buffers per warp (tile pipeline depth)
    static constexpr int r4(int n) { return (n + 3) / 4 * 4; }
    // fp32 tables, one group per direction (forward: A_f = companion(a')^T; backward: A = A_f^T):
    //   K [L][MP] | P [5][M][MP] (P[d][j][i] = X^(L 2^d)[i][j]) | b'[M+1] a'[M+1] c[M] |
    //   Q [M][NPR][32] float2 (Q[j][ip][l] = (X^(l L)[2ip][j], X^(l L)[2ip+1][j]))
    // [0, OQ) is staged in shared memory; Q (each lane reads its own matrix) is read through L1.
    static constexpr int OK_ = 0, OP = r4(L * MP), OC = OP + r4(5 * M * MP), OQ = OC + r4(3 * M + 2);
    static constexpr int STAGE = OQ;
    static constexpr int DIR = OQ + 32 * M * MP;
    static constexpr int SIZE32 = 2 * DIR;
    // fp64 tables: look-back powers A_f^(k 32^l TS) [LEVELS][M*M][32], b'[M+1], a'[M+1], a0
    static constexpr int M2 = M * M;
    static constexpr int PQ = 0, COEF = LEVELS * 32 * M2, A0 = COEF + 2 * (M + 1);
    static constexpr int SIZE64 = (A0 + 1 + 31) / 32 * 32;
    static constexpr int NG = 2 * M + 1;                 // coefficient partial sums per tile
};

constexpr int FLAT_ROWS = 64;   // sets of at most this many tile rows are finalised flat

struct FwdArgs {
    const float* x; float* y; const float* zi; float* zf;
    const float* t32; int64_t t32_stride; const double* t64; int64_t t64_stride;
    CarryWs cw;
    int64_t B, T; int ntiles; int64_t ntot; int vec;
    unsigned long long* trace;                        // debug: 8 %globaltimer stamps per tile (NULL = off)
};
struct BwdArgs {
    const float* gy; const float* gzf; const float* x; const float* y;
    float* gx; float* gzi; float* gb; float* ga; int want_coef;
    const float* t32; int64_t t32_stride; const double* t64; int64_t t64_stride;
    CarryWs cw;
    double* partial; double* partial2; unsigned* gcnt; unsigned* scnt; int64_t ncoef;
    int64_t B, T; int ntiles; int64_t ntot; int vec;
    unsigned long long* trace;
};

// Debug phase stamps (lane 0): [0] aggregate start, [1] data ready, [2] published, [3] look-back
// start, [4] carry known, [5] emit done, [6] stored, [7] warp id.
#define V2_TRACE(tr, t, k)                                                              \
    do {                                                                                \
        if ((tr) != nullptr && lane == 0) (tr)[(size_t)(t) * 8 + (k)] = gtimer();       \
    } while (0)

// One call of the engine (host side): the launch arguments of both directions.
struct Call {
    cudaStream_t st;
    const float* b; const float* a; int64_t cstride;   // raw coefficients (prologue)
    int64_t ncoef; int nlev;
    FwdArgs f;
    BwdArgs g;
};
iir_status_t run(bool fwd, int M, const Call& c);   // lti2.cu
int tile_samples(int M);
size_t tab32_floats(int M);
size_t tab64_doubles(int M);

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned long long ld2(const float* p) {
    return *reinterpret_cast<const unsigned long long*>(p);
}
template <int M>
__device__ __forceinline__ float comp(const unsigned long long (&S)[Cfg<M>::NPR], int j) {
    return (j & 1) ? hi2(S[j >> 1]) : lo2(S[j >> 1]);
}

// acc += (TR ? P^T : P) v, P = A_f^(k 32^l TS) from the fp64 look-back table (global, L1).
template <int M, bool TR>
__device__ __forceinline__ void mv_pq2(const double* __restrict__ t64, int l, int k, const double (&v)[M],
                                       double (&acc)[M]) {
    const double* P = t64 + Cfg<M>::PQ + l * 32 * M * M + k;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double s = acc[i];
#pragma unroll
        for (int j = 0; j < M; ++j) s = fma(__ldg(P + (TR ? j * M + i : i * M + j) * 32), v[j], s);
        acc[i] = s;
    }
}

// Look-back payload publication: a value equal to the all-ones sentinel (a NaN with
// the sign bit set, which a negation of the canonical NaN could produce) is published
// as the canonical NaN, so a NaN input propagates instead of never becoming ready.
template <int M>
__device__ __forceinline__ void publish2(double* dst, const double (&v)[M], int lane) {
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double x = v[i];
            if (is_sentinel(x)) x = __longlong_as_double(0x7ff8000000000000LL);
            __stcg(dst + i, x);
        }
    }
}

// Cross-tile carry of one warp tile (the hierarchical base-32 look-back of lti.cuh
// tile_carry, per warp), in two halves so that a tile's aggregate is published as soon
// as it is known, before the warp waits on the look-back of an earlier tile.
// Publication: tile jt's zero-carry aggregate G (tile 0 of a sequence folds in the
// initial state: G += Q_0 X0) goes to its level-0 slot.
template <int M, bool TR>
__device__ __forceinline__ void warp_publish(const double* __restrict__ t64, int lane, int jt, int64_t seq,
                                             const double (&X0)[M], double (&G)[M], const CarryWs& cw) {
    if (jt == 0) mv_pq2<M, TR>(t64, 0, 1, X0, G);
    publish2<M>(cw.agg[0] + (seq * cw.nblk[0] + jt) * M, G, lane);
}
// Closing publication: a tile whose lower base-32 digits are all 31 completes a block at
// every such level; right after its own aggregate (not at its later look-back) it sums the
// block's other 31 level-l aggregates, T_l = sum_{d<31} Q_l^(30-d) AGG^(l)_{32b+d}, and
// publishes the block's level-(l+1) aggregate Q_l T_l + Own_l (Own_0 = G).  Publishing at
// aggregate time keeps every level's aggregates as prompt as the tile aggregates.
template <int M, bool TR>
__device__ __forceinline__ void warp_close(const double* __restrict__ t64, int lane, int jt, int64_t seq,
                                           const double (&G)[M], const CarryWs& cw) {
    const int nl = cw.nlev;
    if (nl < 2 || (jt & 31) != 31) return;
    double Own[M];
#pragma unroll
    for (int i = 0; i < M; ++i) Own[i] = G[i];
#pragma unroll 1
    for (int l = 0; l + 1 < nl; ++l) {
        if (((jt >> (5 * l)) & 31) != 31) break;
        const int64_t blk = jt >> (5 * l);
        double Tv[M];
#pragma unroll
        for (int i = 0; i < M; ++i) Tv[i] = 0.0;
        if (lane < 31) {
            double V[M];
            const double* slot = cw.agg[l] + (seq * cw.nblk[l] + blk - 31 + lane) * M;
            load_slot<M>(slot, V);
            if (!slot_ready<M>(V)) wait_slot<M>(slot, V, cw.err);
            mv_pq2<M, TR>(t64, l, 30 - lane, V, Tv);
        }
        warp_sum<M>(Tv);
        mv_pq2<M, TR>(t64, l, 1, Tv, Own);                        // Own = Q_l T_l + Own
        publish2<M>(cw.agg[l + 1] + (seq * cw.nblk[l + 1] + (jt >> (5 * (l + 1)))) * M, Own, lane);
    }
}

// Look-back: returns in every lane the state X entering tile jt (scan order) of
// sequence seq.  With base-32 digits d_l of jt, Q_l = A_f^(32^l TS):
//   T_l = sum_{d < d_l} Q_l^(d_l - 1 - d) AGG^(l)_{(jt >> 5l) - d_l + d}     (lane d, one round trip)
//   X   = T_0 + Q_0^d_0 (T_1 + Q_1^d_1 (T_2 + ...))
// Each T_l is a fixed butterfly sum: bitwise deterministic.
template <int M, bool TR>
__device__ __forceinline__ void warp_lookback(const double* __restrict__ t64, int lane, int jt, int64_t seq,
                                              const double (&X0)[M], const CarryWs& cw, double (*sT)[M],
                                              double (&X)[M]) {
    if (jt == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) X[i] = X0[i];
        return;
    }
    const int nl = cw.nlev;
#pragma unroll 1
    for (int l = 0; l < nl; ++l) {
        const int d = (jt >> (5 * l)) & 31;
        const int64_t blk = jt >> (5 * l);
        double Tv[M];
#pragma unroll
        for (int i = 0; i < M; ++i) Tv[i] = 0.0;
        if (d > 0) {
            if (lane < d) {
                double V[M];
                const double* slot = cw.agg[l] + (seq * cw.nblk[l] + blk - d + lane) * M;
                load_slot<M>(slot, V);
                if (!slot_ready<M>(V)) wait_slot<M>(slot, V, cw.err);
                mv_pq2<M, TR>(t64, l, d - 1 - lane, V, Tv);
            }
            warp_sum<M>(Tv);
        }
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) sT[l][i] = Tv[i];
        }
    }
    __syncwarp();
    double R[M];
#pragma unroll
    for (int i = 0; i < M; ++i) R[i] = sT[nl - 1][i];
#pragma unroll 1
    for (int l = nl - 2; l >= 0; --l) {
        double R2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) R2[i] = sT[l][i];
        mv_pq2<M, TR>(t64, l, (jt >> (5 * l)) & 31, R, R2);
#pragma unroll
        for (int i = 0; i < M; ++i) R[i] = R2[i];
    }
#pragma unroll
    for (int i = 0; i < M; ++i) X[i] = R[i];
    __syncwarp();                                    // sT is reused by the warp's next tile
}

// NPR consecutive float pairs from shared memory, 128-bit loads where aligned.
template <int NPR>
__device__ __forceinline__ void ld_pairs(const float* p, unsigned long long (&o)[NPR]) {
    if constexpr (NPR % 2 == 0) {
#pragma unroll
        for (int q = 0; q < NPR / 2; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(p + 4 * q);
            o[2 * q] = pk2(v.x, v.y);
            o[2 * q + 1] = pk2(v.z, v.w);
        }
    } else {
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) o[ip] = ld2(p + 2 * ip);
    }
}

// Load the rows of one tile: lane r's row holds samples [p0 + rL, p0 + (r+1)L) of
// `src` (one sequence, length T); samples outside [0, T) (or src == NULL) read as 0.
// vec: bulk row copies on the TMA engine, completion counted on `bar`; else element
// copies by the lanes and a plain arrive.
template <int M>
__device__ __forceinline__ void load_rows(float* buf, unsigned long long* bar, const float* src, int64_t p0,
                                          int64_t T, bool vec, int lane, int rowmap) {
    using C = Cfg<M>;
    constexpr int L = C::L;
    const int r = rowmap ? 31 - lane : lane;          // any bijection: each lane fills one row
    const int64_t s = p0 + (int64_t)r * L;
    float* row = buf + r * C::PITCH;
    const int64_t lo = s > 0 ? s : 0, hi = (s + L < T) ? s + L : T;
    const bool any = src != nullptr && hi > lo;
    if (vec) {
        if (lane == 0) {
            const int64_t tlo = p0 > 0 ? p0 : 0, thi = (p0 + C::TS < T) ? p0 + C::TS : T;
            const unsigned bytes = (src != nullptr && thi > tlo) ? (unsigned)((thi - tlo) * 4) : 0u;
            mbar_arrive_expect_tx(bar, bytes);
        }
        __syncwarp();
        if (any) bulk_g2s(row + (lo - s), src + lo, (unsigned)((hi - lo) * 4), bar);
        if (!any || lo > s || hi < s + L) {
            for (int g = 0; g < L / 4; ++g) {
                const int64_t e = s + 4 * g;
                if (!any || e < lo || e >= hi) *reinterpret_cast<float4*>(row + 4 * g) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    } else {
        for (int e = 0; e < L; ++e) {
            const int64_t n = s + e;
            row[e] = (src != nullptr && n >= 0 && n < T) ? src[n] : 0.f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar);
    }
}

// w += sum_k K[k] v(k) over one chunk row (the K-form chunk aggregate).
template <int M>
__device__ __forceinline__ void chunk_aggregate(const float* row, const float* K, unsigned long long (&W)[Cfg<M>::NPR]) {
    using C = Cfg<M>;
#pragma unroll 4
    for (int g = 0; g < C::L / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(row + 4 * g);
        const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            unsigned long long Kp[C::NPR];
            ld_pairs<C::NPR>(K + (4 * g + e) * C::MP, Kp);
            const unsigned long long X = pk2(xs[e], xs[e]);
#pragma unroll
            for (int ip = 0; ip < C::NPR; ++ip) W[ip] = ffma2(Kp[ip], X, W[ip]);
        }
    }
}

// Inclusive warp scan S_l <- P^(2^d) S_(l - 2^d) + S_l (fp32, Kogge-Stone), then the
// exclusive prefix E (lane 0: zero) and the tile aggregate G (lane 31's inclusive).
template <int M>
__device__ __forceinline__ void warp_scan32(const float* P0, int lane, unsigned long long (&S)[Cfg<M>::NPR],
                                            float (&E)[M], double (&G)[M]) {
    using C = Cfg<M>;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int off = 1 << d;
        float O[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const float v = __shfl_up_sync(0xffffffffu, comp<M>(S, j), off);
            O[j] = lane >= off ? v : 0.f;
        }
        const float* P = P0 + d * M * C::MP;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const unsigned long long Oj = pk2(O[j], O[j]);
            unsigned long long Pp[C::NPR];
            ld_pairs<C::NPR>(P + j * C::MP, Pp);
#pragma unroll
            for (int ip = 0; ip < C::NPR; ++ip) S[ip] = ffma2(Pp[ip], Oj, S[ip]);
        }
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const float v = comp<M>(S, j);
        const float e = __shfl_up_sync(0xffffffffu, v, 1);
        E[j] = lane == 0 ? 0.f : e;
        G[j] = (double)__shfl_sync(0xffffffffu, v, 31);
    }
}

// State entering this lane's chunk: E + X^(lane L) X (fp32; Q from the tables).
template <int M>
__device__ __forceinline__ void lane_carry(const float* __restrict__ Q, int lane, const float (&E)[M], const double (&X)[M],
                                           float (&v)[M]) {
    using C = Cfg<M>;
    unsigned long long S[C::NPR];
#pragma unroll
    for (int ip = 0; ip < C::NPR; ++ip) S[ip] = pk2(E[2 * ip], 2 * ip + 1 < M ? E[2 * ip + 1] : 0.f);
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const float xj = (float)X[j];
        const unsigned long long Xj = pk2(xj, xj);
#pragma unroll
        for (int ip = 0; ip < C::NPR; ++ip) {
            const float2 q = __ldg(reinterpret_cast<const float2*>(Q) + (j * C::NPR + ip) * 32 + lane);
            S[ip] = ffma2(pk2(q.x, q.y), Xj, S[ip]);
        }
    }
#pragma unroll
    for (int j = 0; j < M; ++j) v[j] = comp<M>(S, j);
}

template <int M>
__device__ __forceinline__ void load_coef32(const float* tab, float (&bc)[M + 1], float (&ac)[M + 1]) {
    using C = Cfg<M>;
#pragma unroll
    for (int k = 0; k <= M; ++k) { bc[k] = tab[C::OC + k]; ac[k] = tab[C::OC + M + 1 + k]; }
}

__device__ __forceinline__ unsigned take_ticket(unsigned* ticket, int lane) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    return __shfl_sync(0xffffffffu, t, 0);
}

// ---------------------------------------------------------------------------
// Forward (a2-a4).  Per warp, a three-deep tile pipeline: while tile t0 looks back
// and emits, tile t1's aggregate is already published and tile t2 streams in, so a
// warp never holds a handed-out tile whose aggregate waits behind its own look-back.
template <int M, int NWP, bool GT>
__global__ void __launch_bounds__(NWP * 32, 1) lti2_fwd_kernel(const FwdArgs p) {
    using C = Cfg<M>;
    constexpr int L = C::L, TS = C::TS;
    extern __shared__ __align__(128) float sm2[];
    __shared__ __align__(8) unsigned long long s_bar[NWP][C::NBUF];
    __shared__ double s_T[NWP][LEVELS][M];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* bA = sm2 + (GT ? 0 : C::STAGE) + warp * C::NBUF * C::BUF;
    float* bB = bA + C::BUF;
    float* bC = bB + C::BUF;
    unsigned long long* rA = &s_bar[warp][0];
    unsigned long long* rB = &s_bar[warp][1];
    unsigned long long* rC = &s_bar[warp][2];
    unsigned pA = 0, pB = 0, pC = 0;
    if (lane == 0) { mbar_init(rA, 1); mbar_init(rB, 1); mbar_init(rC, 1); }
    mbar_fence_init();
    __syncwarp();
    // The kernel before this one on the stream is always this call's prologue, which
    // is launched WITHOUT programmatic serialization: everything enqueued before it
    // (the caller's x, the previous call's use of the workspace) completed before it
    // started.  So the workspace counters and the first x tiles are read before
    // griddepcontrol.wait; only the prologue's tables are read after it.
    CarryWs cw = p.cw;
    const unsigned ep = carry_bank(cw);
    rearm_other_bank(cw, ep, blockIdx.x, gridDim.x);
    const bool vec = p.vec != 0;
    auto issue = [&](float* buf, unsigned long long* bar, unsigned t) {
        load_rows<M>(buf, bar, p.x + (int64_t)(t % (unsigned long long)p.B) * p.T,
                     (int64_t)(t / (unsigned long long)p.B) * TS, p.T, vec, lane, 0);
    };
    unsigned t0 = take_ticket(cw.ticket, lane);
    unsigned t1 = take_ticket(cw.ticket, lane);
    unsigned t2 = take_ticket(cw.ticket, lane);
    if (t0 < p.ntot) issue(bA, rA, t0);
    if (t1 < p.ntot) issue(bB, rB, t1);
    pdl_wait();                                                  // the prologue's tables
    pdl_launch_dependents();
    if constexpr (!GT) {
        for (int i = threadIdx.x; i < C::STAGE / 4; i += blockDim.x) cp_async16_ca(sm2 + 4 * i, p.t32 + 4 * i);
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    // a2 + a3 (intra-warp) of tile t in buf, then its publication: E, G for the look-back
    auto aggregate = [&](float* buf, unsigned long long* bar, unsigned& ph, unsigned t, float (&E)[M]) {
        const int64_t seq = (int64_t)(t % (unsigned long long)p.B);
        const int jt = (int)(t / (unsigned long long)p.B);
        const float* tab = GT ? p.t32 + seq * p.t32_stride : sm2;
        double G[M];
        V2_TRACE(p.trace, t, 0);
        mbar_wait(bar, ph);
        ph ^= 1u;
        V2_TRACE(p.trace, t, 1);
        unsigned long long S[C::NPR];
#pragma unroll
        for (int ip = 0; ip < C::NPR; ++ip) S[ip] = 0ull;
        chunk_aggregate<M>(buf + lane * C::PITCH, tab + C::OK_, S);
        warp_scan32<M>(tab + C::OP, lane, S, E, G);
        double X0[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (p.zi != nullptr && jt == 0) ? (double)p.zi[seq * M + i] : 0.0;
        warp_publish<M, false>(p.t64 + seq * p.t64_stride, lane, jt, seq, X0, G, cw);
        warp_close<M, false>(p.t64 + seq * p.t64_stride, lane, jt, seq, G, cw);
        V2_TRACE(p.trace, t, 2);
    };
    float E0[M];
    if (t0 < p.ntot) aggregate(bA, rA, pA, t0, E0);
    while (t0 < p.ntot) {
        unsigned t3 = 0;
        if (lane == 0) t3 = atomicAdd(cw.ticket, 1u);             // three tiles ahead, in flight
        float E1[M];
        if (t1 < p.ntot) aggregate(bB, rB, pB, t1, E1);
        if (t2 < p.ntot) {
            bulk_wait_read0();                                   // this lane's store from bC has read it
            issue(bC, rC, t2);
        }
        const int64_t seq = (int64_t)(t0 % (unsigned long long)p.B);
        const int jt = (int)(t0 / (unsigned long long)p.B);
        const int64_t p0 = (int64_t)jt * TS;
        const float* tab = GT ? p.t32 + seq * p.t32_stride : sm2;
        float* row = bA + lane * C::PITCH;
        // a3: cross-tile carry, then the state entering this lane's chunk
        double X0[M], X[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (p.zi != nullptr && jt == 0) ? (double)p.zi[seq * M + i] : 0.0;
        V2_TRACE(p.trace, t0, 3);
        warp_lookback<M, false>(p.t64 + seq * p.t64_stride, lane, jt, seq, X0, cw, s_T[warp], X);
        V2_TRACE(p.trace, t0, 4);
        float vin[M];
        lane_carry<M>(p.t32 + seq * p.t32_stride + C::OQ, lane, E0, X, vin);
        float bc[M + 1], ac[M + 1];
        load_coef32<M>(tab, bc, ac);
        // zf = v(T): the lane holding sample T-1 (when it is not its chunk's last)
        const int64_t ez = p.T - 1 - (p0 + (int64_t)lane * L);
        if (p.zf != nullptr && ez >= 0 && ez < L - 1) {
            float w2[M];
#pragma unroll
            for (int i = 0; i < M; ++i) w2[i] = vin[i];
            for (int n = 0; n <= (int)ez; ++n) { float du; fwd_step<float, M, 1>(w2, row[n], bc, ac, du); }
#pragma unroll
            for (int i = 0; i < M; ++i) p.zf[seq * M + i] = w2[i];
        }
        // a4: re-run from the exact carry-in, y in place (paired FMAs)
        {
            Tdf2<M> c2;
            c2.init(bc, ac);
            unsigned long long VP[Tdf2<M>::NP];
            tdf2_pack<M>(vin, VP);
#pragma unroll 4
            for (int g = 0; g < L / 4; ++g) {
                float4 xv = *reinterpret_cast<const float4*>(row + 4 * g);
                tdf2_step<M>(VP, xv.x, xv.y, c2, xv.x, xv.y);
                tdf2_step<M>(VP, xv.z, xv.w, c2, xv.z, xv.w);
                *reinterpret_cast<float4*>(row + 4 * g) = xv;
            }
            if (p.zf != nullptr && ez == L - 1) {
                float v[M];
                tdf2_unpack<M>(VP, v);
#pragma unroll
                for (int i = 0; i < M; ++i) p.zf[seq * M + i] = v[i];
            }
        }
        V2_TRACE(p.trace, t0, 5);
        // store this lane's row of y
        {
            const int64_t s = p0 + (int64_t)lane * L;
            const int64_t lo = s > 0 ? s : 0, hi = (s + L < p.T) ? s + L : p.T;
            float* yrow = p.y + seq * p.T;
            if (hi > lo) {
                if (vec) {
                    fence_proxy_async();
                    bulk_s2g(yrow + lo, row + (lo - s), (unsigned)((hi - lo) * 4));
                    bulk_commit();
                } else {
                    for (int64_t n = lo; n < hi; ++n) yrow[n] = row[n - s];
                }
            }
        }
        V2_TRACE(p.trace, t0, 6);
        if (p.trace != nullptr && lane == 0) p.trace[(size_t)t0 * 8 + 7] = blockIdx.x * NWP + warp;
        // rotate the pipeline
        t0 = t1; t1 = t2; t2 = __shfl_sync(0xffffffffu, t3, 0);
#pragma unroll
        for (int i = 0; i < M; ++i) E0[i] = E1[i];
        float* tb_ = bA; bA = bB; bB = bC; bC = tb_;
        unsigned long long* tr_ = rA; rA = rB; rB = rC; rC = tr_;
        const unsigned tp_ = pA; pA = pB; pB = pC; pC = tp_;
    }
    bulk_wait0();
    cta_exit(cw, ep, gridDim.x);
}

// ---------------------------------------------------------------------------
// Backward (a5-a8).  Tiles are aligned to the END of each sequence and taken last to
// first; lane l owns chunk 31 - l of its tile (so the lane order is the scan order).
template <int M>
__device__ __forceinline__ int tidx(int e) {              // tile-local sample -> shared offset
    return (e / Cfg<M>::L) * Cfg<M>::PITCH + (e % Cfg<M>::L);
}

// Fixed-order fp64 sum of `nrows` rows of NG values (row-major, stride NG): lane l sums
// rows l, l+32, ... in increasing order, then a fixed xor butterfly; all lanes return all sums.
template <int NG>
__device__ __forceinline__ void warp_reduce_rows(const double* src, int64_t nrows, int lane, double (&out)[NG]) {
#pragma unroll
    for (int k = 0; k < NG; ++k) out[k] = 0.0;
    for (int64_t r0 = lane; r0 < nrows; r0 += 64) {
        double v0[NG], v1[NG];
        const int64_t r1 = r0 + 32;
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            v0[k] = __ldcg(src + r0 * NG + k);
            v1[k] = r1 < nrows ? __ldcg(src + r1 * NG + k) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < NG; ++k) out[k] += v0[k] + v1[k];
    }
#pragma unroll
    for (int k = 0; k < NG; ++k)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) out[k] += __shfl_xor_sync(0xffffffffu, out[k], o);
}

// a8: chain rule from the correlation sums G = [C_0 .. C_M, D_1 .. D_M] to (b, a),
// including the a0 un-normalisation (lti.cuh chain_rule):
//   gb'_k = C_k, ga'_k = -D_k;  gb = gb'/a0, ga_k = ga'_k/a0 (k >= 1), ga_0 = -(b'.gb' + a'.ga')/a0.
template <int M>
__device__ __forceinline__ void chain_rule2(const double (&G)[2 * M + 1], const double* __restrict__ t64, float* gb,
                                            float* ga) {
    using C = Cfg<M>;
    double bn[M + 1], an[M + 1];
#pragma unroll
    for (int k = 0; k <= M; ++k) { bn[k] = __ldg(t64 + C::COEF + k); an[k] = __ldg(t64 + C::COEF + M + 1 + k); }
    const double inv_a0 = 1.0 / __ldg(t64 + C::A0);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k <= M; ++k) s += bn[k] * G[k];
#pragma unroll
    for (int k = 1; k <= M; ++k) s -= an[k] * G[M + k];
    if (gb != nullptr)
#pragma unroll
        for (int k = 0; k <= M; ++k) gb[k] = (float)(G[k] * inv_a0);
    if (ga != nullptr) {
        ga[0] = (float)(-s * inv_a0);
#pragma unroll
        for (int k = 1; k <= M; ++k) ga[k] = (float)(-G[M + k] * inv_a0);
    }
}

template <int M>
__device__ __forceinline__ float4 ld_masked4(const float* row, int64_t pos, bool vec) {
    if (row == nullptr || pos + 4 <= 0) return make_float4(0.f, 0.f, 0.f, 0.f);
    if (vec && pos >= 0) return ldg_l2(reinterpret_cast<const float4*>(row + pos));
    float4 r;
    r.x = pos + 0 >= 0 ? row[pos + 0] : 0.f;
    r.y = pos + 1 >= 0 ? row[pos + 1] : 0.f;
    r.z = pos + 2 >= 0 ? row[pos + 2] : 0.f;
    r.w = pos + 3 >= 0 ? row[pos + 3] : 0.f;
    return r;
}

template <int M, int NWP, bool GT>
__global__ void __launch_bounds__(NWP * 32, 1) lti2_bwd_kernel(const BwdArgs p) {
    using C = Cfg<M>;
    constexpr int L = C::L, TS = C::TS, NG = C::NG;
    extern __shared__ __align__(128) float sm2[];
    __shared__ __align__(8) unsigned long long s_bar[NWP][C::NBUF];
    __shared__ double s_T[NWP][LEVELS][M];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* bA = sm2 + (GT ? 0 : C::STAGE) + warp * C::NBUF * C::BUF;
    float* bB = bA + C::BUF;
    float* bC = bB + C::BUF;
    unsigned long long* rA = &s_bar[warp][0];
    unsigned long long* rB = &s_bar[warp][1];
    unsigned long long* rC = &s_bar[warp][2];
    unsigned pA = 0, pB = 0, pC = 0;
    if (lane == 0) { mbar_init(rA, 1); mbar_init(rB, 1); mbar_init(rC, 1); }
    mbar_fence_init();
    __syncwarp();
    // grad_y may be written by the kernel right before this one (the caller's loss):
    // nothing is read before griddepcontrol.wait.
    pdl_wait();
    pdl_launch_dependents();
    CarryWs cw = p.cw;
    const unsigned ep = carry_bank(cw);
    if constexpr (!GT) {
        const float* src = p.t32 + C::DIR;                       // backward table group
        for (int i = threadIdx.x; i < C::STAGE / 4; i += blockDim.x) cp_async16_ca(sm2 + 4 * i, src + 4 * i);
        cp_async_commit();
    }
    rearm_other_bank(cw, ep, blockIdx.x, gridDim.x);
    const bool vec = p.vec != 0;
    const bool shared_set = p.ncoef == 1;
    auto issue = [&](float* buf, unsigned long long* bar, unsigned t) {
        const int64_t seq = (int64_t)(t % (unsigned long long)p.B);
        const int64_t p0 = p.T - (int64_t)(t / (unsigned long long)p.B + 1) * TS;
        const int64_t off = seq * p.T;
        load_rows<M>(buf, bar, p.gy == nullptr ? nullptr : p.gy + off, p0, p.T, vec, lane, 1);
        if (lane == 0 && vec) {                  // x, y are read by pass B: pull them into L2 now
            const int64_t lo = p0 > 0 ? p0 : 0;
            const unsigned bytes = (unsigned)((p0 + TS - lo) * 4);
            prefetch_l2_bulk(p.x + off + lo, bytes);
            prefetch_l2_bulk(p.y + off + lo, bytes);
        }
    };
    unsigned t0 = take_ticket(cw.ticket, lane);
    unsigned t1 = take_ticket(cw.ticket, lane);
    unsigned t2 = take_ticket(cw.ticket, lane);
    if (t0 < p.ntot) issue(bA, rA, t0);
    if (t1 < p.ntot) issue(bB, rB, t1);
    if constexpr (!GT) cp_async_wait<0>();
    __syncthreads();
    // a5 + a6 (intra-warp) of tile t, then its publication (grad_zf folded into the last tile)
    auto aggregate = [&](float* buf, unsigned long long* bar, unsigned& ph, unsigned t, float (&E)[M]) {
        const int64_t seq = (int64_t)(t % (unsigned long long)p.B);
        const int jr = (int)(t / (unsigned long long)p.B);
        const float* tab = GT ? p.t32 + seq * p.t32_stride + C::DIR : sm2;
        double G[M];
        V2_TRACE(p.trace, t, 0);
        mbar_wait(bar, ph);
        ph ^= 1u;
        V2_TRACE(p.trace, t, 1);
        unsigned long long S[C::NPR];
#pragma unroll
        for (int ip = 0; ip < C::NPR; ++ip) S[ip] = 0ull;
        chunk_aggregate<M>(buf + (31 - lane) * C::PITCH, tab + C::OK_, S);
        warp_scan32<M>(tab + C::OP, lane, S, E, G);
        double X0[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (p.gzf != nullptr && jr == 0) ? (double)p.gzf[seq * M + i] : 0.0;
        warp_publish<M, true>(p.t64 + seq * p.t64_stride, lane, jr, seq, X0, G, cw);
        warp_close<M, true>(p.t64 + seq * p.t64_stride, lane, jr, seq, G, cw);
        V2_TRACE(p.trace, t, 2);
    };
    float E0[M];
    if (t0 < p.ntot) aggregate(bA, rA, pA, t0, E0);
    while (t0 < p.ntot) {
        unsigned t3 = 0;
        if (lane == 0) t3 = atomicAdd(cw.ticket, 1u);
        float E1[M];
        if (t1 < p.ntot) aggregate(bB, rB, pB, t1, E1);
        if (t2 < p.ntot) {
            fence_proxy_async();                                 // bC's generic reads / writes before the TMA writes
            issue(bC, rC, t2);
        }
        const int64_t seq = (int64_t)(t0 % (unsigned long long)p.B);
        const int jr = (int)(t0 / (unsigned long long)p.B);      // 0 = last tile in time
        const int jt = p.ntiles - 1 - jr;
        (void)jt;
        const int64_t p0 = p.T - (int64_t)(jr + 1) * TS;          // may be < 0 (first tile in time)
        const float* tab = GT ? p.t32 + seq * p.t32_stride + C::DIR : sm2;
        const double* t64 = p.t64 + seq * p.t64_stride;
        float* row = bA + (31 - lane) * C::PITCH;
        // a6: cross-tile carry (transposed powers), seeded by grad_zf at the last tile
        double X0[M], X[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (p.gzf != nullptr && jr == 0) ? (double)p.gzf[seq * M + i] : 0.0;
        V2_TRACE(p.trace, t0, 3);
        warp_lookback<M, true>(t64, lane, jr, seq, X0, cw, s_T[warp], X);
        V2_TRACE(p.trace, t0, 4);
        float din[M];
        lane_carry<M>(p.t32 + seq * p.t32_stride + C::DIR + C::OQ, lane, E0, X, din);     // [g(e) .. g(e+M-1)], e = this chunk's right end
        float bc[M + 1], ac[M + 1];
        load_coef32<M>(tab, bc, ac);
        {
            float hv = 0.f;
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (lane == i) hv = (float)X[i];
            if (lane < 16) bA[32 * C::PITCH + lane] = hv;           // g(p0 + TS + i) = the tile's right carry
        }
        // a7 pass A: g(n) = dy(n) - sum_k a_k g(n+k), walking the chunk backwards; g over dy
        {
            float g[M];
#pragma unroll
            for (int i = 0; i < M; ++i) g[i] = din[i];
#pragma unroll 4
            for (int q = L / 4 - 1; q >= 0; --q) {
                float4 v = *reinterpret_cast<const float4*>(row + 4 * q);
                float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 3; e >= 0; --e) {
                    float acc = vs[e];
#pragma unroll
                    for (int k = M; k >= 2; --k) acc = fmaf(-ac[k], g[k - 1], acc);
                    const float gn = fmaf(-ac[1], g[0], acc);
#pragma unroll
                    for (int k = M - 1; k >= 1; --k) g[k] = g[k - 1];
                    g[0] = gn;
                    vs[e] = gn;
                }
                *reinterpret_cast<float4*>(row + 4 * q) = make_float4(vs[0], vs[1], vs[2], vs[3]);
            }
        }
        __syncwarp();
        auto gptr = [&](int e) -> const float* { return bA + tidx<M>(e); };   // row 32: the halo
        // grad_zi = d(0) = [g(0) .. g(M-1)] (Eq.9, App. A.3), read back from the tile
        if (p.gzi != nullptr && p0 <= 0 && lane < M) p.gzi[seq * M + lane] = *gptr((int)(-p0) + lane);
        // a7 pass B: dx(n) = sum_k b'_k g(n+k) and the correlation sums, lanes interleaved
        float bk[M + 1];
#pragma unroll
        for (int k = 0; k <= M; ++k) bk[k] = bc[k];
        unsigned long long CD[M];                                // (C_k, D_k), k = 1..M
#pragma unroll
        for (int i = 0; i < M; ++i) CD[i] = 0ull;
        float C0 = 0.f;
        const int64_t off = seq * p.T;
        const float* xrow = p.x + off;
        const float* yrow = p.y + off;
        float* gxrow = p.gx == nullptr ? nullptr : p.gx + off;
#pragma unroll 2
        for (int k = 0; k < TS / 128; ++k) {
            const int n0 = 4 * (lane + 32 * k);
            const int64_t pos = p0 + n0;
            const float4 xv = ld_masked4<M>(xrow, pos, vec);
            const float4 yv = ld_masked4<M>(yrow, pos, vec);
            float gw[12];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const float4 t = *reinterpret_cast<const float4*>(gptr(n0 + 4 * q));
                gw[4 * q] = t.x; gw[4 * q + 1] = t.y; gw[4 * q + 2] = t.z; gw[4 * q + 3] = t.w;
            }
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w}, ys[4] = {yv.x, yv.y, yv.z, yv.w};
            float dx[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float d = bk[0] * gw[e];
#pragma unroll
                for (int k2 = 1; k2 <= M; ++k2) d = fmaf(bk[k2], gw[e + k2], d);
                dx[e] = d;
                C0 = fmaf(gw[e], xs[e], C0);
                const unsigned long long XY = pk2(xs[e], ys[e]);
#pragma unroll
                for (int i = 0; i < M; ++i) CD[i] = ffma2(pk2(gw[e + 1 + i], gw[e + 1 + i]), XY, CD[i]);
            }
            if (gxrow != nullptr) {
                if (vec && pos >= 0) stg_stream(reinterpret_cast<float4*>(gxrow + pos), make_float4(dx[0], dx[1], dx[2], dx[3]));
                else
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (pos + e >= 0) gxrow[pos + e] = dx[e];
            }
        }
        V2_TRACE(p.trace, t0, 5);
        // a8: per-tile row of the coefficient partial sums (fixed order), group / set finalize
        if (p.want_coef) {
            __syncwarp();
            float* scr = bA + lane * C::PITCH;                    // bA is free now: lane rows as scratch
            scr[0] = C0;
#pragma unroll
            for (int i = 0; i < M; ++i) { scr[1 + i] = lo2(CD[i]); scr[M + 1 + i] = hi2(CD[i]); }
            __syncwarp();
            double colsum = 0.0;
            if (lane < NG)
                for (int r = 0; r < 32; ++r) colsum += (double)bA[r * C::PITCH + lane];
            const int64_t per_set = shared_set ? p.ntot : p.ntiles;
            const int64_t cset = shared_set ? 0 : seq;
            const int64_t li = shared_set ? (int64_t)t0 : jr;
            double* part = p.partial + cset * per_set * NG;
            const bool flat = per_set <= FLAT_ROWS;
            const int64_t ngroups = (per_set + 31) >> 5;
            const int64_t gi = li >> 5;
            const int gsize = (int)((per_set - (gi << 5)) < 32 ? (per_set - (gi << 5)) : 32);
            double* part2 = p.partial2 + cset * ngroups * NG;
            if (lane < NG) __stcg(part + li * NG + lane, colsum);
            __threadfence();
            __syncwarp();
            unsigned fin = 0;
            if (lane == 0) {
                if (flat) fin = (atomicAdd(p.scnt + cset, 1u) == (unsigned)per_set - 1u) ? 2u : 0u;
                else fin = (atomicAdd(p.gcnt + cset * ngroups + gi, 1u) == (unsigned)gsize - 1u) ? 1u : 0u;
            }
            fin = __shfl_sync(0xffffffffu, fin, 0);
            if (fin == 1u) {                                  // last tile of its group: reduce the group
                __threadfence();
                double gs[NG];
                warp_reduce_rows<NG>(part + (gi << 5) * NG, gsize, lane, gs);
#pragma unroll
                for (int k = 0; k < NG; ++k)
                    if (lane == k) __stcg(part2 + gi * NG + k, gs[k]);
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    p.gcnt[cset * ngroups + gi] = 0u;
                    fin = (atomicAdd(p.scnt + cset, 1u) == (unsigned)ngroups - 1u) ? 3u : 0u;
                }
                fin = __shfl_sync(0xffffffffu, fin, 0);
            }
            if (fin >= 2u) {                                  // last of the set: final sum + chain rule
                __threadfence();
                double gs[NG];
                if (fin == 2u) warp_reduce_rows<NG>(part, per_set, lane, gs);
                else warp_reduce_rows<NG>(part2, ngroups, lane, gs);
                if (lane == 0) {
                    chain_rule2<M>(gs, t64, p.gb == nullptr ? nullptr : p.gb + cset * (M + 1),
                                   p.ga == nullptr ? nullptr : p.ga + cset * (M + 1));
                    p.scnt[cset] = 0u;
                }
            }
        }
        V2_TRACE(p.trace, t0, 6);
        if (p.trace != nullptr && lane == 0) p.trace[(size_t)t0 * 8 + 7] = blockIdx.x * NWP + warp;
        // rotate the pipeline
        t0 = t1; t1 = t2; t2 = __shfl_sync(0xffffffffu, t3, 0);
#pragma unroll
        for (int i = 0; i < M; ++i) E0[i] = E1[i];
        __syncwarp();
        float* tb_ = bA; bA = bB; bB = bC; bC = tb_;
        unsigned long long* tr_ = rA; rA = rB; rB = rC; rC = tr_;
        const unsigned tp_ = pA; pA = pB; pB = pC; pC = tp_;
    }
    cta_exit(cw, ep, gridDim.x);
}

// ---------------------------------------------------------------------------
// a1: prologue (one CTA per coefficient set, fp64): normalise by a0, A_f = companion(a')^T,
// the chunk weights K, the scan powers, the lane powers and the look-back powers.  Every
// table comes from powers built by batched doubling (about 6 + 5 + 5 nlev dependent
// rounds of independent M x M products), so the prologue is a few microseconds.
template <int M> struct Prep2Slots {
    static constexpr int L = Cfg<M>::L;
    static constexpr int SP = 0 /* L+1: A_f^m */, SL = SP + L + 1 /* 33: A_f^(l L) */, SQ = SL + 33 /* LEVELS x 33 */;
    static constexpr int N = SQ + LEVELS * 33;
    static constexpr size_t bytes() { return (size_t)N * M * M * sizeof(double); }
};

template <int M>
__global__ void __launch_bounds__(256) lti2_prep_kernel(const float* __restrict__ b, const float* __restrict__ a,
                                                       int64_t coef_stride, float* __restrict__ t32,
                                                       int64_t t32_stride, double* __restrict__ t64,
                                                       int64_t t64_stride, int nlev) {
    pdl_launch_dependents();
    using C = Cfg<M>;
    using S = Prep2Slots<M>;
    constexpr int L = C::L, M2 = M * M, MP = C::MP, NPR = C::NPR;
    extern __shared__ __align__(16) unsigned char prep2_raw[];
    double* mat = reinterpret_cast<double*>(prep2_raw);
    __shared__ double bn[M + 1], an[M + 1], cv[M];
    const int set = blockIdx.x, tid = threadIdx.x;
    const float* bb = b + set * coef_stride;
    const float* aa = a + set * coef_stride;
    float* o32 = t32 + set * t32_stride;
    double* o64 = t64 + set * t64_stride;
    if (tid <= M) {
        const double a0 = (double)aa[0];
        bn[tid] = (double)bb[tid] / a0;
        an[tid] = (double)aa[tid] / a0;
    }
    __syncthreads();
    if (tid < M) cv[tid] = bn[tid + 1] - an[tid + 1] * bn[0];
    for (int e = tid; e < M2; e += 256) {
        const int i = e / M, j = e % M;
        mat[(S::SP + 1) * M2 + e] = (j == 0 ? -an[i + 1] : 0.0) + (j == i + 1 ? 1.0 : 0.0);   // A_f[i][j]
        const double id = (i == j) ? 1.0 : 0.0;
        mat[(S::SP + 0) * M2 + e] = id;
        mat[(S::SL + 0) * M2 + e] = id;
        for (int l = 0; l < LEVELS; ++l) mat[(S::SQ + l * 33) * M2 + e] = id;
    }
    __syncthreads();
    auto mm_batch = [&](int n, auto dst, auto lhs, auto rhs) {
        constexpr int R = (32 * M2 + 255) / 256;
        double rr[R];
#pragma unroll
        for (int s = 0; s < R; ++s) {
            const int w = tid + s * 256;
            rr[s] = 0.0;
            if (w < n * M2) {
                const int q = w / M2, e = w % M2, i = e / M, j = e % M;
                const double* A = mat + lhs(q) * M2;
                const double* B = mat + rhs(q) * M2;
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(A[i * M + k], B[k * M + j], acc);
                rr[s] = acc;
            }
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < R; ++s) {
            const int w = tid + s * 256;
            if (w < n * M2) mat[dst(w / M2) * M2 + (w % M2)] = rr[s];
        }
        __syncthreads();
    };
    // slot0 = X^0, slot0 + 1 = X^1 known: fill X^2 .. X^(2^rounds)
    auto powers = [&](int slot0, int rounds) {
        for (int st = 0; st < rounds; ++st) {
            const int h = 1 << st;
            mm_batch(h, [&](int q) { return slot0 + h + 1 + q; }, [&](int) { return slot0 + h; },
                     [&](int q) { return slot0 + 1 + q; });
        }
    };
    auto copy = [&](int dst, int src) {
        for (int e = tid; e < M2; e += 256) mat[dst * M2 + e] = mat[src * M2 + e];
        __syncthreads();
    };
    constexpr int LOG_L = L == 64 ? 6 : L == 32 ? 5 : L == 128 ? 7 : 0;
    static_assert(LOG_L > 0, "chunk length must be 32, 64 or 128");
    powers(S::SP, LOG_L);                                              // A_f^m, m = 0..L
    copy(S::SL + 1, S::SP + L);
    powers(S::SL, 5);                                                  // A_f^(l L), l = 0..32
    copy(S::SQ + 1, S::SL + 32);                                       // A_f^TS
    for (int l = 0; l < nlev; ++l) {
        powers(S::SQ + l * 33, 5);                                     // A_f^(k 32^l TS), k = 0..32
        if (l + 1 < LEVELS) copy(S::SQ + (l + 1) * 33 + 1, S::SQ + l * 33 + 32);
    }
    // chunk weights: KF[k] = A_f^(L-1-k) c (forward), KB[k] = (A_f^T)^k e1 = row 0 of A_f^k (backward)
    for (int w = tid; w < L * MP; w += 256) {
        const int k = w / MP, i = w % MP;
        float kf = 0.f, kb = 0.f;
        if (i < M) {
            const double* X = mat + (S::SP + L - 1 - k) * M2;
            double s = 0.0;
            for (int j = 0; j < M; ++j) s = fma(X[i * M + j], cv[j], s);
            kf = (float)s;
            kb = (float)mat[(S::SP + k) * M2 + i];
        }
        o32[C::OK_ + w] = kf;
        o32[C::DIR + C::OK_ + w] = kb;
    }
    // fp32 tables: P (scan powers) and Q (lane powers), forward (A_f) and backward (A_f^T)
    for (int w = tid; w < 5 * M * MP; w += 256) {
        const int d = w / (M * MP), j = (w / MP) % M, i = w % MP;
        const double* X = mat + (S::SL + (1 << d)) * M2;
        o32[C::OP + w] = i < M ? (float)X[i * M + j] : 0.f;
        o32[C::DIR + C::OP + w] = i < M ? (float)X[j * M + i] : 0.f;
    }
    for (int w = tid; w < 32 * M * NPR; w += 256) {
        const int l = w % 32, ip = (w / 32) % NPR, j = w / (32 * NPR);
        const double* X = mat + (S::SL + l) * M2;
        const int i0 = 2 * ip, i1 = 2 * ip + 1;
        o32[C::OQ + 2 * w] = (float)X[i0 * M + j];
        o32[C::OQ + 2 * w + 1] = i1 < M ? (float)X[i1 * M + j] : 0.f;
        o32[C::DIR + C::OQ + 2 * w] = (float)X[j * M + i0];
        o32[C::DIR + C::OQ + 2 * w + 1] = i1 < M ? (float)X[j * M + i1] : 0.f;
    }
    if (tid <= M) {
        for (int g = 0; g < 2; ++g) {
            o32[g * C::DIR + C::OC + tid] = (float)bn[tid];
            o32[g * C::DIR + C::OC + M + 1 + tid] = (float)an[tid];
            if (tid < M) o32[g * C::DIR + C::OC + 2 * (M + 1) + tid] = (float)cv[tid];
        }
        o64[C::COEF + tid] = bn[tid];
        o64[C::COEF + M + 1 + tid] = an[tid];
        if (tid == 0) o64[C::A0] = (double)aa[0];
    }
    for (int w = tid; w < nlev * 32 * M2; w += 256) {
        const int l = w / (32 * M2), rr = w % (32 * M2), e = rr / 32, k = rr % 32;
        o64[C::PQ + w] = mat[(S::SQ + l * 33 + k) * M2 + e];
    }
}

}  // namespace v2
}  // namespace iirg
