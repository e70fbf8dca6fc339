// lti2.cuh -- round-2 LTI engine for fp32 TDF-II filtering and its closed-form
// backward (arXiv 2511.14390, Eqs.4-9; the BASELINE configs C2, C4, C5).
//
// Same method as lti.cuh (the chunked scan of Eq.10, with a
// deterministic hierarchical look-back across tiles), re-laid out for sm_100a as
// PERSISTENT WARP TILES:
//   * a tile is 32 lane chunks of L samples of one sequence, owned by ONE warp (no
//     block-level scan, no __syncthreads on the per-tile path).  The grid is one
//     resident wave; warp w of the grid takes tiles w, w + W, w + 2W, ... (W warps in the
//     grid; tile t = time tile t / B of sequence t % B), so every tile a warp waits for
//     belongs to a resident warp that reaches it first;
//   * each lane's chunk arrives by one cp.async.bulk row copy (TMA engine, mbarrier
//     completion) into a 16 B-padded shared row;
//   * the chunk aggregate (the zero-state end state, Eq.10's z) is the contraction
//     w = sum_k K[k] x(k) with K[k] = A_f^(L-1-k) c (M FMA per sample, no serial
//     chain) instead of a first run of the recursion;
//   * the intra-warp carry scan runs with paired fp32 FMAs (fma.rn.f32x2) and the
//     prologue's powers A_f^(L 2^d); the cross-tile look-back combines the predecessors'
//     published aggregates in fp32 with per-lane power tables (lane l: A_f^(l 32^v TS));
//   * tile pipeline per warp: tile t1's aggregate is computed and published BEFORE the
//     warp waits on tile t0's look-back, and t0's input is parked in tensor memory
//     (TMEM, 256 KB per SM, unused otherwise) between its aggregate and its emit, so a
//     warp needs only one incoming shared buffer;
//   * forward emit: the TDF recursion re-run from the lane's exact carry-in (paired FMA
//     form, lti.cuh Tdf2) on x read back from TMEM; y leaves by bulk row stores;
//   * backward: the adjoint state of TDF is the shift register d(n) = [g(n) ..
//     g(n+M-1)] with g(n) = dy(n) - sum_k a'_k g(n+k) (Eq.7 with A_f^T = A, C_f = e1).
//     Substituting dy(n) = g(n) + sum_k a'_k g(n+k) into Eq.8 and Eqs.6, 9 gives
//       dx(n) = sum_{k=0..M} b'_k g(n+k)            (reverse-time all-pole, then FIR b'),
//       grad_b'_k = C_k = sum_n g(n+k) x(n) (k = 0..M),   grad_a'_k = -D_k = -sum_n g(n+k) y(n),
//     so one fused pass per lane (dy from TMEM, x and y by TMA rows) produces g, dx and the
//     correlation sums with g(n..n+M) in registers.
#pragma once
#include "../../include/iirgrad.h"
#include "lti.cuh"

#ifndef IIRG_V2_NWF
#define IIRG_V2_NWF 12
#endif
#ifndef IIRG_V2_NWB
#define IIRG_V2_NWB 8
#endif
#ifndef IIRG_V2_L
#define IIRG_V2_L 64
#endif

namespace iirg {
namespace v2 {

template <int M> struct Cfg {
    static constexpr int L = IIRG_V2_L;                 // samples per lane chunk
    static constexpr int TS = 32 * L;                   // samples per warp tile
    static constexpr int MP = (M + 1) & ~1;             // order padded to a pair
    static constexpr int NPR = MP / 2;
    static constexpr int PITCH = L + 4;                 // floats per shared row (16 B pad)
    static constexpr int BUF = 32 * PITCH;              // 32 chunk rows
    static constexpr int r4(int n) { return (n + 3) / 4 * 4; }
    // fp32 tables, one group per direction (forward: X = A_f = companion(a')^T; backward:
    // X = A = A_f^T):
    //   K [L][MP] | P [5][M][MP] (P[d][j][i] = X^(L 2^d)[i][j]) | b'[M+1] a'[M+1] c[M] |
    //   Q  [M][NPR][32] float2: Q[j][ip][l]    = (X^(l L)[2ip][j], X^(l L)[2ip+1][j])
    //   PQ [LEVELS][M][NPR][32] float2: PQ[v][j][ip][k] = the same pairs of X^(k 32^v TS)
    // [0, OQ) is staged in shared memory (broadcast reads); Q and PQ (each lane reads its
    // own matrix) are read through L1.
    // | W: coefficient pairs (JP of each, float2; na = -a', zero outside 0..M), read as pairs
    //   so the hot loops never rebuild them: forward group, the Tdf2 pairs B2, NA2, B1, NA1;
    //   backward group (a7): (na_2j+1, na_2j+2), (na_2j+2, na_2j+3), (b'_2j, b'_2j+1), (b'_2j-1, b'_2j)
    static constexpr int JP = (M + 1) / 2 + 1;
    static constexpr int OK_ = 0, OP = r4(L * MP), OC = OP + r4(5 * M * MP), OW = OC + r4(3 * M + 2);
    static constexpr int OQ = OW + r4(8 * JP);
    static constexpr int OPQ = OQ + 32 * M * MP;
    static constexpr int STAGE = OQ;
    static constexpr int DIR = OPQ + LEVELS * 32 * M * MP;
    static constexpr int SIZE32 = 2 * DIR;
    // fp64: b'[M+1], a'[M+1], a0 (the chain rule of the gradient finalize)
    static constexpr int COEF = 0, A0 = 2 * (M + 1);
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
    int gy_early;                                     // IIR_FLAG_GRAD_Y_EARLY: grad_y / grad_zf complete before the forward
};

// Debug phase stamps (lane 0): [0] aggregate start, [1] data ready, [2] published, [3] look-back
// start, [4] carry known, [5] emit done, [6] stored, [7] warp id.
#define V2_TRACE(tr, t, k)                                                              \
    do {                                                                                \
        if ((tr) != nullptr && lane == 0) (tr)[(size_t)(t) * 8 + (k)] = gtimer();       \
    } while (0)

// Debug CTA stamps (thread 0 of the CTA): [0] entry, [1] setup done, [2] tiles done,
// [3] finalize done, stored after the tile stamps at (ntot + cta) * 8.
#define V2_CTA_TRACE(tr, ntot, k)                                                       \
    do {                                                                                \
        if ((tr) != nullptr && threadIdx.x == 0)                                        \
            (tr)[((size_t)(ntot) + blockIdx.x) * 8 + (k)] = gtimer();                   \
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
template <int NPR>
__device__ __forceinline__ float comp(const unsigned long long (&S)[NPR], int j) {
    return (j & 1) ? hi2(S[j >> 1]) : lo2(S[j >> 1]);
}
template <int M, int NPR>
__device__ __forceinline__ void pack_pairs(const float (&v)[M], unsigned long long (&o)[NPR]) {
#pragma unroll
    for (int ip = 0; ip < NPR; ++ip) o[ip] = pk2(v[2 * ip], 2 * ip + 1 < M ? v[2 * ip + 1] : 0.f);
}
template <int M, int NPR>
__device__ __forceinline__ void unpack_pairs(const unsigned long long (&S)[NPR], float (&v)[M]) {
#pragma unroll
    for (int j = 0; j < M; ++j) v[j] = comp<NPR>(S, j);
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

// ---------------------------------------------------------------------------
// Static persistent schedule: warp w of W takes tiles w, w + W, ...; (seq, j) of tile t =
// (t % B, t / B) are advanced incrementally (no division per tile).
struct Sched {
    unsigned t; int64_t seq; int j;
    unsigned W; int dj; int64_t ds, B;
    __device__ __forceinline__ void init(unsigned t0, unsigned nw, int64_t b) {
        W = nw; B = b;
        t = t0; seq = (int64_t)(t0 % (unsigned long long)b); j = (int)(t0 / (unsigned long long)b);
        dj = (int)(nw / (unsigned long long)b); ds = (int64_t)(nw % (unsigned long long)b);
    }
    __device__ __forceinline__ void next() {
        t += W; seq += ds; j += dj;
        if (seq >= B) { seq -= B; ++j; }
    }
};

// ---------------------------------------------------------------------------
// Cross-tile carry in fp32.  Look-back slots hold M floats (all-ones = not published;
// 4-byte stores and loads are single-copy atomic, a reader re-polls until no element is
// the sentinel).  A value equal to the sentinel (a NaN with the sign bit set) is
// published as the canonical NaN, so a NaN input propagates instead of looking unpublished.
__device__ __forceinline__ float ld_vol_f32(const float* p) {
    float v;
    asm volatile("ld.volatile.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ bool sent32(float v) { return __float_as_uint(v) == 0xffffffffu; }
template <int M>
__device__ __forceinline__ void slot_load(const float* src, float (&v)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = ld_vol_f32(src + i);
}
template <int M>
__device__ __forceinline__ bool slot_ok(const float (&v)[M]) {
    bool r = true;
#pragma unroll
    for (int i = 0; i < M; ++i) r = r && !sent32(v[i]);
    return r;
}
// A slot that is never published (a scheduling fault, e.g. CTAs that cannot all be
// resident) does not hang or trap: after 2 s the waiter sets the workspace error word
// (iir_check_workspace) and continues with NaN.
template <int M>
__device__ __forceinline__ void slot_wait(const float* src, float (&v)[M], unsigned* err) {
    unsigned ns = 32;
    unsigned long long t0 = 0;
    for (;;) {
        __nanosleep(ns);
        slot_load<M>(src, v);
        if (slot_ok<M>(v)) return;
        if (ns < 256) ns *= 2;
        else {
            const unsigned long long now = gtimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 2000000000ull) {
                if (err != nullptr) atomicOr(err, 1u);
#pragma unroll
                for (int i = 0; i < M; ++i) v[i] = __uint_as_float(0x7fc00000u);
                return;
            }
        }
    }
}
template <int M>
__device__ __forceinline__ void slot_publish(float* dst, const float (&v)[M], int lane) {
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) __stcg(dst + i, sent32(v[i]) ? __uint_as_float(0x7fc00000u) : v[i]);
    }
}
template <int M>
__device__ __forceinline__ float* slot_ptr(const CarryWs& cw, int64_t boff, int lev, int64_t seq, int64_t blk) {
    return reinterpret_cast<float*>(cw.agg[lev] + boff) + (seq * cw.nblk[lev] + blk) * M;
}

// acc += Y v with Y = matrix k of a pair table [j][ip][32] (k = lane: each lane its own
// matrix, coalesced; k uniform: broadcast).
template <int M>
__device__ __forceinline__ void mvp(const float* __restrict__ Y, int k, const float (&v)[M],
                                    unsigned long long (&acc)[Cfg<M>::NPR]) {
    constexpr int NPR = Cfg<M>::NPR;
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const unsigned long long Vj = pk2(v[j], v[j]);
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) {
            const float2 q = __ldg(reinterpret_cast<const float2*>(Y) + (j * NPR + ip) * 32 + k);
            acc[ip] = ffma2(pk2(q.x, q.y), Vj, acc[ip]);
        }
    }
}
// Sum over the warp by a fixed xor butterfly: every lane ends with bitwise the same sum
// (each step adds the same two values in both partner lanes).
template <int NPR>
__device__ __forceinline__ void warp_sum2(unsigned long long (&a)[NPR]) {
    const unsigned long long ONE = pk2(1.f, 1.f);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) {
            const float lo = __shfl_xor_sync(0xffffffffu, lo2(a[ip]), o);
            const float hi = __shfl_xor_sync(0xffffffffu, hi2(a[ip]), o);
            a[ip] = ffma2(ONE, pk2(lo, hi), a[ip]);
        }
}

// Publication of tile jt's zero-carry aggregate G (tile 0 of a sequence folds in the
// initial state: G += Y_0^1 X0), then, for a tile whose lower base-32 digits are all 31,
// the aggregates of the blocks it closes: T_v = sum_{l<31} Y_v^l AGG^(v)_{blk-1-l} over the
// block's other 31 members and AGG^(v+1) = Y_v T_v + Own_v (Own_0 = G).  Publishing at
// aggregate time keeps every level as prompt as the tile aggregates.
template <int M>
__device__ __forceinline__ void carry_publish(const float* __restrict__ PQ, int lane, int jt, int64_t seq,
                                              const float (&X0)[M], float (&G)[M], const CarryWs& cw,
                                              int64_t boff) {
    constexpr int NPR = Cfg<M>::NPR, LV = 32 * M * Cfg<M>::MP;
    if (jt == 0) {
        unsigned long long G2[NPR];
        pack_pairs<M, NPR>(G, G2);
        mvp<M>(PQ, 1, X0, G2);
        unpack_pairs<M, NPR>(G2, G);
    }
    slot_publish<M>(slot_ptr<M>(cw, boff, 0, seq, jt), G, lane);
    const int nl = cw.nlev;
    if (nl < 2 || (jt & 31) != 31) return;
    float Own[M];
#pragma unroll
    for (int i = 0; i < M; ++i) Own[i] = G[i];
#pragma unroll 1
    for (int v = 0; v + 1 < nl; ++v) {
        if (((jt >> (5 * v)) & 31) != 31) break;
        const int64_t blk = jt >> (5 * v);
        float V[M];
#pragma unroll
        for (int i = 0; i < M; ++i) V[i] = 0.f;
        if (lane < 31) {
            const float* sp = slot_ptr<M>(cw, boff, v, seq, blk - 1 - lane);
            slot_load<M>(sp, V);
            if (!slot_ok<M>(V)) slot_wait<M>(sp, V, cw.err);
        }
        __syncwarp();
        unsigned long long T2[NPR];
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) T2[ip] = 0ull;
        mvp<M>(PQ + v * LV, lane, V, T2);
        warp_sum2<NPR>(T2);
        float T[M];
        unpack_pairs<M, NPR>(T2, T);
        unsigned long long O2[NPR];
        pack_pairs<M, NPR>(Own, O2);
        mvp<M>(PQ + v * LV, 1, T, O2);                              // Own = Y_v T_v + Own
        unpack_pairs<M, NPR>(O2, Own);
        slot_publish<M>(slot_ptr<M>(cw, boff, v + 1, seq, jt >> (5 * (v + 1))), Own, lane);
    }
}

// Look-back: the state X entering tile jt (scan order) of sequence seq, in every lane.
// With base-32 digits d_v of jt and Y_v = X^(32^v TS):
//   T_v = sum_{l < d_v} Y_v^l AGG^(v)_{(jt >> 5v) - 1 - l}         (lane l, one round trip)
//   X   = T_0 + Y_0^d_0 (T_1 + Y_1^d_1 (T_2 + ...))
// Fixed combination order (per-lane products, a fixed butterfly): bitwise deterministic.
// Level-0 slot of tile jt's look-back, loaded ahead of time (issued before the warp's next
// aggregate so the L2 round trip overlaps it; re-polled in carry_lookback if it was not yet
// published).  Lanes without a slot hold zeros.
template <int M>
__device__ __forceinline__ void lookback_prefetch(int lane, int jt, int64_t seq, const CarryWs& cw, int64_t boff,
                                                  float (&V)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) V[i] = 0.f;
    if (jt > 0 && lane < (jt & 31)) slot_load<M>(slot_ptr<M>(cw, boff, 0, seq, jt - 1 - lane), V);
}
template <int M>
__device__ __forceinline__ void carry_lookback(const float* __restrict__ PQ, int lane, int jt, int64_t seq,
                                               const float (&X0)[M], const CarryWs& cw, int64_t boff,
                                               float (*sT)[M],
                                               float (&X)[M], const float (*V0pre)[M] = nullptr) {
    constexpr int NPR = Cfg<M>::NPR, LV = 32 * M * Cfg<M>::MP;
    if (jt == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) X[i] = X0[i];
        return;
    }
    const int nl = cw.nlev;
#pragma unroll 1
    for (int v = 0; v < nl; ++v) {
        const int d = (jt >> (5 * v)) & 31;
        const int64_t blk = jt >> (5 * v);
        float V[M];
#pragma unroll
        for (int i = 0; i < M; ++i) V[i] = 0.f;
        if (lane < d) {
            const float* sp = slot_ptr<M>(cw, boff, v, seq, blk - 1 - lane);
            if (v == 0 && V0pre != nullptr) {
#pragma unroll
                for (int i = 0; i < M; ++i) V[i] = (*V0pre)[i];
            } else {
                slot_load<M>(sp, V);
            }
            if (!slot_ok<M>(V)) slot_wait<M>(sp, V, cw.err);
        }
        __syncwarp();
        unsigned long long T2[NPR];
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) T2[ip] = 0ull;
        mvp<M>(PQ + v * LV, lane, V, T2);
        warp_sum2<NPR>(T2);
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) sT[v][i] = comp<NPR>(T2, i);
        }
    }
    __syncwarp();
    float R[M];
#pragma unroll
    for (int i = 0; i < M; ++i) R[i] = sT[nl - 1][i];
#pragma unroll 1
    for (int v = nl - 2; v >= 0; --v) {
        unsigned long long R2[NPR];
        float Tv[M];
#pragma unroll
        for (int i = 0; i < M; ++i) Tv[i] = sT[v][i];
        pack_pairs<M, NPR>(Tv, R2);
        mvp<M>(PQ + v * LV, (jt >> (5 * v)) & 31, R, R2);
        unpack_pairs<M, NPR>(R2, R);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) X[i] = R[i];
    __syncwarp();                                                    // sT is reused by the warp's next tile
}

// Re-arm the bank the previous call used (cw unshifted; boff = this call's bank offset).
__device__ __forceinline__ void rearm_other_bank2(const CarryWs& cw, int64_t boff, unsigned cta, unsigned nctas) {
    double* other = cw.agg[0] + (boff != 0 ? 0 : cw.bank);
    for (int64_t i = (int64_t)cta * blockDim.x + threadIdx.x; i < cw.bank; i += (int64_t)nctas * blockDim.x)
        __stcg(other + i, sentinel());
}

template <int N, int I = 0, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<N, I + 1>(f);
    }
}

// ---------------------------------------------------------------------------
// Load the rows of one tile: row r holds samples [p0 + rL, p0 + (r+1)L) of `src` (one
// sequence, length T); samples outside [0, T) (or src == NULL) read as 0.
// vec (rows 16 B aligned, T % 4 == 0): the warp copies the tile's 2048 samples as 512
// coalesced 16-byte cp.async chunks (chunk c -> row c / (L/4), column 4 (c % (L/4)): each
// warp instruction moves 512 contiguous bytes), zero-filling the chunks outside [0, T); the
// copies complete on `bar` (every lane's cp.async.mbarrier.arrive; `arm`: lane 0's plain
// arrive after the whole warp has issued, so with several streams on one barrier the
// arming call comes LAST).  Without vec: element copies by the lanes (lane l fills row l,
// or 31 - l for rowmap 1) and (arm) a plain arrive.
template <int M>
__device__ __forceinline__ void load_rows(float* buf, unsigned long long* bar, const float* src, int64_t p0,
                                          int64_t T, bool vec, int lane, int rowmap, bool arm = true) {
    using C = Cfg<M>;
    constexpr int L = C::L, CPR = L / 4;
    static_assert(32 % CPR == 0, "whole rows per warp instruction");
    if (vec) {
        if (src != nullptr && p0 >= 0 && p0 + C::TS <= T) {        // interior tile: immediate offsets
            const unsigned sb = smem_u32(buf + (lane / CPR) * C::PITCH + 4 * (lane % CPR));
            const float* g = src + p0 + 4 * lane;
            static_for<CPR>([&](auto ic) {
                constexpr int i = decltype(ic)::value;
                asm volatile("cp.async.cg.shared.global [%0+%2], [%1+%3], 16;"
                             :: "r"(sb), "l"(g), "n"(i * (32 / CPR) * C::PITCH * 4), "n"(i * 512) : "memory");
            });
            cp_async_mbar_arrive(bar);
        } else if (src != nullptr) {
#pragma unroll 4
            for (int i = 0; i < CPR; ++i) {
                const int ci = 32 * i + lane;
                const int64_t n = p0 + 4 * (int64_t)ci;
                const bool in = n >= 0 && n < T;
                cp_async16(buf + (ci / CPR) * C::PITCH + 4 * (ci % CPR), in ? src + n : src, in ? 16u : 0u);
            }
            cp_async_mbar_arrive(bar);
        } else {
#pragma unroll
            for (int i = 0; i < CPR; ++i) {
                const int ci = 32 * i + lane;
                *reinterpret_cast<float4*>(buf + (ci / CPR) * C::PITCH + 4 * (ci % CPR)) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncwarp();
        if (arm && lane == 0) mbar_arrive(bar);
    } else {
        const int r = rowmap ? 31 - lane : lane;
        const int64_t s = p0 + (int64_t)r * L;
        float* row = buf + r * C::PITCH;
#pragma unroll 1
        for (int e = 0; e < L; ++e) {
            const int64_t n = s + e;
            row[e] = (src != nullptr && n >= 0 && n < T) ? src[n] : 0.f;
        }
        __syncwarp();
        if (arm && lane == 0) mbar_arrive(bar);
    }
}

// Store the rows of one tile (the inverse of load_rows; samples outside [0, T) dropped).
// vec: coalesced 16-byte stores by the whole warp after a __syncwarp (every lane's row is
// complete); otherwise lane l stores row l (rowmap 0) or 31 - l (rowmap 1).
template <int M>
__device__ __forceinline__ void store_rows(const float* buf, float* dst, int64_t p0, int64_t T, bool vec, int lane,
                                           int rowmap) {
    using C = Cfg<M>;
    constexpr int L = C::L, CPR = L / 4;
    static_assert(32 % CPR == 0, "whole rows per warp instruction");
    if (vec && p0 >= 0 && p0 + C::TS <= T) {                    // interior tile
        __syncwarp();
        const float* sb = buf + (lane / CPR) * C::PITCH + 4 * (lane % CPR);
        float* g = dst + p0 + 4 * lane;
#pragma unroll
        for (int i = 0; i < CPR; ++i)
            *reinterpret_cast<float4*>(g + 128 * i) = *reinterpret_cast<const float4*>(sb + i * (32 / CPR) * C::PITCH);
    } else if (vec) {
        __syncwarp();
#pragma unroll 4
        for (int i = 0; i < CPR; ++i) {
            const int ci = 32 * i + lane;
            const int64_t n = p0 + 4 * (int64_t)ci;
            const float4 v = *reinterpret_cast<const float4*>(buf + (ci / CPR) * C::PITCH + 4 * (ci % CPR));
            if (n >= 0 && n < T) *reinterpret_cast<float4*>(dst + n) = v;
        }
    } else {
        const int r = rowmap ? 31 - lane : lane;
        const int64_t s = p0 + (int64_t)r * L;
        const float* row = buf + r * C::PITCH;
        const int64_t lo = s > 0 ? s : 0, hi = (s + L < T) ? s + L : T;
#pragma unroll 1
        for (int64_t n = lo; n < hi; ++n) dst[n] = row[n - s];
    }
}

// Inclusive warp scan S_l <- P^(2^d) S_(l - 2^d) + S_l (fp32, Kogge-Stone), then the
// exclusive prefix E (lane 0: zero) and the tile aggregate G (lane 31's inclusive).
template <int M>
__device__ __forceinline__ void warp_scan32(const float* P0, int lane, unsigned long long (&S)[Cfg<M>::NPR],
                                            float (&E)[M], float (&G)[M]) {
    using C = Cfg<M>;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int off = 1 << d;
        float O[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const float v = __shfl_up_sync(0xffffffffu, comp<C::NPR>(S, j), off);
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
        const float v = comp<C::NPR>(S, j);
        const float e = __shfl_up_sync(0xffffffffu, v, 1);
        E[j] = lane == 0 ? 0.f : e;
        G[j] = __shfl_sync(0xffffffffu, v, 31);
    }
}

// State entering this lane's chunk: E + X^(lane L) Xc (Q from the tables, through L1).
template <int M>
__device__ __forceinline__ void lane_carry(const float* __restrict__ Q, int lane, const float (&E)[M],
                                           const float (&Xc)[M], float (&v)[M]) {
    using C = Cfg<M>;
    unsigned long long S[C::NPR];
    pack_pairs<M, C::NPR>(E, S);
    mvp<M>(Q, lane, Xc, S);
    unpack_pairs<M, C::NPR>(S, v);
}

template <int M>
__device__ __forceinline__ void load_coef32(const float* tab, float (&bc)[M + 1], float (&ac)[M + 1]) {
    using C = Cfg<M>;
#pragma unroll
    for (int k = 0; k <= M; ++k) { bc[k] = tab[C::OC + k]; ac[k] = tab[C::OC + M + 1 + k]; }
}

// K-form chunk aggregate of 16 samples xs[0..15] at chunk positions k0 .. k0+15.
template <int M>
__device__ __forceinline__ void kform16(const float* K, int k0, const float (&xs)[16],
                                        unsigned long long (&S)[Cfg<M>::NPR]) {
    using C = Cfg<M>;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        unsigned long long Kp[C::NPR];
        ld_pairs<C::NPR>(K + (k0 + e) * C::MP, Kp);
        const unsigned long long X = pk2(xs[e], xs[e]);
#pragma unroll
        for (int ip = 0; ip < C::NPR; ++ip) S[ip] = ffma2(Kp[ip], X, S[ip]);
    }
}

// Chunk aggregates by the recursion itself, from the zero state (the default; IIRG_AGG_KFORM=1
// selects the K-form above).  The K-form moves 8 broadcast table floats per sample and lane
// through the shared-memory pipe (128 B/clk per SM): measured on C5 that pipe, not the FMAs,
// bounded the aggregate (ncu: mio_throttle + short_scoreboard 34 % of stalls).  The
// recursion keeps its 2M+1 coefficients in registers (loaded once per tile).
#ifndef IIRG_AGG_KFORM
#define IIRG_AGG_KFORM 0
#endif
// forward (a2): TDF-II over the lane's row, end state v(L) in scan-pair layout
template <int M>
__device__ __forceinline__ void agg_rec_fwd16(const Tdf2<M>& c2, const float (&xs)[16],
                                              unsigned long long (&VP)[Tdf2<M>::NP]) {
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
        float y0, y1;
        tdf2_step<M>(VP, xs[e], xs[e + 1], c2, y0, y1);
    }
}
// backward (a5): the adjoint g(n) = dy(n) + sum_k na_k g(n+k) over 16 samples of the row,
// newest last (n = k0 + 15 .. k0); Ev[j] = (g(n+2j), g(n+2j+1)) as in the a7 pass
template <int M>
__device__ __forceinline__ void agg_rec_bwd16(const float (&ds)[16], const unsigned long long (&NA1P)[(M + 1) / 2 + 1],
                                              const unsigned long long (&NA0P)[(M + 1) / 2 + 1], float na1,
                                              unsigned long long (&Ev)[(M + 1) / 2 + 1]) {
    constexpr int JE = (M + 1) / 2 + 1;
#pragma unroll
    for (int e = 14; e >= 0; e -= 2) {
        unsigned long long P1 = 0ull, P0 = 0ull;
#pragma unroll
        for (int j = JE - 1; j >= 0; --j) {
            if (2 * j + 1 <= M) P1 = ffma2(NA1P[j], Ev[j], P1);
            if (2 * j + 2 <= M) P0 = ffma2(NA0P[j], Ev[j], P0);
        }
        const float g1 = (ds[e + 1] + lo2(P1)) + hi2(P1);
        const float g0 = fmaf(na1, g1, (ds[e] + lo2(P0)) + hi2(P0));
#pragma unroll
        for (int j = JE - 1; j >= 1; --j) Ev[j] = Ev[j - 1];
        Ev[0] = pk2(g0, g1);
    }
}
// the adjoint state [g(s) .. g(s+M-1)] in scan-pair layout (odd M: the pad slot zero)
template <int M>
__device__ __forceinline__ void ev_to_pairs(const unsigned long long (&Ev)[(M + 1) / 2 + 1],
                                            unsigned long long (&S)[Cfg<M>::NPR]) {
#pragma unroll
    for (int ip = 0; ip < Cfg<M>::NPR; ++ip) S[ip] = (2 * ip + 1 < M) ? Ev[ip] : pk2(lo2(Ev[ip]), 0.f);
}
// the backward a7 coefficient pairs (table W of the backward group)
template <int M>
__device__ __forceinline__ void load_bwd_pairs(const float* tab, unsigned long long (&NA1P)[(M + 1) / 2 + 1],
                                               unsigned long long (&NA0P)[(M + 1) / 2 + 1],
                                               unsigned long long (&B0P)[(M + 1) / 2 + 1],
                                               unsigned long long (&B1P)[(M + 1) / 2 + 1]) {
    constexpr int JE = (M + 1) / 2 + 1;
    const unsigned long long* wp = reinterpret_cast<const unsigned long long*>(tab + Cfg<M>::OW);
#pragma unroll
    for (int j = 0; j < JE; ++j) {
        NA1P[j] = wp[j];
        NA0P[j] = wp[JE + j];
        B0P[j] = wp[2 * JE + j];
        B1P[j] = wp[3 * JE + j];
    }
}

// ---------------------------------------------------------------------------
// Tensor memory (TMEM) as a parking area (sm_100a).  Warp w may access TMEM lanes
// 32 (w % 4) .. 32 (w % 4) + 31; with the 32x32b shape thread i of the warp reads / writes
// its own lane, 16 consecutive 32-bit columns per instruction.
__device__ __forceinline__ void tmem_alloc(unsigned* dst, unsigned ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(unsigned taddr, unsigned ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(unsigned taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(unsigned taddr, float (&v)[16]) {
    unsigned r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------------------
// Forward (a2-a4).  Per warp: one incoming shared buffer (x by TMA), one outgoing buffer
// (y, bulk row stores) and two TMEM slots.  Iteration for tile t0 (aggregate published,
// x parked in TMEM): aggregate + publish t1 (data arrived an iteration ago) and park it,
// issue t2's load, look back for t0, emit t0 from TMEM.
template <int M, int NWP, bool GT>
__global__ void __launch_bounds__(NWP * 32, 1) lti2_fwd_kernel(const __grid_constant__ FwdArgs p) {
    using C = Cfg<M>;
    constexpr int L = C::L, TS = C::TS, NPR = C::NPR;
    static_assert(L % 16 == 0 && NWP <= 16 && 2 * L * ((NWP + 3) / 4) <= 512, "TMEM slots");
    extern __shared__ __align__(128) float sm2[];
    __shared__ __align__(8) unsigned long long s_bar[NWP];
    __shared__ float s_T[NWP][LEVELS][M];
    __shared__ unsigned s_tmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    V2_CTA_TRACE(p.trace, p.ntot, 0);
    float* bX = sm2 + (GT ? 0 : C::STAGE) + warp * 2 * C::BUF;
    float* bY = bX + C::BUF;
    unsigned long long* bar = &s_bar[warp];
    unsigned ph = 0;
    if (lane == 0) mbar_init(bar, 1);
    mbar_fence_init();
    __syncwarp();
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    // The kernel before this one on the stream is always this call's prologue, launched
    // WITHOUT programmatic serialization: everything enqueued before it (the caller's x,
    // the previous call's use of the workspace) completed before it started.  So the
    // workspace and the first x tile are read before griddepcontrol.wait; only the
    // prologue's tables are read after it.
    const CarryWs& cw = p.cw;                                  // grid constant: levels indexed from the param bank
    const unsigned ep = __ldcg(cw.epoch);
    const int64_t boff = (ep & 1u) ? cw.bank : 0;
    rearm_other_bank2(cw, boff, blockIdx.x, gridDim.x);
    const bool vec = p.vec != 0;
    Sched s0, s1;
    s0.init(blockIdx.x * NWP + warp, gridDim.x * NWP, p.B);
    s1 = s0;
    s1.next();
    auto issue = [&](const Sched& s) {
        load_rows<M>(bX, bar, p.x + s.seq * p.T, (int64_t)s.j * TS, p.T, vec, lane, 0);
    };
    if (s0.t < p.ntot) issue(s0);
    pdl_wait();
    pdl_launch_dependents();
    if constexpr (!GT) {
        for (int i = threadIdx.x; i < C::STAGE / 4; i += blockDim.x) cp_async16_ca(sm2 + 4 * i, p.t32 + 4 * i);
        cp_async_commit();
        cp_async_wait<0>();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const unsigned tbase = s_tmem + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 2 * L);
    V2_CTA_TRACE(p.trace, p.ntot, 1);
    auto aggregate = [&](const Sched& s, unsigned slot, float (&E)[M]) {
        const float* tab = GT ? p.t32 + s.seq * p.t32_stride : sm2;
        V2_TRACE(p.trace, s.t, 0);
        mbar_wait(bar, ph);
        ph ^= 1u;
        V2_TRACE(p.trace, s.t, 1);
        const float* row = bX + lane * C::PITCH;
        unsigned long long S[NPR];
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) S[ip] = 0ull;
#if !IIRG_AGG_KFORM
        float bc[M + 1], ac[M + 1];
        load_coef32<M>(tab, bc, ac);
        Tdf2<M> c2;
        c2.init_pairs(tab + C::OW, C::JP, bc, ac);
#endif
#pragma unroll 1
        for (int g = 0; g < L / 16; ++g) {
            float xs[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 v = *reinterpret_cast<const float4*>(row + 16 * g + 4 * q);
                xs[4 * q] = v.x; xs[4 * q + 1] = v.y; xs[4 * q + 2] = v.z; xs[4 * q + 3] = v.w;
            }
            tmem_st16(slot + 16 * g, xs);
#if IIRG_AGG_KFORM
            kform16<M>(tab + C::OK_, 16 * g, xs, S);
#else
            agg_rec_fwd16<M>(c2, xs, S);
#endif
        }
        float G[M];
        warp_scan32<M>(tab + C::OP, lane, S, E, G);
        float X0[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = 0.f;
        if (s.j == 0 && p.zi != nullptr)
#pragma unroll
            for (int i = 0; i < M; ++i) X0[i] = p.zi[s.seq * M + i];
        carry_publish<M>(p.t32 + s.seq * p.t32_stride + C::OPQ, lane, s.j, s.seq, X0, G, cw, boff);
        V2_TRACE(p.trace, s.t, 2);
    };
    float E0[M];
    unsigned sl = 0;                                             // TMEM slot of t0 (0 / 1)
    if (s0.t < p.ntot) {
        aggregate(s0, tbase, E0);
        if (s1.t < p.ntot) { __syncwarp(); issue(s1); }
    }
    while (s0.t < p.ntot) {
        Sched s2 = s1;
        s2.next();
        float V0pre[M];                                          // t0's level-0 look-back slots, in flight
        lookback_prefetch<M>(lane, s0.j, s0.seq, cw, boff, V0pre);   // across t1's aggregate
        float E1[M];
        if (s1.t < p.ntot) {
            aggregate(s1, tbase + (sl ^ 1u) * L, E1);
            if (s2.t < p.ntot) { __syncwarp(); issue(s2); }
        }
        const int64_t seq = s0.seq;
        const int jt = s0.j;
        const int64_t p0 = (int64_t)jt * TS;
        const float* tab = GT ? p.t32 + seq * p.t32_stride : sm2;
        const float* t32s = p.t32 + seq * p.t32_stride;
        const unsigned slot = tbase + sl * L;
        float X0[M], X[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = 0.f;
        if (jt == 0 && p.zi != nullptr)
#pragma unroll
            for (int i = 0; i < M; ++i) X0[i] = p.zi[seq * M + i];
        V2_TRACE(p.trace, s0.t, 3);
        carry_lookback<M>(t32s + C::OPQ, lane, jt, seq, X0, cw, boff, s_T[warp], X, &V0pre);
        V2_TRACE(p.trace, s0.t, 4);
        float vin[M];
        lane_carry<M>(t32s + C::OQ, lane, E0, X, vin);
        float bc[M + 1], ac[M + 1];
        load_coef32<M>(tab, bc, ac);
        tmem_wait_st();                                          // t0's parking (an iteration ago) is complete
        // zf = v(T): the lane holding sample T-1 walks from its carry-in (warp-uniform branch)
        const int64_t ez = p.T - 1 - (p0 + (int64_t)lane * L);
        const bool zwalk = p.zf != nullptr && ez >= 0 && ez < L - 1;
        if (__any_sync(0xffffffffu, zwalk)) {
            float w2[M];
#pragma unroll
            for (int i = 0; i < M; ++i) w2[i] = vin[i];
#pragma unroll 1
            for (int g = 0; g < L / 16; ++g) {
                float xs[16];
                tmem_ld16(slot + 16 * g, xs);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    if (zwalk && 16 * g + e <= ez) { float du; fwd_step<float, M, 1>(w2, xs[e], bc, ac, du); }
            }
            if (zwalk)
#pragma unroll
                for (int i = 0; i < M; ++i) p.zf[seq * M + i] = w2[i];
        }
        // a4: re-run from the exact carry-in, x from TMEM, y into the outgoing buffer
        __syncwarp();                                            // the previous tile's stores have read bY
        float* yr = bY + lane * C::PITCH;
        {
            Tdf2<M> c2;
            c2.init_pairs(tab + C::OW, C::JP, bc, ac);
            unsigned long long VP[Tdf2<M>::NP];
            tdf2_pack<M>(vin, VP);
            float xs[16];
            tmem_ld16(slot, xs);
#pragma unroll 1
            for (int g = 0; g < L / 16; ++g) {
                tmem_wait_ld();
                float ys[16];
#pragma unroll
                for (int e = 0; e < 16; e += 2) tdf2_step<M>(VP, xs[e], xs[e + 1], c2, ys[e], ys[e + 1]);
                if (g + 1 < L / 16) tmem_ld16(slot + 16 * (g + 1), xs);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<float4*>(yr + 16 * g + 4 * q) =
                        make_float4(ys[4 * q], ys[4 * q + 1], ys[4 * q + 2], ys[4 * q + 3]);
            }
            if (p.zf != nullptr && ez == L - 1) {
                float v[M];
                tdf2_unpack<M>(VP, v);
#pragma unroll
                for (int i = 0; i < M; ++i) p.zf[seq * M + i] = v[i];
            }
        }
        V2_TRACE(p.trace, s0.t, 5);
        store_rows<M>(bY, p.y + seq * p.T, p0, p.T, vec, lane, 0);
        V2_TRACE(p.trace, s0.t, 6);
        if (p.trace != nullptr && lane == 0) p.trace[(size_t)s0.t * 8 + 7] = blockIdx.x * NWP + warp;
        s0 = s1;
        s1 = s2;
#pragma unroll
        for (int i = 0; i < M; ++i) E0[i] = E1[i];
        sl ^= 1u;
    }
    V2_CTA_TRACE(p.trace, p.ntot, 2);
    tmem_fence_before();
    cta_exit(cw, ep, gridDim.x);
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 512);
    V2_CTA_TRACE(p.trace, p.ntot, 3);
}

// ---------------------------------------------------------------------------
// Backward (a5-a8).  Tiles are aligned to the END of each sequence and scanned last to
// first; lane l owns chunk 31 - l of its tile (the lane order is the scan order).  Per
// warp: shared buffers dy (incoming), x (-> dx in place, bulk stores) and y, and two TMEM
// slots for the parked dy.  Iteration for tile t0: x, y of t0 go out by TMA, aggregate +
// publish t1 (dy parked), issue dy of t2, look back for t0, then one fused pass per lane.

// Fixed-order fp64 sum of `nrows` rows of NG values (row-major, stride NG): lane l sums
// rows l, l+32, ... in increasing order, then a fixed xor butterfly; all lanes return all sums.
template <int NG>
__device__ __forceinline__ void warp_reduce_rows(const double* src, int64_t nrows, int lane, double (&out)[NG]) {
#pragma unroll
    for (int k = 0; k < NG; ++k) out[k] = 0.0;
#pragma unroll 1
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

// One row of coefficient partial sums (lane k < NG holds value k) joins the fixed-order
// reduction of its set: rows are reduced in groups of 32 by the group's last arrival, the
// groups by the set's last group (flat when the set has at most FLAT_ROWS rows), then the
// chain rule writes grad_b, grad_a.  Deterministic: every sum runs over row indices in a
// fixed order, whatever the arrival order.
template <int M>
__device__ __noinline__ void finalize_row(const BwdArgs& p, int64_t cset, int64_t per_set, int64_t li,
                                             double colsum, int lane, const double* __restrict__ t64) {
    constexpr int NG = Cfg<M>::NG;
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
    if (fin == 1u) {                                  // last row of its group: reduce the group
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
// The 32 lanes' partial sums (C_0, (C_k, D_k) pairs) -> fp64 column sums via lane rows of a
// free shared buffer; lane k < NG returns sum k (fixed order over the lanes).
template <int M>
__device__ __forceinline__ double lane_colsum(float* scratch, int lane, const unsigned long long (&CE)[(M + 1) / 2 + 1],
                                              const unsigned long long (&CO)[(M + 1) / 2 + 1],
                                              const unsigned long long (&DE)[(M + 1) / 2 + 1],
                                              const unsigned long long (&DO)[(M + 1) / 2 + 1]) {
    using C = Cfg<M>;
    __syncwarp();
    float* scr = scratch + lane * C::PITCH;
    auto ck = [&](const unsigned long long (&E)[(M + 1) / 2 + 1], const unsigned long long (&O)[(M + 1) / 2 + 1],
                  int k) {
        return (k & 1) ? lo2(O[(k + 1) / 2]) + hi2(O[(k - 1) / 2]) : lo2(E[k / 2]) + hi2(E[k / 2]);
    };
    scr[0] = ck(CE, CO, 0);
#pragma unroll
    for (int i = 0; i < M; ++i) {
        scr[1 + i] = ck(CE, CO, 1 + i);
        scr[M + 1 + i] = ck(DE, DO, 1 + i);
    }
    __syncwarp();
    double colsum = 0.0;
    if (lane < C::NG)
        for (int r = 0; r < 32; ++r) colsum += (double)scratch[r * C::PITCH + lane];
    __syncwarp();
    return colsum;
}

template <int M, int NWP, bool GT>
__global__ void __launch_bounds__(NWP * 32, 1) lti2_bwd_kernel(const __grid_constant__ BwdArgs p) {
    using C = Cfg<M>;
    constexpr int L = C::L, TS = C::TS, NG = C::NG, NPR = C::NPR;
    static_assert(L % 16 == 0 && NWP <= 16 && 2 * L * ((NWP + 3) / 4) <= 512, "TMEM slots");
    extern __shared__ __align__(128) float sm2[];
    __shared__ __align__(8) unsigned long long s_bar[NWP][2];
    __shared__ float s_T[NWP][LEVELS][M];
    __shared__ unsigned s_tmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    V2_CTA_TRACE(p.trace, p.ntot, 0);
    float* bI = sm2 + (GT ? 0 : C::STAGE) + warp * 3 * C::BUF;    // dy (incoming)
    float* bX = bI + C::BUF;                                      // x -> dx in place
    float* bY = bX + C::BUF;                                      // y, then partial-sum scratch
    unsigned long long* barI = &s_bar[warp][0];
    unsigned long long* barXY = &s_bar[warp][1];
    unsigned phI = 0, phXY = 0;
    if (lane == 0) { mbar_init(barI, 1); mbar_init(barXY, 1); }
    mbar_fence_init();
    __syncwarp();
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    // grad_y may be written by the kernel right before this one (the caller's loss): then
    // nothing the previous kernels wrote is read before griddepcontrol.wait.  With
    // IIR_FLAG_GRAD_Y_EARLY (grad_y, grad_zf written before the forward was enqueued) the
    // first tile's dy load, aggregate and publication run while the forward drains: they read
    // only grad_y, grad_zf, the prologue's tables (complete before the forward passed its own
    // wait and released this grid) and this direction's workspace; the wait comes before the
    // first read of y.
    bool waited = false;
    if (!p.gy_early) { pdl_wait(); waited = true; }
    pdl_launch_dependents();
    const CarryWs& cw = p.cw;                                  // grid constant: levels indexed from the param bank
    const unsigned ep = __ldcg(cw.epoch);
    const int64_t boff = (ep & 1u) ? cw.bank : 0;
    if constexpr (!GT) {
        const float* src = p.t32 + C::DIR;                       // backward table group
        for (int i = threadIdx.x; i < C::STAGE / 4; i += blockDim.x) cp_async16_ca(sm2 + 4 * i, src + 4 * i);
        cp_async_commit();
    }
    rearm_other_bank2(cw, boff, blockIdx.x, gridDim.x);
    if constexpr (!GT) cp_async_wait<0>();
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const unsigned tbase = s_tmem + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 2 * L);
    const bool vec = p.vec != 0;
    V2_CTA_TRACE(p.trace, p.ntot, 1);
    Sched s0, s1;
    s0.init(blockIdx.x * NWP + warp, gridDim.x * NWP, p.B);
    s1 = s0;
    s1.next();
    auto p0_of = [&](const Sched& s) -> int64_t { return p.T - (int64_t)(s.j + 1) * TS; };
    auto issue_dy = [&](const Sched& s) {
        load_rows<M>(bI, barI, p.gy == nullptr ? nullptr : p.gy + s.seq * p.T, p0_of(s), p.T, vec, lane, 1);
    };
    auto issue_xy = [&](const Sched& s) {
        const int64_t off = s.seq * p.T;
        load_rows<M>(bY, barXY, p.y + off, p0_of(s), p.T, vec, lane, 1, false);
        load_rows<M>(bX, barXY, p.x + off, p0_of(s), p.T, vec, lane, 1, true);     // arms last
    };
    // a5 + a6 (intra-warp) of tile t: dy rows -> TMEM slot, K-form aggregate, scan, publication
    auto aggregate = [&](const Sched& s, unsigned slot, float (&E)[M]) {
        const float* tab = GT ? p.t32 + s.seq * p.t32_stride + C::DIR : sm2;
        V2_TRACE(p.trace, s.t, 0);
        mbar_wait(barI, phI);
        phI ^= 1u;
        V2_TRACE(p.trace, s.t, 1);
        const float* row = bI + (31 - lane) * C::PITCH;
        unsigned long long S[NPR];
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) S[ip] = 0ull;
#if IIRG_AGG_KFORM
#pragma unroll 1
        for (int g = 0; g < L / 16; ++g) {
            float xs[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 v = *reinterpret_cast<const float4*>(row + 16 * g + 4 * q);
                xs[4 * q] = v.x; xs[4 * q + 1] = v.y; xs[4 * q + 2] = v.z; xs[4 * q + 3] = v.w;
            }
            tmem_st16(slot + 16 * g, xs);
            kform16<M>(tab + C::OK_, 16 * g, xs, S);
        }
#else
        {
            constexpr int JE = (M + 1) / 2 + 1;
            unsigned long long NA1P[JE], NA0P[JE], B0P[JE], B1P[JE], Ev[JE];
            load_bwd_pairs<M>(tab, NA1P, NA0P, B0P, B1P);
            const float na1 = -tab[C::OC + M + 2];
#pragma unroll
            for (int j = 0; j < JE; ++j) Ev[j] = 0ull;
#pragma unroll 1
            for (int g = L / 16 - 1; g >= 0; --g) {
                float xs[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(row + 16 * g + 4 * q);
                    xs[4 * q] = v.x; xs[4 * q + 1] = v.y; xs[4 * q + 2] = v.z; xs[4 * q + 3] = v.w;
                }
                tmem_st16(slot + 16 * g, xs);
                agg_rec_bwd16<M>(xs, NA1P, NA0P, na1, Ev);
            }
            ev_to_pairs<M>(Ev, S);
        }
#endif
        float G[M];
        warp_scan32<M>(tab + C::OP, lane, S, E, G);
        float X0[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = 0.f;
        if (s.j == 0 && p.gzf != nullptr)
#pragma unroll
            for (int i = 0; i < M; ++i) X0[i] = p.gzf[s.seq * M + i];
        carry_publish<M>(p.t32 + s.seq * p.t32_stride + C::DIR + C::OPQ, lane, s.j, s.seq, X0, G, cw, boff);
        V2_TRACE(p.trace, s.t, 2);
    };
    // coefficient partial sums: SHARED accumulates over all of this warp's tiles (a fixed set
    // in a fixed order under the static schedule) and flushes one row per warp at the end
    // the correlation sums C_k = sum g(n+k) x(n), D_k = sum g(n+k) y(n) in paired partial
    // sums (see a7): C_2j = CE_j.lo + CE_j.hi, C_2j+1 = CO_j+1.lo + CO_j.hi, D likewise
    constexpr int JE = (M + 1) / 2 + 1;
    unsigned long long CE[JE], CO[JE], DE[JE], DO[JE];
#pragma unroll
    for (int j = 0; j < JE; ++j) CE[j] = CO[j] = DE[j] = DO[j] = 0ull;
    float E0[M];
    unsigned sl = 0;
    if (s0.t < p.ntot) {
        issue_dy(s0);
        aggregate(s0, tbase, E0);
        if (s1.t < p.ntot) { __syncwarp(); issue_dy(s1); }
    }
    while (s0.t < p.ntot) {
        Sched s2 = s1;
        s2.next();
        __syncwarp();                                            // the previous tile's dx stores have read bX
        if (!waited) { pdl_wait(); waited = true; }             // y is the forward's output
        issue_xy(s0);
        float V0pre[M];                                          // t0's level-0 look-back slots, in flight
        lookback_prefetch<M>(lane, s0.j, s0.seq, cw, boff, V0pre);   // across t1's aggregate
        float E1[M];
        if (s1.t < p.ntot) {
            aggregate(s1, tbase + (sl ^ 1u) * L, E1);
            if (s2.t < p.ntot) { __syncwarp(); issue_dy(s2); }
        }
        const int64_t seq = s0.seq;
        const int jr = s0.j;                                     // 0 = last tile in time
        const int64_t p0 = p0_of(s0);                            // may be < 0 (first tile in time)
        const float* tab = GT ? p.t32 + seq * p.t32_stride + C::DIR : sm2;
        const float* t32s = p.t32 + seq * p.t32_stride + C::DIR;
        const double* t64 = p.t64 + seq * p.t64_stride;
        const unsigned slot = tbase + sl * L;
        const int c = 31 - lane;                                 // this lane's chunk (time order)
        const int64_t s = p0 + (int64_t)c * L;
        // a6: cross-tile carry (transposed powers), seeded by grad_zf at the last tile
        float X0[M], X[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = 0.f;
        if (jr == 0 && p.gzf != nullptr)
#pragma unroll
            for (int i = 0; i < M; ++i) X0[i] = p.gzf[seq * M + i];
        V2_TRACE(p.trace, s0.t, 3);
        carry_lookback<M>(t32s + C::OPQ, lane, jr, seq, X0, cw, boff, s_T[warp], X, &V0pre);
        V2_TRACE(p.trace, s0.t, 4);
        float din[M];
        lane_carry<M>(t32s + C::OQ, lane, E0, X, din);           // [g(e) .. g(e+M-1)], e = this chunk's right end
        float bk[M + 1], na[M + 1];
        load_coef32<M>(tab, bk, na);
#pragma unroll
        for (int k = 0; k <= M; ++k) na[k] = -na[k];
        // loop-invariant coefficient pairs of the a7 pass, loaded as pairs (table W)
        unsigned long long NA1P[JE], NA0P[JE], B0P[JE], B1P[JE];
        {
            const unsigned long long* wp = reinterpret_cast<const unsigned long long*>(tab + C::OW);
#pragma unroll
            for (int j = 0; j < JE; ++j) {
                NA1P[j] = wp[j];
                NA0P[j] = wp[JE + j];
                B0P[j] = wp[2 * JE + j];
                B1P[j] = wp[3 * JE + j];
            }
        }
        const float na1 = na[1];
        mbar_wait(barXY, phXY);
        phXY ^= 1u;
        tmem_wait_st();
        // grad_zi of a first tile that starts before n = 0: the lane whose chunk straddles
        // n = 0 walks down to it (warp-uniform branch; dy from TMEM)
        const bool zlane = p.gzi != nullptr && s < 0 && s + L > 0;
        if (__any_sync(0xffffffffu, zlane)) {
            float w2[M + 1];                                     // shifted once before each step
#pragma unroll
            for (int k = 0; k < M; ++k) w2[k] = din[k];
            w2[M] = 0.f;
#pragma unroll 1
            for (int g = L / 16 - 1; g >= 0; --g) {
                float ds[16];
                tmem_ld16(slot + 16 * g, ds);
                tmem_wait_ld();
#pragma unroll
                for (int e = 15; e >= 0; --e) {
                    if (zlane && s + 16 * g + e >= 0) {
#pragma unroll
                        for (int k = M; k >= 1; --k) w2[k] = w2[k - 1];
                        float acc = ds[e];
#pragma unroll
                        for (int k = M; k >= 2; --k) acc = fmaf(na[k], w2[k], acc);
                        w2[0] = fmaf(na[1], w2[1], acc);
                    }
                }
            }
            if (zlane)
#pragma unroll
                for (int i = 0; i < M; ++i) p.gzi[seq * M + i] = w2[i];
        }
        // a7: one fused pass per lane, backwards in time, two samples (n, n+1) per step.  The g
        // history is held as even-aligned pairs Ev[j] = (g(n+2j), g(n+2j+1)) only, and every
        // product is a paired FMA on an aligned pair (coefficient pairs are loop-invariant,
        // the (x, y) pairs are used as loaded or half-swapped):
        //   g(n+1) = dy(n+1) + sum_j (na_2j+1, na_2j+2) . Eh[j],                      (Eq.7)
        //   g(n)   = dy(n) + na_1 g(n+1) + sum_j (na_2j+2, na_2j+3) . Eh[j]  (Eh: before the step)
        //   dx(n) = sum_j (b'_2j, b'_2j+1) . Ev[j],  dx(n+1) = sum_j (b'_2j-1, b'_2j) . Ev[j]  (Eq.8)
        //   CE_j += Ev[j] * (x(n), x(n+1))  -> both halves C_2j;
        //   CO_j += Ev[j] * (x(n+1), x(n))  -> halves C_2j-1 (sample n+1), C_2j+1 (sample n);
        //   DE / DO likewise with y.
        if constexpr (GT) {                                     // PER_SEQ: one partial row per tile
#pragma unroll
            for (int j = 0; j < JE; ++j) CE[j] = CO[j] = DE[j] = DO[j] = 0ull;
        }
        unsigned long long Ev[JE];
        {
            auto dv = [&](int i) { return i < M ? din[i] : 0.f; };
#pragma unroll
            for (int j = 0; j < JE; ++j) Ev[j] = pk2(dv(2 * j), dv(2 * j + 1));
        }
        float* xr = bX + c * C::PITCH;
        const float* yr = bY + c * C::PITCH;
        {
            float ds[16];
            tmem_ld16(slot + 16 * (L / 16 - 1), ds);
#pragma unroll 1
            for (int g = L / 16 - 1; g >= 0; --g) {
                tmem_wait_ld();
                float dcur[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) dcur[e] = ds[e];
                if (g > 0) tmem_ld16(slot + 16 * (g - 1), ds);
#pragma unroll
                for (int q = 3; q >= 0; --q) {
                    const float4 xv = *reinterpret_cast<const float4*>(xr + 16 * g + 4 * q);
                    const float4 yv = *reinterpret_cast<const float4*>(yr + 16 * g + 4 * q);
                    float dxs[4];
#pragma unroll
                    for (int h = 1; h >= 0; --h) {               // samples (n, n+1) = 4q + 2h + (0, 1)
                        const float xa = h ? xv.z : xv.x, xb = h ? xv.w : xv.y;
                        const float ya = h ? yv.z : yv.x, yb = h ? yv.w : yv.y;
                        unsigned long long P1 = 0ull, P0 = 0ull;
#pragma unroll
                        for (int j = JE - 1; j >= 0; --j) {      // the newest pair (j = 0) last
                            if (2 * j + 1 <= M) P1 = ffma2(NA1P[j], Ev[j], P1);
                            if (2 * j + 2 <= M) P0 = ffma2(NA0P[j], Ev[j], P0);
                        }
                        const float g1 = (dcur[4 * q + 2 * h + 1] + lo2(P1)) + hi2(P1);
                        const float g0 = fmaf(na1, g1, (dcur[4 * q + 2 * h] + lo2(P0)) + hi2(P0));
#pragma unroll
                        for (int j = JE - 1; j >= 1; --j) Ev[j] = Ev[j - 1];
                        Ev[0] = pk2(g0, g1);
                        const unsigned long long XP = pk2(xa, xb), XS = pk2(xb, xa);
                        const unsigned long long YP = pk2(ya, yb), YS = pk2(yb, ya);
                        unsigned long long A0 = 0ull, A1 = 0ull;
#pragma unroll
                        for (int j = JE - 1; j >= 0; --j) {
                            A0 = ffma2(B0P[j], Ev[j], A0);
                            A1 = ffma2(B1P[j], Ev[j], A1);
                            CE[j] = ffma2(Ev[j], XP, CE[j]);
                            CO[j] = ffma2(Ev[j], XS, CO[j]);
                            DE[j] = ffma2(Ev[j], YP, DE[j]);
                            DO[j] = ffma2(Ev[j], YS, DO[j]);
                        }
                        dxs[2 * h] = lo2(A0) + hi2(A0);
                        dxs[2 * h + 1] = lo2(A1) + hi2(A1);
                    }
                    *reinterpret_cast<float4*>(xr + 16 * g + 4 * q) = make_float4(dxs[0], dxs[1], dxs[2], dxs[3]);
                }
            }
        }
        // grad_zi = d(0) = [g(0) .. g(M-1)] (Eq.9, App. A.3) when this chunk starts at n = 0
        if (p.gzi != nullptr && s == 0)
#pragma unroll
            for (int i = 0; i < M; ++i) p.gzi[seq * M + i] = (i & 1) ? hi2(Ev[i >> 1]) : lo2(Ev[i >> 1]);
        V2_TRACE(p.trace, s0.t, 5);
        // dx rows out
        if (p.gx != nullptr) store_rows<M>(bX, p.gx + seq * p.T, p0, p.T, vec, lane, 1);
        // a8 (PER_SEQ): the tile's partial-sum row joins its sequence's fixed-order reduction
        if constexpr (GT) {
            if (p.want_coef) {
                const double colsum = lane_colsum<M>(bY, lane, CE, CO, DE, DO);
                finalize_row<M>(p, seq, p.ntiles, jr, colsum, lane, t64);
            }
        }
        V2_TRACE(p.trace, s0.t, 6);
        if (p.trace != nullptr && lane == 0) p.trace[(size_t)s0.t * 8 + 7] = blockIdx.x * NWP + warp;
        s0 = s1;
        s1 = s2;
#pragma unroll
        for (int i = 0; i < M; ++i) E0[i] = E1[i];
        sl ^= 1u;
        __syncwarp();
    }
    V2_CTA_TRACE(p.trace, p.ntot, 2);
    // a8 (SHARED): one row per warp of the grid, indexed by the warp's global id
    if constexpr (!GT) {
        if (p.want_coef) {
            const double colsum = lane_colsum<M>(bY, lane, CE, CO, DE, DO);
            finalize_row<M>(p, 0, (int64_t)gridDim.x * NWP, (int64_t)blockIdx.x * NWP + warp, colsum, lane, p.t64);
        }
    }
    V2_CTA_TRACE(p.trace, p.ntot, 4);
    tmem_fence_before();
    cta_exit(cw, ep, gridDim.x);
    V2_CTA_TRACE(p.trace, p.ntot, 5);
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 512);
    V2_CTA_TRACE(p.trace, p.ntot, 3);
}

// ---------------------------------------------------------------------------
// a1: prologue (fp64), one small CTA per (coefficient set, role); the roles are
// independent, so the prologue's latency is the longest role, not their sum:
//   role 0: K weights by vector doubling (U[m] = A_f^m c, R[m] = e1^T A_f^m from the
//           squarings A_f^(2^j)), the scan powers A_f^(L 2^d), the coefficients;
//   role 1: the lane powers A_f^(l L), l = 0..32 (Q);
//   role 2+v: the look-back powers A_f^(k 32^v TS), k = 0..31, of level v (PQ).
// Each role builds its base power by repeated squaring of A_f, then doubles.
constexpr int PREP_NT = 256;
template <int M> struct Prep2Slots {
    static constexpr int NSQ = 32;        // squarings A_f^(2^j), j < NSQ (enough for 32^3 TS)
    static constexpr int SW = NSQ, SPOW = SW + 1, N = SPOW + 33;
    static constexpr size_t bytes() { return (size_t)N * M * M * sizeof(double) + 2 * (size_t)Cfg<M>::L * M * sizeof(double); }
};

template <int M>
__global__ void __launch_bounds__(PREP_NT) lti2_prep_kernel(const float* __restrict__ b, const float* __restrict__ a,
                                                           int64_t coef_stride, float* __restrict__ t32,
                                                           int64_t t32_stride, double* __restrict__ t64,
                                                           int64_t t64_stride, int nlev) {
    pdl_launch_dependents();
    using C = Cfg<M>;
    using S = Prep2Slots<M>;
    constexpr int L = C::L, M2 = M * M, MP = C::MP, NPR = C::NPR;
    constexpr int LOG_L = L == 64 ? 6 : L == 32 ? 5 : L == 128 ? 7 : 0;
    static_assert(LOG_L > 0, "chunk length must be 32, 64 or 128");
    extern __shared__ __align__(16) unsigned char prep2_raw[];
    double* mat = reinterpret_cast<double*>(prep2_raw);
    double* U = mat + S::N * M2;                          // [L][M]: A_f^m c
    double* R = U + L * M;                                // [L][M]: e1^T A_f^m
    __shared__ double bn[M + 1], an[M + 1], cv[M];
    const int set = blockIdx.x, role = blockIdx.y, tid = threadIdx.x;
    if (role >= 2 && role - 2 >= nlev) return;
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
    for (int e = tid; e < M2; e += PREP_NT) {
        const int i = e / M, j = e % M;
        mat[0 * M2 + e] = (j == 0 ? -an[i + 1] : 0.0) + (j == i + 1 ? 1.0 : 0.0);   // A_f[i][j] = squaring 0
        mat[S::SPOW * M2 + e] = (i == j) ? 1.0 : 0.0;                                  // X^0
    }
    __syncthreads();
    // batched products: for q < n: mat[dst(q)] = mat[lhs(q)] * mat[rhs(q)]
    auto mm_batch = [&](int n, auto dst, auto lhs, auto rhs) {
        constexpr int RR = (16 * M2 + PREP_NT - 1) / PREP_NT;
        double rr[RR];
#pragma unroll
        for (int s2 = 0; s2 < RR; ++s2) {
            const int w = tid + s2 * PREP_NT;
            rr[s2] = 0.0;
            if (w < n * M2) {
                const int q = w / M2, e = w % M2, i = e / M, j = e % M;
                const double* A = mat + lhs(q) * M2;
                const double* B = mat + rhs(q) * M2;
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(A[i * M + k], B[k * M + j], acc);
                rr[s2] = acc;
            }
        }
        __syncthreads();
#pragma unroll
        for (int s2 = 0; s2 < RR; ++s2) {
            const int w = tid + s2 * PREP_NT;
            if (w < n * M2) mat[dst(w / M2) * M2 + (w % M2)] = rr[s2];
        }
        __syncthreads();
    };
    auto square_to = [&](int j1) {                      // squarings 1 .. j1 (A_f^(2^j))
        for (int j = 1; j <= j1; ++j)
            mm_batch(1, [&](int) { return j; }, [&](int) { return j - 1; }, [&](int) { return j - 1; });
    };
    // SPOW + k = X^k, k = 0..32, from X = squaring jx (SPOW + 1 set by the caller)
    auto powers32 = [&]() {
        for (int st = 0; st < 5; ++st) {
            const int h = 1 << st;
            mm_batch(h, [&](int q) { return S::SPOW + h + 1 + q; }, [&](int) { return S::SPOW + h; },
                     [&](int q) { return S::SPOW + 1 + q; });
        }
    };
    auto copy = [&](int dst, int src) {
        for (int e = tid; e < M2; e += PREP_NT) mat[dst * M2 + e] = mat[src * M2 + e];
        __syncthreads();
    };
    // pair tables [j][ip][32] of X^k (k = 0..31), forward X and backward X^T
    auto pair_table = [&](int off) {
        for (int w = tid; w < 32 * M * NPR; w += PREP_NT) {
            const int k = w % 32, ip = (w / 32) % NPR, j = w / (32 * NPR);
            const double* X = mat + (S::SPOW + k) * M2;
            const int i0 = 2 * ip, i1 = 2 * ip + 1;
            o32[off + 2 * w] = (float)X[i0 * M + j];
            o32[off + 2 * w + 1] = i1 < M ? (float)X[i1 * M + j] : 0.f;
            o32[C::DIR + off + 2 * w] = (float)X[j * M + i0];
            o32[C::DIR + off + 2 * w + 1] = i1 < M ? (float)X[j * M + i1] : 0.f;
        }
    };
    if (role == 0) {
        square_to(LOG_L + 4);                            // A_f^(2^j), j <= log2(L) + 4
        // vector doubling: U[m] = A_f^m c, R[m] = e1^T A_f^m
        if (tid < M) { U[tid] = cv[tid]; R[tid] = tid == 0 ? 1.0 : 0.0; }
        __syncthreads();
        for (int j = 0; j < LOG_L; ++j) {
            const int h = 1 << j;
            const double* X = mat + j * M2;              // A_f^h
            double ru[(L / 2 * M + PREP_NT - 1) / PREP_NT], rr2[(L / 2 * M + PREP_NT - 1) / PREP_NT];
#pragma unroll
            for (int s2 = 0; s2 < (L / 2 * M + PREP_NT - 1) / PREP_NT; ++s2) {
                const int w = tid + s2 * PREP_NT;
                ru[s2] = rr2[s2] = 0.0;
                if (w < h * M) {
                    const int m = w / M, i = w % M;
                    double su = 0.0, sr = 0.0;
                    for (int k = 0; k < M; ++k) {
                        su = fma(X[i * M + k], U[m * M + k], su);     // (A^h U[m])_i
                        sr = fma(R[m * M + k], X[k * M + i], sr);     // (R[m] A^h)_i
                    }
                    ru[s2] = su;
                    rr2[s2] = sr;
                }
            }
            __syncthreads();
#pragma unroll
            for (int s2 = 0; s2 < (L / 2 * M + PREP_NT - 1) / PREP_NT; ++s2) {
                const int w = tid + s2 * PREP_NT;
                if (w < h * M) { U[(w / M + h) * M + w % M] = ru[s2]; R[(w / M + h) * M + w % M] = rr2[s2]; }
            }
            __syncthreads();
        }
        for (int w = tid; w < L * MP; w += PREP_NT) {       // KF[k] = U[L-1-k], KB[k] = R[k]
            const int k = w / MP, i = w % MP;
            o32[C::OK_ + w] = i < M ? (float)U[(L - 1 - k) * M + i] : 0.f;
            o32[C::DIR + C::OK_ + w] = i < M ? (float)R[k * M + i] : 0.f;
        }
        for (int w = tid; w < 5 * M * MP; w += PREP_NT) {   // P[d][j][i] = X^(L 2^d)[i][j]
            const int d = w / (M * MP), j = (w / MP) % M, i = w % MP;
            const double* X = mat + (LOG_L + d) * M2;
            o32[C::OP + w] = i < M ? (float)X[i * M + j] : 0.f;
            o32[C::DIR + C::OP + w] = i < M ? (float)X[j * M + i] : 0.f;
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
        for (int w = tid; w < 8 * C::JP; w += PREP_NT) {    // W (forward group): the Tdf2 pairs
            const int arr = w / (2 * C::JP), j = (w / 2) % C::JP, h = w & 1;
            const int k = (arr == 0 || arr == 1) ? 2 * j + 2 + h : 2 * j + 1 + h;
            float v = 0.f;
            if (j < (M + 1) / 2 && k <= M) v = (arr & 1) ? -(float)an[k] : (float)bn[k];
            o32[C::OW + w] = v;
        }
        for (int w = tid; w < 8 * C::JP; w += PREP_NT) {    // W (backward group)
            const int arr = w / (2 * C::JP), j = (w / 2) % C::JP, h = w & 1;
            const int k = arr == 0 ? 2 * j + 1 + h : arr == 1 ? 2 * j + 2 + h : arr == 2 ? 2 * j + h : 2 * j - 1 + h;
            float v = 0.f;
            if (arr < 2) { if (k >= 1 && k <= M) v = -(float)an[k]; }
            else if (k >= 0 && k <= M) v = (float)bn[k];
            o32[C::DIR + C::OW + w] = v;
        }
        return;
    }
    // role 1: X = A_f^L;  role 2+v: X = A_f^(32^v TS) = A_f^(2^(LOG_L + 5 + 5 v))
    const int jx = role == 1 ? LOG_L : LOG_L + 5 + 5 * (role - 2);
    square_to(jx);
    copy(S::SPOW + 1, jx);
    powers32();
    pair_table(role == 1 ? C::OQ : C::OPQ + (role - 2) * 32 * M * MP);
}

}  // namespace v2
}  // namespace iirg
