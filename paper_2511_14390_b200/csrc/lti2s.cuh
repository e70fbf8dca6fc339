// lti2s.cuh -- split schedule of the round-2 LTI engine (fp32 TDF-II, orders 1..8):
// two kernels per direction instead of one fused single pass (lti2.cuh).
//
//   carry kernel (a2 + a3 forward, a5 + a6 backward): per warp tile the 32 lane-chunk
//     aggregates (K-form), the warp scan, the publication of the tile aggregate and the
//     hierarchical look-back (Eq.10; the same device functions as the
//     fused kernels), then each lane's carry-in E_l + X^(lane L) X_tile is written to the
//     workspace: carr[t][lane][M] (t = tile in schedule order; M floats per 64-sample
//     chunk, 0.5 B/sample at M = 8).  Only the (small) per-tile work sits between a
//     warp's loads, so its look-back waits are hidden by the other resident warps.
//   emit kernel (a4 forward, a7 backward): per warp tile, no inter-tile dependency: the
//     lane re-runs the recursion from its carry-in (forward: y; backward: g, dx and the
//     correlation sums C_k, D_k of lti2.cuh's a7 pass), the tiles double- (forward) or
//     single-buffered (backward) in shared memory.
//
// Cost against the fused pass: x (forward) and grad_y (backward) are read twice and the
// carries go through L2/HBM: 4 + 2 * 4M / L bytes per sample and direction more traffic
// (DESIGN.md section 6), bought for kernels whose warps never wait on another tile.
#pragma once
#include "lti2.cuh"

namespace iirg {
namespace v2 {

struct CarryArgs {
    const float* src;            // x (forward) or grad_y (backward), (B, T)
    const float* x0;             // zi (forward) or grad_zf (backward), (B, M) or NULL
    const float* t32; int64_t t32_stride;   // table group of this direction (backward: + DIR)
    CarryWs cw;
    int64_t B, T; int ntiles; int64_t ntot; int vec;
    float* carr;                 // [ntot][32][M] lane carry-ins
    unsigned long long* trace;
};

// carr row of tile t, lane l
template <int M>
__device__ __forceinline__ size_t carr_off(unsigned t, int lane) { return ((size_t)t * 32 + lane) * M; }

template <int M>
__device__ __forceinline__ void carr_store(float* dst, const float (&v)[M]) {
    if constexpr (M % 4 == 0) {
#pragma unroll
        for (int q = 0; q < M / 4; ++q)
            __stcg(reinterpret_cast<float4*>(dst) + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    } else if constexpr (M % 2 == 0) {
#pragma unroll
        for (int q = 0; q < M / 2; ++q) __stcg(reinterpret_cast<float2*>(dst) + q, make_float2(v[2 * q], v[2 * q + 1]));
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) __stcg(dst + i, v[i]);
    }
}
template <int M>
__device__ __forceinline__ void carr_load(const float* src, float (&v)[M]) {
    if constexpr (M % 4 == 0) {
#pragma unroll
        for (int q = 0; q < M / 4; ++q) {
            const float4 t = __ldcg(reinterpret_cast<const float4*>(src) + q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    } else if constexpr (M % 2 == 0) {
#pragma unroll
        for (int q = 0; q < M / 2; ++q) {
            const float2 t = __ldcg(reinterpret_cast<const float2*>(src) + q);
            v[2 * q] = t.x; v[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) v[i] = __ldcg(src + i);
    }
}

// ---------------------------------------------------------------------------
// Carry kernel.  Per warp: two incoming shared buffers.  Iteration for tile t0 (aggregate
// published, its buffer already refilled with t2): aggregate + publish t1, issue t3 into
// t1's buffer, look back for t0, write t0's lane carry-ins.  Forward tiles start at
// j TS; backward tiles are aligned to the end of the sequence and lane l owns chunk 31 - l
// (the lane order is the scan order), as in lti2_bwd_kernel.
#ifndef IIRG_S_CNBUF
#define IIRG_S_CNBUF 2
#endif
constexpr int CNBUF = IIRG_S_CNBUF;   // carry kernel: shared tile buffers per warp (1 or 2)
template <int M, int NWP, bool GT, bool BWD>
__global__ void __launch_bounds__(NWP * 32, 1) lti2s_carry_kernel(const __grid_constant__ CarryArgs p) {
    using C = Cfg<M>;
    constexpr int L = C::L, TS = C::TS, NPR = C::NPR;
    extern __shared__ __align__(128) float sm2[];
    __shared__ __align__(8) unsigned long long s_bar[NWP][2];
    __shared__ float s_T[NWP][LEVELS][M];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    V2_CTA_TRACE(p.trace, p.ntot, 0);
    float* buf = sm2 + (GT ? 0 : C::STAGE) + warp * CNBUF * C::BUF;
    if (lane == 0) { mbar_init(&s_bar[warp][0], 1); mbar_init(&s_bar[warp][1], 1); }
    mbar_fence_init();
    __syncwarp();
    // Backward: grad_y may be written by the kernel right before this one, so nothing is
    // read before griddepcontrol.wait.  Forward: the kernel before this one is the call's
    // prologue, launched without programmatic serialization, so x and the workspace are
    // complete and only the prologue's tables wait.
    if constexpr (BWD) pdl_wait();
    const CarryWs& cw = p.cw;
    const unsigned ep = __ldcg(cw.epoch);
    const int64_t boff = (ep & 1u) ? cw.bank : 0;
    const bool vec = p.vec != 0;
    Sched s0, s1, s2;
    s0.init(blockIdx.x * NWP + warp, gridDim.x * NWP, p.B);
    s1 = s0;
    s1.next();
    s2 = s1;
    s2.next();
    auto p0_of = [&](const Sched& s) -> int64_t { return BWD ? p.T - (int64_t)(s.j + 1) * TS : (int64_t)s.j * TS; };
    auto issue = [&](const Sched& s, int b) {
        b = CNBUF == 1 ? 0 : b;
        load_rows<M>(buf + b * C::BUF, &s_bar[warp][b], p.src == nullptr ? nullptr : p.src + s.seq * p.T, p0_of(s),
                     p.T, vec, lane, BWD ? 1 : 0);
    };
    if (s0.t < p.ntot) issue(s0, 0);
    if (CNBUF == 2 && s1.t < p.ntot) issue(s1, 1);
    if constexpr (!BWD) pdl_wait();
    pdl_launch_dependents();
    rearm_other_bank2(cw, boff, blockIdx.x, gridDim.x);
    if constexpr (!GT) {
        for (int i = threadIdx.x; i < C::STAGE / 4; i += blockDim.x) cp_async16_ca(sm2 + 4 * i, p.t32 + 4 * i);
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    V2_CTA_TRACE(p.trace, p.ntot, 1);
    unsigned phm = 0;                                           // mbarrier phase bits of the two buffers
    auto aggregate = [&](const Sched& s, int b, float (&E)[M]) {
        b = CNBUF == 1 ? 0 : b;
        const float* tab = GT ? p.t32 + s.seq * p.t32_stride : sm2;
        V2_TRACE(p.trace, s.t, 0);
        mbar_wait(&s_bar[warp][b], (phm >> b) & 1u);
        phm ^= 1u << b;
        V2_TRACE(p.trace, s.t, 1);
        const float* row = buf + b * C::BUF + (BWD ? 31 - lane : lane) * C::PITCH;
        unsigned long long S[NPR];
#pragma unroll
        for (int ip = 0; ip < NPR; ++ip) S[ip] = 0ull;
        auto ld16 = [&](int g, float (&xs)[16]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 v = *reinterpret_cast<const float4*>(row + 16 * g + 4 * q);
                xs[4 * q] = v.x; xs[4 * q + 1] = v.y; xs[4 * q + 2] = v.z; xs[4 * q + 3] = v.w;
            }
        };
#if IIRG_AGG_KFORM
#pragma unroll 1
        for (int g = 0; g < L / 16; ++g) {
            float xs[16];
            ld16(g, xs);
            kform16<M>(tab + C::OK_, 16 * g, xs, S);
        }
#else
        if constexpr (!BWD) {
            float bc[M + 1], ac[M + 1];
            load_coef32<M>(tab, bc, ac);
            Tdf2<M> c2;
            c2.init_pairs(tab + C::OW, C::JP, bc, ac);
#pragma unroll 1
            for (int g = 0; g < L / 16; ++g) {
                float xs[16];
                ld16(g, xs);
                agg_rec_fwd16<M>(c2, xs, S);
            }
        } else {
            constexpr int JE = (M + 1) / 2 + 1;
            unsigned long long NA1P[JE], NA0P[JE], B0P[JE], B1P[JE], Ev[JE];
            load_bwd_pairs<M>(tab, NA1P, NA0P, B0P, B1P);
            const float na1 = -tab[C::OC + M + 2];
#pragma unroll
            for (int j = 0; j < JE; ++j) Ev[j] = 0ull;
#pragma unroll 1
            for (int g = L / 16 - 1; g >= 0; --g) {
                float xs[16];
                ld16(g, xs);
                agg_rec_bwd16<M>(xs, NA1P, NA0P, na1, Ev);
            }
            ev_to_pairs<M>(Ev, S);
        }
#endif
        V2_TRACE(p.trace, s.t, 5);                              // (carry kernel: [5] = K-form done)
        float G[M];
        warp_scan32<M>(tab + C::OP, lane, S, E, G);
        V2_TRACE(p.trace, s.t, 6);                              // (carry kernel: [6] = scan done)
        float X0[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = 0.f;
        if (s.j == 0 && p.x0 != nullptr)
#pragma unroll
            for (int i = 0; i < M; ++i) X0[i] = p.x0[s.seq * M + i];
        carry_publish<M>(p.t32 + s.seq * p.t32_stride + C::OPQ, lane, s.j, s.seq, X0, G, cw, boff);
        V2_TRACE(p.trace, s.t, 2);
    };
    float E0[M];
    int b0 = 0;                                                  // buffer of t0 (t1: b0 ^ 1)
    if (s0.t < p.ntot) {
        aggregate(s0, 0, E0);
        if (CNBUF == 2 && s2.t < p.ntot) { __syncwarp(); issue(s2, 0); }
        if (CNBUF == 1 && s1.t < p.ntot) { __syncwarp(); issue(s1, 0); }
    }
    while (s0.t < p.ntot) {
        Sched s3 = s2;
        s3.next();
        float E1[M];
        if (s1.t < p.ntot) {
            aggregate(s1, b0 ^ 1, E1);
            if (CNBUF == 2 && s3.t < p.ntot) { __syncwarp(); issue(s3, b0 ^ 1); }
            if (CNBUF == 1 && s2.t < p.ntot) { __syncwarp(); issue(s2, 0); }
        }
        float X0[M], X[M];
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = 0.f;
        if (s0.j == 0 && p.x0 != nullptr)
#pragma unroll
            for (int i = 0; i < M; ++i) X0[i] = p.x0[s0.seq * M + i];
        const float* t32s = p.t32 + s0.seq * p.t32_stride;
        V2_TRACE(p.trace, s0.t, 3);
        carry_lookback<M>(t32s + C::OPQ, lane, s0.j, s0.seq, X0, cw, boff, s_T[warp], X);
        V2_TRACE(p.trace, s0.t, 4);
        float vin[M];
        lane_carry<M>(t32s + C::OQ, lane, E0, X, vin);
        carr_store<M>(p.carr + carr_off<M>(s0.t, lane), vin);
        if (p.trace != nullptr && lane == 0) p.trace[(size_t)s0.t * 8 + 7] = blockIdx.x * NWP + warp;
        s0 = s1;
        s1 = s2;
        s2 = s3;
#pragma unroll
        for (int i = 0; i < M; ++i) E0[i] = E1[i];
        b0 ^= 1;
    }
    V2_CTA_TRACE(p.trace, p.ntot, 2);
    cta_exit(cw, ep, gridDim.x);
    V2_CTA_TRACE(p.trace, p.ntot, 3);
}

// ---------------------------------------------------------------------------
// Forward emit (a4).  Per warp two shared buffers: tile t's x arrives in one while t-1 is
// emitted from the other; y is written over x in the row and leaves by coalesced stores.
template <int M, int NWP, bool GT>
__global__ void __launch_bounds__(NWP * 32, 1) lti2s_emit_fwd_kernel(const __grid_constant__ FwdArgs p) {
    using C = Cfg<M>;
    constexpr int L = C::L, TS = C::TS;
    extern __shared__ __align__(128) float sm2[];
    __shared__ __align__(8) unsigned long long s_bar[NWP][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    V2_CTA_TRACE(p.trace, p.ntot, 0);
    float* buf = sm2 + (GT ? 0 : C::STAGE) + warp * 2 * C::BUF;
    if (lane == 0) { mbar_init(&s_bar[warp][0], 1); mbar_init(&s_bar[warp][1], 1); }
    mbar_fence_init();
    __syncwarp();
    const bool vec = p.vec != 0;
    Sched s0, s1;
    s0.init(blockIdx.x * NWP + warp, gridDim.x * NWP, p.B);
    s1 = s0;
    s1.next();
    auto issue = [&](const Sched& s, int b) {
        load_rows<M>(buf + b * C::BUF, &s_bar[warp][b], p.x + s.seq * p.T, (int64_t)s.j * TS, p.T, vec, lane, 0);
    };
    // x is complete (see lti2s_carry_kernel): the first two tiles load before the wait for
    // the carry kernel; the carry-ins and the tables are read after it.
    if (s0.t < p.ntot) issue(s0, 0);
    if (s1.t < p.ntot) issue(s1, 1);
    pdl_wait();
    pdl_launch_dependents();
    if constexpr (!GT) {
        for (int i = threadIdx.x; i < C::STAGE / 4; i += blockDim.x) cp_async16_ca(sm2 + 4 * i, p.t32 + 4 * i);
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    V2_CTA_TRACE(p.trace, p.ntot, 1);
    unsigned phm = 0;
    int b = 0;
    while (s0.t < p.ntot) {
        const int64_t seq = s0.seq;
        const int64_t p0 = (int64_t)s0.j * TS;
        const float* tab = GT ? p.t32 + seq * p.t32_stride : sm2;
        float vin[M];
        carr_load<M>(p.carr + carr_off<M>(s0.t, lane), vin);
        float bc[M + 1], ac[M + 1];
        load_coef32<M>(tab, bc, ac);
        V2_TRACE(p.trace, s0.t, 0);
        mbar_wait(&s_bar[warp][b], (phm >> b) & 1u);
        phm ^= 1u << b;
        V2_TRACE(p.trace, s0.t, 1);
        float* row = buf + b * C::BUF + lane * C::PITCH;
        // zf = v(T): the lane holding sample T-1 walks from its carry-in (warp-uniform branch)
        const int64_t ez = p.T - 1 - (p0 + (int64_t)lane * L);
        const bool zwalk = p.zf != nullptr && ez >= 0 && ez < L - 1;
        if (__any_sync(0xffffffffu, zwalk)) {
            if (zwalk) {
                float w2[M];
#pragma unroll
                for (int i = 0; i < M; ++i) w2[i] = vin[i];
#pragma unroll 1
                for (int e = 0; e <= (int)ez; ++e) { float du; fwd_step<float, M, 1>(w2, row[e], bc, ac, du); }
#pragma unroll
                for (int i = 0; i < M; ++i) p.zf[seq * M + i] = w2[i];
            }
            __syncwarp();
        }
        {
            Tdf2<M> c2;
            c2.init_pairs(tab + C::OW, C::JP, bc, ac);
            unsigned long long VP[Tdf2<M>::NP];
            tdf2_pack<M>(vin, VP);
#pragma unroll 1
            for (int g = 0; g < L / 16; ++g) {
                float xs[16], ys[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(row + 16 * g + 4 * q);
                    xs[4 * q] = v.x; xs[4 * q + 1] = v.y; xs[4 * q + 2] = v.z; xs[4 * q + 3] = v.w;
                }
#pragma unroll
                for (int e = 0; e < 16; e += 2) tdf2_step<M>(VP, xs[e], xs[e + 1], c2, ys[e], ys[e + 1]);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<float4*>(row + 16 * g + 4 * q) =
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
        store_rows<M>(buf + b * C::BUF, p.y + seq * p.T, p0, p.T, vec, lane, 0);
        V2_TRACE(p.trace, s0.t, 6);
        if (p.trace != nullptr && lane == 0) p.trace[(size_t)s0.t * 8 + 7] = blockIdx.x * NWP + warp;
        Sched s2 = s1;
        s2.next();
        if (s2.t < p.ntot) { __syncwarp(); issue(s2, b); }
        s0 = s1;
        s1 = s2;
        b ^= 1;
    }
    V2_CTA_TRACE(p.trace, p.ntot, 2);
}

// ---------------------------------------------------------------------------
// Backward emit (a7 + a8).  Per warp three shared buffers (dy, x -> dx in place, y), one
// barrier; the fused reverse pass of lti2_bwd_kernel from each lane's carry-in.
template <int M, int NWP, bool GT>
__global__ void __launch_bounds__(NWP * 32, 1) lti2s_emit_bwd_kernel(const __grid_constant__ BwdArgs p) {
    using C = Cfg<M>;
    constexpr int L = C::L, TS = C::TS;
    extern __shared__ __align__(128) float sm2[];
    __shared__ __align__(8) unsigned long long s_bar[NWP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    V2_CTA_TRACE(p.trace, p.ntot, 0);
    float* bI = sm2 + (GT ? 0 : C::STAGE) + warp * 3 * C::BUF;   // dy
    float* bX = bI + C::BUF;                                      // x -> dx in place
    float* bY = bX + C::BUF;                                      // y, then partial-sum scratch
    unsigned long long* bar = &s_bar[warp];
    if (lane == 0) mbar_init(bar, 1);
    mbar_fence_init();
    __syncwarp();
    pdl_wait();
    pdl_launch_dependents();
    const bool vec = p.vec != 0;
    Sched s0;
    s0.init(blockIdx.x * NWP + warp, gridDim.x * NWP, p.B);
    auto p0_of = [&](const Sched& s) -> int64_t { return p.T - (int64_t)(s.j + 1) * TS; };
    auto issue = [&](const Sched& s) {
        const int64_t off = s.seq * p.T;
        load_rows<M>(bI, bar, p.gy == nullptr ? nullptr : p.gy + off, p0_of(s), p.T, vec, lane, 1, false);
        load_rows<M>(bY, bar, p.y + off, p0_of(s), p.T, vec, lane, 1, false);
        load_rows<M>(bX, bar, p.x + off, p0_of(s), p.T, vec, lane, 1, true);     // arms last
    };
    if (s0.t < p.ntot) issue(s0);
    if constexpr (!GT) {
        const float* src = p.t32 + C::DIR;
        for (int i = threadIdx.x; i < C::STAGE / 4; i += blockDim.x) cp_async16_ca(sm2 + 4 * i, src + 4 * i);
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    V2_CTA_TRACE(p.trace, p.ntot, 1);
    constexpr int JE = (M + 1) / 2 + 1;
    unsigned long long CE[JE], CO[JE], DE[JE], DO[JE];
#pragma unroll
    for (int j = 0; j < JE; ++j) CE[j] = CO[j] = DE[j] = DO[j] = 0ull;
    unsigned ph = 0;
    while (s0.t < p.ntot) {
        const int64_t seq = s0.seq;
        const int jr = s0.j;
        const int64_t p0 = p0_of(s0);
        const float* tab = GT ? p.t32 + seq * p.t32_stride + C::DIR : sm2;
        const double* t64 = p.t64 + seq * p.t64_stride;
        const int c = 31 - lane;                                 // this lane's chunk (time order)
        const int64_t s = p0 + (int64_t)c * L;
        float din[M];                                            // [g(e) .. g(e+M-1)], e = chunk end
        carr_load<M>(p.carr + carr_off<M>(s0.t, lane), din);
        float na[M + 1];
        {
            float bk[M + 1];
            load_coef32<M>(tab, bk, na);
        }
#pragma unroll
        for (int k = 0; k <= M; ++k) na[k] = -na[k];
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
        V2_TRACE(p.trace, s0.t, 0);
        mbar_wait(bar, ph);
        ph ^= 1u;
        V2_TRACE(p.trace, s0.t, 1);
        const float* dyr = bI + c * C::PITCH;
        // grad_zi of a first tile that starts before n = 0: the lane whose chunk straddles
        // n = 0 walks down to it (warp-uniform branch)
        const bool zlane = p.gzi != nullptr && s < 0 && s + L > 0;
        if (__any_sync(0xffffffffu, zlane)) {
            if (zlane) {
                float w2[M + 1];
#pragma unroll
                for (int k = 0; k < M; ++k) w2[k] = din[k];
                w2[M] = 0.f;
#pragma unroll 1
                for (int e = L - 1; e >= 0; --e) {
                    if (s + e >= 0) {
#pragma unroll
                        for (int k = M; k >= 1; --k) w2[k] = w2[k - 1];
                        float acc = dyr[e];
#pragma unroll
                        for (int k = M; k >= 2; --k) acc = fmaf(na[k], w2[k], acc);
                        w2[0] = fmaf(na[1], w2[1], acc);
                    }
                }
#pragma unroll
                for (int i = 0; i < M; ++i) p.gzi[seq * M + i] = w2[i];
            }
            __syncwarp();
        }
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
        // a7: the fused pass of lti2_bwd_kernel (see there), dy from the shared row
#pragma unroll 1
        for (int g = L / 16 - 1; g >= 0; --g) {
            float dcur[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 v = *reinterpret_cast<const float4*>(dyr + 16 * g + 4 * q);
                dcur[4 * q] = v.x; dcur[4 * q + 1] = v.y; dcur[4 * q + 2] = v.z; dcur[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int q = 3; q >= 0; --q) {
                const float4 xv = *reinterpret_cast<const float4*>(xr + 16 * g + 4 * q);
                const float4 yv = *reinterpret_cast<const float4*>(yr + 16 * g + 4 * q);
                float dxs[4];
#pragma unroll
                for (int h = 1; h >= 0; --h) {
                    const float xa = h ? xv.z : xv.x, xb = h ? xv.w : xv.y;
                    const float ya = h ? yv.z : yv.x, yb = h ? yv.w : yv.y;
                    unsigned long long P1 = 0ull, P0 = 0ull;
#pragma unroll
                    for (int j = JE - 1; j >= 0; --j) {
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
        if (p.gzi != nullptr && s == 0)
#pragma unroll
            for (int i = 0; i < M; ++i) p.gzi[seq * M + i] = (i & 1) ? hi2(Ev[i >> 1]) : lo2(Ev[i >> 1]);
        V2_TRACE(p.trace, s0.t, 5);
        if (p.gx != nullptr) store_rows<M>(bX, p.gx + seq * p.T, p0, p.T, vec, lane, 1);
        if constexpr (GT) {
            if (p.want_coef) {
                const double colsum = lane_colsum<M>(bY, lane, CE, CO, DE, DO);
                finalize_row<M>(p, seq, p.ntiles, jr, colsum, lane, t64);
            }
        }
        V2_TRACE(p.trace, s0.t, 6);
        if (p.trace != nullptr && lane == 0) p.trace[(size_t)s0.t * 8 + 7] = blockIdx.x * NWP + warp;
        s0.next();
        __syncwarp();
        if (s0.t < p.ntot) issue(s0);
    }
    V2_CTA_TRACE(p.trace, p.ntot, 2);
    if constexpr (!GT) {
        if (p.want_coef) {
            const double colsum = lane_colsum<M>(bY, lane, CE, CO, DE, DO);
            finalize_row<M>(p, 0, (int64_t)gridDim.x * NWP, (int64_t)blockIdx.x * NWP + warp, colsum, lane, p.t64);
        }
    }
    V2_CTA_TRACE(p.trace, p.ntot, 3);
}

}  // namespace v2
}  // namespace iirg
