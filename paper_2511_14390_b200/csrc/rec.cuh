// rec.cuh -- sm_100a kernels for the bare recurrence of Listing 1
// (SURVEY §8(f) f1), the operator the paper benchmarks:
//   v(n+1) = A v(n) + z(n),  n = 0..N-1,  dense M x M A,  output v(1..N)
// and its VJP (Listing 1's backward, Eq.7 on the state itself):
//   g(N-1) = gv(N-1),  g(n) = gv(n) + A^T g(n+1)        (gv(n) = dL/dv(n+1))
//   grad_z = g,  grad_v0 = A^T g(0),  grad_A = sum_n g(n) v(n)^T  (v(0) = v0).
// Same time-parallel machine as the filters (lti.cuh): chunked local pass from
// the zero state, fp64 carries with precomputed powers of A (warp / block /
// hierarchical grid look-back), exact re-run emit; the per-sample state is the
// whole M-vector, stored interleaved (B, N, M) in HBM.
#pragma once
#include "lti.cuh"

namespace iirg {

// samples per thread chunk: a tile holds NT * L samples of M elements
template <typename T, int M> constexpr int rec_L() { return (sizeof(T) == 4 ? 32 : 16) / (M > 2 ? 2 : 1); }

template <typename T, int M>
struct RecSmem {
    static constexpr int L = rec_L<T, M>();
    static constexpr int TS = NT * L;                    // samples per tile
    static constexpr int TE = TS * M;                    // elements per tile
    static constexpr int PT = pidx<T>(TE);
    static constexpr size_t tab_bytes = Smem<T, M>::tab_bytes;
    static constexpr size_t fwd() { return tab_bytes + (size_t)PT * sizeof(T); }
    static constexpr size_t bwd() { return tab_bytes + (size_t)2 * PT * sizeof(T); }
};

template <typename T, int M>
__device__ __forceinline__ void rec_load_A(const T* __restrict__ a, T (&A)[M][M]) {
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) A[i][j] = __ldg(a + i * M + j);
}

// Forward.  p.a = A (row-major, coef_stride 0 SHARED / M*M PER_SEQ), p.x = z,
// p.zi = v0 (NULL = 0), p.y = v(1..N); p.zf unused (v(N) is the last output row).
template <typename T, int M>
__global__ void __launch_bounds__(NT) rec_fwd_kernel(const LtiFwdArgs p) {
    using RS = RecSmem<T, M>;
    constexpr int L = RS::L, TS = RS::TS, TE = RS::TE, W = Vec<T>::W;
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    static_assert((L * M) % W == 0, "vector chunks");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* st = reinterpret_cast<double*>(smem_raw);
    T* zs = reinterpret_cast<T*>(smem_raw + RS::tab_bytes);     // z -> v in place
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned tk = tile_order(p.cw.ticket);
    span_enter(p.span);
    CarryWs cw = p.cw;
    const unsigned ep = carry_bank(cw);
    const int64_t seq = (int64_t)(tk % (unsigned long long)p.B);
    const int jt = (int)(tk / (unsigned long long)p.B);
    const int64_t p0 = (int64_t)jt * TS;
    const int64_t rowlen = p.Tlen * M;
    const T* zrow = static_cast<const T*>(p.x) + seq * rowlen;
    IIRG_TRACE(p.trace, tk, 0);
    tile_load_async<T, TE>(zs, zrow, p0 * M, rowlen, p.vec);
    cp_async_commit();
    pdl_wait();
    pdl_launch_dependents();
    const double* tb = p.tab + seq * p.tab_stride;
    stage_small_async<M>(st, tb);
    cp_async_commit();
    rearm_other_bank(cw, ep, blockIdx.x, gridDim.x);
    T A[M][M];
    rec_load_A<T, M>(static_cast<const T*>(p.a) + seq * p.coef_stride, A);
    cp_async_wait<1>();
    __syncthreads();
    // a2: local pass from the zero state over this thread's chunk
    const int e0 = tid * L * M;
    T v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = T(0);
    auto step = [&](const T (&zz)[M]) {
        T vn[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            T s = zz[i];
#pragma unroll
            for (int j = 0; j < M; ++j) s = fma(A[i][j], v[j], s);
            vn[i] = s;
        }
#pragma unroll
        for (int i = 0; i < M; ++i) v[i] = vn[i];
    };
    {
        T buf[L * M];
#pragma unroll
        for (int g = 0; g < L * M / W; ++g) {
            const V t = *reinterpret_cast<const V*>(zs + pidx<T>(e0 + g * W));
#pragma unroll
            for (int e = 0; e < W; ++e) buf[g * W + e] = vget(t, e);
        }
#pragma unroll
        for (int s2 = 0; s2 < L; ++s2) {
            T zz[M];
#pragma unroll
            for (int i = 0; i < M; ++i) zz[i] = buf[s2 * M + i];
            step(zz);
        }
    }
    IIRG_TRACE(p.trace, tk, 1);
    cp_async_wait<0>();
    __syncthreads();
    double S[M];
#pragma unroll
    for (int i = 0; i < M; ++i) S[i] = (double)v[i];
    warp_scan<M, false>(st, lane, S);
    double E[M];
#pragma unroll
    for (int i = 0; i < M; ++i) { E[i] = shfl_up_d(S[i], 1); if (lane == 0) E[i] = 0.0; }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < M; ++i) s_agg[warp][i] = S[i];
    }
    __syncthreads();
    if (warp == 0) {
        double Jex[M], G[M], X0[M], X[M];
        block_scan<M, false>(st, lane, s_agg, Jex, G);
        const T* v0 = static_cast<const T*>(p.zi);
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (v0 != nullptr && jt == 0) ? (double)v0[seq * M + i] : 0.0;
        IIRG_TRACE(p.trace, tk, 2);
        tile_carry<M, false>(st, tb, lane, jt, seq, X0, G, cw, X, p.trace, tk);
        IIRG_TRACE(p.trace, tk, 3);
        if (lane < NW) {
            double xw[M];
#pragma unroll
            for (int i = 0; i < M; ++i) xw[i] = Jex[i];
            mv_acc_lane_s<M, false>(st + TB::PWT, NW, lane, X, xw);
#pragma unroll
            for (int i = 0; i < M; ++i) s_xw[lane][i] = xw[i];
        }
    }
    __syncthreads();
    {
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
        mv_plt<M, false>(st, tb, lane, xw, E);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = (T)E[i];
    // a4: re-run from the exact carry-in, v(n+1) written over z(n)
    {
        T buf[L * M];
#pragma unroll
        for (int g = 0; g < L * M / W; ++g) {
            const V t = *reinterpret_cast<const V*>(zs + pidx<T>(e0 + g * W));
#pragma unroll
            for (int e = 0; e < W; ++e) buf[g * W + e] = vget(t, e);
        }
#pragma unroll
        for (int s2 = 0; s2 < L; ++s2) {
            T zz[M];
#pragma unroll
            for (int i = 0; i < M; ++i) zz[i] = buf[s2 * M + i];
            step(zz);
#pragma unroll
            for (int i = 0; i < M; ++i) buf[s2 * M + i] = v[i];
        }
#pragma unroll
        for (int g = 0; g < L * M / W; ++g) {
            V t;
#pragma unroll
            for (int e = 0; e < W; ++e) vset(t, e, buf[g * W + e]);
            *reinterpret_cast<V*>(zs + pidx<T>(e0 + g * W)) = t;
        }
    }
    __syncthreads();
    IIRG_TRACE(p.trace, tk, 4);
    tile_store<T, TE>(static_cast<T*>(p.y) + seq * rowlen, zs, p0 * M, rowlen, p.vec);
    IIRG_TRACE(p.trace, tk, 5);
    cta_exit(cw, ep, gridDim.x);
    span_exit(p.span);
}

// Backward.  p.gy = gv (B, N, M), p.y = v(1..N) of the forward, p.zi = v0,
// p.gx = grad_z, p.ga = grad_A (M*M per set), p.gzi = grad_v0.  The state walked
// backwards is s(n) = g(n+1): s <- A^T s + gv(n) emits g(n) = the new s.
template <typename T, int M>
__global__ void __launch_bounds__(NT) rec_bwd_kernel(const LtiBwdArgs p) {
    using RS = RecSmem<T, M>;
    constexpr int L = RS::L, TS = RS::TS, TE = RS::TE, W = Vec<T>::W;
    constexpr int NG = M * M;
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* st = reinterpret_cast<double*>(smem_raw);
    T* gs = reinterpret_cast<T*>(smem_raw + RS::tab_bytes);     // gv -> g in place
    T* vs = gs + RS::PT;                                          // v(n+1), n in the tile
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];
    __shared__ double s_red[NW][NG];
    __shared__ T s_prev[M];                                       // v(p0) = v(1..N)[p0 - 1] or v0
    __shared__ T s_v0[M];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned tk = tile_order(p.cw.ticket);
    span_enter(p.span);
    CarryWs cw = p.cw;
    const unsigned ep = carry_bank(cw);
    const int64_t seq = (int64_t)(tk % (unsigned long long)p.B);
    const int jr = (int)(tk / (unsigned long long)p.B);          // 0 = last tile in time
    const int jt = p.ntiles - 1 - jr;
    const int64_t p0 = p.Tlen - (int64_t)(jr + 1) * TS;          // may be < 0 (first tile)
    const int64_t rowlen = p.Tlen * M;
    const int64_t roff = seq * rowlen;
    const double* tb = p.tab + seq * p.tab_stride;
    const T* v0 = static_cast<const T*>(p.zi);
    IIRG_TRACE(p.trace, tk, 0);
    if (p.gy != nullptr) tile_load_async<T, TE>(gs, static_cast<const T*>(p.gy) + roff, p0 * M, rowlen, p.vec);
    else for (int e = tid; e < TE; e += NT) gs[pidx<T>(e)] = T(0);
    cp_async_commit();
    stage_small_async<M>(st, tb);
    cp_async_commit();
    // v(n) for the tile's samples n = p0 .. p0+TS-1 is the forward output row n-1:
    // the tile of v(1..N) at the same position is v(n+1); v(p0) comes separately
    tile_load_async<T, TE>(vs, static_cast<const T*>(p.y) + roff, p0 * M, rowlen, p.vec);
    cp_async_commit();
    if (tid < M) {
        T pv = T(0);
        if (p0 > 0) pv = static_cast<const T*>(p.y)[roff + (p0 - 1) * M + tid];
        else if (p0 == 0 && v0 != nullptr) pv = v0[seq * M + tid];
        s_prev[tid] = pv;
        s_v0[tid] = v0 != nullptr ? v0[seq * M + tid] : T(0);
    }
    rearm_other_bank(cw, ep, blockIdx.x, gridDim.x);
    T A[M][M];
    rec_load_A<T, M>(static_cast<const T*>(p.a) + seq * p.coef_stride, A);
    cp_async_wait<1>();                                          // gv and the tables
    __syncthreads();
    const int c = NT - 1 - tid;                                  // chunk index (time order)
    const int s0 = c * L, e0 = s0 * M;
    T s[M];
#pragma unroll
    for (int i = 0; i < M; ++i) s[i] = T(0);
    auto step = [&](const T (&gv)[M]) {                          // s <- A^T s + gv
        T sn[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            T a = gv[i];
#pragma unroll
            for (int j = 0; j < M; ++j) a = fma(A[j][i], s[j], a);
            sn[i] = a;
        }
#pragma unroll
        for (int i = 0; i < M; ++i) s[i] = sn[i];
    };
    T buf[L * M];
#pragma unroll
    for (int g = 0; g < L * M / W; ++g) {
        const V t = *reinterpret_cast<const V*>(gs + pidx<T>(e0 + g * W));
#pragma unroll
        for (int e = 0; e < W; ++e) buf[g * W + e] = vget(t, e);
    }
#pragma unroll
    for (int s2 = L - 1; s2 >= 0; --s2) {
        T gg[M];
#pragma unroll
        for (int i = 0; i < M; ++i) gg[i] = buf[s2 * M + i];
        step(gg);
    }
    IIRG_TRACE(p.trace, tk, 1);
    double S[M];
#pragma unroll
    for (int i = 0; i < M; ++i) S[i] = (double)s[i];
    warp_scan<M, true>(st, lane, S);
    double E[M];
#pragma unroll
    for (int i = 0; i < M; ++i) { E[i] = shfl_up_d(S[i], 1); if (lane == 0) E[i] = 0.0; }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < M; ++i) s_agg[warp][i] = S[i];
    }
    __syncthreads();
    if (warp == 0) {
        double Jex[M], G[M], X0[M], X[M];
        block_scan<M, true>(st, lane, s_agg, Jex, G);
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = 0.0;                 // g(N) = 0
        IIRG_TRACE(p.trace, tk, 2);
        tile_carry<M, true>(st, tb, lane, jr, seq, X0, G, cw, X, p.trace, tk);
        IIRG_TRACE(p.trace, tk, 3);
        if (lane < NW) {
            double xw[M];
#pragma unroll
            for (int i = 0; i < M; ++i) xw[i] = Jex[i];
            mv_acc_lane_s<M, true>(st + TB::PWT, NW, lane, X, xw);
#pragma unroll
            for (int i = 0; i < M; ++i) s_xw[lane][i] = xw[i];
        }
    }
    cp_async_wait<0>();                                          // v tile
    __syncthreads();
    {
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
        mv_plt<M, true>(st, tb, lane, xw, E);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) s[i] = (T)E[i];
    // a7: re-run from the exact carry; g(n) over gv(n); grad_A partials g(n) v(n)^T
    T vb[L * M];                                                 // v(n+1) for the chunk's samples
#pragma unroll
    for (int g = 0; g < L * M / W; ++g) {
        const V t = *reinterpret_cast<const V*>(vs + pidx<T>(e0 + g * W));
#pragma unroll
        for (int e = 0; e < W; ++e) vb[g * W + e] = vget(t, e);
    }
    T vprev[M];                                                  // v(s0): the sample before the chunk
#pragma unroll
    for (int i = 0; i < M; ++i) vprev[i] = s0 == 0 ? s_prev[i] : vs[pidx<T>(e0 - M + i)];
    T GA[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) GA[k] = T(0);
#pragma unroll
    for (int s2 = L - 1; s2 >= 0; --s2) {
        T gg[M];
#pragma unroll
        for (int i = 0; i < M; ++i) gg[i] = buf[s2 * M + i];
        step(gg);                                                // s = g(n)
        const int64_t n = p0 + s0 + s2;
        const bool in = n >= 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            buf[s2 * M + i] = s[i];
            if (in) {
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const T vn = n == 0 ? s_v0[j] : (s2 == 0 ? vprev[j] : vb[(s2 - 1) * M + j]);   // v(n)
                    GA[i * M + j] = fma(s[i], vn, GA[i * M + j]);
                }
            }
        }
        if (p.gzi != nullptr && p0 + s0 + s2 == 0) {             // grad_v0 = A^T g(0)
            T* gv0 = static_cast<T*>(p.gzi) + seq * M;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                T a = T(0);
#pragma unroll
                for (int j = 0; j < M; ++j) a = fma(A[j][i], s[j], a);
                gv0[i] = a;
            }
        }
    }
#pragma unroll
    for (int g = 0; g < L * M / W; ++g) {
        V t;
#pragma unroll
        for (int e = 0; e < W; ++e) vset(t, e, buf[g * W + e]);
        *reinterpret_cast<V*>(gs + pidx<T>(e0 + g * W)) = t;
    }
    if (p.want_coef) {
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            double sm = (double)GA[k];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
            if (lane == 0) s_red[warp][k] = sm;
        }
    }
    __syncthreads();
    IIRG_TRACE(p.trace, tk, 4);
    if (p.gx != nullptr) tile_store<T, TE>(static_cast<T*>(p.gx) + roff, gs, p0 * M, rowlen, p.vec);
    IIRG_TRACE(p.trace, tk, 5);
    bwd_finalize<T, M, 2>(p, &cw, ep, tk, seq, jt, tb, s_red);
    span_exit(p.span);
}

}  // namespace iirg
