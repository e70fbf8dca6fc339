// lti.cuh -- sm_100a kernels for batched LTI DF-II / TDF-II filtering and its
// closed-form backward (arXiv 2511.14390, Eqs.4-9).
//
// Time-parallel formulation (Eq.10) as a chunked scan:
//   * a tile of NT*L samples of one sequence per CTA; each thread owns a
//     contiguous chunk of L samples and runs the recursion on it from a zero
//     state (local pass), giving the chunk aggregate w (the z of Eq.10's tuple);
//   * carries are combined in fp64 with the constant transition powers
//     A_f^(L 2^d) (warp Kogge-Stone over shuffles), A_f^(32 L 2^d) (across the
//     warps, shared memory), and A_f^(TS k) (across tiles: single-pass
//     decoupled look-back on per-tile status words);
//   * each thread then re-runs its chunk from the exact carry-in state and
//     emits outputs (and, in the backward pass, the gradient partial sums).
// The backward pass is the same machine run in reverse time on the adjoint
// recursion (Eq.7), whose transition is A_f^T: it reads the same power tables
// transposed ("the backward of DF is a TDF run backwards").
#pragma once
#include "common.cuh"

namespace iirg {

// ---------------------------------------------------------------------------
// fp64 power tables of one coefficient set (computed once per call on device).
template <int M> struct Tab {
    static constexpr int M2 = M * M;
    static constexpr int PL = 0;                      // A_f^(L 2^d), d = 0..4      [d][i][j]
    static constexpr int PLT = PL + 5 * M2;           // A_f^(L t),   t = 0..31     [i][j][t]
    static constexpr int PW = PLT + 32 * M2;          // A_f^(32L 2^d), d < LOG_NW  [d][i][j]
    static constexpr int PWT = PW + LOG_NW * M2;      // A_f^(32L w), w = 0..NW-1   [i][j][w]
    static constexpr int PTK = PWT + NW * M2;         // A_f^(TS k), k = 1..KLB     [k-1][i][j]
    static constexpr int COEF = PTK + KLB * M2;       // b'[0..M], a'[0..M], c[0..M-1]
    static constexpr int A0 = COEF + 3 * M + 2;       // a0 (un-normalised)
    static constexpr int SIZE = (A0 + 1 + 31) / 32 * 32;
};

// acc += P v (TR = false) or P^T v (TR = true); P row-major M x M (fp64).
template <int M, bool TR>
__device__ __forceinline__ void mv_acc(const double* __restrict__ P, const double (&v)[M], double (&acc)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double s = acc[i];
#pragma unroll
        for (int j = 0; j < M; ++j) s = fma(__ldg(P + (TR ? j * M + i : i * M + j)), v[j], s);
        acc[i] = s;
    }
}
// Same with a per-lane matrix stored element-major [i][j][stride] (coalesced).
template <int M, bool TR>
__device__ __forceinline__ void mv_acc_lane(const double* __restrict__ P, int stride, int t,
                                            const double (&v)[M], double (&acc)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double s = acc[i];
#pragma unroll
        for (int j = 0; j < M; ++j) s = fma(__ldg(P + (TR ? j * M + i : i * M + j) * stride + t), v[j], s);
        acc[i] = s;
    }
}

// ---------------------------------------------------------------------------
// a1: coefficient prologue.  Normalise by a0, build A_f (DF: companion(a'),
// TDF: its transpose) and the fp64 power tables.
template <typename T, int M, int FORM>
__global__ void __launch_bounds__(64) lti_prep_kernel(const T* __restrict__ b, const T* __restrict__ a,
                                                     int64_t coef_stride, double* __restrict__ tab,
                                                     int64_t tab_stride) {
    constexpr int L = Chunk<T>::L, M2 = M * M;
    using TB = Tab<M>;
    __shared__ double Af[M2], X[M2], Y[M2], Z[M2], W[M2], bn[M + 1], an[M + 1];
    const int set = blockIdx.x;
    const T* bb = b + set * coef_stride;
    const T* aa = a + set * coef_stride;
    double* tb = tab + set * tab_stride;
    const int tid = threadIdx.x, i = tid / M, j = tid % M;
    const bool act = tid < M2;
    if (tid <= M) {
        const double a0 = (double)aa[0];
        bn[tid] = (double)bb[tid] / a0;
        an[tid] = (double)aa[tid] / a0;
    }
    __syncthreads();
    if (act) {
        const double Aij = (i == 0) ? -an[j + 1] : (i == j + 1 ? 1.0 : 0.0);  // companion(a')
        const double Aji = (j == 0) ? -an[i + 1] : (j == i + 1 ? 1.0 : 0.0);
        Af[tid] = (FORM == 0) ? Aij : Aji;
        Z[tid] = (i == j) ? 1.0 : 0.0;
    }
    if (tid <= M) { tb[TB::COEF + tid] = bn[tid]; tb[TB::COEF + M + 1 + tid] = an[tid]; }
    if (tid < M) tb[TB::COEF + 2 * (M + 1) + tid] = bn[tid + 1] - an[tid + 1] * bn[0];
    if (tid == 0) tb[TB::A0] = (double)aa[0];
    __syncthreads();
    auto mm = [&](double* dst, const double* A, const double* B) {
        double s = 0.0;
        if (act)
#pragma unroll
            for (int k = 0; k < M; ++k) s = fma(A[i * M + k], B[k * M + j], s);
        __syncthreads();
        if (act) dst[tid] = s;
        __syncthreads();
    };
    auto cp = [&](double* dst, const double* src) {
        if (act) dst[tid] = src[tid];
        __syncthreads();
    };
    cp(X, Af);
    for (int p = 1; p < L; p *= 2) mm(X, X, X);                 // X = A_f^L
    cp(Y, X);
    for (int d = 0; d < 5; ++d) {                               // A_f^(L 2^d)
        if (act) tb[TB::PL + d * M2 + tid] = Y[tid];
        mm(Y, Y, Y);
    }                                                           // Y = A_f^(32 L)
    for (int t = 0; t < 32; ++t) {                              // A_f^(L t)
        if (act) tb[TB::PLT + tid * 32 + t] = Z[tid];
        mm(Z, Z, X);
    }
    cp(W, Y);
    for (int d = 0; d < LOG_NW; ++d) {                          // A_f^(32 L 2^d)
        if (act) tb[TB::PW + d * M2 + tid] = W[tid];
        mm(W, W, W);
    }                                                           // W = A_f^(TS)
    if (act) Z[tid] = (i == j) ? 1.0 : 0.0;
    __syncthreads();
    for (int w = 0; w < NW; ++w) {                              // A_f^(32 L w)
        if (act) tb[TB::PWT + tid * NW + w] = Z[tid];
        mm(Z, Z, Y);
    }
    cp(Z, W);
    for (int k = 1; k <= KLB; ++k) {                            // A_f^(TS k)
        if (act) tb[TB::PTK + (k - 1) * M2 + tid] = Z[tid];
        mm(Z, Z, W);
    }
}

// ---------------------------------------------------------------------------
// One-sample recursions.  State v has M entries.
// Forward TDF-II (A^T, c, e1, b0) in its difference-equation form:
//   y = b0 x + v0;  v_i <- v_{i+1} + b_{i+1} x - a_{i+1} y.
// Forward DF-II (A, e1, c, b0), v = [u(n-1) .. u(n-M)] (Eqs.2-3):
//   u = x - sum a_k v_{k-1};  y = b0 u + sum b_k v_{k-1};  shift in u.
template <typename T, int M, int FORM>
__device__ __forceinline__ T fwd_step(T (&v)[M], T x, const T (&bc)[M + 1], const T (&ac)[M + 1], T& u_out) {
    if constexpr (FORM == 1) {
        const T y = fma(bc[0], x, v[0]);
#pragma unroll
        for (int i = 0; i < M - 1; ++i) v[i] = fma(-ac[i + 1], y, fma(bc[i + 1], x, v[i + 1]));
        v[M - 1] = fma(-ac[M], y, bc[M] * x);
        u_out = T(0);
        return y;
    } else {
        T u = x;
#pragma unroll
        for (int k = M; k >= 1; --k) u = fma(-ac[k], v[k - 1], u);   // most recent term last
        T y = bc[0] * u;
#pragma unroll
        for (int k = M; k >= 1; --k) y = fma(bc[k], v[k - 1], y);
#pragma unroll
        for (int k = M - 1; k >= 1; --k) v[k] = v[k - 1];
        v[0] = u;
        u_out = u;
        return y;
    }
}

// Adjoint step of TDF-II (Eq.7 with A_f^T = A, C_f = e1): state d = dz(n),
//   dz(n-1)[0] = dy(n) - sum_k a_k dz(n)[k-1],  dz(n-1)[i] = dz(n)[i-1].
template <typename T, int M>
__device__ __forceinline__ void adj_tdf_step(T (&d)[M], T dy, const T (&ac)[M + 1]) {
    T q = dy;
#pragma unroll
    for (int k = M; k >= 1; --k) q = fma(-ac[k], d[k - 1], q);
#pragma unroll
    for (int k = M - 1; k >= 1; --k) d[k] = d[k - 1];
    d[0] = q;
}
// Adjoint step of DF-II (Eq.7 with A_f^T = A^T, C_f = c): with g = dx(n) =
// dz(n)[0] + b0 dy(n) (Eq.8),  dz(n-1)[i] = dz(n)[i+1] - a_{i+1} g + b_{i+1} dy.
template <typename T, int M>
__device__ __forceinline__ T adj_df_step(T (&d)[M], T dy, const T (&bc)[M + 1], const T (&ac)[M + 1]) {
    const T g = fma(bc[0], dy, d[0]);
#pragma unroll
    for (int i = 0; i < M - 1; ++i) d[i] = fma(-ac[i + 1], g, fma(bc[i + 1], dy, d[i + 1]));
    d[M - 1] = fma(-ac[M], g, bc[M] * dy);
    return g;
}

// ---------------------------------------------------------------------------
struct LtiFwdArgs {
    const void* x; const void* zi; void* y; void* zf; void* u;   // u: DF tape signal
    const double* tab; int64_t tab_stride;                        // 0 for SHARED
    unsigned* ticket; unsigned* flags; double* agg; double* incl;
    int64_t B, Tlen; int ntiles; int vec;
};

struct LtiBwdArgs {
    const void* gy; const void* gzf; const void* x; const void* y; const void* u; const void* zi;
    void* gx; void* gzi; double* partial; int want_coef;
    const double* tab; int64_t tab_stride;
    unsigned* ticket; unsigned* flags; double* agg; double* incl;
    int64_t B, Tlen; int ntiles; int vec;
};

template <typename T, int M>
__device__ __forceinline__ void load_coefs(const double* __restrict__ tb, T (&bc)[M + 1], T (&ac)[M + 1], T (&cc)[M]) {
    using TB = Tab<M>;
#pragma unroll
    for (int k = 0; k <= M; ++k) { bc[k] = (T)__ldg(tb + TB::COEF + k); ac[k] = (T)__ldg(tb + TB::COEF + M + 1 + k); }
#pragma unroll
    for (int k = 0; k < M; ++k) cc[k] = (T)__ldg(tb + TB::COEF + 2 * (M + 1) + k);
}

// Warp-level inclusive Kogge-Stone scan of chunk aggregates in fp64:
//   S_t <- P^(2^d) S_{t-2^d} + S_t, P = A_f^L (TR: transposed for the adjoint).
template <int M, bool TR>
__device__ __forceinline__ void warp_scan(const double* __restrict__ tb, int lane, double (&S)[M]) {
    using TB = Tab<M>;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int off = 1 << d;
        double O[M];
#pragma unroll
        for (int i = 0; i < M; ++i) O[i] = shfl_up_d(S[i], off);
        if (lane >= off) mv_acc<M, TR>(tb + TB::PL + d * M * M, O, S);
    }
}

// Block + grid carry propagation, executed by warp 0 of the CTA.
//   s_agg[w]: warp-local aggregates (zero-start prefix at the end of warp w).
//   Produces s_xw[w]: the exact state entering warp w's first chunk.
//   Decoupled look-back over this sequence's tiles (status 1 = aggregate,
//   2 = inclusive prefix), tiles ordered by ticket so predecessors are running.
template <int M, bool TR>
__device__ __forceinline__ void tile_carry(const double* __restrict__ tb, int lane,
                                           double (*s_agg)[M], double (*s_xw)[M],
                                           int jt, int64_t flat0, const double (&X0)[M],
                                           unsigned* flags, double* agg, double* incl, bool publish_incl) {
    using TB = Tab<M>;
    constexpr int M2 = M * M;
    double J[M];
#pragma unroll
    for (int i = 0; i < M; ++i) J[i] = (lane < NW) ? s_agg[lane][i] : 0.0;
#pragma unroll
    for (int d = 0; d < LOG_NW; ++d) {
        const int off = 1 << d;
        double O[M];
#pragma unroll
        for (int i = 0; i < M; ++i) O[i] = shfl_up_d(J[i], off);
        if (lane >= off && lane < NW) mv_acc<M, TR>(tb + TB::PW + d * M2, O, J);
    }
    double Jex[M], G[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        Jex[i] = shfl_up_d(J[i], 1);
        if (lane == 0) Jex[i] = 0.0;
        G[i] = shfl_d(J[i], NW - 1);           // tile aggregate (all lanes)
    }
    const int64_t me = flat0 + jt;
    double X[M];                               // exclusive prefix = state entering this tile
    if (jt == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) X[i] = X0[i];
    } else {
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) __stcg(agg + me * M + i, G[i]);
            st_release(flags + me, 1u);
        }
#pragma unroll
        for (int i = 0; i < M; ++i) X[i] = 0.0;
        int k = 0;                             // multiplier A_f^(TS k) of the next element
        for (int jj = jt - 1;; --jj, ++k) {
            unsigned f = 0;
            if (lane == 0) {
                const unsigned need = (k >= KLB) ? 2u : 1u;
                do { f = ld_acquire(flags + flat0 + jj); } while (f < need);
            }
            f = __shfl_sync(0xffffffffu, f, 0);
            const double* src = (f == 2u ? incl : agg) + (flat0 + jj) * M;
            double val[M];
#pragma unroll
            for (int i = 0; i < M; ++i) val[i] = __ldcg(src + i);
            if (k == 0) {
#pragma unroll
                for (int i = 0; i < M; ++i) X[i] += val[i];
            } else {
                mv_acc<M, TR>(tb + TB::PTK + (k - 1) * M2, val, X);
            }
            if (f == 2u) break;
        }
    }
    if (publish_incl && lane == 0) {
        double I[M];
#pragma unroll
        for (int i = 0; i < M; ++i) I[i] = G[i];
        mv_acc<M, TR>(tb + TB::PTK, X, I);     // I = A_f^TS X + G
#pragma unroll
        for (int i = 0; i < M; ++i) __stcg(incl + me * M + i, I[i]);
        st_release(flags + me, 2u);
    }
    if (lane < NW) {                           // state entering warp `lane`
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = Jex[i];
        mv_acc_lane<M, TR>(tb + TB::PWT, NW, lane, X, xw);
#pragma unroll
        for (int i = 0; i < M; ++i) s_xw[lane][i] = xw[i];
    }
}

// ---------------------------------------------------------------------------
// Forward: a2-a4.  One CTA per tile (NT*L samples of one sequence).
template <typename T, int M, int FORM>
__global__ void __launch_bounds__(NT) lti_fwd_kernel(const LtiFwdArgs p) {
    constexpr int L = Chunk<T>::L, TS = NT * L, W = Vec<T>::W;
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* xs = reinterpret_cast<T*>(smem_raw);
    T* us = xs + pidx<T>(TS);                  // DF: u tile
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];
    __shared__ unsigned s_ticket;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(p.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    const int64_t seq = (int64_t)(tk % (unsigned long long)p.B);
    const int jt = (int)(tk / (unsigned long long)p.B);
    const int64_t p0 = (int64_t)jt * TS;
    const T* xrow = static_cast<const T*>(p.x) + seq * p.Tlen;
    const double* tb = p.tab + seq * p.tab_stride;

    tile_load<T, TS>(xs, xrow, p0, p.Tlen, p.vec);
    T bc[M + 1], ac[M + 1], cc[M];
    load_coefs<T, M>(tb, bc, ac, cc);
    __syncthreads();

    // a2: local pass from the zero state over this thread's chunk.
    const int s0 = tid * L;
    T v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = T(0);
#pragma unroll
    for (int g = 0; g < L / W; ++g) {
        const V xv = *reinterpret_cast<const V*>(xs + pidx<T>(s0 + g * W));
#pragma unroll
        for (int e = 0; e < W; ++e) { T du; fwd_step<T, M, FORM>(v, vget(xv, e), bc, ac, du); }
    }
    // a3: carries in fp64.
    double S[M];
#pragma unroll
    for (int i = 0; i < M; ++i) S[i] = (double)v[i];
    warp_scan<M, false>(tb, lane, S);
    double E[M];
#pragma unroll
    for (int i = 0; i < M; ++i) { E[i] = shfl_up_d(S[i], 1); if (lane == 0) E[i] = 0.0; }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < M; ++i) s_agg[warp][i] = S[i];
    }
    __syncthreads();
    if (warp == 0) {
        double X0[M];
        const T* zi = static_cast<const T*>(p.zi);
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (zi != nullptr && jt == 0) ? (double)zi[seq * M + i] : 0.0;
        tile_carry<M, false>(tb, lane, s_agg, s_xw, jt, seq * (int64_t)p.ntiles, X0, p.flags, p.agg, p.incl,
                             jt + 1 < p.ntiles);
    }
    __syncthreads();
    // state entering this thread's chunk: E + A_f^(L lane) x_warp
    {
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
        mv_acc_lane<M, false>(tb + TB::PLT, 32, lane, xw, E);
    }
    T vin[M];
#pragma unroll
    for (int i = 0; i < M; ++i) { vin[i] = (T)E[i]; v[i] = vin[i]; }
    // zf = v(T): the thread holding sample T-1 walks its chunk up to it (before
    // the emit pass overwrites x with y).
    if (p.zf != nullptr) {
        const int64_t eL = p.Tlen - 1 - p0;
        if (eL >= s0 && eL < s0 + L) {
            T w2[M];
#pragma unroll
            for (int i = 0; i < M; ++i) w2[i] = vin[i];
            for (int n = s0; n <= (int)eL; ++n) { T du; fwd_step<T, M, FORM>(w2, xs[pidx<T>(n)], bc, ac, du); }
            T* zf = static_cast<T*>(p.zf) + seq * M;
#pragma unroll
            for (int i = 0; i < M; ++i) zf[i] = w2[i];
        }
    }
    // a4: re-run from the exact carry-in, emit y (and u for DF) in place.
#pragma unroll
    for (int g = 0; g < L / W; ++g) {
        V xv = *reinterpret_cast<const V*>(xs + pidx<T>(s0 + g * W));
        V uv;
#pragma unroll
        for (int e = 0; e < W; ++e) {
            T uu;
            const T yy = fwd_step<T, M, FORM>(v, vget(xv, e), bc, ac, uu);
            vset(xv, e, yy);
            vset(uv, e, uu);
        }
        *reinterpret_cast<V*>(xs + pidx<T>(s0 + g * W)) = xv;
        if constexpr (FORM == 0) *reinterpret_cast<V*>(us + pidx<T>(s0 + g * W)) = uv;
    }
    __syncthreads();
    T* yrow = static_cast<T*>(p.y) + seq * p.Tlen;
    tile_store<T, TS>(yrow, xs, p0, p.Tlen, p.vec);
    if constexpr (FORM == 0) {
        T* urow = static_cast<T*>(p.u) + seq * p.Tlen;
        tile_store<T, TS>(urow, us, p0, p.Tlen, p.vec);
    }
}

// ---------------------------------------------------------------------------
// Backward: a5-a7.  Tiles are aligned to the END of each sequence and processed
// last to first; inside a tile thread t owns chunk NT-1-t, walked backwards.
// TDF: smem dy | x | y.  DF: smem dy | u (with HALO samples of history).
template <typename T, int M, int FORM>
__global__ void __launch_bounds__(NT) lti_bwd_kernel(const LtiBwdArgs p) {
    constexpr int L = Chunk<T>::L, TS = NT * L, W = Vec<T>::W;
    constexpr int NG = 2 * M + 1;                       // gradient partial sums
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* dys = reinterpret_cast<T*>(smem_raw);
    T* s2 = dys + pidx<T>(TS);                          // TDF: x        DF: u (+HALO)
    T* s3 = s2 + pidx<T>(TS + HALO);                    // TDF: y
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];
    __shared__ double s_red[NW][NG];
    __shared__ unsigned s_ticket;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(p.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    const int64_t seq = (int64_t)(tk % (unsigned long long)p.B);
    const int jr = (int)(tk / (unsigned long long)p.B);          // 0 = last tile in time
    const int jt = p.ntiles - 1 - jr;                            // time index of the tile
    const int64_t p0 = p.Tlen - (int64_t)(jr + 1) * TS;          // may be < 0 (first tile)
    const double* tb = p.tab + seq * p.tab_stride;
    const int64_t roff = seq * p.Tlen;

    if (p.gy != nullptr) tile_load<T, TS>(dys, static_cast<const T*>(p.gy) + roff, p0, p.Tlen, p.vec);
    else for (int e = tid; e < TS; e += NT) dys[pidx<T>(e)] = T(0);
    if constexpr (FORM == 1) {
        tile_load<T, TS>(s2, static_cast<const T*>(p.x) + roff, p0, p.Tlen, p.vec);
        tile_load<T, TS>(s3, static_cast<const T*>(p.y) + roff, p0, p.Tlen, p.vec);
    }
    T bc[M + 1], ac[M + 1], cc[M];
    load_coefs<T, M>(tb, bc, ac, cc);
    __syncthreads();
    if constexpr (FORM == 0) {
        const T* urow = static_cast<const T*>(p.u) + roff;
        const T* zi = static_cast<const T*>(p.zi);
        // u(p0 - HALO .. p0 + TS) -> s2[pidx(e + HALO)]; u(-k) = zi[k-1] (DF state).
        for (int q = tid; q < (TS + HALO) / W; q += NT) {
            const int e = q * W - HALO;
            const int64_t pos = p0 + e;
            V val;
            if (p.vec && pos >= 0 && pos + W <= p.Tlen) {
                val = ldg_stream(reinterpret_cast<const V*>(urow + pos));
            } else {
#pragma unroll
                for (int r = 0; r < W; ++r) {
                    const int64_t pr = pos + r;
                    T s = T(0);
                    if (pr >= 0 && pr < p.Tlen) s = urow[pr];
                    else if (pr < 0 && pr >= -M && zi != nullptr) s = zi[seq * M + (-pr - 1)];
                    vset(val, r, s);
                }
            }
            *reinterpret_cast<V*>(s2 + pidx<T>(e + HALO)) = val;
        }
        __syncthreads();
    }

    const int c = NT - 1 - tid;          // chunk index within the tile (time order)
    const int s0 = c * L;
    // a5: local adjoint pass from the zero state, walking the chunk backwards.
    T d[M];
#pragma unroll
    for (int i = 0; i < M; ++i) d[i] = T(0);
#pragma unroll
    for (int g = L / W - 1; g >= 0; --g) {
        const V dv = *reinterpret_cast<const V*>(dys + pidx<T>(s0 + g * W));
#pragma unroll
        for (int e = W - 1; e >= 0; --e) {
            if constexpr (FORM == 1) adj_tdf_step<T, M>(d, vget(dv, e), ac);
            else adj_df_step<T, M>(d, vget(dv, e), bc, ac);
        }
    }
    // a6: carries (transposed powers), tiles last -> first.
    double S[M];
#pragma unroll
    for (int i = 0; i < M; ++i) S[i] = (double)d[i];
    warp_scan<M, true>(tb, lane, S);
    double E[M];
#pragma unroll
    for (int i = 0; i < M; ++i) { E[i] = shfl_up_d(S[i], 1); if (lane == 0) E[i] = 0.0; }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < M; ++i) s_agg[warp][i] = S[i];
    }
    __syncthreads();
    if (warp == 0) {
        double X0[M];
        const T* gzf = static_cast<const T*>(p.gzf);
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (gzf != nullptr && jr == 0) ? (double)gzf[seq * M + i] : 0.0;
        tile_carry<M, true>(tb, lane, s_agg, s_xw, jr, seq * (int64_t)p.ntiles, X0, p.flags, p.agg, p.incl,
                            jr + 1 < p.ntiles);
    }
    __syncthreads();
    {
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
        mv_acc_lane<M, true>(tb + TB::PLT, 32, lane, xw, E);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) d[i] = (T)E[i];
    T din[M];
#pragma unroll
    for (int i = 0; i < M; ++i) din[i] = d[i];

    // grad_zi = dz(-1) (Eq.9, A.3): the thread whose chunk holds n = 0 walks down
    // to it before the emit pass overwrites dy with dx.
    if (p.gzi != nullptr && p0 + s0 <= 0 && p0 + s0 + L > 0) {
        T w2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) w2[i] = din[i];
        for (int n = s0 + L - 1; n >= (int)(-p0); --n) {
            const T dy = dys[pidx<T>(n)];
            if constexpr (FORM == 1) adj_tdf_step<T, M>(w2, dy, ac);
            else (void)adj_df_step<T, M>(w2, dy, bc, ac);
        }
        T* gzi = static_cast<T*>(p.gzi) + seq * M;
#pragma unroll
        for (int i = 0; i < M; ++i) gzi[i] = w2[i];
    }
    // a7: re-run with the exact carry, emit dx, accumulate the coefficient sums.
    T G[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) G[k] = T(0);
    const bool has_neg = (p0 + s0) < 0;                 // chunk reaches before n = 0
#pragma unroll
    for (int g = L / W - 1; g >= 0; --g) {
        V dv = *reinterpret_cast<const V*>(dys + pidx<T>(s0 + g * W));
        if constexpr (FORM == 1) {
            const V xv = *reinterpret_cast<const V*>(s2 + pidx<T>(s0 + g * W));
            const V yv = *reinterpret_cast<const V*>(s3 + pidx<T>(s0 + g * W));
#pragma unroll
            for (int e = W - 1; e >= 0; --e) {
                const T dy = vget(dv, e), xx = vget(xv, e), yy = vget(yv, e);
                T dx = bc[0] * dy;
#pragma unroll
                for (int i = 0; i < M; ++i) dx = fma(cc[i], d[i], dx);     // Eq.8: c^T dz + b0 dy
#pragma unroll
                for (int i = 0; i < M; ++i) { G[i] = fma(d[i], xx, G[i]); G[M + i] = fma(d[i], yy, G[M + i]); }
                G[2 * M] = fma(dy, xx, G[2 * M]);
                vset(dv, e, dx);
                adj_tdf_step<T, M>(d, dy, ac);
            }
        } else {
#pragma unroll
            for (int e = W - 1; e >= 0; --e) {
                const int n = s0 + g * W + e;                 // tile-local time index
                const T dy = vget(dv, e);
                const T dx = adj_df_step<T, M>(d, dy, bc, ac); // dx(n), then d <- dz(n-1)
                const T gmask = (!has_neg || p0 + n >= 0) ? dx : T(0);
#pragma unroll
                for (int k = 0; k <= M; ++k) {
                    const T uk = s2[pidx<T>(n - k + HALO)];
                    G[k] = fma(dy, uk, G[k]);                          // Gb[k] = sum dy u(n-k)
                    if (k >= 1) G[M + k] = fma(gmask, uk, G[M + k]);  // Ga[k] = sum dx u(n-k)
                }
                vset(dv, e, dx);
            }
        }
        *reinterpret_cast<V*>(dys + pidx<T>(s0 + g * W)) = dv;   // dx in place
    }
    // block reduction of the partial sums (fp64, fixed order) -> per-tile partial
    if (p.want_coef) {
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            double s = (double)G[k];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) s_red[warp][k] = s;
        }
    }
    __syncthreads();
    if (p.want_coef && tid < NG) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += s_red[w][tid];
        p.partial[(seq * (int64_t)p.ntiles + jt) * NG + tid] = s;
    }
    if (p.gx != nullptr) tile_store<T, TS>(static_cast<T*>(p.gx) + roff, dys, p0, p.Tlen, p.vec);
}

// ---------------------------------------------------------------------------
// a8: gradient finalize.  One CTA per coefficient set: fixed-order fp64 sum of
// the per-tile partials (over the whole local batch for SHARED), then the
// chain rule from the state-space sums to (b', a') and the a0 un-normalisation.
//   TDF: G = [Gx(M), Gy(M), Gd]:  gb'_k = Gx[k-1], ga'_k = -Gy[k-1],
//        gb'_0 = Gd - sum_k a'_k Gx[k-1]            (Eqs.6,9 with C_f = e1)
//   DF : G = [Gb(0..M), Ga(1..M)]:  gb'_k = Gb[k],  ga'_k = -Ga[k]
//   gb = gb'/a0;  ga_k = ga'_k/a0 (k>=1);  ga_0 = -(b'.gb' + a'.ga')/a0.
template <typename T, int M, int FORM>
__global__ void __launch_bounds__(256) lti_finalize_kernel(const double* __restrict__ partial, int64_t tiles_per_set,
                                                           const double* __restrict__ tab, int64_t tab_stride,
                                                           T* __restrict__ gb, T* __restrict__ ga) {
    constexpr int NG = 2 * M + 1;
    using TB = Tab<M>;
    __shared__ double red[256];
    __shared__ double Gs[NG];
    const int set = blockIdx.x, tid = threadIdx.x;
    const double* part = partial + (int64_t)set * tiles_per_set * NG;
    for (int k = 0; k < NG; ++k) {
        double s = 0.0;
        for (int64_t t = tid; t < tiles_per_set; t += 256) s += part[t * NG + k];
        red[tid] = s;
        __syncthreads();
        for (int o = 128; o >= 1; o >>= 1) {
            if (tid < o) red[tid] += red[tid + o];
            __syncthreads();
        }
        if (tid == 0) Gs[k] = red[0];
        __syncthreads();
    }
    if (tid == 0) {
        const double* tb = tab + set * tab_stride + TB::COEF;
        const double* bn = tb;
        const double* an = tb + M + 1;
        double gbn[M + 1], gan[M + 1];
        gan[0] = 0.0;
        if (FORM == 1) {
            gbn[0] = Gs[2 * M];
            for (int k = 1; k <= M; ++k) {
                gbn[k] = Gs[k - 1];
                gan[k] = -Gs[M + k - 1];
                gbn[0] -= an[k] * Gs[k - 1];
            }
        } else {
            for (int k = 0; k <= M; ++k) gbn[k] = Gs[k];
            for (int k = 1; k <= M; ++k) gan[k] = -Gs[M + k];
        }
        const double a0 = tab[set * tab_stride + TB::A0];
        double s = 0.0;
        for (int k = 0; k <= M; ++k) s += bn[k] * gbn[k];
        for (int k = 1; k <= M; ++k) s += an[k] * gan[k];
        if (gb != nullptr)
            for (int k = 0; k <= M; ++k) gb[set * (M + 1) + k] = (T)(gbn[k] / a0);
        if (ga != nullptr) {
            ga[set * (M + 1)] = (T)(-s / a0);
            for (int k = 1; k <= M; ++k) ga[set * (M + 1) + k] = (T)(gan[k] / a0);
        }
    }
}

}  // namespace iirg
