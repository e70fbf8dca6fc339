// lti.cuh -- sm_100a kernels for batched LTI DF-II / TDF-II filtering and its
// closed-form backward (arXiv 2511.14390, Eqs.4-9).
//
// Time-parallel formulation (Eq.10) as a chunked scan:
//   * a tile of TS = NT*L samples of one sequence per CTA; each thread owns a
//     contiguous chunk of L samples and runs the recursion on it from a zero
//     state (local pass), giving the chunk aggregate w (the z of Eq.10's tuple);
//   * carries are combined in fp64 with constant transition powers: A_f^(L 2^d)
//     (warp Kogge-Stone over shuffles), A_f^(32 L 2^d) (across the warps), and
//     A_f^(k 32^l TS) (across tiles: a deterministic hierarchical look-back in
//     base 32, see tile_carry);
//   * each thread then re-runs its chunk from the exact carry-in state and
//     emits outputs (and, in the backward pass, the gradient partial sums).
// The backward pass is the same machine run in reverse time on the adjoint
// recursion (Eq.7), whose transition is A_f^T: it reads the same power tables
// transposed ("the backward of DF is a TDF run backwards").
#pragma once
#include "common.cuh"

namespace iirg {

constexpr int PREP_THREADS = 256;

// ---------------------------------------------------------------------------
// fp64 power tables of one coefficient set (computed on device, once per call).
template <int M> struct Tab {
    static constexpr int M2 = M * M;
    static constexpr int PL = 0;                       // A_f^(L 2^d), d = 0..4          [d][i][j]
    static constexpr int PW = PL + 5 * M2;             // A_f^(32L 2^d), d < LOG_NW      [d][i][j]
    static constexpr int PWT = PW + LOG_NW * M2;       // A_f^(32L w), w = 0..NW-1       [i][j][w]
    static constexpr int SMALL = PWT + NW * M2;        // [0, SMALL): staged in shared memory per CTA
    static constexpr int PLT = SMALL;                  // A_f^(L t),   t = 0..31         [i][j][t]
    static constexpr int PQ = PLT + 32 * M2;           // A_f^(k TS), k = 0..31          [i][j][k]
    static constexpr int PC = PQ + 32 * M2;            // A_f^(4 TS 2^d), d = 0..8 (carry pass) [d][i][j]
    static constexpr int COEF = PC + 9 * M2;           // b'[0..M], a'[0..M], c[0..M-1]
    static constexpr int A0 = COEF + 3 * M + 2;        // a0 (un-normalised)
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
// Same with one matrix per index t, stored element-major [i][j][stride] (lanes coalesce).
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

// Shared-memory versions (tables staged once per CTA).
template <int M, bool TR>
__device__ __forceinline__ void mv_acc_s(const double* P, const double (&v)[M], double (&acc)[M]) {
    if constexpr (M % 2 == 0) {
        // 128-bit shared loads (two matrix elements each); P is 16-byte aligned
        const double2* P2 = reinterpret_cast<const double2*>(P);
        if constexpr (!TR) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double s = acc[i];
#pragma unroll
                for (int j = 0; j < M; j += 2) {
                    const double2 q = P2[(i * M + j) / 2];
                    s = fma(q.x, v[j], s);
                    s = fma(q.y, v[j + 1], s);
                }
                acc[i] = s;
            }
        } else {
#pragma unroll
            for (int j = 0; j < M; ++j)
#pragma unroll
                for (int i = 0; i < M; i += 2) {
                    const double2 q = P2[(j * M + i) / 2];       // P[j][i], P[j][i+1] = (P^T)[i][j], [i+1][j]
                    acc[i] = fma(q.x, v[j], acc[i]);
                    acc[i + 1] = fma(q.y, v[j], acc[i + 1]);
                }
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double s = acc[i];
#pragma unroll
            for (int j = 0; j < M; ++j) s = fma(P[TR ? j * M + i : i * M + j], v[j], s);
            acc[i] = s;
        }
    }
}
template <int M, bool TR>
__device__ __forceinline__ void mv_acc_lane_s(const double* P, int stride, int t, const double (&v)[M],
                                              double (&acc)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double s = acc[i];
#pragma unroll
        for (int j = 0; j < M; ++j) s = fma(P[(TR ? j * M + i : i * M + j) * stride + t], v[j], s);
        acc[i] = s;
    }
}

// Programmatic dependent launch (PTX griddepcontrol).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---------------------------------------------------------------------------
// a1: coefficient prologue.  Normalise by a0, build A_f (DF: companion(a'),
// TDF: its transpose) and every fp64 power table by batched
// doubling (log depth): about 30 dependent matrix-product steps.
template <int M> struct PrepSlots {
    static constexpr int P1 = 0, PLT = 1 /* 33 */, YP = PLT + 33 /* 5 */, Q = YP + 5 /* 33 */, C = Q + 33 /* 9 */;
    static constexpr int N = C + 9;
    static constexpr size_t bytes() { return (size_t)N * M * M * sizeof(double); }
};

template <typename T, int M, int FORM>
__global__ void __launch_bounds__(PREP_THREADS) lti_prep_kernel(const T* __restrict__ b, const T* __restrict__ a,
                                                               int64_t coef_stride, double* __restrict__ tab,
                                                               int64_t tab_stride, int nlev) {
    // Let the dependent scan kernel start its prologue (tile loads, local pass);
    // it waits for this grid's completion (griddepcontrol.wait) before reading tables.
    pdl_launch_dependents();
    constexpr int L = Chunk<T>::L, M2 = M * M;
    using TB = Tab<M>;
    using S = PrepSlots<M>;
    extern __shared__ __align__(16) unsigned char prep_raw[];
    double* mat = reinterpret_cast<double*>(prep_raw);
    __shared__ double bn[M + 1], an[M + 1];
    const int set = blockIdx.x;
    const T* bb = b + set * coef_stride;
    const T* aa = a + set * coef_stride;
    double* tb = tab + set * tab_stride;
    const int tid = threadIdx.x;
    if (tid <= M) {
        const double a0 = (double)aa[0];
        bn[tid] = (double)bb[tid] / a0;
        an[tid] = (double)aa[tid] / a0;
    }
    __syncthreads();
    for (int e = tid; e < M2; e += PREP_THREADS) {
        const int i = e / M, j = e % M;
        const double Aij = (i == 0) ? -an[j + 1] : (i == j + 1 ? 1.0 : 0.0);  // companion(a'), row 0 = -a'
        const double Aji = (j == 0) ? -an[i + 1] : (j == i + 1 ? 1.0 : 0.0);
        mat[S::P1 * M2 + e] = (FORM == 0) ? Aij : Aji;
        const double id = (i == j) ? 1.0 : 0.0;
        mat[(S::PLT + 0) * M2 + e] = id;
        mat[(S::YP + 0) * M2 + e] = id;
        mat[S::Q * M2 + e] = id;
    }
    if (tid <= M) { tb[TB::COEF + tid] = bn[tid]; tb[TB::COEF + M + 1 + tid] = an[tid]; }
    if (tid < M) tb[TB::COEF + 2 * (M + 1) + tid] = bn[tid + 1] - an[tid + 1] * bn[0];
    if (tid == 0) tb[TB::A0] = (double)aa[0];
    __syncthreads();
    // batched product: for q < n: mat[dst(q)] = mat[lhs(q)] * mat[rhs(q)]
    auto mm_batch = [&](int n, auto dst, auto lhs, auto rhs) {
        constexpr int R = (16 * M2 + PREP_THREADS - 1) / PREP_THREADS;
        double r[R];
#pragma unroll
        for (int s = 0; s < R; ++s) {
            const int w = tid + s * PREP_THREADS;
            r[s] = 0.0;
            if (w < n * M2) {
                const int q = w / M2, e = w % M2, i = e / M, j = e % M;
                const double* A = mat + lhs(q) * M2;
                const double* B = mat + rhs(q) * M2;
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(A[i * M + k], B[k * M + j], acc);
                r[s] = acc;
            }
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < R; ++s) {
            const int w = tid + s * PREP_THREADS;
            if (w < n * M2) mat[dst(w / M2) * M2 + (w % M2)] = r[s];
        }
        __syncthreads();
    };
    // doubling: slot0 = X^0 and slot0+1 = X^1 known; fill slot0+2 .. slot0+2^nsteps
    auto powers = [&](int slot0, int nsteps) {
        for (int st = 0; st < nsteps; ++st) {
            const int h = 1 << st;  // known X^0..X^h; X^(h+1+q) = X^h X^(1+q), q < h
            mm_batch(h, [&](int q) { return slot0 + h + 1 + q; }, [&](int) { return slot0 + h; },
                     [&](int q) { return slot0 + 1 + q; });
        }
    };
    auto copy = [&](int dst, int src) {
        for (int e = tid; e < M2; e += PREP_THREADS) mat[dst * M2 + e] = mat[src * M2 + e];
        __syncthreads();
    };
    for (int p = 1; p < L; p *= 2)                                      // P1 = A_f^L
        mm_batch(1, [&](int) { return S::P1; }, [&](int) { return S::P1; }, [&](int) { return S::P1; });
    copy(S::PLT + 1, S::P1);
    powers(S::PLT, 5);                                                  // A_f^(L t), t = 0..32
    copy(S::YP + 1, S::PLT + 32);
    powers(S::YP, LOG_NW);                                              // A_f^(32 L w), w = 0..NW
    copy(S::Q + 1, S::YP + NW);                                         // A_f^TS
    powers(S::Q, 5);                                                    // A_f^(k TS), k = 0..32
    copy(S::C, S::Q + 4);                                               // A_f^(4 TS 2^d), d = 0..8
    for (int d = 1; d < 9; ++d)
        mm_batch(1, [&](int) { return S::C + d; }, [&](int) { return S::C + d - 1; }, [&](int) { return S::C + d - 1; });
    (void)nlev;
    // write out in the kernels' layouts
    for (int e = tid; e < M2; e += PREP_THREADS) {
        for (int d = 0; d < 5; ++d) tb[TB::PL + d * M2 + e] = mat[(S::PLT + (1 << d)) * M2 + e];
        for (int d = 0; d < LOG_NW; ++d) tb[TB::PW + d * M2 + e] = mat[(S::YP + (1 << d)) * M2 + e];
        for (int w = 0; w < NW; ++w) tb[TB::PWT + e * NW + w] = mat[(S::YP + w) * M2 + e];
    }
    for (int w = tid; w < 32 * M2; w += PREP_THREADS) {
        const int e = w / 32, t = w % 32;
        tb[TB::PLT + w] = mat[(S::PLT + t) * M2 + e];
    }
    (void)0;
    for (int w = tid; w < 32 * M2; w += PREP_THREADS) {
        const int e = w / 32, k = w % 32;
        tb[TB::PQ + w] = mat[(S::Q + k) * M2 + e];
    }
    for (int w = tid; w < 9 * M2; w += PREP_THREADS) tb[TB::PC + w] = mat[(S::C + w / M2) * M2 + (w % M2)];
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
// a8: gradient finalize, fused into the backward kernel.  Fixed-order fp64 sum
// of the per-tile partials (groups of 32 tiles, then the groups; over the
// whole local batch for SHARED), then the chain rule from the state-space sums
// to (b', a') and the a0 un-normalisation:
//   TDF: G = [Gx(M), Gy(M), Gd]:  gb'_k = Gx[k-1], ga'_k = -Gy[k-1],
//        gb'_0 = Gd - sum_k a'_k Gx[k-1]            (Eqs.6,9 with C_f = e1)
//   DF : G = [Gb(0..M), Ga(1..M)]:  gb'_k = Gb[k],  ga'_k = -Ga[k]
//   gb = gb'/a0;  ga_k = ga'_k/a0 (k>=1);  ga_0 = -(b'.gb' + a'.ga')/a0.
template <typename T, int M, int FORM>
__device__ __forceinline__ void chain_rule(const double* __restrict__ G, const double* __restrict__ tb, T* gb, T* ga) {
    using TB = Tab<M>;
    const double* bn = tb + TB::COEF;
    const double* an = tb + TB::COEF + M + 1;
    const double a0 = tb[TB::A0];
    double gbn[M + 1], gan[M + 1];
    gan[0] = 0.0;
    if constexpr (FORM == 1) {
        gbn[0] = G[2 * M];
        for (int k = 1; k <= M; ++k) {
            gbn[k] = G[k - 1];
            gan[k] = -G[M + k - 1];
            gbn[0] -= an[k] * G[k - 1];
        }
    } else {
        for (int k = 0; k <= M; ++k) gbn[k] = G[k];
        for (int k = 1; k <= M; ++k) gan[k] = -G[M + k];
    }
    double s = 0.0;
    for (int k = 0; k <= M; ++k) s += bn[k] * gbn[k];
    for (int k = 1; k <= M; ++k) s += an[k] * gan[k];
    if (gb != nullptr)
        for (int k = 0; k <= M; ++k) gb[k] = (T)(gbn[k] / a0);
    if (ga != nullptr) {
        ga[0] = (T)(-s / a0);
        for (int k = 1; k <= M; ++k) ga[k] = (T)(gan[k] / a0);
    }
}

// ---------------------------------------------------------------------------
// Kernel arguments.  Scan order: forward tiles in time order (tile jt covers
// [jt TS, (jt+1) TS)), backward tiles in reverse time order (tile jr covers
// [T - (jr+1) TS, T - jr TS)).  agg / carry are indexed [seq][scan index][M].
struct LtiFwdArgs {
    const void* b; const void* a; int64_t coef_stride;           // raw coefficients (local pass)
    const void* x; const void* zi; void* y; void* zf; void* u;    // u: DF tape signal
    const double* tab; int64_t tab_stride;                        // 0 for SHARED
    double* agg;                                                  // tile aggregates (phase 1)
    const double* carry;                                          // state entering each tile (phase 3)
    int64_t B, Tlen; int ntiles; int vec;
    unsigned long long* trace;                                    // debug: per-tile phase times
};

struct LtiBwdArgs {
    const void* gy; const void* gzf; const void* x; const void* y; const void* u; const void* zi;
    void* gx; void* gzi; void* gb; void* ga; int want_coef;
    double* partial; double* partial2; unsigned* gcnt; unsigned* scnt;   // fused finalize
    int64_t ncoef;
    const double* tab; int64_t tab_stride;
    double* agg; const double* carry;
    int64_t B, Tlen; int ntiles; int vec;
    unsigned long long* trace;
};

struct CarryArgs {
    const double* agg; double* carry;
    const void* x0; int x0_f64;                                   // zi (fwd) / grad_zf (bwd), may be NULL
    const double* tab; int64_t tab_stride;
    int64_t B; int ntiles;
};

// Normalised coefficients in T, straight from the caller's b, a (the same
// rounding as the prologue's fp64 b/a0, a/a0 cast to T).
template <typename T, int M>
__device__ __forceinline__ void raw_coefs(const T* __restrict__ b, const T* __restrict__ a, T (&bc)[M + 1],
                                          T (&ac)[M + 1]) {
    const double a0 = (double)__ldg(a);
#pragma unroll
    for (int k = 0; k <= M; ++k) { bc[k] = (T)((double)__ldg(b + k) / a0); ac[k] = (T)((double)__ldg(a + k) / a0); }
}
template <typename T, int M>
__device__ __forceinline__ void load_coefs(const double* __restrict__ tb, T (&bc)[M + 1], T (&ac)[M + 1], T (&cc)[M]) {
    using TB = Tab<M>;
#pragma unroll
    for (int k = 0; k <= M; ++k) { bc[k] = (T)__ldg(tb + TB::COEF + k); ac[k] = (T)__ldg(tb + TB::COEF + M + 1 + k); }
#pragma unroll
    for (int k = 0; k < M; ++k) cc[k] = (T)__ldg(tb + TB::COEF + 2 * (M + 1) + k);
}

// Stage the small power tables (PL | PW | PWT) of this tile's coefficient set.
template <int M>
__device__ __forceinline__ void stage_small(double* st, const double* __restrict__ tb) {
    for (int i = threadIdx.x; i < Tab<M>::SMALL; i += blockDim.x) st[i] = __ldg(tb + i);
}

// Warp-level inclusive Kogge-Stone scan of chunk aggregates in fp64:
//   S_t <- P^(2^d) S_{t-2^d} + S_t, P = A_f^L (TR: transposed for the adjoint).
template <int M, bool TR>
__device__ __forceinline__ void warp_scan(const double* st, int lane, double (&S)[M]) {
    using TB = Tab<M>;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int off = 1 << d;
        double O[M];
#pragma unroll
        for (int i = 0; i < M; ++i) O[i] = shfl_up_d(S[i], off);
        if (lane >= off) mv_acc_s<M, TR>(st + TB::PL + d * M * M, O, S);
    }
}

// Block level (warp 0): inclusive scan of the NW warp aggregates with
// A_f^(32 L 2^d); returns the exclusive prefix Jex (lanes < NW) and the tile
// aggregate G (all lanes).
template <int M, bool TR>
__device__ __forceinline__ void block_scan(const double* st, int lane, double (*s_agg)[M], double (&Jex)[M],
                                           double (&G)[M]) {
    using TB = Tab<M>;
    double J[M];
#pragma unroll
    for (int i = 0; i < M; ++i) J[i] = (lane < NW) ? s_agg[lane][i] : 0.0;
#pragma unroll
    for (int d = 0; d < LOG_NW; ++d) {
        const int off = 1 << d;
        double O[M];
#pragma unroll
        for (int i = 0; i < M; ++i) O[i] = shfl_up_d(J[i], off);
        if (lane >= off && lane < NW) mv_acc_s<M, TR>(st + TB::PW + d * M * M, O, J);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        Jex[i] = shfl_up_d(J[i], 1);
        if (lane == 0) Jex[i] = 0.0;
        G[i] = shfl_d(J[i], NW - 1);
    }
}

template <int M>
__device__ __forceinline__ void warp_sum(double (&v)[M]) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int i = 0; i < M; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

// Phase 1 needs only the tile aggregate, a reduction rather than a scan:
//   G = sum_t A_f^(L (NT-1-t)) w_t   (t in scan order; TR: transposed powers)
// lane term with A_f^(L (31-lane)), fixed butterfly sum per warp, then warp 0
// combines the NW warp sums with A_f^(32 L (NW-1-w)).  Writes G to dst.
template <int M, bool TR>
__device__ __forceinline__ void tile_reduce(const double* __restrict__ tb, const double* st, int lane, int warp,
                                            const double (&w)[M], double (*s_agg)[M], double* dst) {
    using TB = Tab<M>;
    double t[M];
#pragma unroll
    for (int i = 0; i < M; ++i) t[i] = 0.0;
    mv_acc_lane<M, TR>(tb + TB::PLT, 32, 31 - lane, w, t);
    warp_sum<M>(t);
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) s_agg[warp][i] = t[i];
    }
    __syncthreads();
    if (warp == 0) {
        double v[M], g[M];
#pragma unroll
        for (int i = 0; i < M; ++i) { v[i] = (lane < NW) ? s_agg[lane][i] : 0.0; g[i] = 0.0; }
        if (lane < NW) mv_acc_lane_s<M, TR>(st + TB::PWT, NW, NW - 1 - lane, v, g);
        warp_sum<M>(g);
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) dst[i] = g[i];
        }
    }
}

// ---------------------------------------------------------------------------
// Phase 2 (a3/a6 across tiles): per sequence, the exact state entering every
// tile from the tile aggregates:  X_0 = x0,  X_{j+1} = Q X_j + agg_j, Q = A_f^TS.
// One CTA per sequence walks the tiles in chunks of CARRY_CHUNK staged in
// shared memory; thread t owns CARRY_K consecutive tiles of a chunk: a Horner
// pass gives its aggregate, a block-wide Kogge-Stone scan with Q^(K 2^d)
// (fp64) gives its entering state, a second Horner pass writes X per tile.
// Fixed order throughout: bitwise deterministic.
constexpr int CARRY_THREADS = 256;
constexpr int CARRY_K = 4;
constexpr int CARRY_CHUNK = CARRY_THREADS * CARRY_K;

template <int M>
constexpr size_t carry_smem() { return (size_t)CARRY_CHUNK * M * sizeof(double); }

template <int M, bool TR>
__global__ void __launch_bounds__(CARRY_THREADS) lti_carry_kernel(const CarryArgs c) {
    constexpr int M2 = M * M;
    constexpr int NWC = CARRY_THREADS / 32;
    using TB = Tab<M>;
    extern __shared__ __align__(16) unsigned char carry_raw[];
    double* sA = reinterpret_cast<double*>(carry_raw);     // [CARRY_CHUNK][M] aggregates of a chunk
    __shared__ __align__(16) double sQ[M2];                 // Q = A_f^TS (transposed for the adjoint)
    __shared__ __align__(16) double sR[9][M2];              // Q^(K 2^d), d = 0..8
    __shared__ double sW[NWC][M];
    __shared__ double sX[M];
    pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t seq = blockIdx.x;
    const double* tb = c.tab + seq * c.tab_stride;
    const int n = c.ntiles;
    for (int e = tid; e < M2; e += CARRY_THREADS) {
        const int i = e / M, j = e % M;
        const int src = TR ? j * M + i : e;
        sQ[e] = __ldg(tb + TB::PQ + src * 32 + 1);                                  // A_f^TS
#pragma unroll
        for (int d = 0; d < 9; ++d) sR[d][e] = __ldg(tb + TB::PC + d * M2 + src); // A_f^(K TS 2^d)
    }
    static_assert(CARRY_K == 4, "PC tables hold A_f^(4 TS 2^d)");
    if (tid < M) {
        double x0 = 0.0;
        if (c.x0 != nullptr)
            x0 = c.x0_f64 ? static_cast<const double*>(c.x0)[seq * M + tid]
                          : (double)static_cast<const float*>(c.x0)[seq * M + tid];
        sX[tid] = x0;
    }
    __syncthreads();
    pdl_wait();                                                                 // phase-1 aggregates
    const double* agg = c.agg + seq * (int64_t)n * M;
    double* carry = c.carry + seq * (int64_t)n * M;
    for (int cs = 0; cs < n; cs += CARRY_CHUNK) {
        const int cnt = min(CARRY_CHUNK, n - cs);
        for (int e = tid; e < CARRY_CHUNK * M; e += CARRY_THREADS)
            sA[e] = (e < cnt * M) ? __ldcg(agg + (int64_t)cs * M + e) : 0.0;
        __syncthreads();
        // Horner over this thread's tiles
        double S[M];
#pragma unroll
        for (int i = 0; i < M; ++i) S[i] = 0.0;
#pragma unroll
        for (int q = 0; q < CARRY_K; ++q) {
            double Sn[M];
#pragma unroll
            for (int i = 0; i < M; ++i) Sn[i] = sA[(tid * CARRY_K + q) * M + i];
            mv_acc_s<M, false>(sQ, S, Sn);
#pragma unroll
            for (int i = 0; i < M; ++i) S[i] = Sn[i];
        }
        // inclusive scan across threads: warp level then across warps
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const int off = 1 << d;
            double O[M];
#pragma unroll
            for (int i = 0; i < M; ++i) O[i] = shfl_up_d(S[i], off);
            if (lane >= off) mv_acc_s<M, false>(sR[d], O, S);
        }
        if (lane == 31) {
#pragma unroll
            for (int i = 0; i < M; ++i) sW[warp][i] = S[i];
        }
        __syncthreads();
        if (warp == 0) {
            double Wv[M];
#pragma unroll
            for (int i = 0; i < M; ++i) Wv[i] = (lane < NWC) ? sW[lane][i] : 0.0;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int off = 1 << d;
                double O[M];
#pragma unroll
                for (int i = 0; i < M; ++i) O[i] = shfl_up_d(Wv[i], off);
                if (lane >= off && lane < NWC) mv_acc_s<M, false>(sR[5 + d], O, Wv);
            }
            double We[M];
#pragma unroll
            for (int i = 0; i < M; ++i) { We[i] = shfl_up_d(Wv[i], 1); if (lane == 0) We[i] = 0.0; }
            __syncwarp();
            if (lane < NWC) {
#pragma unroll
                for (int i = 0; i < M; ++i) sW[lane][i] = We[i];
            }
        }
        __syncthreads();
        // entering state: exclusive lane prefix + Q^(K lane) (warp prefix) + Q^(K tid) X_chunk
        double E[M], Y[M], Z[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            E[i] = shfl_up_d(S[i], 1);
            if (lane == 0) E[i] = 0.0;
            Y[i] = sW[warp][i];
            Z[i] = sX[i];
        }
#pragma unroll
        for (int d = 0; d < 8; ++d) {                 // Z <- Q^(K tid) X,  Y <- Q^(K lane) Y
            if ((tid >> d) & 1) {
                double Zn[M];
#pragma unroll
                for (int i = 0; i < M; ++i) Zn[i] = 0.0;
                mv_acc_s<M, false>(sR[d], Z, Zn);
#pragma unroll
                for (int i = 0; i < M; ++i) Z[i] = Zn[i];
            }
            if (d < 5 && ((lane >> d) & 1)) {
                double Yn[M];
#pragma unroll
                for (int i = 0; i < M; ++i) Yn[i] = 0.0;
                mv_acc_s<M, false>(sR[d], Y, Yn);
#pragma unroll
                for (int i = 0; i < M; ++i) Y[i] = Yn[i];
            }
        }
#pragma unroll
        for (int i = 0; i < M; ++i) E[i] += Y[i] + Z[i];
        __syncthreads();                                        // everyone has read sX / sW
        // second Horner pass: state entering each tile
#pragma unroll
        for (int q = 0; q < CARRY_K; ++q) {
            const int t = tid * CARRY_K + q;
            double Sn[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                if (t < cnt) carry[(int64_t)(cs + t) * M + i] = E[i];
                Sn[i] = sA[t * M + i];
            }
            mv_acc_s<M, false>(sQ, E, Sn);
#pragma unroll
            for (int i = 0; i < M; ++i) E[i] = Sn[i];
        }
        if (tid == CARRY_THREADS - 1) {                          // state at the end of the chunk
#pragma unroll
            for (int i = 0; i < M; ++i) sX[i] = E[i];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
template <typename T, int M>
struct Smem {
    static constexpr int TS = NT * Chunk<T>::L;
    static constexpr int PT = pidx<T>(TS);               // one padded tile
    static constexpr int PTH = pidx<T>(TS + HALO);       // padded tile with u history
    static constexpr size_t tab_bytes = ((size_t)Tab<M>::SMALL * 8 + 15) / 16 * 16;
    // forward: 2 stages of x (-> y), plus the u tile for DF emits
    static constexpr size_t fwd(int form, int phase) {
        return tab_bytes + (size_t)(2 * PT + (form == 0 && phase == 3 ? PT : 0)) * sizeof(T);
    }
    // backward: 2 stages of dy (-> dx) [+ one x, y (TDF) or u (DF) tile in phase 3]
    static constexpr int bwd_xy(int form, int phase) { return phase == 3 ? PTH + (form == 1 ? PT : 0) : 0; }
    static constexpr size_t bwd(int form, int phase) {
        return tab_bytes + (size_t)(2 * PT + bwd_xy(form, phase)) * sizeof(T);
    }
};

// Per-CTA coefficient state (tables staged in shared memory, coefficients in registers).
template <typename T, int M>
struct CoefRegs {
    T bc[M + 1], ac[M + 1], cc[M];
};

// ---------------------------------------------------------------------------
// Forward, phases 1 and 3 (a2-a4).  Persistent CTAs stride over the tiles
// (tile = seq * ntiles + jt, TS samples each) and double-buffer them: tile k+1
// streams into shared memory (cp.async) while tile k is scanned.
//   PHASE 1: local pass, warp + block scans -> tile aggregate (no outputs).
//   PHASE 3: the same scans again (x now comes from L2), plus the state
//            entering the tile from phase 2 -> exact per-thread carry-in,
//            re-run and emit y (and u for DF), zf.
template <typename T, int M, int FORM, int PHASE>
__global__ void __launch_bounds__(NT) lti_fwd_kernel(const LtiFwdArgs p) {
    constexpr int L = Chunk<T>::L, TS = NT * L, W = Vec<T>::W;
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    using SM = Smem<T, M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* st = reinterpret_cast<double*>(smem_raw);
    T* xb = reinterpret_cast<T*>(smem_raw + SM::tab_bytes);     // 2 stages, x -> y in place
    T* us = xb + 2 * SM::PT;                                      // DF: u tile (phase 3)
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];

    pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntot = p.B * (int64_t)p.ntiles;
    int64_t tile = blockIdx.x;
    if (tile < ntot) {
        const int64_t sq = tile / p.ntiles;
        tile_load_async<T, TS>(xb, static_cast<const T*>(p.x) + sq * p.Tlen, (tile - sq * p.ntiles) * TS,
                               p.Tlen, p.vec);
    }
    cp_async_commit();
    int64_t staged = -1;
    bool waited = false;
    T bc[M + 1], ac[M + 1], cc[M];
    for (int it = 0; tile < ntot; ++it, tile += gridDim.x) {
        const int64_t next = tile + gridDim.x;
        if (next < ntot) {
            const int64_t sq = next / p.ntiles;
            tile_load_async<T, TS>(xb + ((it + 1) & 1) * SM::PT, static_cast<const T*>(p.x) + sq * p.Tlen,
                                   (next - sq * p.ntiles) * TS, p.Tlen, p.vec);
        }
        cp_async_commit();
        const int64_t seq = tile / p.ntiles;
        const int jt = (int)(tile - seq * p.ntiles);
        const int64_t p0 = (int64_t)jt * TS;
        const double* tb = p.tab + seq * p.tab_stride;
        T* xs = xb + (it & 1) * SM::PT;
        const int64_t set = p.tab_stride == 0 ? 0 : seq;
        if (set != staged) {
            // previous grid: phase 1 waits for the prologue (tables), phase 3 for phase 2
            if (!waited) { pdl_wait(); waited = true; }
            stage_small<M>(st, tb);
            load_coefs<T, M>(tb, bc, ac, cc);
            staged = set;
        }
        IIRG_TRACE(p.trace, tile, 0);
        cp_async_wait<1>();
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
        IIRG_TRACE(p.trace, tile, 1);
        // a3: carries in fp64
        double S[M];
#pragma unroll
        for (int i = 0; i < M; ++i) S[i] = (double)v[i];
        if constexpr (PHASE == 1) {
            tile_reduce<M, false>(tb, st, lane, warp, S, s_agg, p.agg + tile * M);
            IIRG_TRACE(p.trace, tile, 2);
        } else {
            warp_scan<M, false>(st, lane, S);
            if (lane == 31) {
#pragma unroll
                for (int i = 0; i < M; ++i) s_agg[warp][i] = S[i];
            }
            __syncthreads();
            double E[M];
#pragma unroll
            for (int i = 0; i < M; ++i) { E[i] = shfl_up_d(S[i], 1); if (lane == 0) E[i] = 0.0; }
            if (warp == 0) {
                double Jex[M], G[M];
                block_scan<M, false>(st, lane, s_agg, Jex, G);
                if (lane < NW) {                           // state entering warp `lane`
                    double X[M], xw[M];
#pragma unroll
                    for (int i = 0; i < M; ++i) { X[i] = p.carry[tile * M + i]; xw[i] = Jex[i]; }
                    mv_acc_lane_s<M, false>(st + TB::PWT, NW, lane, X, xw);
#pragma unroll
                    for (int i = 0; i < M; ++i) s_xw[lane][i] = xw[i];
                }
            }
            __syncthreads();
            IIRG_TRACE(p.trace, tile, 2);
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
            // zf = v(T): the thread holding sample T-1 walks its chunk up to it.
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
            IIRG_TRACE(p.trace, tile, 3);
            T* yrow = static_cast<T*>(p.y) + seq * p.Tlen;
            tile_store<T, TS>(yrow, xs, p0, p.Tlen, p.vec);
            if constexpr (FORM == 0) {
                T* urow = static_cast<T*>(p.u) + seq * p.Tlen;
                tile_store<T, TS>(urow, us, p0, p.Tlen, p.vec);
            }
        }
        __syncthreads();                                  // this stage may be refilled
    }
    if (!waited) pdl_wait();
}

// ---------------------------------------------------------------------------
// Backward, phases 1 and 3 (a5-a8).  Tiles are aligned to the END of each
// sequence; scan index jr = 0 is the last tile in time; inside a tile thread t
// owns chunk NT-1-t, walked backwards.  Persistent, double-buffered like the
// forward kernel.
//   PHASE 1: local adjoint pass over dy, warp + block scans -> tile aggregate.
//   PHASE 3: dy again (from L2) plus x, y (TDF) or u (DF): carry-in from phase
//            2, re-run, emit dx and grad_zi, coefficient partial sums, fused a8.
template <typename T, int M, int FORM>
__device__ __forceinline__ void bwd_load_u(const LtiBwdArgs& p, int64_t seq, int64_t p0, T* s2) {
    constexpr int TS = NT * Chunk<T>::L, W = Vec<T>::W;
    using V = typename Vec<T>::type;
    // u(p0 - HALO .. p0 + TS) -> s2[pidx(e + HALO)]; u(-k) = zi[k-1] (DF state).
    const T* urow = static_cast<const T*>(p.u) + seq * p.Tlen;
    const T* zi = static_cast<const T*>(p.zi);
    for (int q = threadIdx.x; q < (TS + HALO) / W; q += NT) {
        const int e = q * W - HALO;
        const int64_t pos = p0 + e;
        if (p.vec && pos >= 0 && pos + W <= p.Tlen) {
            cp_async16(s2 + pidx<T>(e + HALO), urow + pos, 16u);
        } else {
            V val;
#pragma unroll
            for (int r = 0; r < W; ++r) {
                const int64_t pr = pos + r;
                T s = T(0);
                if (pr >= 0 && pr < p.Tlen) s = urow[pr];
                else if (pr < 0 && pr >= -M && zi != nullptr) s = zi[seq * M + (-pr - 1)];
                vset(val, r, s);
            }
            *reinterpret_cast<V*>(s2 + pidx<T>(e + HALO)) = val;
        }
    }
}

template <typename T>
__device__ __forceinline__ void bwd_issue_dy(const LtiBwdArgs& p, int64_t tile, T* dys) {
    constexpr int TS = NT * Chunk<T>::L;
    const int64_t seq = tile / p.ntiles;
    const int jr = (int)(tile - seq * p.ntiles);
    const int64_t p0 = p.Tlen - (int64_t)(jr + 1) * TS;
    if (p.gy != nullptr) tile_load_async<T, TS>(dys, static_cast<const T*>(p.gy) + seq * p.Tlen, p0, p.Tlen, p.vec);
    else for (int e = threadIdx.x; e < TS; e += NT) dys[pidx<T>(e)] = T(0);
}
template <typename T, int M, int FORM>
__device__ __forceinline__ void bwd_issue_xy(const LtiBwdArgs& p, int64_t tile, T* s2, T* s3) {
    constexpr int TS = NT * Chunk<T>::L;
    const int64_t seq = tile / p.ntiles;
    const int jr = (int)(tile - seq * p.ntiles);
    const int64_t p0 = p.Tlen - (int64_t)(jr + 1) * TS;
    const int64_t roff = seq * p.Tlen;
    if constexpr (FORM == 1) {
        tile_load_async<T, TS>(s2, static_cast<const T*>(p.x) + roff, p0, p.Tlen, p.vec);
        tile_load_async<T, TS>(s3, static_cast<const T*>(p.y) + roff, p0, p.Tlen, p.vec);
    } else {
        bwd_load_u<T, M, FORM>(p, seq, p0, s2);
    }
}

template <typename T, int M, int FORM, int PHASE>
__global__ void __launch_bounds__(NT) lti_bwd_kernel(const LtiBwdArgs p) {
    constexpr int L = Chunk<T>::L, TS = NT * L, W = Vec<T>::W;
    constexpr int NG = 2 * M + 1;                       // gradient partial sums
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    using SM = Smem<T, M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* st = reinterpret_cast<double*>(smem_raw);
    T* sb = reinterpret_cast<T*>(smem_raw + SM::tab_bytes);    // 2 stages of dy -> dx
    T* s2 = sb + 2 * SM::PT;                                   // TDF: x        DF: u (+HALO)
    T* s3 = s2 + SM::PTH;                                      // TDF: y
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];
    __shared__ double s_red[NW][NG];
    __shared__ double s_G[NG];
    __shared__ unsigned s_fin;

    pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntot = p.B * (int64_t)p.ntiles;
    int64_t tile = blockIdx.x;
    if (tile < ntot) bwd_issue_dy<T>(p, tile, sb);
    cp_async_commit();
    int64_t staged = -1;
    bool waited = false;
    T bc[M + 1], ac[M + 1], cc[M];
    for (int it = 0; tile < ntot; ++it, tile += gridDim.x) {
        const int64_t next = tile + gridDim.x;
        // groups in flight: dy(this) [earlier], x/y(this), dy(next)
        if constexpr (PHASE == 3) bwd_issue_xy<T, M, FORM>(p, tile, s2, s3);
        cp_async_commit();
        if (next < ntot) bwd_issue_dy<T>(p, next, sb + ((it + 1) & 1) * SM::PT);
        cp_async_commit();
        const int64_t seq = tile / p.ntiles;
        const int jr = (int)(tile - seq * p.ntiles);                 // 0 = last tile in time
        const int jt = p.ntiles - 1 - jr;                            // time index of the tile
        const int64_t p0 = p.Tlen - (int64_t)(jr + 1) * TS;          // may be < 0 (first tile)
        const double* tb = p.tab + seq * p.tab_stride;
        const int64_t roff = seq * p.Tlen;
        T* dys = sb + (it & 1) * SM::PT;
        const int64_t set = p.tab_stride == 0 ? 0 : seq;
        if (set != staged) {                   // tables live in the tape (written by the forward)
            stage_small<M>(st, tb);
            load_coefs<T, M>(tb, bc, ac, cc);
            staged = set;
        }
        IIRG_TRACE(p.trace, tile, 0);
        cp_async_wait<2>();                                          // dy of this tile
        __syncthreads();

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
        IIRG_TRACE(p.trace, tile, 1);
        // a6: carries (transposed powers)
        double S[M];
#pragma unroll
        for (int i = 0; i < M; ++i) S[i] = (double)d[i];
        if constexpr (PHASE == 1) {
            tile_reduce<M, true>(tb, st, lane, warp, S, s_agg, p.agg + tile * M);
            IIRG_TRACE(p.trace, tile, 2);
        } else {
            warp_scan<M, true>(st, lane, S);
            if (lane == 31) {
#pragma unroll
                for (int i = 0; i < M; ++i) s_agg[warp][i] = S[i];
            }
            __syncthreads();
            double E[M];
#pragma unroll
            for (int i = 0; i < M; ++i) { E[i] = shfl_up_d(S[i], 1); if (lane == 0) E[i] = 0.0; }
            if (!waited) { pdl_wait(); waited = true; }          // tile carries of phase 2
            if (warp == 0) {
                double Jex[M], G[M];
                block_scan<M, true>(st, lane, s_agg, Jex, G);
                if (lane < NW) {                                 // state entering warp `lane`
                    double X[M], xw[M];
#pragma unroll
                    for (int i = 0; i < M; ++i) { X[i] = p.carry[tile * M + i]; xw[i] = Jex[i]; }
                    mv_acc_lane_s<M, true>(st + TB::PWT, NW, lane, X, xw);
#pragma unroll
                    for (int i = 0; i < M; ++i) s_xw[lane][i] = xw[i];
                }
            }
            __syncthreads();
            IIRG_TRACE(p.trace, tile, 2);
            {
                double xw[M];
#pragma unroll
                for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
                mv_acc_lane<M, true>(tb + TB::PLT, 32, lane, xw, E);
            }
            T din[M];
#pragma unroll
            for (int i = 0; i < M; ++i) { din[i] = (T)E[i]; d[i] = din[i]; }
            cp_async_wait<1>();                                      // x, y / u of this tile
            __syncthreads();

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
            T Gs[NG];
#pragma unroll
            for (int k = 0; k < NG; ++k) Gs[k] = T(0);
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
                        for (int i = 0; i < M; ++i) { Gs[i] = fma(d[i], xx, Gs[i]); Gs[M + i] = fma(d[i], yy, Gs[M + i]); }
                        Gs[2 * M] = fma(dy, xx, Gs[2 * M]);
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
                            Gs[k] = fma(dy, uk, Gs[k]);                          // Gb[k] = sum dy u(n-k)
                            if (k >= 1) Gs[M + k] = fma(gmask, uk, Gs[M + k]);  // Ga[k] = sum dx u(n-k)
                        }
                        vset(dv, e, dx);
                    }
                }
                *reinterpret_cast<V*>(dys + pidx<T>(s0 + g * W)) = dv;   // dx in place
            }
            // warp reduction of the partial sums (fp64, fixed order)
            if (p.want_coef) {
#pragma unroll
                for (int k = 0; k < NG; ++k) {
                    double s = (double)Gs[k];
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    if (lane == 0) s_red[warp][k] = s;
                }
            }
            __syncthreads();
            IIRG_TRACE(p.trace, tile, 3);
            if (p.gx != nullptr) tile_store<T, TS>(static_cast<T*>(p.gx) + roff, dys, p0, p.Tlen, p.vec);

            if (p.want_coef) {
                // fused a8: group of 32 tiles -> group sum; last group of the set -> chain rule.
                const bool shared = p.ncoef == 1;
                const int64_t per_set = shared ? p.B * p.ntiles : p.ntiles;
                const int64_t cset = shared ? 0 : seq;
                const int64_t li = shared ? seq * p.ntiles + jt : jt;          // index within the set
                const int64_t gi = li >> 5;
                const int64_t ngroups = (per_set + 31) >> 5;
                const int gsize = (int)min((int64_t)32, per_set - (gi << 5));
                double* part = p.partial + cset * per_set * NG;
                double* part2 = p.partial2 + cset * ngroups * NG;
                if (tid < NG) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < NW; ++w) s += s_red[w][tid];
                    __stcg(part + li * NG + tid, s);
                    __threadfence();
                }
                __syncthreads();
                if (tid == 0) s_fin = (atomicAdd(p.gcnt + cset * ngroups + gi, 1u) == (unsigned)gsize - 1u) ? 1u : 0u;
                __syncthreads();
                if (s_fin) {                                   // last tile of its group
                    __threadfence();
                    if (tid < NG) {
                        double s = 0.0;
                        for (int t = 0; t < gsize; ++t) s += __ldcg(part + ((gi << 5) + t) * NG + tid);
                        __stcg(part2 + gi * NG + tid, s);
                        __threadfence();
                    }
                    __syncthreads();
                    if (tid == 0) {
                        p.gcnt[cset * ngroups + gi] = 0u;
                        s_fin = (atomicAdd(p.scnt + cset, 1u) == (unsigned)ngroups - 1u) ? 2u : 0u;
                    }
                    __syncthreads();
                    if (s_fin == 2u) {                          // last group of the set
                        __threadfence();
                        if (tid < NG) {
                            double s = 0.0;
                            for (int64_t g2 = 0; g2 < ngroups; ++g2) s += __ldcg(part2 + g2 * NG + tid);
                            s_G[tid] = s;
                        }
                        __syncthreads();
                        if (tid == 0) {
                            chain_rule<T, M, FORM>(s_G, tb,
                                                   p.gb == nullptr ? nullptr : static_cast<T*>(p.gb) + cset * (M + 1),
                                                   p.ga == nullptr ? nullptr : static_cast<T*>(p.ga) + cset * (M + 1));
                            p.scnt[cset] = 0u;
                        }
                    }
                }
            }
        }
        __syncthreads();                                  // this stage may be refilled
    }
    if (!waited) pdl_wait();
}

}  // namespace iirg
