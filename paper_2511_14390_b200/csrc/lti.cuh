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

constexpr int LEVELS = 4;          // hierarchical carry levels: ntiles <= 32^4 per sequence
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
    static constexpr int PQ = PLT + 32 * M2;           // A_f^(k 32^l TS), k = 0..31     [l][i][j][k]
    static constexpr int COEF = PQ + LEVELS * 32 * M2; // b'[0..M], a'[0..M], c[0..M-1]
    static constexpr int A0 = COEF + 3 * M + 2;        // a0 (un-normalised)
    static constexpr int SIZE = (A0 + 1 + 31) / 32 * 32;
    // [0, STAGE) is staged in shared memory: the small tables always, the
    // per-lane carry-in powers A_f^(L t) for M <= 4 and the look-back powers of
    // levels 0, 1 for M <= 2 (smaller orders: the round trips they save sit on
    // every tile's critical path; larger orders: they would cost occupancy)
    static constexpr int STAGE = M <= 2 ? PQ + 2 * 32 * M2 : (M <= 4 ? PQ : SMALL);
};

// acc += P v with P = A_f^(L t) (the carry into lane t's chunk), staged or global.
template <int M, bool TR>
__device__ __forceinline__ void mv_plt(const double* st, const double* __restrict__ tb, int t, const double (&v)[M],
                                       double (&acc)[M]);
// acc += P v with P = A_f^(k 32^l TS) (look-back level l), staged or global.
template <int M, bool TR>
__device__ __forceinline__ void mv_pq(const double* st, const double* __restrict__ tb, int l, int k,
                                      const double (&v)[M], double (&acc)[M]);

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

template <int M, bool TR>
__device__ __forceinline__ void mv_plt(const double* st, const double* __restrict__ tb, int t, const double (&v)[M],
                                       double (&acc)[M]) {
    if constexpr (Tab<M>::STAGE > Tab<M>::PLT) mv_acc_lane_s<M, TR>(st + Tab<M>::PLT, 32, t, v, acc);
    else mv_acc_lane<M, TR>(tb + Tab<M>::PLT, 32, t, v, acc);
}
template <int M, bool TR>
__device__ __forceinline__ void mv_pq(const double* st, const double* __restrict__ tb, int l, int k,
                                      const double (&v)[M], double (&acc)[M]) {
    constexpr int M2 = M * M;
    if (Tab<M>::STAGE >= Tab<M>::PQ + (l + 1) * 32 * M2) mv_acc_lane_s<M, TR>(st + Tab<M>::PQ + l * 32 * M2, 32, k, v, acc);
    else mv_acc_lane<M, TR>(tb + Tab<M>::PQ + l * 32 * M2, 32, k, v, acc);
}

// Programmatic dependent launch (PTX griddepcontrol).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---------------------------------------------------------------------------
// a1: coefficient prologue.  Normalise by a0, build A_f (DF: companion(a'),
// TDF: its transpose) and every fp64 power table by batched
// doubling (log depth): about 30 dependent matrix-product steps.
template <int M> struct PrepSlots {
    static constexpr int P1 = 0, PLT = 1 /* 33 */, YP = PLT + 33 /* 5 */, Q = YP + 5 /* LEVELS x 33 */;
    static constexpr int N = Q + LEVELS * 33;
    static constexpr size_t bytes() { return (size_t)N * M * M * sizeof(double); }
};

// FORM 0 / 1: companion(a') (DF) or its transpose (TDF) from (b, a); FORM 2: the
// dense A itself (the bare recurrence, rec.cuh), given row-major in `a`.  LC is
// the chunk length of the consuming scan kernel.
template <typename T, int M, int FORM, int LC = Chunk<T, M>::L>
__global__ void __launch_bounds__(PREP_THREADS) lti_prep_kernel(const T* __restrict__ b, const T* __restrict__ a,
                                                               int64_t coef_stride, double* __restrict__ tab,
                                                               int64_t tab_stride, int nlev,
                                                               unsigned long long* span = nullptr) {
    // Let the dependent scan kernel start its prologue (tile loads, local pass);
    // it waits for this grid's completion (griddepcontrol.wait) before reading tables.
    pdl_launch_dependents();
    span_enter(span);
    constexpr int L = LC, M2 = M * M;
    using TB = Tab<M>;
    using S = PrepSlots<M>;
    extern __shared__ __align__(16) unsigned char prep_raw[];
    double* mat = reinterpret_cast<double*>(prep_raw);
    __shared__ double bn[M + 1], an[M + 1];
    const int set = blockIdx.x;
    const T* bb = FORM == 2 ? nullptr : b + set * coef_stride;
    const T* aa = a + set * coef_stride;
    double* tb = tab + set * tab_stride;
    const int tid = threadIdx.x;
    if (FORM != 2 && tid <= M) {
        const double a0 = (double)aa[0];
        bn[tid] = (double)bb[tid] / a0;
        an[tid] = (double)aa[tid] / a0;
    }
    __syncthreads();
    for (int e = tid; e < M2; e += PREP_THREADS) {
        const int i = e / M, j = e % M;
        if constexpr (FORM == 2) {
            mat[S::P1 * M2 + e] = (double)aa[e];
        } else {
            const double Aij = (i == 0) ? -an[j + 1] : (i == j + 1 ? 1.0 : 0.0);  // companion(a'), row 0 = -a'
            const double Aji = (j == 0) ? -an[i + 1] : (j == i + 1 ? 1.0 : 0.0);
            mat[S::P1 * M2 + e] = (FORM == 0) ? Aij : Aji;
        }
        const double id = (i == j) ? 1.0 : 0.0;
        mat[(S::PLT + 0) * M2 + e] = id;
        mat[(S::YP + 0) * M2 + e] = id;
        for (int l = 0; l < LEVELS; ++l) mat[(S::Q + l * 33) * M2 + e] = id;
    }
    if constexpr (FORM != 2) {
        if (tid <= M) { tb[TB::COEF + tid] = bn[tid]; tb[TB::COEF + M + 1 + tid] = an[tid]; }
        if (tid < M) tb[TB::COEF + 2 * (M + 1) + tid] = bn[tid + 1] - an[tid + 1] * bn[0];
        if (tid == 0) tb[TB::A0] = (double)aa[0];
    }
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
    for (int l = 0; l < nlev; ++l) {                                    // A_f^(k 32^l TS), k = 0..32
        powers(S::Q + l * 33, 5);
        if (l + 1 < LEVELS) copy(S::Q + (l + 1) * 33 + 1, S::Q + l * 33 + 32);
    }
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
    for (int w = tid; w < nlev * 32 * M2; w += PREP_THREADS) {
        const int l = w / (32 * M2), r = w % (32 * M2), e = r / 32, k = r % 32;
        tb[TB::PQ + w] = mat[(S::Q + l * 33 + k) * M2 + e];
    }
    __syncthreads();
    span_exit(span);
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

// Forward TDF-II, fp32, two samples per step with paired FMAs.  Unrolling by two
// turns the state shift into a shift by one PAIR, so with the state held as
// pairs V_k = (v_2k, v_2k+1) (zero-padded to an even length) every update is
// aligned:  v''_i = v_(i+2) + b_(i+2) x0 - a_(i+2) y0 + b_(i+1) x1 - a_(i+1) y1
// (the difference equation of Eqs.4-5 applied twice), four FFMA2 per pair with
// the sample values as broadcast operands, plus the two outputs
// y0 = b0 x0 + v0,  y1 = b0 x1 + (v1 + b1 x0 - a1 y0).
// 1.5 + M instructions per sample instead of 2M + 1.
template <int M> struct Tdf2 {
    static constexpr int NP = (M + 1) / 2;
    unsigned long long B2[NP], NA2[NP], B1[NP], NA1[NP];
    float b0, b1, na1;
    __device__ __forceinline__ void init(const float (&bc)[M + 1], const float (&ac)[M + 1]) {
        auto cb = [&](int k) { return k <= M ? bc[k] : 0.f; };
        auto ca = [&](int k) { return k <= M ? -ac[k] : 0.f; };
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            B2[k] = pk2(cb(2 * k + 2), cb(2 * k + 3));
            NA2[k] = pk2(ca(2 * k + 2), ca(2 * k + 3));
            B1[k] = pk2(cb(2 * k + 1), cb(2 * k + 2));
            NA1[k] = pk2(ca(2 * k + 1), ca(2 * k + 2));
        }
        b0 = bc[0]; b1 = bc[1]; na1 = -ac[1];
    }
    // the same pairs from a table laid out [B2 | NA2 | B1 | NA1], stride jp pairs (lti2.cuh W)
    __device__ __forceinline__ void init_pairs(const float* w, int jp, const float (&bc)[M + 1], const float (&ac)[M + 1]) {
        const unsigned long long* wp = reinterpret_cast<const unsigned long long*>(w);
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            B2[k] = wp[k];
            NA2[k] = wp[jp + k];
            B1[k] = wp[2 * jp + k];
            NA1[k] = wp[3 * jp + k];
        }
        b0 = bc[0]; b1 = bc[1]; na1 = -ac[1];
    }
};
template <int M>
__device__ __forceinline__ void tdf2_pack(const float (&v)[M], unsigned long long (&V)[Tdf2<M>::NP]) {
#pragma unroll
    for (int k = 0; k < Tdf2<M>::NP; ++k) V[k] = pk2(v[2 * k], 2 * k + 1 < M ? v[2 * k + 1] : 0.f);
}
template <int M>
__device__ __forceinline__ void tdf2_unpack(const unsigned long long (&V)[Tdf2<M>::NP], float (&v)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = (i & 1) ? hi2(V[i >> 1]) : lo2(V[i >> 1]);
}
template <int M>
__device__ __forceinline__ void tdf2_step(unsigned long long (&V)[Tdf2<M>::NP], float x0, float x1, const Tdf2<M>& c,
                                          float& y0, float& y1) {
    constexpr int NP = Tdf2<M>::NP;
    y0 = fmaf(c.b0, x0, lo2(V[0]));
    y1 = fmaf(c.b0, x1, fmaf(c.na1, y0, fmaf(c.b1, x0, hi2(V[0]))));
    const unsigned long long X0 = pk2(x0, x0), Y0 = pk2(y0, y0), X1 = pk2(x1, x1), Y1 = pk2(y1, y1);
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        unsigned long long acc = (k + 1 < NP) ? V[k + 1] : 0ull;
        acc = ffma2(c.B2[k], X0, acc);
        acc = ffma2(c.NA2[k], Y0, acc);
        acc = ffma2(c.B1[k], X1, acc);
        acc = ffma2(c.NA1[k], Y1, acc);
        V[k] = acc;
    }
}
template <typename T, int FORM> constexpr bool use_tdf2() { return FORM == 1 && sizeof(T) == 4; }

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
    double bn[M + 1], an[M + 1];                 // every load issued up front (one round trip)
#pragma unroll
    for (int k = 0; k <= M; ++k) { bn[k] = __ldg(tb + TB::COEF + k); an[k] = __ldg(tb + TB::COEF + M + 1 + k); }
    const double inv_a0 = 1.0 / __ldg(tb + TB::A0);
    double gbn[M + 1], gan[M + 1];
    gan[0] = 0.0;
    if constexpr (FORM == 1) {
        gbn[0] = G[2 * M];
#pragma unroll
        for (int k = 1; k <= M; ++k) {
            gbn[k] = G[k - 1];
            gan[k] = -G[M + k - 1];
            gbn[0] -= an[k] * G[k - 1];
        }
    } else {
#pragma unroll
        for (int k = 0; k <= M; ++k) gbn[k] = G[k];
#pragma unroll
        for (int k = 1; k <= M; ++k) gan[k] = -G[M + k];
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k <= M; ++k) s += bn[k] * gbn[k];
#pragma unroll
    for (int k = 1; k <= M; ++k) s += an[k] * gan[k];
    if (gb != nullptr) {
#pragma unroll
        for (int k = 0; k <= M; ++k) gb[k] = (T)(gbn[k] * inv_a0);
    }
    if (ga != nullptr) {
        ga[0] = (T)(-s * inv_a0);
#pragma unroll
        for (int k = 1; k <= M; ++k) ga[k] = (T)(gan[k] * inv_a0);
    }
}

// ---------------------------------------------------------------------------
// Grid-level carry bookkeeping (workspace pointers), shared by fwd and bwd.
struct CarryWs {
    unsigned* ticket;            // tile ticket counter (IIRG_TICKETS only)
    unsigned* done;              // CTAs finished (the last one advances the epoch)
    unsigned* epoch;             // call counter: slot bank = epoch & 1
    int64_t bank;                // elements between the two slot banks
    double* agg[LEVELS];         // bank 0 level-l block aggregates [seq][block][M]; all-ones NaN = not published
    int64_t nblk[LEVELS];        // blocks per sequence at level l (ceil(ntiles / 32^l))
    int nlev;                    // levels in use
    unsigned* err;               // workspace error word (a look-back wait that timed out)
};

struct LtiFwdArgs {
    const void* b; const void* a; int64_t coef_stride;           // raw coefficients (local pass)
    const void* x; const void* zi; void* y; void* zf; void* u;    // u: DF tape, chunk-entry states
    const double* tab; int64_t tab_stride;                        // 0 for SHARED
    CarryWs cw;
    int64_t B, Tlen; int ntiles; int vec;
    unsigned long long* trace;                                    // debug: per-tile phase times
    unsigned long long* span;                                     // debug: kernel span
};

struct LtiBwdArgs {
    const void* gy; const void* gzf; const void* x; const void* y; const void* u; const void* zi;
    const void* a; int64_t coef_stride;                           // bare recurrence (rec.cuh): A
    void* gx; void* gzi; void* gb; void* ga; int want_coef; int gy_early;
    double* partial; double* partial2; unsigned* gcnt; unsigned* scnt;   // fused finalize
    int64_t ncoef;
    const double* tab; int64_t tab_stride;
    CarryWs cw;
    int64_t B, Tlen; int ntiles; int vec;
    unsigned long long* trace;
    unsigned long long* span;
};

// Normalised coefficients in T, straight from the caller's b, a (the same
// rounding as the prologue's fp64 b/a0, a/a0 cast to T): the forward local pass
// runs before the prologue's tables are ready.
template <typename T, int M>
__device__ __forceinline__ void raw_coefs(const T* __restrict__ b, const T* __restrict__ a, T (&bc)[M + 1],
                                          T (&ac)[M + 1]) {
    double bb[M + 1], aa[M + 1];                 // every load issued before the one division
#pragma unroll
    for (int k = 0; k <= M; ++k) { bb[k] = (double)__ldg(b + k); aa[k] = (double)__ldg(a + k); }
    const double inv_a0 = 1.0 / aa[0];
#pragma unroll
    for (int k = 0; k <= M; ++k) { bc[k] = (T)(bb[k] * inv_a0); ac[k] = (T)(aa[k] * inv_a0); }
}
template <typename T, int M>
__device__ __forceinline__ void load_coefs(const double* __restrict__ tb, T (&bc)[M + 1], T (&ac)[M + 1], T (&cc)[M]) {
    using TB = Tab<M>;
#pragma unroll
    for (int k = 0; k <= M; ++k) { bc[k] = (T)__ldg(tb + TB::COEF + k); ac[k] = (T)__ldg(tb + TB::COEF + M + 1 + k); }
#pragma unroll
    for (int k = 0; k < M; ++k) cc[k] = (T)__ldg(tb + TB::COEF + 2 * (M + 1) + k);
}

template <int M>
__device__ __forceinline__ void stage_small_async(double* st, const double* __restrict__ tb) {
    // 16 B copies through L1 (every CTA of the SM reads the same tables; st and tb
    // are 16 B aligned: tables start on 256 B boundaries)
    constexpr int N2 = Tab<M>::STAGE / 2;
    for (int i = threadIdx.x; i < N2; i += blockDim.x) cp_async16_ca(st + 2 * i, tb + 2 * i);
    if constexpr (Tab<M>::STAGE % 2 != 0) {
        if (threadIdx.x == 0) cp_async8(st + Tab<M>::STAGE - 1, tb + Tab<M>::STAGE - 1);
    }
}
// Stage the small power tables (PL | PW | PWT) of this tile's coefficient set.
template <int M>
__device__ __forceinline__ void stage_small(double* st, const double* __restrict__ tb) {
    for (int i = threadIdx.x; i < Tab<M>::STAGE; i += blockDim.x) st[i] = __ldg(tb + i);
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

// dst[k] = sum_r src[r NG + k] (r < nrows) in a fixed order: warp w owns the
// columns k = w (mod NW); lane l sums rows l, l+32, ... and a xor butterfly
// combines the lanes.  All loads of a row sweep are independent (one round trip
// for up to 32 rows), and the result is bitwise reproducible.
template <int NG>
__device__ __forceinline__ void reduce_rows(const double* src, int64_t nrows, double* dst, int lane, int warp) {
    constexpr int KQ = (NG + NW - 1) / NW;
    constexpr int RB = 2;                        // rows per lane loaded together
    double acc[KQ];
#pragma unroll
    for (int q = 0; q < KQ; ++q) acc[q] = 0.0;
    for (int64_t r0 = lane; r0 < nrows; r0 += 32 * RB) {
        double v[RB][KQ];
#pragma unroll
        for (int b = 0; b < RB; ++b)
#pragma unroll
            for (int q = 0; q < KQ; ++q) {
                const int k = warp + q * NW;
                const int64_t r = r0 + 32 * b;
                v[b][q] = (k < NG && r < nrows) ? __ldcg(src + r * NG + k) : 0.0;
            }
#pragma unroll
        for (int b = 0; b < RB; ++b)
#pragma unroll
            for (int q = 0; q < KQ; ++q) acc[q] += v[b][q];
    }
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
        double v = acc[q];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int k = warp + q * NW;
        if (lane == 0 && k < NG) dst[k] = v;
    }
}

template <int M>
__device__ __forceinline__ void warp_sum(double (&v)[M]) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int i = 0; i < M; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

template <int M>
__device__ __forceinline__ void publish(double* dst, const double (&v)[M], int lane) {
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) __stcg(dst + i, v[i]);
    }
}

// Look-back payload slots.  A read is one round trip: all M elements are
// loaded at once (volatile: never hoisted, never served from a stale L1 line)
// and the slot is ready when none is the sentinel.
template <int M>
__device__ __forceinline__ void load_slot(const double* src, double (&v)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = ld_relaxed(src + i);
}
template <int M>
__device__ __forceinline__ bool slot_ready(const double (&v)[M]) {
    bool r = true;
#pragma unroll
    for (int i = 0; i < M; ++i) r = r && !is_sentinel(v[i]);
    return r;
}
// Re-poll a slot whose first read was not ready, with exponential back-off.  A
// slot that is never published (a scheduling or library bug) does not hang the GPU
// and does not trap (which would poison the whole CUDA context): after 2 s the
// waiter sets the workspace error word (reported by iir_check_workspace) and
// continues with NaN, so the call completes with NaN outputs.
template <int M>
__device__ __forceinline__ void wait_slot(const double* src, double (&v)[M], unsigned* err) {
    unsigned ns = 32;
    unsigned long long t0 = 0;
    for (;;) {
        __nanosleep(ns);
        load_slot<M>(src, v);
        if (slot_ready<M>(v)) return;
        if (ns < 256) ns *= 2;
        else {
            const unsigned long long now = gtimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 2000000000ull) {
                if (err != nullptr) atomicOr(err, 1u);
#pragma unroll
                for (int i = 0; i < M; ++i) v[i] = __longlong_as_double(0x7ff8000000000000LL);
                return;
            }
        }
    }
}

// Grid-level carry (warp 0).  Tile j (scan order within its sequence) has
// base-32 digits d_l.  With AGG^(0) = tile aggregates (tile 0's includes the
// initial state X0) and AGG^(l+1)_b = sum_{d<32} Q_l^(31-d) AGG^(l)_{32b+d},
// Q_l = A_f^(32^l TS):
//   T_l = sum_{d < d_l} Q_l^(d_l - 1 - d) AGG^(l)_{(j >> 5l) - d_l + d}
//   X_j = T_0 + Q_0^d_0 (T_1 + Q_1^d_1 (T_2 + ...))     (state entering tile j)
// Lane d reads slot d of EVERY level at once, so a tile whose inputs are all
// published pays one round trip for the whole look-back (the levels are not
// waited for one after the other).  Each T_l is then a fixed butterfly sum:
// bitwise deterministic.  A tile that closes a level-(l+1) block publishes
// AGG^(l+1) = Q_l T_l + AGG^(l)_own as soon as T_l is known.
template <int M, bool TR>
__device__ __forceinline__ void tile_carry(const double* st, const double* __restrict__ tb, int lane, int jt, int64_t seq,
                                           const double (&X0)[M], double (&G)[M], const CarryWs& cw,
                                           double (&X)[M], unsigned long long* trace = nullptr,
                                           unsigned tk = 0) {
    using TB = Tab<M>;
    constexpr int M2 = M * M;
    __shared__ double s_T[LEVELS][M];
#pragma unroll
    for (int i = 0; i < M; ++i) X[i] = X0[i];
    if (jt == 0) mv_pq<M, TR>(st, tb, 0, 1, X0, G);               // tile 0 carries the initial state
    publish<M>(cw.agg[0] + (seq * cw.nblk[0] + jt) * M, G, lane);
    if (jt == 0) return;
    // levels 0 and 1 are read up front (one round trip); deeper levels, used only
    // by sequences of more than 32^2 tiles, when they are reached
    constexpr int PF = LEVELS < 2 ? LEVELS : 2;
    int dl[LEVELS];
    double V[LEVELS][M];
#pragma unroll
    for (int l = 0; l < LEVELS; ++l) {
        dl[l] = l < cw.nlev ? (jt >> (5 * l)) & 31 : 0;
        if (l < PF && lane < dl[l])
            load_slot<M>(cw.agg[l] + (seq * cw.nblk[l] + (jt >> (5 * l)) - dl[l] + lane) * M, V[l]);
    }
    bool closing = true;                   // all lower digits were 31 so far
    double Own[M];
#pragma unroll
    for (int i = 0; i < M; ++i) Own[i] = G[i];
#pragma unroll
    for (int l = 0; l < LEVELS; ++l) {
        double Tv[M];
#pragma unroll
        for (int i = 0; i < M; ++i) Tv[i] = 0.0;
        if (dl[l] > 0) {
            if (lane < dl[l]) {
                if (l >= PF) load_slot<M>(cw.agg[l] + (seq * cw.nblk[l] + (jt >> (5 * l)) - dl[l] + lane) * M, V[l]);
                if (!slot_ready<M>(V[l]))
                    wait_slot<M>(cw.agg[l] + (seq * cw.nblk[l] + (jt >> (5 * l)) - dl[l] + lane) * M, V[l], cw.err);
                mv_pq<M, TR>(st, tb, l, dl[l] - 1 - lane, V[l], Tv);
            }
            warp_sum<M>(Tv);
        }
        if (l < 2 && trace != nullptr && lane == 0) trace[(size_t)tk * 16 + 6 + l] = gtimer();
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) s_T[l][i] = Tv[i];
        }
        closing = closing && dl[l] == 31;
        if (closing && l + 1 < cw.nlev) {
            mv_pq<M, TR>(st, tb, l, 1, Tv, Own);                          // Own = Q_l T_l + Own
            const int64_t bi = seq * cw.nblk[l + 1] + (jt >> (5 * (l + 1)));
            publish<M>(cw.agg[l + 1] + bi * M, Own, lane);
        }
    }
    __syncwarp();
    double R[M];
#pragma unroll
    for (int i = 0; i < M; ++i) R[i] = 0.0;
#pragma unroll
    for (int l = LEVELS - 1; l >= 0; --l) {
        if (l < cw.nlev) {
            double R2[M];
#pragma unroll
            for (int i = 0; i < M; ++i) R2[i] = s_T[l][i];
            if (l + 1 < cw.nlev) mv_pq<M, TR>(st, tb, l, dl[l], R, R2);
#pragma unroll
            for (int i = 0; i < M; ++i) R[i] = R2[i];
        }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) X[i] = R[i];
}

// Scan order of this CTA's tile.  Tiles are scanned in CTA launch order: the
// hardware dispatches the CTAs of a 1-D grid in increasing blockIdx, so every
// tile a CTA waits for belongs to a CTA that is already resident (the single-
// pass look-back of CUB-style scans relies on the same order).  IIRG_TICKETS=1
// takes an atomic ticket instead (one more round trip before the tile load).
#ifndef IIRG_TICKETS
#define IIRG_TICKETS 0
#endif
__device__ __forceinline__ unsigned tile_order(unsigned* ticket) {
#if IIRG_TICKETS
    __shared__ unsigned s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    return s_ticket;
#else
    (void)ticket;
    return blockIdx.x;
#endif
}

// Look-back slots live in two banks used by alternate calls (epoch parity).
// Every CTA re-arms its share of the OTHER bank (last used by the previous
// call on this workspace, which has completed) with sentinels, and the last
// CTA to finish advances the epoch, so a call leaves the workspace ready for
// the next one without a serial clean-up tail.
__device__ __forceinline__ unsigned carry_bank(CarryWs& cw) {
    const unsigned ep = __ldcg(cw.epoch);
    if (ep & 1u)
        for (int l = 0; l < LEVELS; ++l)
            if (cw.agg[l] != nullptr) cw.agg[l] += cw.bank;
    return ep;
}
__device__ __forceinline__ void rearm_other_bank(const CarryWs& cw, unsigned ep, unsigned cta, unsigned nctas) {
    // the other bank is one contiguous range starting at agg[0] -/+ bank
    double* other = cw.agg[0] + ((ep & 1u) ? -cw.bank : cw.bank);
    for (int64_t i = (int64_t)cta * blockDim.x + threadIdx.x; i < cw.bank; i += (int64_t)nctas * blockDim.x)
        __stcg(other + i, sentinel());
}
__device__ __forceinline__ void cta_exit(const CarryWs& cw, unsigned ep, unsigned nctas) {
    __shared__ unsigned s_last;
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(cw.done, 1u) == nctas - 1u) ? 1u : 0u;
    __syncthreads();
    if (s_last && threadIdx.x == 0) { *cw.ticket = 0u; *cw.done = 0u; *cw.epoch = ep + 1u; }
}

template <typename T, int M>
struct Smem {
    static constexpr int TS = NT * Chunk<T, M>::L;
    static constexpr int PT = pidx<T>(TS);               // one padded tile
    static constexpr int PTH = pidx<T>(TS + HALO);       // padded tile with u history
    static constexpr size_t tab_bytes = ((size_t)Tab<M>::STAGE * 8 + 15) / 16 * 16;
    static constexpr size_t fwd(int) { return tab_bytes + (size_t)PT * sizeof(T); }
    static constexpr size_t bwd_tdf() { return tab_bytes + (size_t)PT * sizeof(T); }
    static constexpr size_t bwd(int form) {
        return tab_bytes + (size_t)(PT + PTH + (form == 1 ? PT : 0)) * sizeof(T);
    }
};

// ---------------------------------------------------------------------------
// Forward: a2-a4.  One CTA per tile of TS samples; tiles are taken in ticket
// order (ticket t = tile t / B of sequence t % B), so every tile a CTA waits
// for belongs to a CTA that is already running.
// Minimum resident CTAs per SM requested from ptxas (caps the registers of the
// high-order instantiations, whose occupancy is otherwise register-bound).
// (counts for 128-thread CTAs, scaled to NT)
#ifndef IIRG_MINB2
#define IIRG_MINB2 8
#endif
template <int M> constexpr int fwd_min_blocks() { return (M <= 2 ? IIRG_MINB2 : (M <= 4 ? 6 : 4)) * 128 / NT; }
template <int M> constexpr int bwd_min_blocks() { return (M <= 4 ? 4 : 3) * 128 / NT > 0 ? (M <= 4 ? 4 : 3) * 128 / NT : 1; }
template <int M> constexpr int bwd_tdf_min_blocks() { return (M <= 2 ? IIRG_MINB2 : (M <= 4 ? 6 : 4)) * 128 / NT; }

template <typename T, int M, int FORM>
__global__ void __launch_bounds__(NT, fwd_min_blocks<M>()) lti_fwd_kernel(const LtiFwdArgs p) {
    constexpr int L = Chunk<T, M>::L, TS = NT * L, W = Vec<T>::W;
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    using SM = Smem<T, M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* st = reinterpret_cast<double*>(smem_raw);
    T* xs = reinterpret_cast<T*>(smem_raw + SM::tab_bytes);     // x -> y in place
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
    const T* xrow = static_cast<const T*>(p.x) + seq * p.Tlen;
    IIRG_TRACE(p.trace, tk, 0);
    tile_load_async<T, TS>(xs, xrow, p0, p.Tlen, p.vec);
    cp_async_commit();
    // the power tables come from the prologue kernel (PDL): wait, then stage them
    // asynchronously so that their load overlaps the tile's and the local pass
    pdl_wait();
    // the prologue has completed: a dependent backward may start (it reads the
    // tables, never this kernel's outputs, before its own griddepcontrol.wait)
    pdl_launch_dependents();
    const double* tb = p.tab + seq * p.tab_stride;
    stage_small_async<M>(st, tb);
    cp_async_commit();
    rearm_other_bank(cw, ep, blockIdx.x, gridDim.x);
    T bc[M + 1], ac[M + 1];
    raw_coefs<T, M>(static_cast<const T*>(p.b) + seq * p.coef_stride,
                    static_cast<const T*>(p.a) + seq * p.coef_stride, bc, ac);
    cp_async_wait<1>();                                // x tile
    __syncthreads();

    // a2: local pass from the zero state over this thread's chunk.
    const int s0 = tid * L;
    T v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = T(0);
    if constexpr (use_tdf2<T, FORM>()) {
        Tdf2<M> c2;
        c2.init(bc, ac);
        unsigned long long VP[Tdf2<M>::NP];
        tdf2_pack<M>(v, VP);
#pragma unroll
        for (int g = 0; g < L / W; ++g) {
            const float4 xv = *reinterpret_cast<const float4*>(xs + pidx<T>(s0 + g * W));
            float ya, yb;
            tdf2_step<M>(VP, xv.x, xv.y, c2, ya, yb);
            tdf2_step<M>(VP, xv.z, xv.w, c2, ya, yb);
        }
        tdf2_unpack<M>(VP, v);
    } else {
#pragma unroll
        for (int g = 0; g < L / W; ++g) {
            const V xv = *reinterpret_cast<const V*>(xs + pidx<T>(s0 + g * W));
#pragma unroll
            for (int e = 0; e < W; ++e) { T du; fwd_step<T, M, FORM>(v, vget(xv, e), bc, ac, du); }
        }
    }
    IIRG_TRACE(p.trace, tk, 1);
    // a3: carries in fp64
    cp_async_wait<0>();                                // power tables
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
        const T* zi = static_cast<const T*>(p.zi);
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (zi != nullptr && jt == 0) ? (double)zi[seq * M + i] : 0.0;
        IIRG_TRACE(p.trace, tk, 2);
        tile_carry<M, false>(st, tb, lane, jt, seq, X0, G, cw, X, p.trace, tk);
        IIRG_TRACE(p.trace, tk, 3);
        if (lane < NW) {                           // state entering warp `lane`
            double xw[M];
#pragma unroll
            for (int i = 0; i < M; ++i) xw[i] = Jex[i];
            mv_acc_lane_s<M, false>(st + TB::PWT, NW, lane, X, xw);
#pragma unroll
            for (int i = 0; i < M; ++i) s_xw[lane][i] = xw[i];
        }
    }
    __syncthreads();
    // state entering this thread's chunk: E + A_f^(L lane) x_warp
    {
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
        mv_plt<M, false>(st, tb, lane, xw, E);
    }
    T vin[M];
#pragma unroll
    for (int i = 0; i < M; ++i) { vin[i] = (T)E[i]; v[i] = vin[i]; }
    if constexpr (FORM == 0) {
        // DF: the tape keeps the state entering every chunk, [u(n-1) .. u(n-M)] at n = the
        // chunk's first sample (M values per L samples), not the signal u itself: the
        // backward re-runs the recursion from it (df_regen_u) -- the same fwd_step from the
        // same T state, so the regenerated u is bit-identical to the one emitted here.
        if (p0 + s0 < p.Tlen) {
            T* ust = static_cast<T*>(p.u) + (seq * ((p.Tlen + L - 1) / L) + (p0 + s0) / L) * M;
#pragma unroll
            for (int i = 0; i < M; ++i) ust[i] = vin[i];
        }
    }
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
    // a4: re-run from the exact carry-in, emit y in place.
    if constexpr (use_tdf2<T, FORM>()) {
        Tdf2<M> c2;
        c2.init(bc, ac);
        unsigned long long VP[Tdf2<M>::NP];
        tdf2_pack<M>(v, VP);
#pragma unroll
        for (int g = 0; g < L / W; ++g) {
            float4 xv = *reinterpret_cast<const float4*>(xs + pidx<T>(s0 + g * W));
            tdf2_step<M>(VP, xv.x, xv.y, c2, xv.x, xv.y);
            tdf2_step<M>(VP, xv.z, xv.w, c2, xv.z, xv.w);
            *reinterpret_cast<float4*>(xs + pidx<T>(s0 + g * W)) = xv;
        }
    } else {
#pragma unroll
        for (int g = 0; g < L / W; ++g) {
            V xv = *reinterpret_cast<const V*>(xs + pidx<T>(s0 + g * W));
#pragma unroll
            for (int e = 0; e < W; ++e) {
                T uu;
                vset(xv, e, fwd_step<T, M, FORM>(v, vget(xv, e), bc, ac, uu));
            }
            *reinterpret_cast<V*>(xs + pidx<T>(s0 + g * W)) = xv;
        }
    }
    __syncthreads();
    IIRG_TRACE(p.trace, tk, 4);
    T* yrow = static_cast<T*>(p.y) + seq * p.Tlen;
    tile_store<T, TS>(yrow, xs, p0, p.Tlen, p.vec);
    IIRG_TRACE(p.trace, tk, 5);
    cta_exit(cw, ep, gridDim.x);
    span_exit(p.span);
}

// DF backward: x(p0 .. p0 + TS) -> s2[pidx(e + HALO)] (the slots of u, regenerated in place by
// df_regen_u; samples before n = 0 are never read from x).
template <typename T, int M>
__device__ __forceinline__ void bwd_load_x_df(const LtiBwdArgs& p, int64_t seq, int64_t p0, T* s2) {
    constexpr int TS = NT * Chunk<T, M>::L, W = Vec<T>::W;
    using V = typename Vec<T>::type;
    const T* xrow = static_cast<const T*>(p.x) + seq * p.Tlen;
    for (int q = threadIdx.x; q < TS / W; q += NT) {
        const int e = q * W;
        const int64_t pos = p0 + e;
        if (pos < 0 && pos + W <= 0) continue;
        if (p.vec && pos >= 0) {
            cp_async16(s2 + pidx<T>(e + HALO), xrow + pos, 16u);
        } else {
            V val;
#pragma unroll
            for (int r = 0; r < W; ++r) vset(val, r, pos + r >= 0 ? xrow[pos + r] : T(0));
            *reinterpret_cast<V*>(s2 + pidx<T>(e + HALO)) = val;
        }
    }
}

// DF backward: u(n) for this thread's chunk [p0 + s0, p0 + s0 + L) re-run from the chunk-entry
// state the forward saved (Eqs.2-3: u = x - sum a_k u(n-k)), written over x in s2; u(-k) =
// zi[k-1], zero beyond.  The tile's first chunk also writes the tile's u history u(n-1 .. n-M)
// (the state itself).  A chunk that does not start on the forward's chunk grid (backward tiles
// are aligned to the sequence end) first walks from the grid point before it on x read from
// global memory (fewer than L samples; none when L divides T).
template <typename T, int M>
__device__ __forceinline__ void df_regen_u(const LtiBwdArgs& p, int64_t seq, int64_t p0, int s0, T* s2,
                                           const T (&bc)[M + 1], const T (&ac)[M + 1]) {
    constexpr int L = Chunk<T, M>::L, W = Vec<T>::W;
    using V = typename Vec<T>::type;
    const T* xrow = static_cast<const T*>(p.x) + seq * p.Tlen;
    const T* zi = static_cast<const T*>(p.zi);
    const int64_t ns = p0 + s0, hi = ns + L;                 // the chunk [ns, hi)
    for (int64_t n = ns - (s0 == 0 ? HALO : 0); n < min(hi, (int64_t)0); ++n)
        s2[pidx<T>((int)(n - p0) + HALO)] = (n >= -M && zi != nullptr) ? zi[seq * M + (-n - 1)] : T(0);
    if (hi <= 0) return;
    const int64_t first = max(ns, (int64_t)0);
    const int64_t g = first / L * L;                         // forward chunk grid point <= first
    const T* ust = static_cast<const T*>(p.u) + (seq * ((p.Tlen + L - 1) / L) + g / L) * M;
    T v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = ust[i];
    T uu;
#pragma unroll 8
    for (int64_t n = g; n < first; ++n) (void)fwd_step<T, M, 0>(v, __ldg(xrow + n), bc, ac, uu);
    if (s0 == 0 && ns > 0) {                                 // the tile's history u(ns-1 .. ns-M)
#pragma unroll
        for (int k = 1; k <= M; ++k) s2[pidx<T>(HALO - k)] = v[k - 1];
    }
    constexpr int RU = IIRG_DF_GU;
    if (first == ns) {                                       // the whole chunk, W-wide groups
#pragma unroll RU
        for (int q = 0; q < L / W; ++q) {
            V* slot = reinterpret_cast<V*>(s2 + pidx<T>(s0 + HALO + q * W));
            V xv = *slot;
#pragma unroll
            for (int e = 0; e < W; ++e) {
                (void)fwd_step<T, M, 0>(v, vget(xv, e), bc, ac, uu);
                vset(xv, e, uu);
            }
            *slot = xv;
        }
    } else {                                                 // the chunk holding n = 0 (first tile)
        for (int64_t n = first; n < hi; ++n) {
            T* slot = s2 + pidx<T>((int)(n - p0) + HALO);
            (void)fwd_step<T, M, 0>(v, *slot, bc, ac, uu);
            *slot = uu;
        }
    }
}

// a8 (fused): the CTA's fp64 partial sums (s_red, per warp) -> per-tile row ->
// group of 32 tiles -> set -> chain rule.  SHARED groups are consecutive tiles
// in scan order (they complete, and are reduced, while the kernel runs);
// PER_SEQ groups are a sequence's tiles.  Fixed reduction order throughout.
template <int M, int FORM> constexpr int n_partials() { return FORM == 2 ? M * M : 2 * M + 1; }
constexpr int64_t FLAT_MAX = 8192;   // partial values of a set reduced flat (one round trip) by its last CTA


template <typename T, int M, int FORM>
// Also counts the CTA out of the look-back (cw != NULL): its atomic and the
// partial-sum publication run concurrently (warps 0 and 1).
__device__ __forceinline__ void bwd_finalize(const LtiBwdArgs& p, const CarryWs* cw, unsigned ep, unsigned tk,
                                             int64_t seq, int jt, const double* __restrict__ tb,
                                             const double (*s_red)[n_partials<M, FORM>()]) {
    constexpr int NG = n_partials<M, FORM>();
    static_assert(NG <= 32, "one lane of warp 1 per partial sum");
    __shared__ double s_G[NG];
    __shared__ unsigned s_fin, s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // fused a8: group of 32 tiles -> group sum; last group of the set -> chain rule.
    // SHARED groups are consecutive tiles in scan order (they complete, and are
    // reduced, while the kernel runs); PER_SEQ groups are a sequence's tiles.
    const bool shared = p.ncoef == 1;
    const int64_t per_set = shared ? p.B * p.ntiles : p.ntiles;
    const int64_t cset = shared ? 0 : seq;
    const int64_t li = shared ? (int64_t)tk : jt;                  // index within the set
    const int64_t gi = li >> 5;
    const int64_t ngroups = (per_set + 31) >> 5;
    const int gsize = (int)min((int64_t)32, per_set - (gi << 5));
    double* part = p.partial + cset * per_set * NG;
    double* part2 = p.partial2 + cset * ngroups * NG;
    // small sets: one counter per set and a flat fixed-order reduction of every
    // per-tile row by the set's last CTA (one load round trip; no group level)
    const bool flat = per_set * NG <= FLAT_MAX;
    __syncthreads();                               // s_red complete; the look-back slots are no longer read
    if (p.want_coef && warp == 1) {
        if (lane < NG) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += s_red[w][lane];
            __stcg(part + li * NG + lane, s);
            __threadfence();
        }
        __syncwarp();
        if (lane == 0) {
            if (flat) s_fin = (atomicAdd(p.scnt + cset, 1u) == (unsigned)per_set - 1u) ? 3u : 0u;
            else s_fin = (atomicAdd(p.gcnt + cset * ngroups + gi, 1u) == (unsigned)gsize - 1u) ? 1u : 0u;
        }
    }
    if (cw != nullptr && tid == 0) s_last = (atomicAdd(cw->done, 1u) == gridDim.x - 1u) ? 1u : 0u;
    __syncthreads();
    IIRG_TRACE(p.trace, tk, 8);
    if (cw != nullptr && s_last && tid == 0) { *cw->ticket = 0u; *cw->done = 0u; *cw->epoch = ep + 1u; }
    if (p.want_coef && s_fin == 3u) {              // flat: last tile of the set
        constexpr int FLAT_RB = (24 / NG) > 0 ? 24 / NG : 1;   // rows per thread per load round trip
        __threadfence();
        double acc[NG];
#pragma unroll
        for (int k = 0; k < NG; ++k) acc[k] = 0.0;
        for (int64_t r0 = 0; r0 < per_set; r0 += (int64_t)NT * FLAT_RB) {   // rows tid, tid + NT, ... in order
            double v[FLAT_RB][NG];
#pragma unroll
            for (int b = 0; b < FLAT_RB; ++b) {
                const int64_t r = r0 + (int64_t)b * NT + tid;
#pragma unroll
                for (int k = 0; k < NG; ++k) v[b][k] = r < per_set ? __ldcg(part + r * NG + k) : 0.0;
            }
#pragma unroll
            for (int b = 0; b < FLAT_RB; ++b)
#pragma unroll
                for (int k = 0; k < NG; ++k) acc[k] += v[b][k];
        }
        __shared__ double s_w[NW][NG];
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            double v = acc[k];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) s_w[warp][k] = v;
        }
        __syncthreads();
        if (tid < NG) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += s_w[w][tid];
            s_G[tid] = v;
        }
        __syncthreads();
        if (tid == 0) {
            if constexpr (FORM == 2) {
                if (p.ga != nullptr)
                    for (int e = 0; e < NG; ++e) static_cast<T*>(p.ga)[cset * NG + e] = (T)s_G[e];
            } else {
                chain_rule<T, M, FORM>(s_G, tb, p.gb == nullptr ? nullptr : static_cast<T*>(p.gb) + cset * (M + 1),
                                       p.ga == nullptr ? nullptr : static_cast<T*>(p.ga) + cset * (M + 1));
            }
            p.scnt[cset] = 0u;
        }
        return;
    }
    if (p.want_coef && s_fin == 1u) {              // last tile of its group
        __threadfence();
        reduce_rows<NG>(part + (gi << 5) * NG, gsize, part2 + gi * NG, lane, warp);
        __threadfence();
        __syncthreads();
        IIRG_TRACE(p.trace, tk, 9);
        if (tid == 0) {
            p.gcnt[cset * ngroups + gi] = 0u;
            s_fin = (atomicAdd(p.scnt + cset, 1u) == (unsigned)ngroups - 1u) ? 2u : 0u;
        }
        __syncthreads();
        if (s_fin == 2u) {                          // last group of the set
            __threadfence();
            IIRG_TRACE(p.trace, tk, 12);
            reduce_rows<NG>(part2, ngroups, s_G, lane, warp);
            __syncthreads();
            IIRG_TRACE(p.trace, tk, 13);
            if (tid == 0) {
                if constexpr (FORM == 2) {                   // bare recurrence: grad_A is the sum itself
                    if (p.ga != nullptr)
                        for (int e = 0; e < NG; ++e) static_cast<T*>(p.ga)[cset * NG + e] = (T)s_G[e];
                } else {
                    chain_rule<T, M, FORM>(s_G, tb,
                                       p.gb == nullptr ? nullptr : static_cast<T*>(p.gb) + cset * (M + 1),
                                       p.ga == nullptr ? nullptr : static_cast<T*>(p.ga) + cset * (M + 1));
                }
                p.scnt[cset] = 0u;
                IIRG_TRACE(p.trace, tk, 14);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Backward: a5-a8.  Tiles are aligned to the END of each sequence and taken in
// ticket order last to first; inside a tile thread t owns chunk NT-1-t, walked
// backwards.  TDF: smem dy | x | y.  DF: smem dy | u (with HALO samples of history).
template <typename T, int M, int FORM>
__global__ void __launch_bounds__(NT, bwd_min_blocks<M>()) lti_bwd_kernel(const LtiBwdArgs p) {
    constexpr int L = Chunk<T, M>::L, TS = NT * L, W = Vec<T>::W;
    constexpr int NG = 2 * M + 1;                       // gradient partial sums
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    using SM = Smem<T, M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* st = reinterpret_cast<double*>(smem_raw);
    T* dys = reinterpret_cast<T*>(smem_raw + SM::tab_bytes);   // dy -> dx in place
    T* s2 = dys + SM::PT;                                      // TDF: x        DF: u (+HALO)
    T* s3 = s2 + SM::PTH;                                      // TDF: y
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];
    __shared__ double s_red[NW][NG];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned tk = tile_order(p.cw.ticket);
    span_enter(p.span);
    CarryWs cw = p.cw;
    const unsigned ep = carry_bank(cw);
    const int64_t seq = (int64_t)(tk % (unsigned long long)p.B);
    const int jr = (int)(tk / (unsigned long long)p.B);          // 0 = last tile in time
    const int jt = p.ntiles - 1 - jr;                            // time index of the tile
    const int64_t p0 = p.Tlen - (int64_t)(jr + 1) * TS;          // may be < 0 (first tile)
    const double* tb = p.tab + seq * p.tab_stride;
    const int64_t roff = seq * p.Tlen;
    IIRG_TRACE(p.trace, tk, 0);

    // group 0: dy;  group 1: the power tables (in the tape, written by the forward's
    // prologue);  group 2: x, y (TDF) or u (DF).  All in flight at once.
    if (p.gy != nullptr) tile_load_async<T, TS>(dys, static_cast<const T*>(p.gy) + roff, p0, p.Tlen, p.vec);
    else for (int e = tid; e < TS; e += NT) dys[pidx<T>(e)] = T(0);
    cp_async_commit();
    stage_small_async<M>(st, tb);
    cp_async_commit();
    if constexpr (FORM == 1) {
        tile_load_async<T, TS>(s2, static_cast<const T*>(p.x) + roff, p0, p.Tlen, p.vec);
        tile_load_async<T, TS>(s3, static_cast<const T*>(p.y) + roff, p0, p.Tlen, p.vec);
    } else {
        bwd_load_x_df<T, M>(p, seq, p0, s2);
    }
    cp_async_commit();
    rearm_other_bank(cw, ep, blockIdx.x, gridDim.x);
    T bc[M + 1], ac[M + 1], cc[M];
    load_coefs<T, M>(tb, bc, ac, cc);
    cp_async_wait<2>();                              // dy
    __syncthreads();

    const int c = NT - 1 - tid;          // chunk index within the tile (time order)
    const int s0 = c * L;
    // DF: the fully unrolled chunk loops overflow the instruction cache at M = 8 (ncu: 40 % of
    // stalls "no_instructions"); the group loops are unrolled by IIRG_DF_GU only
    constexpr int GU = FORM == 0 ? IIRG_DF_GU : L / W;
    // a5: local adjoint pass from the zero state, walking the chunk backwards.
    T d[M];
#pragma unroll
    for (int i = 0; i < M; ++i) d[i] = T(0);
#pragma unroll GU
    for (int g = L / W - 1; g >= 0; --g) {
        const V dv = *reinterpret_cast<const V*>(dys + pidx<T>(s0 + g * W));
#pragma unroll
        for (int e = W - 1; e >= 0; --e) {
            if constexpr (FORM == 1) adj_tdf_step<T, M>(d, vget(dv, e), ac);
            else adj_df_step<T, M>(d, vget(dv, e), bc, ac);
        }
    }
    IIRG_TRACE(p.trace, tk, 1);
    // a6: carries (transposed powers), tiles last -> first.
    cp_async_wait<FORM == 0 ? 0 : 1>();              // power tables (DF: and x)
    __syncthreads();
    double S[M];
#pragma unroll
    for (int i = 0; i < M; ++i) S[i] = (double)d[i];
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
        const T* gzf = static_cast<const T*>(p.gzf);
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (gzf != nullptr && jr == 0) ? (double)gzf[seq * M + i] : 0.0;
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
    } else if constexpr (FORM == 0) {
        // DF: while warp 0 looks back, the other warps re-run u over the tile (x -> u in place)
        static_assert(NT > 32, "warps 1.. re-run u");
        for (int c = tid - 32; c < NT; c += NT - 32) df_regen_u<T, M>(p, seq, p0, c * L, s2, bc, ac);
    }
    __syncthreads();
    {
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
        mv_plt<M, true>(st, tb, lane, xw, E);
    }
    T din[M];
#pragma unroll
    for (int i = 0; i < M; ++i) { din[i] = (T)E[i]; d[i] = din[i]; }
    cp_async_wait<0>();                              // x, y (TDF)
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
#pragma unroll GU
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
            // u(n - k), k = 0..M, of the group's W samples: one window of vector loads
            // u(s0 + gW - MW .. s0 + gW + W - 1) (MW = M rounded up to W <= HALO)
            constexpr int MW = (M + W - 1) / W * W;
            static_assert(MW <= HALO, "u history window inside the halo");
            T uw[MW + W];
#pragma unroll
            for (int q = 0; q < (MW + W) / W; ++q) {
                const V t = *reinterpret_cast<const V*>(s2 + pidx<T>(s0 + g * W + HALO - MW + q * W));
#pragma unroll
                for (int r = 0; r < W; ++r) uw[q * W + r] = vget(t, r);
            }
#pragma unroll
            for (int e = W - 1; e >= 0; --e) {
                const int n = s0 + g * W + e;                 // tile-local time index
                const T dy = vget(dv, e);
                const T dx = adj_df_step<T, M>(d, dy, bc, ac); // dx(n), then d <- dz(n-1)
                const T gmask = (!has_neg || p0 + n >= 0) ? dx : T(0);
#pragma unroll
                for (int k = 0; k <= M; ++k) {
                    const T uk = uw[MW + e - k];
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
    IIRG_TRACE(p.trace, tk, 4);
    if (p.gx != nullptr) tile_store<T, TS>(static_cast<T*>(p.gx) + roff, dys, p0, p.Tlen, p.vec);
    IIRG_TRACE(p.trace, tk, 5);

    // the look-back slots are no longer needed: count this CTA out first, so the
    // gradient finalize of the last CTAs is the kernel's only tail
    IIRG_TRACE(p.trace, tk, 10);
    bwd_finalize<T, M, FORM>(p, &cw, ep, tk, seq, jt, tb, s_red);
    IIRG_TRACE(p.trace, tk, 11);
    span_exit(p.span);
}

// ---------------------------------------------------------------------------
// TDF backward (a5-a8) with a single shared-memory tile.  The TDF adjoint state
// is a shift register: dz(n)[i] = g(n+i) with g(n) = dz(n)[0] (Eq.7 with
// A_f^T = A, C_f = e1), so after the carry the emit pass only has to produce
// g(n) (written in place of dy), and a second, coalesced pass forms
//   dx(n) = b0 dy(n) + sum_i c_i g(n+i)                       (Eq.8)
//   Gx[i] = sum_n g(n+i) x(n),  Gy[i] = sum_n g(n+i) y(n),  Gd = sum dy x   (Eqs.6, 9)
// reading dy, x, y straight from global memory (x, y are prefetched into L2 at
// tile start) and storing dx straight to global memory.  The tile's shared
// footprint drops from three tiles to one, so about twice as many tiles are in
// flight.  g beyond the tile end comes from the carry: g(p0+TS+j) = X[j+1].
template <typename T, int M>
__global__ void __launch_bounds__(NT, bwd_tdf_min_blocks<M>()) lti_bwd_tdf_kernel(const LtiBwdArgs p) {
    constexpr int L = Chunk<T, M>::L, TS = NT * L, W = Vec<T>::W;
    constexpr int NG = 2 * M + 1;
    using V = typename Vec<T>::type;
    using TB = Tab<M>;
    using SM = Smem<T, M>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* st = reinterpret_cast<double*>(smem_raw);
    T* gs = reinterpret_cast<T*>(smem_raw + SM::tab_bytes);    // dy -> g in place
    __shared__ double s_agg[NW][M];
    __shared__ double s_xw[NW][M];
    __shared__ double s_red[NW][NG];
    __shared__ T s_halo[8];                                     // g(p0 + TS + j), j < M - 1

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned tk = tile_order(p.cw.ticket);
    span_enter(p.span);
    CarryWs cw = p.cw;
    const unsigned ep = carry_bank(cw);
    const int64_t seq = (int64_t)(tk % (unsigned long long)p.B);
    const int jr = (int)(tk / (unsigned long long)p.B);          // 0 = last tile in time
    const int jt = p.ntiles - 1 - jr;
    const int64_t p0 = p.Tlen - (int64_t)(jr + 1) * TS;          // may be < 0 (first tile)
    const double* tb = p.tab + seq * p.tab_stride;
    const int64_t roff = seq * p.Tlen;
    const T* gyrow = static_cast<const T*>(p.gy) + roff;
    const T* xrow = static_cast<const T*>(p.x) + roff;
    const T* yrow = static_cast<const T*>(p.y) + roff;
    IIRG_TRACE(p.trace, tk, 0);

    // grad_y / grad_zf may be written by the kernel right before this one (the caller's
    // loss): without IIR_FLAG_GRAD_Y_EARLY they are read only after griddepcontrol.wait.
    // (The tables, x and the workspace were complete before this call's forward began.)
    if (!p.gy_early) pdl_wait();
    if (p.gy != nullptr) tile_load_async<T, TS>(gs, gyrow, p0, p.Tlen, p.vec);
    else for (int e = tid; e < TS; e += NT) gs[pidx<T>(e)] = T(0);
    cp_async_commit();
    const int64_t pa = p0 < 0 ? 0 : p0;              // x, y are read after the carry: pull them into L2
    const unsigned pbytes = (unsigned)((p0 + TS - pa) * (int64_t)sizeof(T));
    if (tid == 0 && p.vec) prefetch_l2_bulk(xrow + pa, pbytes);
    stage_small_async<M>(st, tb);                    // tables live in the tape (written by the forward)
    cp_async_commit();
    rearm_other_bank(cw, ep, blockIdx.x, gridDim.x);
    T bc[M + 1], ac[M + 1], cc[M];
    load_coefs<T, M>(tb, bc, ac, cc);
    cp_async_wait<0>();
    __syncthreads();

    const int c = NT - 1 - tid;          // chunk index within the tile (time order)
    const int s0 = c * L;
    // a5: local adjoint pass from the zero state, walking the chunk backwards.
    T d[M];
#pragma unroll
    for (int i = 0; i < M; ++i) d[i] = T(0);
#pragma unroll
    for (int g = L / W - 1; g >= 0; --g) {
        const V dv = *reinterpret_cast<const V*>(gs + pidx<T>(s0 + g * W));
#pragma unroll
        for (int e = W - 1; e >= 0; --e) adj_tdf_step<T, M>(d, vget(dv, e), ac);
    }
    IIRG_TRACE(p.trace, tk, 1);
    // a6: carries (transposed powers), tiles last -> first.
    double S[M];
#pragma unroll
    for (int i = 0; i < M; ++i) S[i] = (double)d[i];
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
        const T* gzf = static_cast<const T*>(p.gzf);
#pragma unroll
        for (int i = 0; i < M; ++i) X0[i] = (gzf != nullptr && jr == 0) ? (double)gzf[seq * M + i] : 0.0;
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
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j + 1 < M; ++j) s_halo[j] = (T)X[j + 1];
        }
    }
    __syncthreads();
    {
        double xw[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xw[i] = s_xw[warp][i];
        mv_plt<M, true>(st, tb, lane, xw, E);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) d[i] = (T)E[i];
    // a7, pass A: re-run with the exact carry, write g(n) = dz(n)[0] over dy(n).
    // The chunk holding n = 0 also yields grad_zi = dz(-1) (Eq.9, A.3).
    if (p.gzi != nullptr && p0 + s0 <= 0 && p0 + s0 + L > 0) {   // this chunk holds n = 0: walk down to it
        T w2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) w2[i] = d[i];
        for (int n = s0 + L - 1; n >= (int)(-p0); --n) adj_tdf_step<T, M>(w2, gs[pidx<T>(n)], ac);
        T* gzi = static_cast<T*>(p.gzi) + seq * M;
#pragma unroll
        for (int i = 0; i < M; ++i) gzi[i] = w2[i];
    }
#pragma unroll
    for (int g = L / W - 1; g >= 0; --g) {
        V dv = *reinterpret_cast<const V*>(gs + pidx<T>(s0 + g * W));
#pragma unroll
        for (int e = W - 1; e >= 0; --e) {
            const T dy = vget(dv, e);
            vset(dv, e, d[0]);
            adj_tdf_step<T, M>(d, dy, ac);           // d <- dz(n-1)
        }
        *reinterpret_cast<V*>(gs + pidx<T>(s0 + g * W)) = dv;
    }
    // y is the forward's output: with PDL this kernel may have started while the
    // forward was still running (its dy-only phases above overlap it)
    pdl_wait();
    if (tid == 0 && p.vec) prefetch_l2_bulk(yrow + pa, pbytes);
    __syncthreads();
    IIRG_TRACE(p.trace, tk, 4);
    // a7, pass B: coalesced.  Thread t owns the W-sample groups q = t + NT k.
    auto gat = [&](int m) -> T { return m < TS ? gs[pidx<T>(m)] : s_halo[m - TS]; };
    T Gs[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) Gs[k] = T(0);
    T* gxrow = p.gx == nullptr ? nullptr : static_cast<T*>(p.gx) + roff;
    const bool fast = p.vec && p0 >= 0 && p.gy != nullptr;   // interior tile: no clipping, no NULL dy
#pragma unroll 4
    for (int k = 0; k < L / W; ++k) {
        const int n0 = (tid + NT * k) * W;             // tile-local
        const int64_t pos = p0 + n0;
        V xv, yv, dyv;
        if (fast) {
            xv = ldg_l2(reinterpret_cast<const V*>(xrow + pos));
            yv = ldg_l2(reinterpret_cast<const V*>(yrow + pos));
            dyv = ldg_l2(reinterpret_cast<const V*>(gyrow + pos));
        } else if (p.vec && pos >= 0) {
            xv = ldg_l2(reinterpret_cast<const V*>(xrow + pos));
            yv = ldg_l2(reinterpret_cast<const V*>(yrow + pos));
            dyv = p.gy != nullptr ? ldg_l2(reinterpret_cast<const V*>(gyrow + pos)) : V{};
        } else {
#pragma unroll
            for (int e = 0; e < W; ++e) {
                const bool in = pos + e >= 0;
                vset(xv, e, in ? xrow[pos + e] : T(0));
                vset(yv, e, in ? yrow[pos + e] : T(0));
                vset(dyv, e, (in && p.gy != nullptr) ? gyrow[pos + e] : T(0));
            }
        }
        constexpr int NQ = (2 * W + M - 2) / W;       // W-vectors covering g(n0 .. n0 + W + M - 2)
        T gw[NQ * W];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {                 // 128-bit shared loads: conflict free
            const int m = n0 + q * W;
            if (m + W <= TS) {
                const V t = *reinterpret_cast<const V*>(gs + pidx<T>(m));
#pragma unroll
                for (int e = 0; e < W; ++e) gw[q * W + e] = vget(t, e);
            } else {
#pragma unroll
                for (int e = 0; e < W; ++e) gw[q * W + e] = gat(m + e);
            }
        }
        V dxv;
#pragma unroll
        for (int e = 0; e < W; ++e) {
            const T dy = vget(dyv, e), xx = vget(xv, e), yy = vget(yv, e);
            T dx = bc[0] * dy;
#pragma unroll
            for (int i = 0; i < M; ++i) dx = fma(cc[i], gw[e + i], dx);
#pragma unroll
            for (int i = 0; i < M; ++i) { Gs[i] = fma(gw[e + i], xx, Gs[i]); Gs[M + i] = fma(gw[e + i], yy, Gs[M + i]); }
            Gs[2 * M] = fma(dy, xx, Gs[2 * M]);
            vset(dxv, e, dx);
        }
        if (gxrow != nullptr) {
            if (fast || (p.vec && pos >= 0)) stg_stream(reinterpret_cast<V*>(gxrow + pos), dxv);
            else
#pragma unroll
                for (int e = 0; e < W; ++e)
                    if (pos + e >= 0) gxrow[pos + e] = vget(dxv, e);
        }
    }
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
    IIRG_TRACE(p.trace, tk, 5);
    IIRG_TRACE(p.trace, tk, 10);
    bwd_finalize<T, M, 1>(p, &cw, ep, tk, seq, jt, tb, s_red);
    IIRG_TRACE(p.trace, tk, 11);
    span_exit(p.span);
}


}  // namespace iirg
