// tv.cuh -- per-sample ("parameter-varying") all-pole DF filter:
//   y(n) = x(n) - sum_{i=1..M} a_i(n) y(n-i),   v(n) = [y(n-1) .. y(n-M)],  v(0) = zi
// and its closed-form backward (Eq.7 with time-varying A(n) = companion(a(n)),
// C(n) = -a(n), D = 1; readings R10/R11):
//   g(n) = dz(n)[0] + dy(n)        (= grad_x(n), Eq.8)
//   dz(n-1)[i] = dz(n)[i+1] - a_{i+1}(n) g(n),   dz(N-1) = grad_zf,  grad_zi = dz(-1)
//   grad_a_i(n) = -g(n) y(n-i)     (Eq.9's dA(n) = dz(n) v(n)^T and Eq.6's dC)
//
// Time parallelism (Eq.10) with time-varying transitions: the sequence is cut
// into segments of TV_SEG samples.  Segment k's transition Phi_k = A(n1-1)..A(n0)
// and zero-state response w_k are built by one warp, lane j propagating the
// basis state e_j (lane M propagates x from the zero state): M^2 FMA per sample,
// the price of a matrix-valued scan element.  A per-sequence fp64
// chain s_{k+1} = Phi_k s_k + w_k gives every segment's entering state, and one
// thread per segment re-runs the plain recursion from it.  The backward reuses
// Phi_k^T from the tape (the adjoint segment map is exactly Phi_k^T).
#pragma once
#include "common.cuh"

namespace iirg {

constexpr int TV_SEG = 512;          // samples per segment
constexpr int TV_THREADS = 128;      // thread-per-segment kernels
constexpr int TV_PHI_WARPS = 4;      // warps (segments) per CTA of the Phi kernel
constexpr int TV_CH = 32;            // samples per staged coefficient chunk (Phi kernel)
constexpr int TV_U = 8;              // unroll of the sequential recursions

struct TvArgs {
    const void* a; const void* x; const void* zi;     // a: (B, T, M)
    void* y; void* zf;                                // forward outputs
    const void* gy; const void* gzf; const void* yin; // backward inputs (yin = forward y)
    void* gx; void* ga; void* gzi;                    // backward outputs
    void* phi;                                        // tape: [B][nseg][M][M]  (Phi[i][j])
    double* w;                                        // ws: [B][nseg][M] segment aggregates
    double* carry;                                    // ws: [B][nseg][M] entering states
    int64_t B, T; int nseg;
};

// ---------------------------------------------------------------------------
// Forward phase 1: one warp per segment builds Phi_k (lanes 0..M-1) and w_k
// (lane M).  Coefficients are staged per chunk of TV_CH samples in shared
// memory and read by broadcast.
template <typename T, int M>
__global__ void __launch_bounds__(32 * TV_PHI_WARPS) tv_phi_kernel(const TvArgs p) {
    static_assert(M + 1 <= 32, "one lane per basis state plus one for the input");
    __shared__ __align__(16) T sa[TV_PHI_WARPS][TV_CH * M];
    __shared__ T sx[TV_PHI_WARPS][TV_CH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t seg = (int64_t)blockIdx.x * TV_PHI_WARPS + warp;
    if (seg >= p.B * p.nseg) return;
    const int64_t seq = seg / p.nseg;
    const int k = (int)(seg - seq * p.nseg);
    const int64_t n0 = (int64_t)k * TV_SEG, n1 = min(n0 + TV_SEG, p.T);
    const T* arow = static_cast<const T*>(p.a) + seq * p.T * M;
    const T* xrow = static_cast<const T*>(p.x) + seq * p.T;
    T v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = (lane == i) ? T(1) : T(0);
    for (int64_t c = n0; c < n1; c += TV_CH) {
        const int cnt = (int)min((int64_t)TV_CH, n1 - c);
        __syncwarp();
        for (int e = lane; e < TV_CH * M; e += 32) sa[warp][e] = (e < cnt * M) ? arow[c * M + e] : T(0);
        sx[warp][lane] = (lane < cnt) ? xrow[c + lane] : T(0);
        __syncwarp();
        if (cnt == TV_CH) {
#pragma unroll
            for (int s2 = 0; s2 < TV_CH; ++s2) {
                T yn = (lane == M) ? sx[warp][s2] : T(0);
#pragma unroll
                for (int i = M - 1; i >= 0; --i) yn = fma(-sa[warp][s2 * M + i], v[i], yn);   // newest term last
#pragma unroll
                for (int i = M - 1; i >= 1; --i) v[i] = v[i - 1];
                v[0] = yn;
            }
        } else {                                   // ragged last chunk: exactly cnt samples
            for (int s2 = 0; s2 < cnt; ++s2) {
                T yn = (lane == M) ? sx[warp][s2] : T(0);
#pragma unroll
                for (int i = M - 1; i >= 0; --i) yn = fma(-sa[warp][s2 * M + i], v[i], yn);
#pragma unroll
                for (int i = M - 1; i >= 1; --i) v[i] = v[i - 1];
                v[0] = yn;
            }
        }
    }
    const T (&vf)[M] = v;
    if (lane < M) {
        T* ph = static_cast<T*>(p.phi) + seg * M * M;
#pragma unroll
        for (int i = 0; i < M; ++i) ph[i * M + lane] = vf[i];              // column `lane`
    } else if (lane == M) {
#pragma unroll
        for (int i = 0; i < M; ++i) p.w[seg * M + i] = (double)vf[i];
    }
}

// ---------------------------------------------------------------------------
// Phase 2: per-sequence fp64 chain over the segments (one warp per sequence,
// lane i = row i).  FWD: s_0 = zi, s_{k+1} = Phi_k s_k + w_k.
// BWD: d_{nseg-1} = grad_zf, d_{k-1} = Phi_k^T d_k + w_k.  carry[k] = entering state.
template <typename T, int M, bool BWD>
__global__ void __launch_bounds__(32) tv_chain_kernel(const TvArgs p) {
    __shared__ double ss[M];
    const int lane = threadIdx.x;
    const int64_t seq = blockIdx.x;
    const T* x0 = static_cast<const T*>(BWD ? p.gzf : p.zi);
    double s = (lane < M && x0 != nullptr) ? (double)x0[seq * M + lane] : 0.0;
    const T* phi = static_cast<const T*>(p.phi) + seq * p.nseg * M * M;
    for (int q = 0; q < p.nseg; ++q) {
        const int k = BWD ? p.nseg - 1 - q : q;
        if (lane < M) {
            p.carry[(seq * p.nseg + k) * M + lane] = s;
            ss[lane] = s;
        }
        __syncwarp();
        double acc = (lane < M) ? p.w[(seq * p.nseg + k) * M + lane] : 0.0;
        if (lane < M) {
            const T* ph = phi + (int64_t)k * M * M;
#pragma unroll
            for (int j = 0; j < M; ++j) acc = fma((double)(BWD ? ph[j * M + lane] : ph[lane * M + j]), ss[j], acc);
        }
        __syncwarp();
        s = acc;
    }
}

// Coefficient row of sample n (M values).
template <typename T, int M>
__device__ __forceinline__ void load_row(const T* __restrict__ ar, T (&c)[M]) {
    if constexpr (sizeof(T) == 4 && M % 4 == 0) {
#pragma unroll
        for (int q = 0; q < M / 4; ++q) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(ar) + q);
            c[4 * q] = t.x; c[4 * q + 1] = t.y; c[4 * q + 2] = t.z; c[4 * q + 3] = t.w;
        }
    } else if constexpr (sizeof(T) == 8 && M % 2 == 0) {
#pragma unroll
        for (int q = 0; q < M / 2; ++q) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(ar) + q);
            c[2 * q] = t.x; c[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) c[i] = __ldg(ar + i);
    }
}

// ---------------------------------------------------------------------------
// Forward phase 3: one thread per segment re-runs the recursion from its
// entering state and writes y (and zf from the segment holding sample T-1).
// The thread-per-segment recursions accumulate in fp64 (R = double) with T I/O:
// they are bound by the 4M bytes of coefficients per sample, and fp64 removes the
// O(TV_SEG) fp32 rounding growth of a 24-tap feedback loop ("TV precision").
template <typename T, int M>
__global__ void __launch_bounds__(TV_THREADS) tv_emit_kernel(const TvArgs p) {
    using R = double;
    const int64_t seg = (int64_t)blockIdx.x * TV_THREADS + threadIdx.x;
    if (seg >= p.B * p.nseg) return;
    const int64_t seq = seg / p.nseg;
    const int k = (int)(seg - seq * p.nseg);
    const int64_t n0 = (int64_t)k * TV_SEG, n1 = min(n0 + TV_SEG, p.T);
    const T* arow = static_cast<const T*>(p.a) + seq * p.T * M;
    const T* xrow = static_cast<const T*>(p.x) + seq * p.T;
    T* yrow = static_cast<T*>(p.y) + seq * p.T;
    R v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = p.carry[seg * M + i];
    int64_t n = n0;
    for (; n + TV_U <= n1; n += TV_U) {
#pragma unroll
        for (int u = 0; u < TV_U; ++u) {
            T c[M];
            load_row<T, M>(arow + (n + u) * M, c);
            R yn = (R)__ldg(xrow + n + u);
#pragma unroll
            for (int i = M - 1; i >= 0; --i) yn = fma(-(R)c[i], v[i], yn);
#pragma unroll
            for (int i = M - 1; i >= 1; --i) v[i] = v[i - 1];
            v[0] = yn;
            yrow[n + u] = (T)yn;
        }
    }
    for (; n < n1; ++n) {
        T c[M];
        load_row<T, M>(arow + n * M, c);
        R yn = (R)__ldg(xrow + n);
#pragma unroll
        for (int i = M - 1; i >= 0; --i) yn = fma(-(R)c[i], v[i], yn);
#pragma unroll
        for (int i = M - 1; i >= 1; --i) v[i] = v[i - 1];
        v[0] = yn;
        yrow[n] = (T)yn;
    }
    if (p.zf != nullptr && n1 == p.T) {
        T* zf = static_cast<T*>(p.zf) + seq * M;
#pragma unroll
        for (int i = 0; i < M; ++i) zf[i] = (T)v[i];
    }
}

// ---------------------------------------------------------------------------
// Backward phase 1: one thread per segment, adjoint from the zero state at the
// segment's end, walking back: w_k = dz(n0-1) given dz(n1-1) = 0.
template <typename T, int M>
__global__ void __launch_bounds__(TV_THREADS) tv_bwd_agg_kernel(const TvArgs p) {
    using R = double;
    const int64_t seg = (int64_t)blockIdx.x * TV_THREADS + threadIdx.x;
    if (seg >= p.B * p.nseg) return;
    const int64_t seq = seg / p.nseg;
    const int k = (int)(seg - seq * p.nseg);
    const int64_t n0 = (int64_t)k * TV_SEG, n1 = min(n0 + TV_SEG, p.T);
    const T* arow = static_cast<const T*>(p.a) + seq * p.T * M;
    const T* gyrow = p.gy == nullptr ? nullptr : static_cast<const T*>(p.gy) + seq * p.T;
    R d[M];
#pragma unroll
    for (int i = 0; i < M; ++i) d[i] = 0.0;
    for (int64_t n = n1 - 1; n >= n0; --n) {
        T c[M];
        load_row<T, M>(arow + n * M, c);
        const R g = d[0] + (gyrow ? (R)__ldg(gyrow + n) : 0.0);
#pragma unroll
        for (int i = 0; i < M - 1; ++i) d[i] = fma(-(R)c[i], g, d[i + 1]);
        d[M - 1] = -(R)c[M - 1] * g;
    }
#pragma unroll
    for (int i = 0; i < M; ++i) p.w[seg * M + i] = (double)d[i];
}

// Backward phase 3: one thread per segment from its entering adjoint state:
// grad_x, grad_a (M per sample), and grad_zi from the first segment.
template <typename T, int M>
__global__ void __launch_bounds__(TV_THREADS) tv_bwd_emit_kernel(const TvArgs p) {
    using R = double;
    const int64_t seg = (int64_t)blockIdx.x * TV_THREADS + threadIdx.x;
    if (seg >= p.B * p.nseg) return;
    const int64_t seq = seg / p.nseg;
    const int k = (int)(seg - seq * p.nseg);
    const int64_t n0 = (int64_t)k * TV_SEG, n1 = min(n0 + TV_SEG, p.T);
    const T* arow = static_cast<const T*>(p.a) + seq * p.T * M;
    const T* gyrow = p.gy == nullptr ? nullptr : static_cast<const T*>(p.gy) + seq * p.T;
    const T* yrow = static_cast<const T*>(p.yin) + seq * p.T;
    const T* zi = p.zi == nullptr ? nullptr : static_cast<const T*>(p.zi) + seq * M;
    T* gxrow = p.gx == nullptr ? nullptr : static_cast<T*>(p.gx) + seq * p.T;
    T* garow = p.ga == nullptr ? nullptr : static_cast<T*>(p.ga) + seq * p.T * M;
    auto yat = [&](int64_t m) -> R {                 // y(m), m >= -M; y(-k) = zi[k-1]
        if (m >= 0) return (R)__ldg(yrow + m);
        return zi != nullptr ? (R)zi[-m - 1] : 0.0;
    };
    R d[M], yw[M];                                   // yw[i] = y(n-1-i)
#pragma unroll
    for (int i = 0; i < M; ++i) { d[i] = p.carry[seg * M + i]; yw[i] = yat(n1 - 2 - i); }
    for (int64_t n = n1 - 1; n >= n0; --n) {
        T c[M];
        load_row<T, M>(arow + n * M, c);
        const R g = d[0] + (gyrow ? (R)__ldg(gyrow + n) : 0.0);
        if (gxrow) gxrow[n] = (T)g;
        if (garow) {
#pragma unroll
            for (int i = 0; i < M; ++i) garow[n * M + i] = (T)(-g * yw[i]);
        }
#pragma unroll
        for (int i = 0; i < M - 1; ++i) d[i] = fma(-(R)c[i], g, d[i + 1]);
        d[M - 1] = -(R)c[M - 1] * g;
#pragma unroll
        for (int i = 0; i < M - 1; ++i) yw[i] = yw[i + 1];
        yw[M - 1] = yat(n - 2 - (M - 1));
    }
    if (p.gzi != nullptr && k == 0) {
        T* gzi = static_cast<T*>(p.gzi) + seq * M;
#pragma unroll
        for (int i = 0; i < M; ++i) gzi[i] = (T)d[i];
    }
}

}  // namespace iirg
