// tvtdf.cuh -- general time-varying TDF-II filter (reading R20):
// the TDF realisation of PAPER.md:67-68 at every sample,
//     y(n) = b_0(n) x(n) + v_1(n),   v_i(n+1) = v_{i+1}(n) + b_i(n) x(n) - a_i(n) y(n).
// Unrolled, y(n) = sum_k b_k(n-k) x(n-k) - sum_i a_i(n-i) y(n-i) + zi[n] (n < M): the
// zeros-then-poles (DF-I) structure on SKEWED coefficient rows
//     b~_k(n) = b_k(n - k),   a~_i(n) = a_i(n - i)      (zero before n = 0),
// so the path reuses the per-sample kernels of the DF filter: the FIR stage (tv_fir on the
// skewed rows b~, read in place from b; zero history) gives f, zi is added to f(0..M-1), and the all-pole recursion (rows a~,
// zero history) gives y.  zf = v(N) is the tail sum
//     zf_i = zi_{i+N} + sum_{d=0}^{min(N-1, M-i)} [b_{i+d}(m) x(m) - a_{i+d}(m) y(m)],  m = N-1-d.
// Backward: the all-pole adjoint on rows a~ (input grad_y plus the zf tail terms) gives
// g = dL/df and grad_a~; the FIR adjoint on rows b~ gives grad_x and grad_b (= grad_b~ at the
// skewed rows, written unskewed); the skew of a is undone (grad_a_i(m) = grad_a~_i(m + i)) and
// the zf tail terms are added.
#pragma once
#include "common.cuh"

namespace iirg {
namespace tdf {

constexpr int NT = 256;

constexpr int SR = 128;    // rows (samples) per block of the skew kernels

// dst[q] = src[q] for q in [q_lo, q_hi), zero elsewhere, q in [0, cnt): a block's contiguous run of
// rows staged into shared memory, four independent loads in flight per thread (the runs are read
// once: streaming hint)
template <typename T>
__device__ __forceinline__ void stage_rows(T* __restrict__ dst, const T* __restrict__ src, int64_t base, int cnt,
                                           int q_lo, int q_hi) {
    int q = threadIdx.x;
    for (; q + 3 * NT < cnt; q += 4 * NT) {
        T v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = q + u * NT;
            v[u] = (e >= q_lo && e < q_hi) ? __ldcs(src + base + e) : T(0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) dst[q + u * NT] = v[u];
    }
    for (; q < cnt; q += NT) dst[q] = (q >= q_lo && q < q_hi) ? __ldcs(src + base + q) : T(0);
}

// out[e] = s[e + off(c)], c = e mod W, for e in [0, cnt) (the column index c advanced
// incrementally: no division in the loop)
template <typename T, typename Off>
__device__ __forceinline__ void emit_rows(T* __restrict__ out, const T* __restrict__ s, int cnt, int W, Off off) {
    const int st = NT % W;
    int c = threadIdx.x % W;
    for (int e = threadIdx.x; e < cnt; e += NT) {
        __stcs(out + e, s[e + off(c)]);
        c += st;
        if (c >= W) c -= W;
    }
}

// a~ (B, N, M) from a.  Block (tile, sequence): rows [n0, n0 + SR) of the output need input
// rows [n0 - M, n0 + SR); they are staged through shared memory so every global access is a
// contiguous run of rows.  (b~ is never materialised: the FIR stage reads b at skewed rows,
// tv_impl.cuh.)
template <typename T>
__global__ void __launch_bounds__(NT) skew_kernel(const T* __restrict__ a, T* __restrict__ as, int64_t N, int M) {
    extern __shared__ __align__(16) unsigned char skew_raw[];
    T* sa = reinterpret_cast<T*>(skew_raw);                 // (SR + M) x M
    const int64_t s = blockIdx.y, n0 = (int64_t)blockIdx.x * SR;
    const int64_t lo = n0 - M;                               // first staged input row
    const int rows = (int)min((int64_t)SR + M, N - lo);      // staged rows inside the sequence
    const int r0 = lo < 0 ? (int)-lo : 0;                    // staged rows before n = 0 (zero)
    stage_rows(sa, a, (s * N + lo) * M, (SR + M) * M, r0 * M, rows * M);
    __syncthreads();
    const int nout = (int)min((int64_t)SR, N - n0);
    // a~_i(n) = a_i(n - i), column c = i - 1: staged row r + M - i  ->  offset (M - 1 - c) M
    emit_rows(as + (s * N + n0) * M, sa, nout * M, M, [=](int c) { return (M - 1 - c) * M; });
}
template <typename T>
constexpr size_t skew_smem(int M) { return (size_t)(SR + M) * M * sizeof(T); }

// grad_a from the gradient of the skewed rows: g_i(m) = g~_i(m + i) (zero past N);
// block (tile, sequence) stages input rows [m0, m0 + SR + M)
template <typename T>
__global__ void __launch_bounds__(NT) unskew_kernel(const T* __restrict__ gas, T* __restrict__ ga, int64_t N, int M) {
    extern __shared__ __align__(16) unsigned char skew_raw[];
    T* sa = reinterpret_cast<T*>(skew_raw);
    const int64_t s = blockIdx.y, m0 = (int64_t)blockIdx.x * SR;
    const int rows = (int)min((int64_t)SR + M, N - m0);
    const int nout = (int)min((int64_t)SR, N - m0);
    stage_rows(sa, gas, (s * N + m0) * M, (SR + M) * M, 0, rows * M);
    __syncthreads();
    // column c = i - 1: staged row r + i  ->  offset (c + 1) M
    emit_rows(ga + (s * N + m0) * M, sa, nout * M, M, [=](int c) { return (c + 1) * M; });
}

// f(n) += zi[n], n < min(M, N); one thread per (sequence, n)
template <typename T>
__global__ void zi_add_kernel(T* __restrict__ f, const T* __restrict__ zi, int64_t B, int64_t N, int M) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= B * M) return;
    const int64_t s = e / M;
    const int n = (int)(e - s * M);
    if (n < N) f[s * N + n] = f[s * N + n] + zi[e];
}

// zf = v(N) by the tail sum (fp64 accumulation); one thread per (sequence, i)
template <typename T>
__global__ void zf_kernel(const T* __restrict__ a, const T* __restrict__ b, const T* __restrict__ x,
                          const T* __restrict__ y, const T* __restrict__ zi, T* __restrict__ zf, int64_t B, int64_t N,
                          int M) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= B * M) return;
    const int64_t s = e / M;
    const int i = (int)(e - s * M) + 1;               // 1-based state index
    const int64_t K = M + 1;
    double acc = (zi != nullptr && i + N <= M) ? (double)zi[s * M + i + N - 1] : 0.0;
    for (int d = 0; d <= M - i && d < N; ++d) {
        const int64_t m = N - 1 - d, r = s * N + m;
        const int j = i + d;
        acc += (double)b[r * K + j] * (double)x[r] - (double)a[r * M + j - 1] * (double)y[r];
    }
    zf[e] = (T)acc;
}

// gye(n) = gy(n) - sum_{i=1}^{M-d} a_{i+d}(n) gzf_i  (d = N-1-n; the zf tail's y terms);
// block (tile, sequence), one thread per n
template <typename T>
__global__ void __launch_bounds__(NT) gy_eff_kernel(const T* __restrict__ gy, const T* __restrict__ gzf,
                                                    const T* __restrict__ a, T* __restrict__ gye, int64_t N, int M) {
    const int64_t s = blockIdx.y, n = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (n >= N) return;
    const int64_t r = s * N + n, d = N - 1 - n;
    double v = gy != nullptr ? (double)gy[r] : 0.0;
    if (gzf != nullptr && d < M)
        for (int i = 1; i + d <= M; ++i) v -= (double)a[r * M + i + d - 1] * (double)gzf[s * M + i - 1];
    gye[r] = (T)v;
}

// After the FIR adjoint and the unskew: the zf tail's x / coefficient terms and grad_zi.
//   gx(m) += sum_{i} b_{i+d}(m) gzf_i,  gb_{i+d}(m) += gzf_i x(m),  ga_{i+d}(m) -= gzf_i y(m)  (m = N-1-d)
//   gzi[k] = g(k) (k < N: zi adds into f(k))  +  gzf[k - N] (k >= N: zi_{k} reaches zf directly)
// One thread per (sequence, k), k = 0..M-1 (k doubles as the tail offset d).
template <typename T>
__global__ void tail_kernel(const T* __restrict__ gzf, const T* __restrict__ a, const T* __restrict__ b,
                            const T* __restrict__ x, const T* __restrict__ y, const T* __restrict__ g,
                            T* __restrict__ gx, T* __restrict__ ga, T* __restrict__ gb, T* __restrict__ gzi,
                            int64_t B, int64_t N, int M) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= B * M) return;
    const int64_t s = e / M;
    const int k = (int)(e - s * M);
    const int64_t K = M + 1;
    if (gzi != nullptr) {
        double v = k < N ? (double)g[s * N + k] : 0.0;
        if (gzf != nullptr && k >= N) v += (double)gzf[s * M + k - N];
        gzi[e] = (T)v;
    }
    const int d = k;
    if (gzf == nullptr || d >= N) return;
    const int64_t m = N - 1 - d, r = s * N + m;
    double dx = 0.0;
    for (int i = 1; i + d <= M; ++i) {
        const double gz = (double)gzf[s * M + i - 1];
        const int j = i + d;
        dx += (double)b[r * K + j] * gz;
        if (gb != nullptr) gb[r * K + j] = (T)((double)gb[r * K + j] + gz * (double)x[r]);
        if (ga != nullptr) ga[r * M + j - 1] = (T)((double)ga[r * M + j - 1] - gz * (double)y[r]);
    }
    if (gx != nullptr) gx[r] = (T)((double)gx[r] + dx);
}

}  // namespace tdf
}  // namespace iirg
