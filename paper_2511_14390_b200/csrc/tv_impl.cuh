// tv_impl.cuh -- the per-order templates of the per-sample (time-varying) paths
// (IIR_COEF_PER_SAMPLE): the FIR stage of the general DF filter and the
// all-pole scan launches.  Instantiated per order in tv_o*.cu (split for parallel
// compilation: every order 1..31 is compiled), dispatched from tv.cu.
#pragma once
#include <type_traits>

#include "host.h"
#include "tv.cuh"

namespace iirg {

// ---- general time-varying DF (IIR_FLAG_PER_SAMPLE_B) ---------
// The filter factors into the all-pole recursion on the internal signal u
// (tv_* kernels above, whose "y" is u) and a per-sample FIR stage
// y(n) = sum_k b_k(n) u(n-k), u(-k) = zi[k-1] (Eqs.2-3 with b(n), a(n)).  The
// FIR stage's adjoint is  du(m) = sum_k b_k(m+k) dy(m+k)  (m >= -M; m < 0 are
// the zi entries) and  grad_b_k(n) = dy(n) u(n-k);  the all-pole backward then
// runs with grad_y = du, and grad_zi gains the FIR's direct terms du(-1..-M).
// One CTA per tile of FIR_TS consecutive samples of one sequence (compile-time
// order: every loop unrolled, no runtime division): the tile's b rows
// (contiguous in global memory) and the u / dy windows are staged in shared
// memory by coalesced loads (row stride padded to an odd count: the per-thread
// row reads are conflict free); grad_b rows leave through shared memory by
// coalesced stores.
// skew != 0 (the general TDF filter, tvtdf.cuh, reading R20): the stage runs on the SKEWED
// rows b~_k(n) = b_k(n - k) (zero before n = 0) without materialising them: the forward
// stages b rows [n0 - M, n0 + FIR_TS) and reads b~_k(n) as row n - k; the adjoint uses
// b~_k(m + k) = b_k(m) (rows of the tile only) and writes grad_b_k(m) = grad_b~_k(m + k)
// = dy(m + k) u(m) directly (the unskewed gradient; u's history is zero: no du(-1..-M)).
constexpr int FIR_TS = 256;
template <int M> struct Fir {
    static constexpr int K = M + 1, RS = K | 1;
};
template <typename T, int M>
__device__ __forceinline__ void fir_stage_rows(T* sb, const T* __restrict__ b, int64_t seq, int64_t Tlen, int64_t r0,
                                               int nr) {
    constexpr int K = Fir<M>::K, RS = Fir<M>::RS, W = 16 / (int)sizeof(T);
    const int nv = (int)max((int64_t)0, min((int64_t)nr, Tlen - r0));   // rows inside the sequence
    const int z = r0 < 0 ? (int)-r0 : 0;                                 // rows before n = 0 (skew: zero)
    const T* src = b + (seq * Tlen + r0) * K;
    // asynchronous copies (no register round trip: every load of the tile is in
    // flight at once); rows past the sequence end are zero-filled
    if (z == 0 && RS == K && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {     // same layout: 16 B chunks
        const int nvalid = nv * K;
        for (int e = threadIdx.x * W; e < nr * K; e += FIR_TS * W) {
            if (e + W <= nr * K) {
                const int left = nvalid - e;
                const unsigned bytes = left <= 0 ? 0u : (unsigned)(min(left, W) * (int)sizeof(T));
                cp_async16(sb + e, bytes ? (const void*)(src + e) : (const void*)src, bytes);
            } else {                   // the tile's last partial chunk: never write past nr * K
                for (int q = e; q < nr * K; ++q) {
                    if (q < nvalid) cp_async_elem(sb + q, src + q);
                    else sb[q] = T(0);
                }
            }
        }
    } else {
        for (int e = threadIdx.x; e < nr * K; e += FIR_TS) {
            const int r = e / K, k = e - r * K;
            if (r >= z && r < nv) cp_async_elem(sb + r * RS + k, src + e);
            else sb[r * RS + k] = T(0);
        }
    }
    cp_async_commit();
}
template <typename T, int M>
__device__ __forceinline__ T u_at(const T* __restrict__ u, const T* __restrict__ zi, int64_t seq, int64_t Tlen,
                                  int64_t m) {
    if (m >= 0) return m < Tlen ? u[seq * Tlen + m] : T(0);
    return zi != nullptr ? zi[seq * M + (-m - 1)] : T(0);
}
template <typename T, int M>
constexpr size_t fir_fwd_smem() { return ((size_t)(FIR_TS + M) * Fir<M>::RS + FIR_TS + M) * sizeof(T); }
template <typename T, int M>
constexpr size_t fir_bwd_smem() {
    return ((size_t)(FIR_TS + M) * Fir<M>::RS + (size_t)FIR_TS * Fir<M>::K + 2 * (FIR_TS + M)) * sizeof(T);
}

template <typename T, int M>
__global__ void __launch_bounds__(FIR_TS) tv_fir_fwd_kernel(const T* __restrict__ b, const T* __restrict__ u,
                                                            const T* __restrict__ zi, T* __restrict__ y,
                                                            int64_t Tlen, int64_t ntile, int skew) {
    constexpr int RS = Fir<M>::RS;
    extern __shared__ __align__(16) unsigned char fir_raw[];
    T* sb = reinterpret_cast<T*>(fir_raw);
    T* su = sb + (FIR_TS + M) * RS;                 // u(n0 - M .. n0 + FIR_TS - 1)
    const int64_t seq = blockIdx.x / ntile, n0 = (blockIdx.x - seq * ntile) * (int64_t)FIR_TS;
    const int t = threadIdx.x;
    if (skew) fir_stage_rows<T, M>(sb, b, seq, Tlen, n0 - M, FIR_TS + M);   // rows n0 - M ..
    else fir_stage_rows<T, M>(sb, b, seq, Tlen, n0, FIR_TS);
    for (int e = t; e < FIR_TS + M; e += FIR_TS) su[e] = u_at<T, M>(u, zi, seq, Tlen, n0 - M + e);
    cp_async_wait<0>();
    __syncthreads();
    if (n0 + t >= Tlen) return;
    double acc = 0.0;
    if (skew) {                                     // b~_k(n) = b_k(n - k): staged row t + M - k
#pragma unroll
        for (int k = 0; k <= M; ++k) acc = fma((double)sb[(t + M - k) * RS + k], (double)su[M + t - k], acc);
    } else {
#pragma unroll
        for (int k = 0; k <= M; ++k) acc = fma((double)sb[t * RS + k], (double)su[M + t - k], acc);
    }
    y[seq * Tlen + n0 + t] = (T)acc;
}

template <typename T, int M>
__global__ void __launch_bounds__(FIR_TS) tv_fir_bwd_kernel(const T* __restrict__ b, const T* __restrict__ u,
                                                            const T* __restrict__ zi, const T* __restrict__ gy,
                                                            T* __restrict__ du, T* __restrict__ duneg,
                                                            T* __restrict__ gb, int64_t Tlen, int64_t ntile,
                                                            int skew) {
    constexpr int K = Fir<M>::K, RS = Fir<M>::RS;
    extern __shared__ __align__(16) unsigned char fir_raw[];
    T* sb = reinterpret_cast<T*>(fir_raw);         // b rows n0 .. n0 + FIR_TS + M - 1
    T* sg = sb + (FIR_TS + M) * RS;                // grad_b rows of the tile, contiguous (stride K)
    T* sdy = sg + FIR_TS * K;                      // dy(n0 .. n0 + FIR_TS + M - 1)
    T* su = sdy + FIR_TS + M;                      // u(n0 - M .. n0 + FIR_TS - 1)
    const int64_t seq = blockIdx.x / ntile, n0 = (blockIdx.x - seq * ntile) * (int64_t)FIR_TS;
    const int t = threadIdx.x;
    fir_stage_rows<T, M>(sb, b, seq, Tlen, n0, skew ? FIR_TS : FIR_TS + M);
    for (int e = t; e < FIR_TS + M; e += FIR_TS) {
        const int64_t n = n0 + e;
        sdy[e] = (gy != nullptr && n < Tlen) ? gy[seq * Tlen + n] : T(0);
        su[e] = u_at<T, M>(u, zi, seq, Tlen, n0 - M + e);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (skew) {
        if (n0 + t < Tlen) {                        // du(m) = sum_k b~_k(m+k) dy(m+k) = sum_k b_k(m) dy(m+k)
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k <= M; ++k) acc = fma((double)sb[t * RS + k], (double)sdy[t + k], acc);
            du[seq * Tlen + n0 + t] = (T)acc;
            const double un = (double)su[M + t];    // grad_b_k(m) = grad_b~_k(m+k) = dy(m+k) u(m)
#pragma unroll
            for (int k = 0; k <= M; ++k) sg[t * K + k] = (T)((double)sdy[t + k] * un);
        }
    } else if (n0 + t < Tlen) {                     // du(m) = sum_k b_k(m+k) dy(m+k)
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k <= M; ++k) acc = fma((double)sb[(t + k) * RS + k], (double)sdy[t + k], acc);
        du[seq * Tlen + n0 + t] = (T)acc;
        const double dyn = (double)sdy[t];          // grad_b_k(m) = dy(m) u(m-k)
#pragma unroll
        for (int k = 0; k <= M; ++k) sg[t * K + k] = (T)(dyn * (double)su[M + t - k]);
    }
    if (!skew && n0 == 0 && t < M) {               // du(-1-t) (the zi entries): sum_{k > t} b_k(k-1-t) dy(k-1-t)
        double acc = 0.0;
#pragma unroll
        for (int k = 1; k <= M; ++k)
            if (k > t) acc = fma((double)sb[(k - 1 - t) * RS + k], (double)sdy[k - 1 - t], acc);
        duneg[seq * M + t] = (T)acc;
    }
    if (gb == nullptr) return;
    __syncthreads();
    const int nv = (int)min((int64_t)FIR_TS, Tlen - n0);
    T* gbt = gb + (seq * Tlen + n0) * K;            // the tile's grad_b rows are contiguous
    for (int e = t; e < nv * K; e += FIR_TS) gbt[e] = sg[e];
}

template <typename T, int M>
static iir_status_t fir_run(bool fwd, int skew, const iir_desc_t* d, const void* b, const void* u, const void* zi,
                            const void* gy, void* y, void* du, void* duneg, void* gb, cudaStream_t st) {
    const int64_t ntile = (d->length + FIR_TS - 1) / FIR_TS;
    const unsigned grid = (unsigned)(d->batch * ntile);
    static PerDevice attrs;
    attrs.once([] {
        cudaFuncSetAttribute(tv_fir_fwd_kernel<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fir_fwd_smem<T, M>());
        cudaFuncSetAttribute(tv_fir_bwd_kernel<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fir_bwd_smem<T, M>());
    });
    return launch(K_TV_FIR, st, [&] {
        if (fwd)
            tv_fir_fwd_kernel<T, M><<<grid, FIR_TS, fir_fwd_smem<T, M>(), st>>>(static_cast<const T*>(b),
                static_cast<const T*>(u), static_cast<const T*>(zi), static_cast<T*>(y), d->length, ntile, skew);
        else
            tv_fir_bwd_kernel<T, M><<<grid, FIR_TS, fir_bwd_smem<T, M>(), st>>>(static_cast<const T*>(b),
                static_cast<const T*>(u), static_cast<const T*>(zi), static_cast<const T*>(gy), static_cast<T*>(du),
                static_cast<T*>(duneg), static_cast<T*>(gb), d->length, ntile, skew);
    });
}
template <typename T>
__global__ void tv_add_kernel(T* __restrict__ dst, const T* __restrict__ src, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = dst[i] + src[i];
}

template <typename T, int M, int MODE>
static void tv_seq_launch(unsigned nseg_tot, const TvArgs& a, cudaStream_t st) {
    const size_t smem = TvStage<T, M, MODE>::bytes(MODE);
    static PerDevice attrs;
    attrs.once([&] {
        cudaFuncSetAttribute(tv_seq_kernel<T, M, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    const unsigned per = 32 * TV_SEQ_WARPS;
    tv_seq_kernel<T, M, MODE><<<(nseg_tot + per - 1) / per, per, smem, st>>>(a);
}

// phase 2 (both directions): group maps, chain over the groups, expansion
template <typename T, int M, bool BWD>
static iir_status_t tv_chain2(const TvArgs& a, const void* x0, cudaStream_t st) {
    const unsigned ng = (unsigned)(a.B * a.ngrp);
    const unsigned blocks = (ng + TV_GRP_WARPS - 1) / TV_GRP_WARPS;
    iir_status_t s = launch(K_TV_CHAIN, st, [&] {
        tv_group_kernel<T, M, BWD><<<blocks, 32 * TV_GRP_WARPS, 0, st>>>(a);
    });
    if (s != IIR_OK) return s;
    s = launch(K_TV_CHAIN, st, [&] {
        tv_groupchain_kernel<M, BWD><<<(unsigned)a.B, 32, 0, st>>>(a, x0, (int)sizeof(T));
    });
    if (s != IIR_OK) return s;
    return launch(K_TV_CHAIN, st, [&] { tv_expand_kernel<T, M, BWD><<<blocks, 32 * TV_GRP_WARPS, 0, st>>>(a); });
}

#ifndef IIRG_TV_PHI_F64
#define IIRG_TV_PHI_F64 0
#endif
template <typename T, int M>
static iir_status_t tv_fwd_m(const Layout& L, TvArgs& a, cudaStream_t st) {
    const unsigned nseg_tot = (unsigned)L.ntot;
    iir_status_t s;
    if constexpr (sizeof(T) == 4 && !IIRG_TV_PHI_F64) {
        // fp32 data: the segment transitions Phi_k in fp32 (their entries are tiny against the
        // carried states: measured 6e-14 absolute on config 3) and the zero-state responses w_k,
        // which carry the fp32-sequential error into the carries (R18), by an fp64 re-run of
        // the recursion (TV_FWD_AGG) that overwrites tv_phi's fp32 w.  The fp64 tv_phi was
        // bound by its fp64 coefficient broadcasts (twice the shared-memory traffic of fp32).
        // The two are independent (both read a and x): the fp64 re-run (few, latency-bound warps)
        // runs on a side stream beside the transitions (many warps, FMA / shared-memory bound).
        SideStream& ss = side_stream();
        if (cudaEventRecord(ss.fork, st) != cudaSuccess || cudaStreamWaitEvent(ss.st, ss.fork, 0) != cudaSuccess)
            return fail(IIR_ECUDA, "side-stream fork failed");
        s = launch(K_TV_WAGG, ss.st, [&] { tv_seq_launch<T, M, TV_FWD_AGG>(nseg_tot, a, ss.st); });
        if (s != IIR_OK) return s;
        if (cudaEventRecord(ss.join, ss.st) != cudaSuccess) return fail(IIR_ECUDA, "side-stream join failed");
        TvArgs aphi = a;
        aphi.w = nullptr;                                   // w is the side stream's
        s = launch(K_TV_PHI, st, [&] {
            tv_phi_kernel<T, M, T><<<(nseg_tot + TV_PHI_WARPS - 1) / TV_PHI_WARPS, 32 * TV_PHI_WARPS, 0, st>>>(aphi);
        });
        if (s != IIR_OK) return s;
        if (cudaStreamWaitEvent(st, ss.join, 0) != cudaSuccess) return fail(IIR_ECUDA, "side-stream join failed");
    } else {
        s = launch(K_TV_PHI, st, [&] {
            tv_phi_kernel<T, M, double><<<(nseg_tot + TV_PHI_WARPS - 1) / TV_PHI_WARPS, 32 * TV_PHI_WARPS, 0, st>>>(a);
        });
    }
    if (s != IIR_OK) return s;
    s = tv_chain2<T, M, false>(a, a.zi, st);
    if (s != IIR_OK) return s;
    return launch(K_TV_FWD, st, [&] { tv_seq_launch<T, M, TV_FWD_EMIT>(nseg_tot, a, st); });
}

template <typename T, int M>
static iir_status_t tv_bwd_m(const Layout& L, TvArgs& a, cudaStream_t st) {
    const unsigned nseg_tot = (unsigned)L.ntot;
    iir_status_t s = launch(K_TV_BWD_AGG, st, [&] { tv_seq_launch<T, M, TV_BWD_AGG>(nseg_tot, a, st); });
    if (s != IIR_OK) return s;
    s = tv_chain2<T, M, true>(a, a.gzf, st);
    if (s != IIR_OK) return s;
    return launch(K_TV_BWD, st, [&] { tv_seq_launch<T, M, TV_BWD_EMIT>(nseg_tot, a, st); });
}

// one entry per (dtype, order): op 0 / 1 = all-pole scan forward / backward,
// op 2 / 3 = FIR stage forward / backward
template <typename T, int M>
iir_status_t tv_order(int op, const iir_desc_t* d, const Layout& L, TvArgs& a, const void* b, const void* u,
                      const void* zi, const void* gy, void* y, void* du, void* duneg, void* gb, cudaStream_t st) {
    switch (op) {
        case 0: return tv_fwd_m<T, M>(L, a, st);
        case 1: return tv_bwd_m<T, M>(L, a, st);
        case 2: return fir_run<T, M>(true, 0, d, b, u, zi, gy, y, du, duneg, gb, st);
        case 3: return fir_run<T, M>(false, 0, d, b, u, zi, gy, y, du, duneg, gb, st);
        case 4: return fir_run<T, M>(true, 1, d, b, u, zi, gy, y, du, duneg, gb, st);    // skewed rows (TDF)
        default: return fir_run<T, M>(false, 1, d, b, u, zi, gy, y, du, duneg, gb, st);
    }
}

#define IIRG_TV_INST(m)                                                                                        \
    template iir_status_t tv_order<float, m>(int, const iir_desc_t*, const Layout&, TvArgs&, const void*,      \
                                             const void*, const void*, const void*, void*, void*, void*,      \
                                             void*, cudaStream_t);                                            \
    template iir_status_t tv_order<double, m>(int, const iir_desc_t*, const Layout&, TvArgs&, const void*,     \
                                              const void*, const void*, const void*, void*, void*, void*,     \
                                              void*, cudaStream_t);

}  // namespace iirg
