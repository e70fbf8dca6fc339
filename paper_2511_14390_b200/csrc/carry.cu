// carry.cu -- time-sharded sequences: the exact state entering
// a segment from the other segments' zero-carry aggregates, Eq.10 (PAPER.md:
// 121-130) with the whole segment as the chunk: P = A_f^seg_len by binary
// powering in fp64, then a Horner sum over the segments (include/iirgrad.h,
// iir_state_carry).
#include <cuda_runtime.h>

#include <string>

#include "../../include/iirgrad.h"
#include "host.h"

namespace iirg {

constexpr int SC_THREADS = 64;                 // >= M^2 for M <= 8

// C = A B (M x M, row-major, shared memory); thread e < M^2 owns element e.
template <int M>
__device__ __forceinline__ void mm(double* C, const double* A, const double* B) {
    const int e = threadIdx.x;
    double acc = 0.0;
    if (e < M * M) {
        const int i = e / M, j = e % M;
#pragma unroll
        for (int k = 0; k < M; ++k) acc = fma(A[i * M + k], B[k * M + j], acc);
    }
    __syncthreads();
    if (e < M * M) C[e] = acc;
    __syncthreads();
}

template <typename T, int M>
__global__ void __launch_bounds__(SC_THREADS) state_carry_kernel(const T* __restrict__ a, int64_t cstride, int form,
                                                                const T* __restrict__ w, int nseg, int rank,
                                                                int64_t seg_len, int reverse, T* __restrict__ out,
                                                                int64_t B) {
    __shared__ double P[M * M], X[M * M], an[M + 1], s[M];
    const int64_t seq = blockIdx.x;
    const int tid = threadIdx.x;
    const T* aa = a + seq * cstride;
    if (tid <= M) an[tid] = (double)aa[tid] / (double)aa[0];
    __syncthreads();
    // base X = A_f (DF: companion(a'), row 0 = -a'[1..M], ones below the diagonal;
    // TDF: its transpose), transposed once more for the adjoint direction
    if (tid < M * M) {
        int i = tid / M, j = tid % M;
        if ((form == 1) != (reverse != 0)) { const int t = i; i = j; j = t; }
        X[tid] = (i == 0) ? -an[j + 1] : (i == j + 1 ? 1.0 : 0.0);
        P[tid] = (tid / M == tid % M) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int64_t e = seg_len; e > 0; e >>= 1) {    // P = X^seg_len
        if (e & 1) mm<M>(P, P, X);
        if (e > 1) mm<M>(X, X, X);
    }
    if (tid < M) s[tid] = 0.0;
    __syncthreads();
    const int j0 = reverse ? nseg - 1 : 0, j1 = rank, dj = reverse ? -1 : 1;
    for (int j = j0; j != j1; j += dj) {            // s <- P s + w_j (segments before `rank` in scan order)
        double v = 0.0;
        if (tid < M) {
#pragma unroll
            for (int k = 0; k < M; ++k) v = fma(P[tid * M + k], s[k], v);
            v += (double)w[((int64_t)j * B + seq) * M + tid];
        }
        __syncthreads();
        if (tid < M) s[tid] = v;
        __syncthreads();
    }
    if (tid < M) out[seq * M + tid] = (T)s[tid];
}

template <typename T>
static void launch_sc(int M, unsigned grid, cudaStream_t st, const T* a, int64_t cs, int form, const T* w, int nseg,
                      int rank, int64_t len, int rev, T* out, int64_t B) {
#define IIRG_SC(MM) case MM: state_carry_kernel<T, MM><<<grid, SC_THREADS, 0, st>>>(a, cs, form, w, nseg, rank, len, rev, out, B); break;
    switch (M) { IIRG_SC(1) IIRG_SC(2) IIRG_SC(3) IIRG_SC(4) IIRG_SC(5) IIRG_SC(6) IIRG_SC(7) IIRG_SC(8) }
#undef IIRG_SC
}

}  // namespace iirg

using namespace iirg;

extern "C" iir_status_t iir_state_carry(const iir_desc_t* d, const void* a, const void* w, int32_t nseg, int32_t rank,
                                        int64_t seg_len, int32_t reverse, void* out, iir_stream_t stream) {
    if (d == nullptr) return fail(IIR_EINVAL, "desc is NULL");
    if (d->batch < 1) return fail(IIR_EINVAL, "batch must be >= 1");
    if (d->form != IIR_DF2 && d->form != IIR_TDF2) return fail(IIR_EUNSUPPORTED, "state carry: DF2 / TDF2 only");
    if (d->coef_mode != IIR_COEF_SHARED && d->coef_mode != IIR_COEF_PER_SEQ)
        return fail(IIR_EUNSUPPORTED, "state carry: SHARED or PER_SEQ coefficients");
    if (d->order < 1 || d->order > 8) return fail(IIR_EUNSUPPORTED, "state carry: order must be 1..8");
    if (d->dtype != IIR_F32 && d->dtype != IIR_F64) return fail(IIR_EINVAL, "dtype must be IIR_F32 or IIR_F64");
    if (nseg < 1 || rank < 0 || rank >= nseg) return fail(IIR_EINVAL, "need 0 <= rank < nseg");
    if (seg_len < 0) return fail(IIR_EINVAL, "seg_len must be >= 0");
    if (a == nullptr || w == nullptr || out == nullptr) return fail(IIR_EINVAL, "a, w and out must be non-NULL");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t cs = d->coef_mode == IIR_COEF_SHARED ? 0 : d->order + 1;
    return launch(K_STATE_CARRY, st, [&] {
        if (d->dtype == IIR_F32)
            launch_sc<float>(d->order, (unsigned)d->batch, st, static_cast<const float*>(a), cs, d->form,
                             static_cast<const float*>(w), nseg, rank, seg_len, reverse,
                             static_cast<float*>(out), d->batch);
        else
            launch_sc<double>(d->order, (unsigned)d->batch, st, static_cast<const double*>(a), cs, d->form,
                              static_cast<const double*>(w), nseg, rank, seg_len, reverse,
                              static_cast<double*>(out), d->batch);
    });
}
