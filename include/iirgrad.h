/*
 * iirgrad.h -- C ABI of the B200-native differentiable IIR filter library
 * (libiirgrad.so), the hot path of arXiv 2511.14390.
 *
 * What it computes (citations are /root/reference/PAPER.md lines):
 *   Eq.1 (l.46-51)   H(z) = (b0 + b1 z^-1 + .. + bM z^-M) / (a0 + a1 z^-1 + .. + aM z^-M)
 *                    (a0 != 0; the library normalises by a0 -- Eq.1 is monic).
 *   Eq.2-3 (l.53-56) DF-II:  u(n) = x(n) - sum a_i u(n-i),  y(n) = sum b_i u(n-i)
 *   TDF-II (l.58,67) the transposed form, state space (A^T, C, B, D)
 *                    == scipy.signal.lfilter(b, a, x, zi).
 *   Eq.4-5 (l.60-63) state space v(n+1) = A v(n) + B x(n),  y(n) = C^T v(n) + D x(n),
 *                    companion realisation (l.66).  zi = v(0), zf = v(N).
 *   Eq.6-9 (l.89-111) closed-form backward: the adjoint recursion (Eq.7) run in
 *                    reverse time from dz(N-1) = grad_zf, dx (Eq.8), dv(0) = grad_zi
 *                    (Eq.9, App. A.3 l.277-294), dA/dB/dC/dD sums (Eqs.6,9), chained to
 *                    grad_b, grad_a (including grad_a[0]).
 *   l.178            per-sample ("parameter-varying") all-pole DF:
 *                    y(n) = x(n) - sum_i a_i(n) y(n-i)   (IIR_COEF_PER_SAMPLE).
 *   l.121-130 (Eq.10) time parallelism by an associative scan over (A, z) tuples:
 *                    realised as a chunked scan with fp64 carries and a single-pass,
 *                    deterministic hierarchical look-back across tiles.
 *
 * The loss whose gradient iir_backward returns is
 *   L = sum_{b,n} grad_y[b,n] * y[b,n] + sum_{b,i} grad_zf[b,i] * zf[b,i].
 *
 * Memory / layout / ownership
 *   - Every data pointer is DEVICE memory owned by the caller.  The library never
 *     allocates device memory and never synchronises the host: every call only
 *     enqueues work on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - All tensors are C-contiguous and share the descriptor's dtype (fp32 / fp64).
 *       x, y, grad_x, grad_y : (batch, length)            time is the last axis
 *       zi, zf, grad_zi, grad_zf : (batch, order)
 *       b, a, grad_b, grad_a : (order+1,) for IIR_COEF_SHARED,
 *                              (batch, order+1) for IIR_COEF_PER_SEQ
 *       a, grad_a           : (batch, length, order) for IIR_COEF_PER_SAMPLE (b = NULL,
 *                              monic a0 = 1 implied, form must be IIR_DF2)
 *     The caller zero-pads b / a to equal length ("padding if necessary").
 *   - zi / zf are the state-space v(0) / v(N) of the chosen form: TDF = scipy's zi;
 *     DF = [u(-1) .. u(-M)]; per-sample all-pole = [y(-1) .. y(-M)].
 *   - `tape` (iir_tape_bytes) is written by iir_forward and read by iir_backward; it
 *     must stay untouched in between.  `ws` (iir_workspace_bytes) is scratch used by
 *     both calls; one ws must not be used by two calls that may run concurrently.
 *     Every completed call leaves ws in its initialised (zeroed-counter) state.
 *   - Gradient outputs are OVERWRITTEN, not accumulated.  SHARED-coefficient
 *     gradients are sums over the local batch (a multi-GPU driver all-reduces them).
 *   - Optional pointers may be NULL: zi (zeros), zf (not written), grad_y (zeros),
 *     grad_zf (zeros), grad_x / grad_b / grad_a / grad_zi (not written).
 *   - Results are deterministic: same inputs and descriptor -> bitwise-identical
 *     outputs (fixed reduction order, no floating-point atomics).
 *
 * Errors
 *   Descriptor / pointer / size checks run on the host before any launch and return
 *   IIR_EINVAL / IIR_EUNSUPPORTED / IIR_EWORKSPACE; a failed launch returns
 *   IIR_ECUDA.  iir_last_error() returns a thread-local message for the last
 *   failure.  Data-dependent conditions (a0 == 0, unstable filters, NaN inputs) are
 *   NOT checked (that would need a device->host sync): they propagate as inf / nan.
 */
#ifndef IIRGRAD_H
#define IIRGRAD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IIRGRAD_ABI_VERSION 2

typedef enum { IIR_OK = 0, IIR_EINVAL = 1, IIR_EUNSUPPORTED = 2, IIR_ECUDA = 3, IIR_EWORKSPACE = 4 } iir_status_t;
typedef enum {
    IIR_DF2 = 0,   /* direct form II (Eqs.2-3)                        PAPER.md:52 footnote: type-II forms */
    IIR_TDF2 = 1,  /* transposed direct form II (= scipy lfilter)                                          */
    IIR_SS = 2     /* bare state-space recurrence of Listing 1 (the paper's benchmark op):
                    *   v(n+1) = A v(n) + z(n), dense A (order M = 1..4), SHARED (M, M) or PER_SEQ (B, M, M),
                    *   row-major.  Argument mapping: a = A, b = NULL, x = z (B, T, M), zi = v0 (B, M) or NULL,
                    *   y = v(1..T) (B, T, M), zf unused (NULL).  Backward: grad_y = dL/dv(1..T) (B, T, M),
                    *   grad_zf = NULL, y = the forward's v, zi = v0; grad_x = dL/dz (B, T, M),
                    *   grad_a = dL/dA (shape of A; SHARED: summed over the batch), grad_zi = dL/dv0,
                    *   grad_b = NULL.  Listing 1's VJP: g(n) = gv(n) + A^T g(n+1),
                    *   dL/dv0 = A^T g(0), dL/dA = sum_n g(n) v(n)^T.                                       */
} iir_form_t;
typedef enum { IIR_F32 = 0, IIR_F64 = 1 } iir_dtype_t;
typedef enum {
    IIR_COEF_SHARED = 0,     /* b, a: (M+1); one filter for the whole batch          */
    IIR_COEF_PER_SEQ = 1,    /* b, a: (B, M+1); one filter per sequence              */
    IIR_COEF_PER_SAMPLE = 2  /* all-pole DF only: a: (B, T, M), b = NULL */
} iir_coef_mode_t;

typedef void *iir_stream_t;  /* a cudaStream_t */

typedef struct {
    int64_t batch;      /* B >= 1                                                  */
    int64_t length;     /* T >= 1 samples per sequence                             */
    int32_t order;      /* M: 1..8 (SHARED / PER_SEQ); PER_SAMPLE: 1..32                  */
    int32_t form;       /* iir_form_t                                              */
    int32_t dtype;      /* iir_dtype_t                                             */
    int32_t coef_mode;  /* iir_coef_mode_t                                         */
    int32_t flags;      /* bitwise OR of iir_flags_t (0 = defaults)                */
} iir_desc_t;

typedef enum {
    /* The workspace is known to be in its initialised state (fresh from
     * iir_workspace_init, or left by a previous completed call: every call restores
     * it), so iir_forward / iir_backward skip their cudaMemsetAsync of it.  Without
     * this flag every call first clears the workspace's counters itself.           */
    IIR_FLAG_WS_READY = 1,
    /* Bit 1 is accepted and ignored (it named the single-pass LTI schedule, the only
     * one).  Bit 2 named a three-phase schedule (tile aggregates, a separate carry scan,
     * then emission) that lost on every measured shape; it was removed in ABI 2 and is
     * rejected with IIR_EUNSUPPORTED. */
    IIR_FLAG_SINGLE_PASS = 2,
    IIR_FLAG_THREE_PHASE_REMOVED = 4,
    /* IIR_COEF_PER_SAMPLE with a per-sample numerator; b (B, T, M+1) and
     * grad_b (B, T, M+1) are then required / returned.
     *   form IIR_DF2: the general time-varying DF-II filter u(n) = x(n) - sum_i a_i(n) u(n-i),
     *     y(n) = sum_k b_k(n) u(n-k), both rows applied at output time n (R19);
     *     zi, zf are the internal signal history [u(-1)..u(-M)].
     *   form IIR_TDF2: the TDF-II realisation built from the rows of sample n (PAPER.md:67-68,
     *     DESIGN.md R20): y(n) = b_0(n) x(n) + v_1(n), v_i(n+1) = v_{i+1}(n) + b_i(n) x(n)
     *     - a_i(n) y(n); zi = v(0), zf = v(N) (scipy's zi for constant rows); iir_backward
     *     needs the forward's x.
     * Without the flag, PER_SAMPLE is the all-pole DF filter (form IIR_DF2, b must be NULL). */
    IIR_FLAG_PER_SAMPLE_B = 8,
    /* Engine of fp32 TDF-II with SHARED / PER_SEQ coefficients.
     * Default: the round-2 engine (persistent warp tiles, TMEM parking, fused backward)
     * from order 4 up, the round-1 engine (one CTA per tile) below, by measured speed.
     * IIR_FLAG_LEGACY_LTI forces the round-1 engine, IIR_FLAG_ENGINE_V2 the round-2 one
     * (both compute the same filter and gradients; they differ in rounding only). */
    IIR_FLAG_LEGACY_LTI = 16,
    IIR_FLAG_ENGINE_V2 = 32,
    /* The caller asserts that grad_y and grad_zf of iir_backward were written before the
     * matching iir_forward was enqueued (e.g. resident buffers, host copies), so the
     * backward may read them while the forward is still draining (programmatic dependent
     * launch).  Without it the backward reads nothing the previous kernel on the stream
     * may have written before griddepcontrol.wait -- required when a kernel producing
     * grad_y (a loss) runs between the two calls. */
    IIR_FLAG_GRAD_Y_EARLY = 64,
    /* Bare recurrence (form IIR_SS), orders 1..4: the paper's Diag-EXT variant (PAPER.md:
     * 132-134, 145, 167).  A = V diag(lam) V^-1 is decomposed on device
     * (fp64: closed form for M <= 2; characteristic polynomial, Durand-Kerner roots and null
     * vectors for M = 3, 4); the recursion and its VJP run element-wise in the eigenbasis
     * (complex first-order scans) with the eigen-space projection of the inputs and outputs.
     * Same outputs and gradients as the dense path; where A is defective or its eigenbasis is
     * ill-conditioned (kappa(V) > 100 for fp32, 1e4 for fp64) the same kernels run the dense
     * transition instead (per coefficient set, no host round trip). */
    IIR_FLAG_DIAG = 128
} iir_flags_t;

/* Bytes of the forward->backward tape / of the scratch workspace (0 on a bad desc). */
size_t iir_tape_bytes(const iir_desc_t *desc);
size_t iir_workspace_bytes(const iir_desc_t *desc);

/* Initialise a workspace (stream-ordered cudaMemsetAsync: counters to 0, look-back
 * payload slots to the all-ones NaN sentinel). */
iir_status_t iir_workspace_init(const iir_desc_t *desc, void *ws, size_t ws_bytes, iir_stream_t stream);

/* Forward: y = filter(b, a, x; zi), zf = final state.  Eqs.1-5. */
iir_status_t iir_forward(const iir_desc_t *desc, const void *b, const void *a, const void *x,
                         const void *zi, void *y, void *zf, void *tape, size_t tape_bytes,
                         void *ws, size_t ws_bytes, iir_stream_t stream);

/* Backward: gradients of L (above) w.r.t. x, b, a, zi.  Eqs.6-9 + App. A.
 * b, a, x, y, zi must be the forward's inputs / output (unmodified), tape its tape. */
iir_status_t iir_backward(const iir_desc_t *desc, const void *grad_y, const void *grad_zf,
                          const void *b, const void *a, const void *x, const void *y,
                          const void *zi, const void *tape, size_t tape_bytes,
                          void *grad_x, void *grad_b, void *grad_a, void *grad_zi,
                          void *ws, size_t ws_bytes, iir_stream_t stream);

/* Time-sharded sequences (Eq.10, with the
 * segment as the chunk).  One sequence is split into `nseg` consecutive segments
 * of `seg_len` samples (the last may be shorter), one per rank.  Each segment is
 * first filtered with a zero carry: its forward gives the final state w_j (zf;
 * segment 0 uses the true zi), its backward the adjoint state at its start
 * (grad_zi; the last segment uses the true grad_zf).  With P = A_f^seg_len
 * (A_f = companion(a / a0) for DF, its transpose for TDF):
 *   reverse = 0:  out = sum_{j < rank} P^(rank-1-j) w_j       (zi of segment rank)
 *   reverse = 1:  out = sum_{j > rank} (P^T)^(j-rank-1) w_j   (grad_zf of segment rank)
 * i.e. the exact carry into the segment, after which the segment's forward /
 * backward with that zi / grad_zf equals the unsharded computation on it.
 *   desc: the per-segment descriptor (batch B, order M, form DF2 / TDF2, dtype,
 *         coef_mode SHARED or PER_SEQ); a: (M+1) or (B, M+1), device;
 *   w:    (nseg, B, M) device, the gathered aggregates; out: (B, M) device
 *         (zeros for rank 0 forward / rank nseg-1 reverse).
 * fp64 arithmetic (binary powering of A_f, Horner over the segments), one
 * launch, no host sync.  IIR_EINVAL on a bad rank / nseg / seg_len / NULL. */
iir_status_t iir_state_carry(const iir_desc_t *desc, const void *a, const void *w, int32_t nseg, int32_t rank,
                             int64_t seg_len, int32_t reverse, void *out, iir_stream_t stream);

/* Synchronises `stream`, then reports (and clears) the workspace's error word: a
 * look-back wait that did not see its predecessor's aggregate within 2 s (a
 * scheduling fault, e.g. CTAs that can never become co-resident) does not hang or
 * trap; it completes the call with NaN outputs and sets this word.  Returns IIR_OK,
 * or IIR_ECUDA with iir_last_error() describing the fault.  The word is cleared by
 * the next call that does not pass IIR_FLAG_WS_READY (check right after the call).
 * Host-synchronising: a diagnostic, not part of the hot path. */
iir_status_t iir_check_workspace(const iir_desc_t *desc, void *ws, size_t ws_bytes, iir_stream_t stream);

/* Thread-local message describing the last non-IIR_OK status of this thread. */
const char *iir_last_error(void);
int iir_abi_version(void);

/* ---- instrumentation (host side only; no effect on results) -------------------
 * Every kernel the library launches is counted.  When profiling is enabled each
 * launch is additionally bracketed by cudaEventRecord on its own stream, so the
 * per-kernel device time can be read back after the caller synchronised.        */
int64_t iir_launch_count(void);                     /* kernels launched since load  */
int iir_num_kernels(void);                          /* number of kernel kinds       */
const char *iir_kernel_name(int kind);
void iir_profile_enable(int on);
void iir_profile_reset(void);
/* Accumulated device milliseconds and launch count of kernel kind `kind` over the
 * profiled launches; syncs on the recorded events (call after a stream sync). */
int iir_profile_query(int kind, double *total_ms, int64_t *launches);
/* Debug: when buf (device, >= 8 u64 per tile) is non-NULL, the scan kernels record
 * %globaltimer at 8 phase points per tile (indexed by tile ticket).  NULL = off.  */
void iir_debug_trace(void *buf);

#ifdef __cplusplus
}
#endif
#endif /* IIRGRAD_H */
