// diag.cu -- SURVEY 8(f) f3: the paper's Diag-EXT variant of the bare recurrence
// (form IIR_SS with IIR_FLAG_DIAG; Eq.4 and Listing 1,
// PAPER.md:60-63, 296-343), orders M = 1..4 (the paper benchmarks M = 2; closed-form eigenbasis for
// M <= 2, characteristic polynomial + Durand-Kerner roots + null vectors for M = 3, 4).
//
//   A = V diag(lam) V^-1  ("decomposing A into diagonal and invertible matrices, reducing
//   matrix multiplications to element-wise multiplications"):
//   forward   w = V^-1 v,  w(n+1) = lam * w(n) + V^-1 z(n),  v(n+1) = Re V w(n+1)
//   backward  h = V^T g,   h(n) = V^T gv(n) + lam * h(n+1),   g(n) = Re V^-T h(n)   (Listing 1's VJP)
//             grad_z = g,  grad_v0 = A^T g(0),  grad_A = sum_n g(n) v(n)^T  (v(0) = v0)
// Time parallelism: chunks of DG_C samples per thread, the chunk aggregates scanned per
// sequence by one warp (Kogge-Stone over 32 chunks with the transition's powers, fp64), then
// each chunk re-runs from its exact carry-in.  The eigen-decomposition is computed on device
// (closed form for M <= 2, fp64) by a prologue that also estimates kappa(V) = ||V|| ||V^-1||:
// a defective or ill-conditioned eigenbasis ("only applicable when A is diagonalisable",
// PAPER.md:134) falls back, per coefficient set and without a host round trip, to the dense
// transition (V = I, lam -> A), i.e. the plain recurrence run by the same kernels.
#include <cuda_runtime.h>

#include "host.h"
#include "lti.cuh"

namespace iirg {
namespace dg {

#ifndef IIRG_DG_C
#define IIRG_DG_C 256
#endif
constexpr int DG_C = IIRG_DG_C;    // samples per thread chunk
constexpr int DG_NT = 128;         // threads per CTA of the chunk kernels

template <typename T> struct cx { T r, i; };
template <typename T> __device__ __forceinline__ cx<T> cmad(cx<T> a, cx<T> b, cx<T> c) {
    return {fma(a.r, b.r, fma(-a.i, b.i, c.r)), fma(a.r, b.i, fma(a.i, b.r, c.i))};
}

// Per coefficient set (fp64, in the tape): flag (1 = diagonal basis, 0 = dense fallback),
// lam[M], V[M][M], Vi[M][M] (complex), A[M][M] (real), and the transition powers used by the
// carry scan: Pw[d] = X^(DG_C 2^d), d = 0..6, complex M x M (X = diag(lam) or A).
template <int M> struct Tb {
    static constexpr int FLAG = 0, LAM = 2, V = LAM + 2 * M, VI = V + 2 * M * M, A = VI + 2 * M * M;
    static constexpr int NPW = 7;
    static constexpr int PW = A + M * M, SIZE = (PW + NPW * 2 * M * M + 31) / 32 * 32;
};

// ---- prologue: closed-form eigen-decomposition, conditioning test, powers ------------------
template <int M>
__device__ void cmatmul(const double* X, const double* Y, double* Z) {   // complex M x M, interleaved re/im
    double t[2 * M * M];
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            double re = 0, im = 0;
            for (int k = 0; k < M; ++k) {
                const double ar = X[2 * (i * M + k)], ai = X[2 * (i * M + k) + 1];
                const double br = Y[2 * (k * M + j)], bi = Y[2 * (k * M + j) + 1];
                re += ar * br - ai * bi;
                im += ar * bi + ai * br;
            }
            t[2 * (i * M + j)] = re;
            t[2 * (i * M + j) + 1] = im;
        }
    for (int e = 0; e < 2 * M * M; ++e) Z[e] = t[e];
}

// General eigen-decomposition for M = 3, 4 (fp64, one thread per coefficient set):
//   characteristic polynomial by Faddeev-LeVerrier (M_k = A M_{k-1} + c_{M-k+1} I,
//   c_{M-k} = -tr(A M_k) / k), roots by Durand-Kerner iterations polished with Newton steps,
//   each eigenvector as the null vector of A - lam I by Gaussian elimination with complete
//   pivoting (free variable = the last pivot), unit 2-norm; V^-1 by Gauss-Jordan with partial
//   pivoting.  A defective or nearly defective A gives an ill-conditioned V: kappa(V) decides
//   the dense fallback exactly as for the closed form.
struct cd { double r, i; };
__device__ __forceinline__ cd cd_add(cd a, cd b) { return {a.r + b.r, a.i + b.i}; }
__device__ __forceinline__ cd cd_sub(cd a, cd b) { return {a.r - b.r, a.i - b.i}; }
__device__ __forceinline__ cd cd_mul(cd a, cd b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ double cd_abs2(cd a) { return a.r * a.r + a.i * a.i; }
__device__ __forceinline__ cd cd_div(cd a, cd b) {
    const double d = cd_abs2(b);
    return {(a.r * b.r + a.i * b.i) / d, (a.i * b.r - a.r * b.i) / d};
}

template <int M>
__device__ bool eig_general(const double (&Ar)[M * M], double (&lr)[M], double (&li)[M], double (&Vr)[M][M],
                            double (&Vim)[M][M]) {
    // characteristic polynomial p(x) = sum_k c[k] x^k, c[M] = 1
    double c[M + 1], Mk[M * M], AM[M * M];
    c[M] = 1.0;
    for (int e = 0; e < M * M; ++e) Mk[e] = 0.0;
    for (int k = 1; k <= M; ++k) {
        for (int i = 0; i < M; ++i)                       // Mk = A Mk + c[M-k+1] I
            for (int j = 0; j < M; ++j) {
                double s = (i == j) ? c[M - k + 1] : 0.0;
                for (int q = 0; q < M; ++q) s += Ar[i * M + q] * Mk[q * M + j];
                AM[i * M + j] = s;
            }
        for (int e = 0; e < M * M; ++e) Mk[e] = AM[e];
        double tr = 0.0;                                  // tr(A Mk)
        for (int i = 0; i < M; ++i)
            for (int q = 0; q < M; ++q) tr += Ar[i * M + q] * Mk[q * M + i];
        c[M - k] = -tr / k;
    }
    auto peval = [&](cd x, cd& dp) {                      // p(x) and p'(x) by Horner
        cd pv = {c[M], 0.0};
        dp = {0.0, 0.0};
        for (int k = M - 1; k >= 0; --k) {
            dp = cd_add(cd_mul(dp, x), pv);
            pv = cd_add(cd_mul(pv, x), cd{c[k], 0.0});
        }
        return pv;
    };
    double rad = 1.0;
    for (int k = 0; k < M; ++k) rad = fmax(rad, 1.0 + fabs(c[k]));
    cd z[M];
    for (int k = 0; k < M; ++k) {                         // start on a circle, off the real axis
        const double th = 0.4 + 6.283185307179586 * k / M;
        z[k] = {0.5 * rad * cos(th), 0.5 * rad * sin(th)};
    }
    for (int it = 0; it < 500; ++it) {                    // Durand-Kerner
        double mv = 0.0;
        for (int k = 0; k < M; ++k) {
            cd dp;
            const cd pv = peval(z[k], dp);
            cd den = {1.0, 0.0};
            for (int j = 0; j < M; ++j)
                if (j != k) den = cd_mul(den, cd_sub(z[k], z[j]));
            if (cd_abs2(den) == 0.0) den = {1e-300, 0.0};
            const cd dz = cd_div(pv, den);
            z[k] = cd_sub(z[k], dz);
            mv = fmax(mv, cd_abs2(dz) / fmax(cd_abs2(z[k]), 1e-300));
        }
        if (mv < 1e-30) break;
    }
    for (int k = 0; k < M; ++k)                           // Newton polish
        for (int it = 0; it < 3; ++it) {
            cd dp;
            const cd pv = peval(z[k], dp);
            if (cd_abs2(dp) > 0.0) z[k] = cd_sub(z[k], cd_div(pv, dp));
        }
    bool ok = true;
    for (int k = 0; k < M; ++k) {
        lr[k] = z[k].r;
        li[k] = z[k].i;
        // null vector of B = A - lam I: elimination with complete pivoting
        cd Bm[M][M];
        int col[M];
        for (int i = 0; i < M; ++i) {
            col[i] = i;
            for (int j = 0; j < M; ++j) Bm[i][j] = {Ar[i * M + j] - (i == j ? z[k].r : 0.0), i == j ? -z[k].i : 0.0};
        }
        for (int q = 0; q < M - 1; ++q) {
            int pi = q, pj = q;
            double best = -1.0;
            for (int i = q; i < M; ++i)
                for (int j = q; j < M; ++j)
                    if (cd_abs2(Bm[i][j]) > best) { best = cd_abs2(Bm[i][j]); pi = i; pj = j; }
            for (int j = 0; j < M; ++j) { const cd t = Bm[q][j]; Bm[q][j] = Bm[pi][j]; Bm[pi][j] = t; }
            for (int i = 0; i < M; ++i) { const cd t = Bm[i][q]; Bm[i][q] = Bm[i][pj]; Bm[i][pj] = t; }
            { const int t = col[q]; col[q] = col[pj]; col[pj] = t; }
            if (best <= 0.0) { ok = false; continue; }
            for (int i = q + 1; i < M; ++i) {
                const cd f = cd_div(Bm[i][q], Bm[q][q]);
                for (int j = q; j < M; ++j) Bm[i][j] = cd_sub(Bm[i][j], cd_mul(f, Bm[q][j]));
            }
        }
        cd y[M];
        y[M - 1] = {1.0, 0.0};
        for (int q = M - 2; q >= 0; --q) {
            cd sacc = {0.0, 0.0};
            for (int j = q + 1; j < M; ++j) sacc = cd_add(sacc, cd_mul(Bm[q][j], y[j]));
            y[q] = cd_abs2(Bm[q][q]) > 0.0 ? cd_div(cd{-sacc.r, -sacc.i}, Bm[q][q]) : cd{0.0, 0.0};
        }
        double nrm = 0.0;
        for (int j = 0; j < M; ++j) nrm += cd_abs2(y[j]);
        nrm = sqrt(nrm);
        ok = ok && nrm > 0.0 && nrm == nrm;
        const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
        for (int j = 0; j < M; ++j) { Vr[col[j]][k] = y[j].r * inv; Vim[col[j]][k] = y[j].i * inv; }
    }
    return ok;
}

// V^-1 by Gauss-Jordan with partial pivoting (complex); false when singular
template <int M>
__device__ bool cinv(const double (&Vr)[M][M], const double (&Vim)[M][M], double (&Wr)[M][M], double (&Wi)[M][M]) {
    cd a[M][2 * M];
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            a[i][j] = {Vr[i][j], Vim[i][j]};
            a[i][M + j] = {i == j ? 1.0 : 0.0, 0.0};
        }
    for (int q = 0; q < M; ++q) {
        int pi = q;
        for (int i = q + 1; i < M; ++i)
            if (cd_abs2(a[i][q]) > cd_abs2(a[pi][q])) pi = i;
        if (cd_abs2(a[pi][q]) == 0.0) return false;
        for (int j = 0; j < 2 * M; ++j) { const cd t = a[q][j]; a[q][j] = a[pi][j]; a[pi][j] = t; }
        const cd piv = a[q][q];
        for (int j = 0; j < 2 * M; ++j) a[q][j] = cd_div(a[q][j], piv);
        for (int i = 0; i < M; ++i) {
            if (i == q) continue;
            const cd f = a[i][q];
            for (int j = 0; j < 2 * M; ++j) a[i][j] = cd_sub(a[i][j], cd_mul(f, a[q][j]));
        }
    }
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) { Wr[i][j] = a[i][M + j].r; Wi[i][j] = a[i][M + j].i; }
    return true;
}

template <typename T, int M>
__global__ void dg_prep_kernel(const T* __restrict__ a, int64_t stride, int64_t nsets, double* __restrict__ tab,
                               double kmax) {
    using TB = Tb<M>;
    const int64_t set = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (set >= nsets) return;
    const T* A = a + set * stride;
    double* t = tab + set * TB::SIZE;
    double Ar[M * M];
    for (int e = 0; e < M * M; ++e) Ar[e] = (double)A[e];
    double lr[M], li[M], Vr[M][M], Vim[M][M];
    bool ok = true;
    if constexpr (M >= 3) {
        ok = eig_general<M>(Ar, lr, li, Vr, Vim);
        // accept the iterative eigen-decomposition only if it reproduces A: max |A V - V Lambda|
        // small against ||A|| (a repeated root converges to ~eps^(1/m) and its null vectors are
        // not eigenvectors; the dense fallback is exact)
        double an = 0.0, res = 0.0;
        for (int e = 0; e < M * M; ++e) an += Ar[e] * Ar[e];
        for (int i = 0; i < M; ++i)
            for (int k = 0; k < M; ++k) {
                double rr = -(Vr[i][k] * lr[k] - Vim[i][k] * li[k]), ri = -(Vr[i][k] * li[k] + Vim[i][k] * lr[k]);
                for (int q = 0; q < M; ++q) { rr += Ar[i * M + q] * Vr[q][k]; ri += Ar[i * M + q] * Vim[q][k]; }
                res = fmax(res, rr * rr + ri * ri);
            }
        ok = ok && sqrt(res) <= 1e-12 * (1.0 + sqrt(an));
    } else if (M == 1) {
        lr[0] = Ar[0]; li[0] = 0; Vr[0][0] = 1; Vim[0][0] = 0;
    } else {
        const double a0 = Ar[0], b0 = Ar[1], c0 = Ar[2], d0 = Ar[3];
        const double h = 0.5 * (a0 + d0), disc = 0.25 * (a0 - d0) * (a0 - d0) + b0 * c0;
        const double s = sqrt(fabs(disc));
        if (disc >= 0) { lr[0] = h + s; lr[1] = h - s; li[0] = li[1] = 0; }
        else { lr[0] = lr[1] = h; li[0] = s; li[1] = -s; }
        for (int k = 0; k < 2; ++k) {                  // eigenvector columns, unit 2-norm
            double x0r, x0i, x1r, x1i;
            if (b0 == 0 && c0 == 0) { x0r = k == 0; x1r = k == 1; x0i = x1i = 0; }
            else if (fabs(b0) >= fabs(c0)) { x0r = b0; x0i = 0; x1r = lr[k] - a0; x1i = li[k]; }
            else { x0r = lr[k] - d0; x0i = li[k]; x1r = c0; x1i = 0; }
            const double nrm = sqrt(x0r * x0r + x0i * x0i + x1r * x1r + x1i * x1i);
            ok = ok && nrm > 0;
            const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
            Vr[0][k] = x0r * inv; Vim[0][k] = x0i * inv; Vr[1][k] = x1r * inv; Vim[1][k] = x1i * inv;
        }
    }
    // inverse (M <= 2) and kappa(V) ~ ||V||_F ||V^-1||_F
    double Wr[M][M], Wi[M][M];
    if constexpr (M >= 3) {
        ok = ok && cinv<M>(Vr, Vim, Wr, Wi);
    } else if (M == 1) { Wr[0][0] = 1; Wi[0][0] = 0; }
    else {
        const double dr = Vr[0][0] * Vr[1][1] - Vim[0][0] * Vim[1][1] - (Vr[0][1] * Vr[1][0] - Vim[0][1] * Vim[1][0]);
        const double di = Vr[0][0] * Vim[1][1] + Vim[0][0] * Vr[1][1] - (Vr[0][1] * Vim[1][0] + Vim[0][1] * Vr[1][0]);
        const double den = dr * dr + di * di;
        ok = ok && den > 0;
        const double ir = den > 0 ? dr / den : 0, ii = den > 0 ? -di / den : 0;   // 1 / det
        auto mul = [&](double xr, double xi, double& orr, double& oi) { orr = xr * ir - xi * ii; oi = xr * ii + xi * ir; };
        mul(Vr[1][1], Vim[1][1], Wr[0][0], Wi[0][0]);
        mul(-Vr[0][1], -Vim[0][1], Wr[0][1], Wi[0][1]);
        mul(-Vr[1][0], -Vim[1][0], Wr[1][0], Wi[1][0]);
        mul(Vr[0][0], Vim[0][0], Wr[1][1], Wi[1][1]);
    }
    double nv = 0, nw = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            nv += Vr[i][j] * Vr[i][j] + Vim[i][j] * Vim[i][j];
            nw += Wr[i][j] * Wr[i][j] + Wi[i][j] * Wi[i][j];
        }
    const double kappa = sqrt(nv * nw);
    ok = ok && kappa <= kmax && kappa == kappa;
    // dense fallback: V = V^-1 = I and the transition is A itself
    t[TB::FLAG] = ok ? 1.0 : 0.0;
    for (int i = 0; i < M; ++i) {
        t[TB::LAM + 2 * i] = ok ? lr[i] : 0.0;
        t[TB::LAM + 2 * i + 1] = ok ? li[i] : 0.0;
        for (int j = 0; j < M; ++j) {
            t[TB::V + 2 * (i * M + j)] = ok ? Vr[i][j] : (i == j);
            t[TB::V + 2 * (i * M + j) + 1] = ok ? Vim[i][j] : 0.0;
            t[TB::VI + 2 * (i * M + j)] = ok ? Wr[i][j] : (i == j);
            t[TB::VI + 2 * (i * M + j) + 1] = ok ? Wi[i][j] : 0.0;
            t[TB::A + i * M + j] = Ar[i * M + j];
        }
    }
    double X[2 * M * M];                               // the transition: diag(lam) or A
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            X[2 * (i * M + j)] = ok ? (i == j ? lr[i] : 0.0) : Ar[i * M + j];
            X[2 * (i * M + j) + 1] = ok ? (i == j ? li[i] : 0.0) : 0.0;
        }
    for (int q = 1; q < DG_C; q *= 2) cmatmul<M>(X, X, X);           // X^C
    for (int d = 0; d < TB::NPW; ++d) {
        for (int e = 0; e < 2 * M * M; ++e) t[TB::PW + d * 2 * M * M + e] = X[e];
        cmatmul<M>(X, X, X);
    }
}

// ---- chunk kernels ---------------------------------------------------------------------------
struct Args {
    const void* a; const void* z; const void* v0; void* v;          // forward
    const void* gv; const void* vout; void* gz; void* gv0;          // backward
    const double* tab; int64_t tab_stride, coef_stride;
    double* agg; double* carry; double* gpart;                      // workspace
    int64_t B, T; int nch; int ncoef;
};

template <typename T, int M>
struct Par {                                                         // one set's parameters in T
    bool diag;
    cx<T> lam[M], V[M][M], Vi[M][M];
    T A[M][M];
    __device__ void load(const double* t) {
        using TB = Tb<M>;
        diag = t[TB::FLAG] != 0.0;
        for (int i = 0; i < M; ++i) {
            lam[i] = {(T)t[TB::LAM + 2 * i], (T)t[TB::LAM + 2 * i + 1]};
            for (int j = 0; j < M; ++j) {
                V[i][j] = {(T)t[TB::V + 2 * (i * M + j)], (T)t[TB::V + 2 * (i * M + j) + 1]};
                Vi[i][j] = {(T)t[TB::VI + 2 * (i * M + j)], (T)t[TB::VI + 2 * (i * M + j) + 1]};
                A[i][j] = (T)t[TB::A + i * M + j];
            }
        }
    }
};

// one step of the state recursion in the working basis (BWD: the transposed operator)
template <typename T, int M, bool BWD>
__device__ __forceinline__ void dg_step(const Par<T, M>& P, cx<T> (&w)[M], const T (&in)[M]) {
    cx<T> nw[M];
    if (P.diag) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            cx<T> acc = {T(0), T(0)};
#pragma unroll
            for (int j = 0; j < M; ++j) {                  // projection: V^-1 z (fwd) or V^T gv (bwd)
                const cx<T> q = BWD ? P.V[j][i] : P.Vi[i][j];
                acc.r = fma(q.r, in[j], acc.r);
                acc.i = fma(q.i, in[j], acc.i);
            }
            nw[i] = cmad(P.lam[i], w[i], acc);            // element-wise
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            T acc = in[i];
#pragma unroll
            for (int j = 0; j < M; ++j) acc = fma(BWD ? P.A[j][i] : P.A[i][j], w[j].r, acc);
            nw[i] = {acc, T(0)};
        }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) w[i] = nw[i];
}
// back to the real state: Re V w (fwd) or Re V^-T h (bwd)
template <typename T, int M, bool BWD>
__device__ __forceinline__ void dg_out(const Par<T, M>& P, const cx<T> (&w)[M], T (&out)[M]) {
#pragma unroll
    for (int k = 0; k < M; ++k) {
        if (P.diag) {
            T s = T(0);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const cx<T> q = BWD ? P.Vi[i][k] : P.V[k][i];
                s = fma(q.r, w[i].r, fma(-q.i, w[i].i, s));
            }
            out[k] = s;
        } else {
            out[k] = w[k].r;
        }
    }
}

template <typename T, int M>
__device__ __forceinline__ void ld_vec(const T* p, int64_t idx, T (&v)[M]) {
#pragma unroll
    for (int j = 0; j < M; ++j) v[j] = p[idx * M + j];
}

// phase 1: chunk aggregates from the zero state (forward in time / backward in reverse time).
// Forward chunks start at 0 (the ragged chunk is the last); backward chunks, scanned last to
// first, end at T (the ragged chunk is the first in time): every scanned chunk but the final
// one spans exactly DG_C samples, the span of the scan's transition X^C.  The CTA's chunks
// advance together DG_S samples per step with their input rows staged through shared memory
// (cooperative 16 B copies, cp.async double buffer), as in the emit kernels below.
template <typename T, int M, bool BWD>
__global__ void __launch_bounds__(DG_NT) dg_agg_kernel(const Args p);

// phase 2: one warp per sequence scans the chunk aggregates in fp64 (blocks of 32 chunks:
// Kogge-Stone with X^(C 2^d), the block's carry-in folded into its first chunk) and writes
// the state entering every chunk (forward: chunk order; backward: reverse chunk order)
template <int M, bool BWD>
__device__ __forceinline__ void cmv(const double* P, const double (&v)[2 * M], double (&acc)[2 * M]) {
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const int e = BWD ? (j * M + i) : (i * M + j);     // the transposed operator for the adjoint
            const double pr = P[2 * e], pi = P[2 * e + 1];
            acc[2 * i] += pr * v[2 * j] - pi * v[2 * j + 1];
            acc[2 * i + 1] += pr * v[2 * j + 1] + pi * v[2 * j];
        }
}

template <typename T, int M, bool BWD>
__global__ void __launch_bounds__(32) dg_scan_kernel(const Args p) {
    using TB = Tb<M>;
    const int64_t seq = blockIdx.x;
    const int lane = threadIdx.x;
    const double* t = p.tab + (p.ncoef > 1 ? seq : 0) * p.tab_stride;
    const bool diag = t[TB::FLAG] != 0.0;
    double X[2 * M];                                       // state entering the current block
#pragma unroll
    for (int i = 0; i < 2 * M; ++i) X[i] = 0.0;
    if (!BWD && p.v0 != nullptr) {                         // forward: the projected initial state V^-1 v0
        const T* v0 = static_cast<const T*>(p.v0) + seq * M;
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) {
                const double q0 = diag ? t[TB::VI + 2 * (i * M + j)] : (i == j), q1 = diag ? t[TB::VI + 2 * (i * M + j) + 1] : 0.0;
                X[2 * i] += q0 * (double)v0[j];
                X[2 * i + 1] += q1 * (double)v0[j];
            }
    }
    // Each lane owns DG_K consecutive chunks of a block of 32 DG_K: it folds them serially with
    // X^C, the lanes' inclusive states are scanned with X^(DG_K C 2^d) (levels log2 DG_K + d of
    // the table), and each lane then walks its chunks' entering states forward.  The powers are
    // staged once in shared memory (read by broadcast) and the next block's aggregates are
    // loaded one block ahead: the loop's only serial dependency is the carry X.
    constexpr int DG_K = 4, LK = 2;                      // chunks per lane, log2
    static_assert(LK + 4 < TB::NPW, "scan levels in the table");
    constexpr int NPW = TB::NPW * 2 * M * M;
    __shared__ double spw[NPW];
    for (int e = lane; e < NPW; e += 32) spw[e] = t[TB::PW + e];
    __syncwarp();
    auto lvl = [&](int d) -> const double* { return spw + d * 2 * M * M; };
    double An[DG_K][2 * M];
    auto load = [&](int b0, double (&dst)[DG_K][2 * M]) {
#pragma unroll
        for (int j = 0; j < DG_K; ++j) {
            const int cc = b0 + lane * DG_K + j;
#pragma unroll
            for (int i = 0; i < 2 * M; ++i) dst[j][i] = cc < p.nch ? p.agg[(seq * p.nch + cc) * 2 * M + i] : 0.0;
        }
    };
    load(0, An);
    for (int b0 = 0; b0 < p.nch; b0 += 32 * DG_K) {
        double Ag[DG_K][2 * M];
#pragma unroll
        for (int j = 0; j < DG_K; ++j)
#pragma unroll
            for (int i = 0; i < 2 * M; ++i) Ag[j][i] = An[j][i];
        load(b0 + 32 * DG_K, An);
        double S[2 * M];                                   // the lane's inclusive aggregate (zero carry-in)
#pragma unroll
        for (int i = 0; i < 2 * M; ++i) S[i] = Ag[0][i];
#pragma unroll
        for (int j = 1; j < DG_K; ++j) {
            double acc[2 * M];
#pragma unroll
            for (int i = 0; i < 2 * M; ++i) acc[i] = Ag[j][i];
            cmv<M, BWD>(lvl(0), S, acc);
#pragma unroll
            for (int i = 0; i < 2 * M; ++i) S[i] = acc[i];
        }
        if (lane == 0) cmv<M, BWD>(lvl(LK), X, S);         // fold the block's carry-in
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            double O[2 * M], acc[2 * M];
#pragma unroll
            for (int i = 0; i < 2 * M; ++i) { O[i] = __shfl_up_sync(0xffffffffu, S[i], 1 << d); acc[i] = 0.0; }
            cmv<M, BWD>(lvl(LK + d), O, acc);
            if (lane >= (1 << d))
#pragma unroll
                for (int i = 0; i < 2 * M; ++i) S[i] += acc[i];
        }
        double E[2 * M];                                   // state entering the lane's first chunk
#pragma unroll
        for (int i = 0; i < 2 * M; ++i) {
            const double e = __shfl_up_sync(0xffffffffu, S[i], 1);
            E[i] = lane == 0 ? X[i] : e;
        }
#pragma unroll
        for (int j = 0; j < DG_K; ++j) {
            const int cc = b0 + lane * DG_K + j;
            if (cc < p.nch)
#pragma unroll
                for (int i = 0; i < 2 * M; ++i) p.carry[(seq * p.nch + cc) * 2 * M + i] = E[i];
            if (j + 1 < DG_K) {
                double acc[2 * M];
#pragma unroll
                for (int i = 0; i < 2 * M; ++i) acc[i] = Ag[j][i];
                cmv<M, BWD>(lvl(0), E, acc);
#pragma unroll
                for (int i = 0; i < 2 * M; ++i) E[i] = acc[i];
            }
        }
#pragma unroll
        for (int i = 0; i < 2 * M; ++i) X[i] = __shfl_sync(0xffffffffu, S[i], 31);
    }
}

// phase 3, forward: re-run every chunk from its carry-in, v(n+1) = Re V w(n+1).  The CTA's 128
// chunks advance together DG_S samples per step: their z rows are staged into shared memory by
// cooperative 16 B copies (every chunk's step is one contiguous 8M-element run), double-buffered
// with cp.async, and their v rows leave the same way, instead of every lane streaming its own
// rows 2 KB away from its neighbours' (ncu: 95 % long-scoreboard stalls).
// samples per step: the largest of 8 / 4 / 2 whose three staged buffers fit 48 KB of static shared memory
template <typename T, int M> constexpr bool dg_s_fits(int S) {
    return (S * M) % (16 / (int)sizeof(T)) == 0 &&
           3 * DG_NT * (S * M + 16 / (int)sizeof(T)) * (int)sizeof(T) <= 48 * 1024;
}
template <typename T, int M> constexpr int dg_s() { return dg_s_fits<T, M>(8) ? 8 : dg_s_fits<T, M>(4) ? 4 : 2; }
template <typename T, int M, bool BWD>
__global__ void __launch_bounds__(DG_NT) dg_agg_kernel(const Args p) {
    constexpr int DG_S = dg_s<T, M>();
    constexpr int ROW = DG_S * M, W = 16 / (int)sizeof(T), RS = ROW + W, PPC = ROW / W;
    __shared__ __align__(16) T zs[2][DG_NT * RS];
    const int64_t ntot = p.B * p.nch, cbase = (int64_t)blockIdx.x * DG_NT;
    const int64_t c = cbase + threadIdx.x;
    const bool valid = c < ntot;
    const T* in = static_cast<const T*>(BWD ? p.gv : p.z);
    // the chunk's sample range [n0, n1) and the first sample of step `step`'s rows
    auto range = [&](int64_t cc, int64_t& n0, int64_t& n1) {
        const int64_t sq = cc / p.nch;
        const int kk = (int)(cc - sq * p.nch);
        n0 = BWD ? max((int64_t)0, p.T - (int64_t)(kk + 1) * DG_C) : (int64_t)kk * DG_C;
        n1 = BWD ? p.T - (int64_t)kk * DG_C : min(n0 + DG_C, p.T);
        return sq;
    };
    auto stage = [&](int step, T* dst) {
        for (int q = threadIdx.x; q < DG_NT * PPC; q += DG_NT) {
            const int lc = q / PPC, part = q - (q / PPC) * PPC;
            const int64_t cc = cbase + lc;
            T* d = dst + lc * RS + part * W;
            int64_t n0 = 0, n1 = 0, sq = 0;
            if (cc < ntot && in != nullptr) sq = range(cc, n0, n1);
            const int64_t a = BWD ? n1 - (int64_t)(step + 1) * DG_S : n0 + (int64_t)step * DG_S;   // buffer row 0
            const int e0 = part * W;
            // valid samples of the piece: n in [max(a, n0), min(a + S, n1))
            const int64_t lo = max(a, n0), hi = min(a + DG_S, n1);
            const int64_t elo = (lo - a) * M, ehi = (hi - a) * M;           // valid elements [elo, ehi)
            const T* g = in + (sq * p.T + a) * M + e0;
            if (cc < ntot && in != nullptr && e0 >= elo && e0 + W <= ehi &&
                (reinterpret_cast<uintptr_t>(g) & 15u) == 0) {
                cp_async16(d, g, 16u);
            } else {
#pragma unroll
                for (int r = 0; r < W; ++r)
                    d[r] = (cc < ntot && in != nullptr && e0 + r >= elo && e0 + r < ehi) ? g[r] : T(0);
            }
        }
        cp_async_commit();
    };
    Par<T, M> P;
    int64_t n0 = 0, n1 = 0;
    if (valid) {
        const int64_t sq = range(c, n0, n1);
        P.load(p.tab + (p.ncoef > 1 ? sq : 0) * p.tab_stride);
    }
    cx<T> w[M];
#pragma unroll
    for (int i = 0; i < M; ++i) w[i] = {T(0), T(0)};
    constexpr int NSTEP = DG_C / DG_S;
    stage(0, zs[0]);
    for (int step = 0; step < NSTEP; ++step) {
        const int b = step & 1;
        if (step + 1 < NSTEP) { stage(step + 1, zs[b ^ 1]); cp_async_wait<1>(); }
        else cp_async_wait<0>();
        __syncthreads();
        if (valid && in != nullptr) {
            const int64_t a = BWD ? n1 - (int64_t)(step + 1) * DG_S : n0 + (int64_t)step * DG_S;
            const T* zr = zs[b] + threadIdx.x * RS;
#pragma unroll
            for (int uu = 0; uu < DG_S; ++uu) {
                const int u = BWD ? DG_S - 1 - uu : uu;
                const int64_t n = a + u;
                if (n >= n0 && n < n1) {
                    T zz[M];
#pragma unroll
                    for (int j = 0; j < M; ++j) zz[j] = zr[u * M + j];
                    dg_step<T, M, BWD>(P, w, zz);
                }
            }
        }
        __syncthreads();                                   // zs[b] free for step + 2
    }
    if (!valid) return;
    double* o = p.agg + c * 2 * M;
#pragma unroll
    for (int i = 0; i < M; ++i) { o[2 * i] = (double)w[i].r; o[2 * i + 1] = (double)w[i].i; }
}

template <typename T, int M>
__device__ __forceinline__ int64_t dg_row0(const Args& p, int64_t cc, int step) {   // first element of a step
    const int64_t sq = cc / p.nch;
    const int kk = (int)(cc - sq * p.nch);
    return (sq * p.T + (int64_t)kk * DG_C + (int64_t)step * dg_s<T, M>()) * M;
}
template <typename T, int M>
__device__ __forceinline__ int dg_rows_valid(const Args& p, int64_t cc, int step) {  // samples of the step < T
    const int64_t sq = cc / p.nch;
    const int kk = (int)(cc - sq * p.nch);
    const int64_t n = (int64_t)kk * DG_C + (int64_t)step * dg_s<T, M>();
    return (int)max((int64_t)0, min((int64_t)dg_s<T, M>(), p.T - n));
}
template <typename T, int M>
__global__ void __launch_bounds__(DG_NT) dg_fwd_emit_kernel(const Args p) {
    constexpr int DG_S = dg_s<T, M>();
    static_assert(dg_s_fits<T, M>(DG_S), "staged buffers fit");
    constexpr int ROW = DG_S * M, W = 16 / (int)sizeof(T), RS = ROW + W, PPC = ROW / W;
    static_assert(ROW % W == 0, "whole 16 B pieces per chunk step");
    __shared__ __align__(16) T zs[2][DG_NT * RS];
    __shared__ __align__(16) T vs[DG_NT * RS];
    const int64_t ntot = p.B * p.nch, cbase = (int64_t)blockIdx.x * DG_NT;
    const int64_t c = cbase + threadIdx.x;
    const bool valid = c < ntot;
    const T* z = static_cast<const T*>(p.z);
    T* v = static_cast<T*>(p.v);
    auto stage = [&](int step, T* dst) {
        for (int q = threadIdx.x; q < DG_NT * PPC; q += DG_NT) {
            const int lc = q / PPC, part = q - (q / PPC) * PPC;
            const int64_t cc = cbase + lc;
            T* d = dst + lc * RS + part * W;
            const int nv = cc < ntot ? dg_rows_valid<T, M>(p, cc, step) * M - part * W : 0;   // valid elements
            if (nv <= 0) {
#pragma unroll
                for (int r = 0; r < W; ++r) d[r] = T(0);
                continue;
            }
            const T* src = z + dg_row0<T, M>(p, cc, step) + part * W;
            if (nv >= W && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
                cp_async16(d, src, 16u);
            } else {
#pragma unroll
                for (int r = 0; r < W; ++r) d[r] = r < nv ? src[r] : T(0);
            }
        }
        cp_async_commit();
    };
    Par<T, M> P;
    cx<T> w[M];
    if (valid) {
        P.load(p.tab + (p.ncoef > 1 ? c / p.nch : 0) * p.tab_stride);
#pragma unroll
        for (int i = 0; i < M; ++i) w[i] = {(T)p.carry[c * 2 * M + 2 * i], (T)p.carry[c * 2 * M + 2 * i + 1]};
    }
    constexpr int NSTEP = DG_C / DG_S;
    stage(0, zs[0]);
    for (int step = 0; step < NSTEP; ++step) {
        const int b = step & 1;
        if (step + 1 < NSTEP) { stage(step + 1, zs[b ^ 1]); cp_async_wait<1>(); }
        else cp_async_wait<0>();
        __syncthreads();                                   // step's z rows landed; vs free
        if (valid) {
            const int nvs = dg_rows_valid<T, M>(p, c, step);
            const T* zr = zs[b] + threadIdx.x * RS;
            T* vr = vs + threadIdx.x * RS;
#pragma unroll
            for (int u = 0; u < DG_S; ++u) {
                if (u < nvs) {
                    T zz[M], o[M];
#pragma unroll
                    for (int j = 0; j < M; ++j) zz[j] = zr[u * M + j];
                    dg_step<T, M, false>(P, w, zz);
                    dg_out<T, M, false>(P, w, o);
#pragma unroll
                    for (int j = 0; j < M; ++j) vr[u * M + j] = o[j];
                }
            }
        }
        __syncthreads();                                   // vs complete; zs[b] free for step + 2
        for (int q = threadIdx.x; q < DG_NT * PPC; q += DG_NT) {   // cooperative store of the v rows
            const int lc = q / PPC, part = q - (q / PPC) * PPC;
            const int64_t cc = cbase + lc;
            if (cc >= ntot) continue;
            const int nv = dg_rows_valid<T, M>(p, cc, step) * M - part * W;
            if (nv <= 0) continue;
            T* dst = v + dg_row0<T, M>(p, cc, step) + part * W;
            const T* sv = vs + lc * RS + part * W;
            if (nv >= W && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
                using V = typename Vec<T>::type;
                *reinterpret_cast<V*>(dst) = *reinterpret_cast<const V*>(sv);
            } else {
#pragma unroll
                for (int r = 0; r < W; ++r)
                    if (r < nv) dst[r] = sv[r];
            }
        }
    }
}

// phase 3, backward: h from the carry at the chunk's end, g(n) = Re V^-T h(n); grad_z = g;
// per-chunk partial sums of grad_A = sum g(n) v(n)^T (fixed-order reduction later);
// the chunk holding n = 0 writes grad_v0 = A^T g(0).  Staged like the forward emit, walking
// back from the chunk's end: step s holds rows [b - S, b), b = n1 - s S, of gv and of the
// forward's v (whose row n - 1 is v(n)); the first sample of a step pairs with the last row
// of the next step (kept pending), the chunk's first sample with v(n0 - 1) or v0.
template <typename T, int M>
__global__ void __launch_bounds__(DG_NT) dg_bwd_emit_kernel(const Args p) {
    constexpr int DG_S = dg_s<T, M>();
    constexpr int ROW = DG_S * M, W = 16 / (int)sizeof(T), RS = ROW + W, PPC = ROW / W;
    static_assert(ROW % W == 0, "whole 16 B pieces per chunk step");
    // gv, v (double-buffered) and gz staging: 5 buffers
    static_assert(5 * DG_NT * RS * (int)sizeof(T) <= 80 * 1024, "staged buffers");
    extern __shared__ __align__(16) unsigned char dg_raw[];
    T* sg = reinterpret_cast<T*>(dg_raw);                  // [2][DG_NT * RS] gv rows
    T* sv = sg + 2 * DG_NT * RS;                           // [2][DG_NT * RS] forward v rows
    T* so = sv + 2 * DG_NT * RS;                           // [DG_NT * RS] gz rows out
    const int64_t ntot = p.B * p.nch, cbase = (int64_t)blockIdx.x * DG_NT;
    const int64_t c = cbase + threadIdx.x;
    const bool valid = c < ntot;
    const T* gv = static_cast<const T*>(p.gv);
    const T* vo = static_cast<const T*>(p.vout);
    const T* v0 = static_cast<const T*>(p.v0);
    T* gz = static_cast<T*>(p.gz);
    // rows of step `step` of chunk cc: [a, b) of its sequence, the valid part [max(a, n0), b)
    auto span = [&](int64_t cc, int step, int64_t& rowbase, int& lo) {
        const int64_t sq = cc / p.nch;
        const int kk = (int)(cc - sq * p.nch);
        const int64_t n0 = max((int64_t)0, p.T - (int64_t)(kk + 1) * DG_C), n1 = p.T - (int64_t)kk * DG_C;
        const int64_t b = n1 - (int64_t)step * DG_S, a = b - DG_S;
        rowbase = sq * p.T + a;                            // global row of buffer row 0
        lo = (int)min((int64_t)DG_S, max((int64_t)0, n0 - a));   // buffer rows below lo are invalid
        if (b <= n0) lo = DG_S;
    };
    auto stage_one = [&](const T* src, int step, T* dst) {
        for (int q = threadIdx.x; q < DG_NT * PPC; q += DG_NT) {
            const int lc = q / PPC, part = q - (q / PPC) * PPC;
            const int64_t cc = cbase + lc;
            T* d = dst + lc * RS + part * W;
            int64_t rb = 0;
            int lo = DG_S;
            if (cc < ntot && src != nullptr) span(cc, step, rb, lo);
            const int e0 = part * W;                       // first element of the piece
            if (lo * M <= e0 && lo < DG_S) {
                const T* g = src + rb * M + e0;
                if ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) { cp_async16(d, g, 16u); continue; }
#pragma unroll
                for (int r = 0; r < W; ++r) d[r] = g[r];
            } else {
#pragma unroll
                for (int r = 0; r < W; ++r) d[r] = (lo < DG_S && e0 + r >= lo * M) ? src[rb * M + e0 + r] : T(0);
            }
        }
    };
    auto stage = [&](int step, int b) {
        stage_one(gv, step, sg + b * DG_NT * RS);
        stage_one(vo, step, sv + b * DG_NT * RS);
        cp_async_commit();
    };
    Par<T, M> P;
    cx<T> h[M];
    int64_t n0 = 0, n1 = 0;
    if (valid) {
        const int64_t sq = c / p.nch;
        const int kk = (int)(c - sq * p.nch);
        n0 = max((int64_t)0, p.T - (int64_t)(kk + 1) * DG_C);
        n1 = p.T - (int64_t)kk * DG_C;
        P.load(p.tab + (p.ncoef > 1 ? sq : 0) * p.tab_stride);
#pragma unroll
        for (int i = 0; i < M; ++i) h[i] = {(T)p.carry[c * 2 * M + 2 * i], (T)p.carry[c * 2 * M + 2 * i + 1]};
    }
    double gA[M][M];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) gA[i][j] = 0.0;
    T g[M], gpend[M];
    bool pending = false;
    constexpr int NSTEP = DG_C / DG_S;
    stage(0, 0);
    for (int step = 0; step < NSTEP; ++step) {
        const int b = step & 1;
        if (step + 1 < NSTEP) { stage(step + 1, b ^ 1); cp_async_wait<1>(); }
        else cp_async_wait<0>();
        __syncthreads();                                   // this step's rows landed; so free
        const int64_t bb = n1 - (int64_t)step * DG_S, aa = bb - DG_S;
        const T* gr = sg + b * DG_NT * RS + threadIdx.x * RS;
        const T* vr = sv + b * DG_NT * RS + threadIdx.x * RS;
        T* orow = so + threadIdx.x * RS;
        if (valid && bb > n0) {
            if (pending) {                                 // v(aa_prev) = forward row aa_prev - 1 = this step's last row
#pragma unroll
                for (int i = 0; i < M; ++i)
#pragma unroll
                    for (int j = 0; j < M; ++j) gA[i][j] = fma((double)gpend[i], (double)vr[(DG_S - 1) * M + j], gA[i][j]);
                pending = false;
            }
#pragma unroll
            for (int u = DG_S - 1; u >= 0; --u) {
                const int64_t n = aa + u;
                if (n >= n0) {
                    T gg[M];
#pragma unroll
                    for (int j = 0; j < M; ++j) gg[j] = gr[u * M + j];
                    dg_step<T, M, true>(P, h, gg);
                    dg_out<T, M, true>(P, h, g);
#pragma unroll
                    for (int j = 0; j < M; ++j) orow[u * M + j] = g[j];
                    if (u > 0 && n - 1 >= n0) {            // v(n) = forward row n - 1, staged
#pragma unroll
                        for (int i = 0; i < M; ++i)
#pragma unroll
                            for (int j = 0; j < M; ++j) gA[i][j] = fma((double)g[i], (double)vr[(u - 1) * M + j], gA[i][j]);
                    } else {
                        pending = true;
#pragma unroll
                        for (int j = 0; j < M; ++j) gpend[j] = g[j];
                    }
                }
            }
        }
        __syncthreads();                                   // so complete
        if (gz != nullptr)
            for (int q = threadIdx.x; q < DG_NT * PPC; q += DG_NT) {   // cooperative store of the gz rows
                const int lc = q / PPC, part = q - (q / PPC) * PPC;
                const int64_t cc = cbase + lc;
                if (cc >= ntot) continue;
                int64_t rb;
                int lo;
                span(cc, step, rb, lo);
                if (lo >= DG_S) continue;
                const int e0 = part * W;
                T* dst = gz + rb * M + e0;
                const T* s2 = so + lc * RS + e0;
                if (lo * M <= e0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
                    using V = typename Vec<T>::type;
                    *reinterpret_cast<V*>(dst) = *reinterpret_cast<const V*>(s2);
                } else {
#pragma unroll
                    for (int r = 0; r < W; ++r)
                        if (e0 + r >= lo * M) dst[r] = s2[r];
                }
            }
    }
    if (!valid) return;
    if (pending) {                                         // the chunk's first sample n0: v(n0)
        T vp[M];
        const int64_t sq = c / p.nch;
#pragma unroll
        for (int j = 0; j < M; ++j)
            vp[j] = n0 > 0 ? vo[(sq * p.T + n0 - 1) * M + j] : (v0 != nullptr ? v0[sq * M + j] : T(0));
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) gA[i][j] = fma((double)gpend[i], (double)vp[j], gA[i][j]);
    }
    if (n0 == 0 && p.gv0 != nullptr) {                     // g now holds g(0)
        T* o = static_cast<T*>(p.gv0) + (c / p.nch) * M;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            T s = T(0);
#pragma unroll
            for (int j = 0; j < M; ++j) s = fma(P.A[j][i], g[j], s);
            o[i] = s;
        }
    }
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) p.gpart[c * M * M + i * M + j] = gA[i][j];
}
template <typename T, int M>
constexpr size_t dg_bwd_smem() { return (size_t)5 * DG_NT * (dg_s<T, M>() * M + 16 / sizeof(T)) * sizeof(T); }

// grad_A: fixed-order sum of the chunk partials (SHARED: every chunk; PER_SEQ: per sequence)
template <typename T, int M>
__global__ void __launch_bounds__(256) dg_reduce_kernel(const Args p, T* __restrict__ gA) {
    // block (set, entry e of grad_A): every thread sums its fixed strided rows with four
    // independent partial sums (loads in flight), then a fixed-order tree: deterministic
    __shared__ double red[256];
    const int64_t set = blockIdx.x;
    const int e = blockIdx.y;
    const int64_t r0 = p.ncoef > 1 ? set * p.nch : 0, nr = p.ncoef > 1 ? p.nch : p.B * p.nch;
    const double* g = p.gpart + r0 * M * M + e;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t r = threadIdx.x;
    for (; r + 3 * 256 < nr; r += 4 * 256) {
        s0 += g[r * M * M];
        s1 += g[(r + 256) * M * M];
        s2 += g[(r + 512) * M * M];
        s3 += g[(r + 768) * M * M];
    }
    for (; r < nr; r += 256) s0 += g[r * M * M];
    red[threadIdx.x] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) gA[set * M * M + e] = (T)red[0];
}

template <typename T, int M>
static iir_status_t run(bool fwd, const iir_desc_t* d, Args& a, void* gA, cudaStream_t st) {
    const unsigned nchunk = (unsigned)(a.B * a.nch), grid = (nchunk + DG_NT - 1) / DG_NT;
    const double kmax = sizeof(T) == 4 ? 100.0 : 1e4;     // kappa(V) beyond which the dense fallback runs
    iir_status_t s;
    if (fwd) {
        s = launch(K_DIAG_PREP, st, [&] {
            dg_prep_kernel<T, M><<<(unsigned)((a.ncoef + 63) / 64), 64, 0, st>>>(static_cast<const T*>(a.a),
                                                                                  a.coef_stride, a.ncoef,
                                                                                  const_cast<double*>(a.tab), kmax);
        });
        if (s != IIR_OK) return s;
        s = launch(K_DIAG_AGG, st, [&] { dg_agg_kernel<T, M, false><<<grid, DG_NT, 0, st>>>(a); });
        if (s != IIR_OK) return s;
        s = launch(K_DIAG_SCAN, st, [&] { dg_scan_kernel<T, M, false><<<(unsigned)a.B, 32, 0, st>>>(a); });
        if (s != IIR_OK) return s;
        return launch(K_DIAG_FWD, st, [&] { dg_fwd_emit_kernel<T, M><<<grid, DG_NT, 0, st>>>(a); });
    }
    s = launch(K_DIAG_AGG, st, [&] { dg_agg_kernel<T, M, true><<<grid, DG_NT, 0, st>>>(a); });
    if (s != IIR_OK) return s;
    s = launch(K_DIAG_SCAN, st, [&] { dg_scan_kernel<T, M, true><<<(unsigned)a.B, 32, 0, st>>>(a); });
    if (s != IIR_OK) return s;
    static PerDevice attrs;
    attrs.once([] {
        cudaFuncSetAttribute(dg_bwd_emit_kernel<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dg_bwd_smem<T, M>());
    });
    s = launch(K_DIAG_BWD, st, [&] { dg_bwd_emit_kernel<T, M><<<grid, DG_NT, dg_bwd_smem<T, M>(), st>>>(a); });
    if (s != IIR_OK || gA == nullptr) return s;
    return launch(K_DIAG_RED, st, [&] {
        dg_reduce_kernel<T, M><<<dim3((unsigned)a.ncoef, M * M), 256, 0, st>>>(a, static_cast<T*>(gA));
    });
    (void)d;
}

}  // namespace dg

size_t diag_tab_doubles(int M) {
    switch (M) {
        case 1: return dg::Tb<1>::SIZE; case 2: return dg::Tb<2>::SIZE;
        case 3: return dg::Tb<3>::SIZE; case 4: return dg::Tb<4>::SIZE;
    }
    return 0;
}
int diag_chunk() { return dg::DG_C; }

iir_status_t diag_run(bool fwd, const iir_desc_t* d, const void* A, const void* z, const void* v0, void* v,
                      const void* gv, const void* vout, void* gz, void* gA, void* gv0, double* tab, double* agg,
                      double* carry, double* gpart, cudaStream_t st) {
    dg::Args a{};
    a.a = A; a.z = z; a.v0 = v0; a.v = v; a.gv = gv; a.vout = vout; a.gz = gz; a.gv0 = gv0;
    a.tab = tab; a.tab_stride = (int64_t)diag_tab_doubles(d->order);
    a.coef_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : (int64_t)d->order * d->order;
    a.agg = agg; a.carry = carry; a.gpart = gpart;
    a.B = d->batch; a.T = d->length; a.nch = (int)((d->length + dg::DG_C - 1) / dg::DG_C);
    a.ncoef = d->coef_mode == IIR_COEF_SHARED ? 1 : (int)d->batch;
    switch (d->order * 2 + (d->dtype == IIR_F64 ? 1 : 0)) {
        case 2: return dg::run<float, 1>(fwd, d, a, gA, st);
        case 3: return dg::run<double, 1>(fwd, d, a, gA, st);
        case 4: return dg::run<float, 2>(fwd, d, a, gA, st);
        case 5: return dg::run<double, 2>(fwd, d, a, gA, st);
        case 6: return dg::run<float, 3>(fwd, d, a, gA, st);
        case 7: return dg::run<double, 3>(fwd, d, a, gA, st);
        case 8: return dg::run<float, 4>(fwd, d, a, gA, st);
        case 9: return dg::run<double, 4>(fwd, d, a, gA, st);
    }
    return fail(IIR_EUNSUPPORTED, "Diag-EXT: order must be 1..4");
}

}  // namespace iirg
