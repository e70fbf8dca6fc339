// host.h -- internal host-side helpers shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/iirgrad.h"

namespace iirg {

iir_status_t fail(iir_status_t st, const std::string& msg);

enum Kind { K_LTI_PREP = 0, K_LTI_FWD, K_LTI_BWD, K_TV_PHI, K_TV_CHAIN, K_TV_FWD, K_TV_BWD_AGG, K_TV_BWD, K_REC_FWD,
            K_REC_BWD, K_STATE_CARRY, K_TV_FIR, K_DIAG_PREP, K_DIAG_AGG, K_DIAG_SCAN, K_DIAG_FWD, K_DIAG_BWD, K_DIAG_RED,
            K_TV_SKEW, K_TV_WAGG, K_NUM };

// Launch bookkeeping: counts every kernel and (when profiling is on) brackets it
// with CUDA events on its stream.
struct LaunchGuard {
    int kind; cudaStream_t st; cudaEvent_t e0 = nullptr, e1 = nullptr;
    LaunchGuard(int k, cudaStream_t s);
    iir_status_t done();
};
template <typename F>
iir_status_t launch(int kind, cudaStream_t st, F&& f) {
    LaunchGuard g(kind, st);
    f();
    return g.done();
}

inline size_t al256(size_t n) { return (n + 255) / 256 * 256; }

// Once-per-device setup (kernel attributes such as the max dynamic shared memory are
// per device: a process driving several GPUs must set them on each).
struct PerDevice {
    std::mutex mu;
    bool done[64] = {};
    template <typename F>
    void once(F&& f) {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        if (!done[dev & 63]) { f(); done[dev & 63] = true; }
    }
};

// A second stream per (host thread, device) for work of one call that is independent of the
// caller stream's current work (fork: event on the caller stream -> side stream; join: event on
// the side stream -> caller stream).  Works under stream capture (the events become graph edges).
struct SideStream {
    cudaStream_t st = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream();

constexpr int MAX_LEVELS = 4;
struct Layout {
    int64_t ntiles = 0, ntot = 0, ncoef = 0, ngroups = 0;
    int nlev = 0;
    int64_t nblk[MAX_LEVELS] = {0, 0, 0, 0};
    // workspace: counters + flags (cleared region), then payloads
    size_t ws_ticket = 0, ws_done = 0, ws_epoch = 0, ws_gcnt = 0, ws_scnt = 0, ws_bank = 0;
    size_t ws_clear = 0;                                   // [0, ws_clear): counters, initialised to 0
    size_t ws_sent = 0, ws_sent_bytes = 0;                 // look-back slots, initialised to all-ones (NaN)
    size_t ws_agg[MAX_LEVELS] = {0, 0, 0, 0}, ws_part = 0, ws_part2 = 0, ws_bytes = 0;
    size_t ws_du = 0, ws_duneg = 0;                        // general TV DF: FIR-stage adjoint of u
    size_t ws_f = 0, ws_as = 0, ws_gas = 0;   // general TV TDF (tvtdf.cuh)
    size_t ws_psi = 0, ws_omega = 0, ws_sgrp = 0;          // TV two-level chain
    size_t tp_tab = 0, tp_u = 0, tp_extra = 0, tp_bytes = 0;
    size_t tp_t64 = 0, tp_t32 = 0;                         // v2 engine tables (lti2.cuh)
    size_t ws_err = 0;                                     // error word (look-back timeout)
    bool v2 = false;
};

// Diag-EXT bare recurrence (IIR_SS + IIR_FLAG_DIAG, M <= 2), diag.cu
size_t diag_tab_doubles(int M);
int diag_chunk();
iir_status_t diag_run(bool fwd, const iir_desc_t* d, const void* A, const void* z, const void* v0, void* v,
                      const void* gv, const void* vout, void* gz, void* gA, void* gv0, double* tab, double* agg,
                      double* carry, double* gpart, cudaStream_t st);

// per-sample (time-varying all-pole) path, tv.cu
constexpr int TV_MAX_M = 32;   // per-sample orders 1..32 (the Phi kernel: one lane per column, two column blocks at 32)
bool tv_supported(int M);
Layout tv_layout(const iir_desc_t* d);
iir_status_t tv_forward(const iir_desc_t* d, const Layout& L, const void* b, const void* a, const void* x,
                        const void* zi, void* y, void* zf, char* tape, char* ws, bool vec, cudaStream_t st);
iir_status_t tv_backward(const iir_desc_t* d, const Layout& L, const void* gy, const void* gzf, const void* b,
                         const void* a, const void* y, const void* zi, const char* tape, void* gx, void* gb,
                         void* ga, void* gzi, char* ws, bool vec, cudaStream_t st,
                         const void* x);

}  // namespace iirg
