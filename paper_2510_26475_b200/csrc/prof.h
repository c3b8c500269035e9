// prof.h -- opt-in per-kernel-class timing with CUDA events on the launching stream.
// Each profiled launch records a start/end event pair; prof_collect() (after a stream sync)
// folds them into per-class totals {launches, ms, flops, bytes}. Used by bench.py for the
// roofline (achieved FLOP/s or GB/s of the dominant kernel) and by tools/ for breakdowns.
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace rs {

bool prof_enabled();
void prof_set_scope(const char *scope);  // e.g. "verify", "draft", "prefill"
void prof_begin(const char *kind, double flops, double bytes, cudaStream_t st);
void prof_end(cudaStream_t st);
void prof_collect();  // requires the profiled work to have completed
std::string prof_json();
void prof_reset();
void prof_enable(bool on);

struct ProfScope {
    cudaStream_t st;
    bool on;
    ProfScope(const char *kind, double flops, double bytes, cudaStream_t s) : st(s), on(prof_enabled()) {
        if (on) prof_begin(kind, flops, bytes, st);
    }
    ~ProfScope() {
        if (on) prof_end(st);
    }
};

}  // namespace rs
