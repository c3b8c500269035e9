// prof.cpp -- see prof.h.
#include "prof.h"

#include <nvtx3/nvToolsExt.h>

#include <cstdio>
#include <map>
#include <vector>

#include "common.cuh"

namespace rs {

namespace {
struct Rec {
    std::string cls;
    double flops, bytes;
    cudaEvent_t a, b;
};
struct Tot {
    long n = 0;
    double ms = 0, flops = 0, bytes = 0;
};
thread_local bool g_on = false;
thread_local std::string g_scope = "step";
thread_local std::vector<Rec> g_open;     // recorded, not yet collected
thread_local std::vector<cudaEvent_t> g_pool;
thread_local std::map<std::string, Tot> g_tot;
thread_local int g_depth = 0;

cudaEvent_t take() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    RS_CUDA(cudaEventCreate(&e));
    return e;
}
}  // namespace

bool prof_enabled() { return g_on && g_depth == 0; }
void prof_enable(bool on) { g_on = on; }
// Scopes double as NVTX ranges ("draft", "verify", "accept", ...) so ncu can target a phase:
// ncu --nvtx --nvtx-include "verify/" ...
void prof_set_scope(const char *s) {
    static thread_local bool open = false;
    if (open) nvtxRangePop();
    nvtxRangePushA(s);
    open = true;
    g_scope = s;
}

void prof_begin(const char *kind, double flops, double bytes, cudaStream_t st) {
    Rec r{g_scope + "." + kind, flops, bytes, take(), take()};
    RS_CUDA(cudaEventRecord(r.a, st));
    g_open.push_back(r);
    ++g_depth;  // nested launches (e.g. a GEMM inside a profiled helper) are not double counted
}

void prof_end(cudaStream_t st) {
    --g_depth;
    RS_CUDA(cudaEventRecord(g_open.back().b, st));
}

void prof_collect() {
    for (auto &r : g_open) {
        float ms = 0.f;
        RS_CUDA(cudaEventSynchronize(r.b));
        RS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        Tot &t = g_tot[r.cls];
        t.n += 1;
        t.ms += ms;
        t.flops += r.flops;
        t.bytes += r.bytes;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_open.clear();
}

std::string prof_json() {
    std::string s = "{";
    bool first = true;
    char buf[256];
    for (auto &[k, t] : g_tot) {
        std::snprintf(buf, sizeof(buf), "%s\"%s\": {\"launches\": %ld, \"ms\": %.6f, \"flops\": %.6e, \"bytes\": %.6e}",
                      first ? "" : ", ", k.c_str(), t.n, t.ms, t.flops, t.bytes);
        s += buf;
        first = false;
    }
    return s + "}";
}

void prof_reset() {
    g_open.clear();
    g_tot.clear();
}

}  // namespace rs
