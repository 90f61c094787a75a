#include <cstdlib>
// prof.cu — per-kernel-class CUDA-event timing and launch counting (the
// library's own tracing; used by bench.py to time the dominant kernel live on
// the stream it is launched on).
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "internal.h"

namespace nrlsh {

static const char *kSlotNames[kNumSlots] = {
    "norms", "partition", "scatter", "codes", "qcodes", "pilot", "scan", "fallback",
    "select", "gt_score", "gt_topk", "gt_norms", "gt_filter", "rerank", "rerank_topk", "other"};

static std::atomic<long long> g_launches{0};
static std::atomic<int> g_prof_on{0};
static std::mutex g_mu;
struct Pending { int slot; cudaEvent_t a, b; };
static std::vector<Pending> g_pending;
static std::vector<cudaEvent_t> g_free;
static double g_ms[kNumSlots];
static long long g_cnt[kNumSlots];

void note_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
bool pdl_enabled() {
    static const bool on = !(getenv("NRLSH_NO_PDL") && atoi(getenv("NRLSH_NO_PDL")) != 0);
    return on;
}
long long launch_count() { return g_launches.load(); }

static cudaEvent_t get_event() {
    if (!g_free.empty()) { cudaEvent_t e = g_free.back(); g_free.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

ProfScope::ProfScope(int slot, cudaStream_t s) : slot_(slot), s_(s), a_(nullptr) {
    if (!g_prof_on.load()) return;
    std::lock_guard<std::mutex> g(g_mu);
    a_ = get_event();
    cudaEventRecord((cudaEvent_t)a_, s);
}

ProfScope::~ProfScope() {
    if (!a_) return;
    std::lock_guard<std::mutex> g(g_mu);
    cudaEvent_t b = get_event();
    cudaEventRecord(b, s_);
    g_pending.push_back({slot_, (cudaEvent_t)a_, b});
}

void prof_collect() {
    std::lock_guard<std::mutex> g(g_mu);
    for (auto &p : g_pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            g_ms[p.slot] += ms;
            g_cnt[p.slot] += 1;
        }
        g_free.push_back(p.a);
        g_free.push_back(p.b);
    }
    g_pending.clear();
}

}  // namespace nrlsh

extern "C" {

void nrlsh_profile_enable(int on) {
    nrlsh::prof_collect();
    nrlsh::g_prof_on.store(on ? 1 : 0);
}

int nrlsh_profile_read(double *ms, int64_t *counts, int32_t nslots, int reset) {
    nrlsh::prof_collect();
    std::lock_guard<std::mutex> g(nrlsh::g_mu);
    for (int i = 0; i < nslots && i < nrlsh::kNumSlots; ++i) {
        if (ms) ms[i] = nrlsh::g_ms[i];
        if (counts) counts[i] = nrlsh::g_cnt[i];
        if (reset) { nrlsh::g_ms[i] = 0.0; nrlsh::g_cnt[i] = 0; }
    }
    return nrlsh::kNumSlots;
}

const char *nrlsh_profile_slot_name(int32_t slot) {
    if (slot < 0 || slot >= nrlsh::kNumSlots) return "";
    return nrlsh::kSlotNames[slot];
}

int64_t nrlsh_launch_count(void) { return nrlsh::launch_count(); }

}  // extern "C"
