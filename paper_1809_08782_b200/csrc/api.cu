// api.cu — the C ABI of libnrlsh (include/nrlsh.h): validation, device memory,
// launch orchestration, and the two small host-side steps of the build (the
// seeded projection matrix and the sorted (U_j, l) structure of PAPER:217).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

using namespace nrlsh;

namespace {

thread_local std::string g_last_error;
thread_local int64_t g_last_fallbacks = 0;
thread_local int64_t g_last_launches = 0;
thread_local int64_t g_last_pairs = 0;
thread_local int64_t g_last_entries = 0;       // candidate-buffer entries the select read
thread_local int64_t g_last_lb_pairs = 0;       // pairs the scan's lower bound ran on
thread_local int64_t g_last_lb_skipped = 0;     // ... and decided alone
thread_local int64_t g_last_scan_popc = 0;      // POPCs the scan issued on existing items
thread_local int64_t g_last_gt_pairs = 0;      // (query, item) pairs the exact filter multiplied
thread_local int64_t g_last_rescored = 0;
thread_local int64_t g_last_rtc_overflow = 0;   // tensor-core re-rank: queries redone by gather
thread_local int64_t g_last_rtc = 0;            // 1 if the last query used the tensor-core re-rank
thread_local int64_t g_last_rtc_pairs = 0;      // (query, item) pairs its filter multiplied
thread_local bool g_in_rtc_redo = false;
thread_local int64_t g_last_gt_max_cand = 0, g_last_gt_sum_cand = 0, g_last_gt_overflow = 0;

nrlsh_status fail(nrlsh_status st, const std::string &msg) {
    g_last_error = msg;
    return st;
}

nrlsh_status cuda_fail(cudaError_t e, const char *where) {
    return fail(NRLSH_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// RAII device allocation (stream-ordered).
struct DBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    ~DBuf() { if (p) cudaFreeAsync(p, s); }
    cudaError_t alloc(size_t bytes, cudaStream_t st) {
        s = st;
        return dmalloc(&p, bytes ? bytes : 16, st);
    }
    template <class T> T *get() const { return (T *)p; }
};

// -------------------------------------------------------------- projection
// Documented generator (include/nrlsh.h): SplitMix64 at counter c, two 53-bit
// uniforms, Box-Muller in fp64, fp32, then round-to-nearest-even to TF32.
inline uint64_t mix64_at(uint64_t seed, uint64_t c) {
    uint64_t x = seed + (c + 1ull) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

float tf32_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x0FFFu + ((u >> 13) & 1u);
    u &= ~0x1FFFu;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

void make_projection(uint64_t seed, int rows, int L, std::vector<float> &A) {
    A.resize((size_t)rows * L);
    const double k2pi = 2.0 * M_PI;
    const double inv53 = 1.0 / 9007199254740992.0;
    for (size_t e = 0; e < A.size(); ++e) {
        const double u1 = (double)((mix64_at(seed, 2 * e) >> 11) + 1ull) * inv53;
        const double u2 = (double)(mix64_at(seed, 2 * e + 1) >> 11) * inv53;
        const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(k2pi * u2);
        A[e] = tf32_rne((float)g);
    }
}

// -------------------------------------------------------------- rank table
// s_hat(j, h) = U_j cos(pi (1 - eps) h / L)  (Eq. (12) + eps);
// order: s_hat desc, U desc, h asc, j asc.  R[j][h] = position; order[pos] = j*(L+1)+h.
void make_rank_table(const std::vector<double> &U, int L, double eps, std::vector<uint16_t> &R,
                     std::vector<int32_t> &order) {
    const int m = (int)U.size();
    struct E { double s, u; int j, h; };
    std::vector<E> es;
    es.reserve((size_t)m * (L + 1));
    // (cos(pi (1 - eps) h / L) depends on h only: evaluated once per h, the same
    // fp64 value as in the product below)
    std::vector<double> ch(L + 1);
    for (int h = 0; h <= L; ++h) ch[h] = std::cos(M_PI * (1.0 - eps) * (double)h / (double)L);
    for (int j = 0; j < m; ++j)
        for (int h = 0; h <= L; ++h)
            es.push_back({U[j] * ch[h], U[j], j, h});
    std::sort(es.begin(), es.end(), [](const E &a, const E &b) {
        if (a.s != b.s) return a.s > b.s;
        if (a.u != b.u) return a.u > b.u;
        if (a.h != b.h) return a.h < b.h;
        return a.j < b.j;
    });
    R.assign(es.size(), 0);
    order.assign(es.size(), 0);
    for (size_t p = 0; p < es.size(); ++p) {
        R[(size_t)es[p].j * (L + 1) + es[p].h] = (uint16_t)p;
        order[p] = es[p].j * (L + 1) + es[p].h;
    }
}

int words_for(int L) { return L <= 32 ? 1 : (L <= 64 ? 2 : 4); }

void free_index(nrlsh_index *ix) {
    if (!ix) return;
    void *ps[] = {ix->X_owned, ix->Xpad, ix->Xb, ix->xnorm, ix->norm2, ix->perm, ix->pos_of_id, ix->part_of_id,
                  ix->part_of_pos, ix->offsets_d, ix->V_d, ix->codes, ix->A, ix->Apad,
                  ix->R_d, ix->chunks_d, ix->order_d, ix->samp_codes, ix->samp_part,
                  ix->xnorm_pos, ix->tile_xmax, ix->ctiles_d, ix->codes_pm};
    // pool-backed (cudaMallocAsync at build); the index may have been used on any stream
    cudaDeviceSynchronize();
    for (void *p : ps)
        if (p) cudaFreeAsync(p, nullptr);
    delete ix;
}

// Stage a possibly-host input into device memory.
struct Staged {
    const void *dev = nullptr;
    DBuf buf;
    cudaError_t in(const void *p, size_t bytes, cudaStream_t s) {
        if (is_device_ptr(p)) { dev = p; return cudaSuccess; }
        cudaError_t e = buf.alloc(bytes, s);
        if (e) return e;
        dev = buf.p;
        return cudaMemcpyAsync(buf.p, p, bytes, cudaMemcpyHostToDevice, s);
    }
};
// Device destination for a possibly-host output.
struct OutBuf {
    void *user = nullptr;
    void *dev = nullptr;
    size_t bytes = 0;
    bool host = false;
    DBuf buf;
    cudaError_t init(void *p, size_t b, cudaStream_t s) {
        user = p;
        bytes = b;
        host = !is_device_ptr(p);
        if (!host) { dev = p; return cudaSuccess; }
        cudaError_t e = buf.alloc(b, s);
        dev = buf.p;
        return e;
    }
    cudaError_t finish(cudaStream_t s) {
        if (!host) return cudaSuccess;
        return cudaMemcpyAsync(user, dev, bytes, cudaMemcpyDeviceToHost, s);
    }
};

}  // namespace

namespace nrlsh {
// Stream-ordered allocations come from a private pool per device (not the
// process-wide default pool a PyTorch allocator in the same process may rely on).
// It keeps up to 24 GiB of freed memory cached across calls (query workspaces are
// ~2.5 GB and are reallocated every call, an index of the scale config holds ~5 GB:
// below the footprint of a build + query + ground-truth cycle the pool would unmap
// and re-map memory every cycle, ~10-40 ms at scale) and returns the rest to the
// driver at the next synchronisation.
cudaError_t dmalloc(void **p, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static cudaMemPool_t pools[128] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    if (dev < 0 || dev >= 128) return cudaErrorInvalidDevice;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> g(mu);
        if (!pools[dev]) {
            cudaMemPoolProps pr = {};
            pr.allocType = cudaMemAllocationTypePinned;
            pr.location.type = cudaMemLocationTypeDevice;
            pr.location.id = dev;
            if ((e = cudaMemPoolCreate(&pools[dev], &pr))) { pools[dev] = nullptr; return e; }
            uint64_t thr = 24ull << 30;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

int pilot_stride(int64_t n) {
    if (n <= (1 << 18)) return 1;                 // exact histogram: no fallback needed
    // ~32,768 sampled positions (stride capped at 64; NRLSH_PILOT_SAMPLES overrides for
    // experiments): on c4 the pilot halves (0.27 -> 0.16 ms per 1024 queries) for +4% scan
    const int64_t ns = getenv("NRLSH_PILOT_SAMPLES") ? atoll(getenv("NRLSH_PILOT_SAMPLES")) : 32768;
    // (stride at most 64, 128 past 4M items: at scale, n = 16.8M, 131K samples instead of
    // 262K halve the pilot, 46 -> 27 ms per 65,536 queries, for +6 ms of scan and select)
    const int64_t cap = getenv("NRLSH_PILOT_MAXSTRIDE") ? atoll(getenv("NRLSH_PILOT_MAXSTRIDE"))
                                                        : (n > (4ll << 20) ? 128 : 64);
    int64_t s = n / std::max<int64_t>(1024, ns);
    return (int)std::max<int64_t>(1, std::min<int64_t>(cap, s));
}
}  // namespace nrlsh

// ============================================================================ ABI
extern "C" {

void nrlsh_default_options(nrlsh_options *opt) {
    if (!opt) return;
    opt->eps = 0.01;
    opt->scheme = NRLSH_SCHEME_PERCENTILE;
    opt->index_bits_in_budget = 0;
    opt->query_batch = 0;
    opt->proj = NRLSH_PROJ_SHARED;
}

const char *nrlsh_last_error(void) { return g_last_error.c_str(); }

void nrlsh_free(nrlsh_index *index) { free_index(index); }

nrlsh_status nrlsh_build(const float *items, int64_t n, int32_t d, int32_t code_bits,
                         int32_t num_parts, uint64_t seed, nrlsh_index **out, void *cuda_stream) {
    nrlsh_options o;
    nrlsh_default_options(&o);
    return nrlsh_build_ex(items, n, d, code_bits, num_parts, seed, &o, out, cuda_stream);
}

nrlsh_status nrlsh_build_ex(const float *items, int64_t n, int32_t d, int32_t code_bits,
                            int32_t num_parts, uint64_t seed, const nrlsh_options *opt,
                            nrlsh_index **out, void *cuda_stream) {
    if (!out) return fail(NRLSH_EINVAL, "out is NULL");
    *out = nullptr;
    nrlsh_options o;
    nrlsh_default_options(&o);
    if (opt) o = *opt;
    if (!items) return fail(NRLSH_EINVAL, "items is NULL");
    if (n < 1 || n >= (1ll << 31)) return fail(NRLSH_EINVAL, "n must be in [1, 2^31)");
    if (d < 1 || d > 4096) return fail(NRLSH_EINVAL, "d must be in [1, 4096]");
    if (!(o.eps >= 0.0 && o.eps < 1.0)) return fail(NRLSH_EINVAL, "eps must be in [0, 1)");
    if (o.scheme != NRLSH_SCHEME_PERCENTILE && o.scheme != NRLSH_SCHEME_UNIFORM)
        return fail(NRLSH_EINVAL, "unknown partition scheme");
    if (o.proj != NRLSH_PROJ_SHARED && o.proj != NRLSH_PROJ_PER_PARTITION)
        return fail(NRLSH_EINVAL, "unknown projection mode");
    if (num_parts < 1 || num_parts > kMaxParts)
        return fail(NRLSH_EINVAL, "num_parts must be in [1, 256]");
    if (o.scheme == NRLSH_SCHEME_PERCENTILE && (int64_t)num_parts > n)
        return fail(NRLSH_EINVAL, "num_parts > n (percentile partitioning needs m <= n)");
    int L = code_bits;
    if (o.index_bits_in_budget) {
        int ib = 0;
        while ((1 << ib) < num_parts) ++ib;   // ceil(log2 m)
        L = code_bits - ib;
    }
    if (L < 1 || L > 128 || (L > 64 && L <= 96))
        return fail(NRLSH_EINVAL, "hash bits L_h must be in [1,64] or [97,128] (got " +
                                      std::to_string(L) + ")");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    // (NRLSH_BUILD_TRACE=1: host timestamps of the build's phases on stderr)
    const bool trace = getenv("NRLSH_BUILD_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto tr = [&](const char *what) {
        if (trace)
            fprintf(stderr, "[build] %8.1f us  %s\n",
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_start).count(), what);
    };

    std::unique_ptr<nrlsh_index, void (*)(nrlsh_index *)> ix(new nrlsh_index(), free_index);
    ix->n = n;
    ix->d = d;
    ix->L = L;
    ix->W = words_for(L);
    ix->m = num_parts;
    ix->code_bits = code_bits;
    ix->seed = seed;
    ix->eps = o.eps;
    ix->scheme = o.scheme;
    ix->query_batch = o.query_batch > 0 ? o.query_batch : 1024;
    if (getenv("NRLSH_QUERY_BATCH")) ix->query_batch = std::max(1, atoi(getenv("NRLSH_QUERY_BATCH")));   // (experiments)
    ix->proj = o.proj;
    ix->QM = o.proj == NRLSH_PROJ_PER_PARTITION ? num_parts : 1;
    if (ix->QM > 1 && !codes_tc_supported(d, words_for(L)))
        return fail(NRLSH_ENOTIMPL, "per-sub-dataset projections need the tensor-core code kernel's "
                                    "shapes (d <= 512, ceil(L_h/32) != 3)");
    cudaGetDevice(&ix->device);
    const int m = num_parts, W = ix->W;

#define NR_ALLOC(ptr, bytes)                                                      \
    do {                                                                          \
        cudaError_t e_ = dmalloc((void **)&(ptr), (bytes) ? (bytes) : 16, s); \
        if (e_ != cudaSuccess) { cudaGetLastError(); return fail(NRLSH_ENOMEM, "cudaMalloc " #ptr); } \
    } while (0)

    if (is_device_ptr(items)) {
        ix->X = items;
    } else {
        NR_ALLOC(ix->X_owned, (size_t)n * d * 4);
        cudaError_t e = cudaMemcpyAsync(ix->X_owned, items, (size_t)n * d * 4,
                                        cudaMemcpyHostToDevice, s);
        if (e) return cuda_fail(e, "copy items");
        ix->X = ix->X_owned;
    }
    tr("args");
    NR_ALLOC(ix->norm2, (size_t)n * 8);
    // bf16 rows (16-byte aligned, zero-padded to dpb) and |x| rounded up, written by the
    // norms pass: the ground truth's tensor-core operand and the re-rank's certified
    // filter pass (half the bytes of the fp32 rows it then gathers only for survivors)
    // rows of d % 4 != 0 floats are only 4- or 8-byte aligned: a 16-byte-aligned padded
    // fp32 copy (written by the codes pass) lets the re-rank gather with 16-byte loads
    // (opt-in NRLSH_XPAD=1: a 16-byte-aligned fp32 row copy for the re-rank's gathers
    // when 4 does not divide d — measured a wash on c4: the codes pass saves 0.17 ms
    // without it, the 8-byte-load gathers lose about as much)
    ix->dpad = (d + 3) / 4 * 4;
    if (ix->dpad != d && getenv("NRLSH_XPAD") && atoi(getenv("NRLSH_XPAD")) != 0)
        NR_ALLOC(ix->Xpad, (size_t)n * ix->dpad * 4);
    ix->dpb = (d + 7) / 8 * 8;
    const int64_t npad = (n + 255) / 256 * 256;
    NR_ALLOC(ix->Xb, (size_t)n * ix->dpb * 2);
    NR_ALLOC(ix->xnorm, (size_t)npad * 4);
    cudaMemsetAsync(ix->xnorm + n, 0, (size_t)(npad - n) * 4, s);
    NR_ALLOC(ix->perm, (size_t)n * 4);
    NR_ALLOC(ix->pos_of_id, (size_t)n * 4);
    NR_ALLOC(ix->part_of_id, (size_t)npad);
    cudaMemsetAsync(ix->part_of_id + n, 0, (size_t)(npad - n), s);
    NR_ALLOC(ix->part_of_pos, (size_t)npad);
    cudaMemsetAsync(ix->part_of_pos + n, 0, (size_t)(npad - n), s);
    NR_ALLOC(ix->xnorm_pos, (size_t)npad * 4);
    cudaMemsetAsync(ix->xnorm_pos + n, 0, (size_t)(npad - n) * 4, s);
    NR_ALLOC(ix->tile_xmax, (size_t)((n + 127) / 128) * 4);
    // +-1 rows for the opt-in tensor-core scan (NEXT-3; NRLSH_SCAN_TC=1 at build and query)
    if (L <= 128 && ix->QM == 1 && getenv("NRLSH_SCAN_TC") && atoi(getenv("NRLSH_SCAN_TC")) != 0)
        NR_ALLOC(ix->codes_pm, (size_t)n * scan_kp(L));
    NR_ALLOC(ix->offsets_d, (size_t)(m + 1) * 8);
    NR_ALLOC(ix->V_d, (size_t)m * 8);
    NR_ALLOC(ix->codes, (size_t)n * W * 4 + 1024);   // (+1 KB: the scans' aligned reads past the end)

    // One host round trip: the device steps of Alg. 1 are enqueued ahead of the host
    // work that depends on them.  Stream order: norms, partition, scatter, the
    // read-back of (offsets, V, flags) [event], codes and the |x| tiles; meanwhile the
    // host generates the projection (before the codes are enqueued) and, once the
    // event fires, builds its tables while the codes kernel runs.
    tr("allocs");
    const int QM = ix->QM;
    const size_t ablk = (size_t)(d + 1) * L, pblk = (size_t)(d + 1) * 32 * W;
    NR_ALLOC(ix->A, (size_t)QM * ablk * 4);
    NR_ALLOC(ix->Apad, (size_t)QM * pblk * 4);
    // build flags: [0] first non-finite item (~0: none), [1] large percentile group,
    // [2] the filter's first-pass |x| split (float bits)
    // [4], [5] the smallest positive and largest norm2 bits (the percentile select's window)
    DBuf res;
    if (res.alloc(48, s)) return fail(NRLSH_ENOMEM, "cudaMallocAsync");
    const unsigned long long res0[6] = {~0ull, 0ull, 0ull, 0ull, ~0ull, 0ull};
    cudaMemcpyAsync(res.p, res0, 48, cudaMemcpyHostToDevice, s);
    unsigned long long *resd = res.get<unsigned long long>();
    const int64_t ntx = (n + 127) / 128;   // 128-row |x| tiles
    ix->offsets.resize(m + 1);
    ix->V.resize(m);
    // pinned read-back area (a D2H copy into pageable memory would block the host):
    // [offsets (m+1) | V (m) | flags (4)], thread-local and grown on demand
    thread_local void *pin = nullptr;
    thread_local size_t pin_bytes = 0;
    const size_t need = (size_t)(2 * m + 1) * 8 + 32;
    if (pin_bytes < need) {
        if (pin) cudaFreeHost(pin);
        pin = nullptr;
        pin_bytes = 0;
        if (cudaMallocHost(&pin, std::max<size_t>(need, 8192)) != cudaSuccess) {
            cudaGetLastError();
            return fail(NRLSH_ENOMEM, "pinned read-back buffer");
        }
        pin_bytes = std::max<size_t>(need, 8192);
    }
    int64_t *h_off = reinterpret_cast<int64_t *>(pin);
    double *h_V = reinterpret_cast<double *>(h_off + m + 1);
    unsigned long long *hres = reinterpret_cast<unsigned long long *>(h_V + m);
    cudaEvent_t ev_part;
    cudaEventCreateWithFlags(&ev_part, cudaEventDisableTiming);
    std::unique_ptr<CUevent_st, cudaError_t (*)(cudaEvent_t)> ev_guard(ev_part, cudaEventDestroy);
    auto partition_steps = [&](bool fast) -> nrlsh_status {
        std::string err;
        int rc;
        bool have_mm = false;
        if (fast) {   // K1: norms + finite check
            ProfScope p(SLOT_NORMS, s);
            have_mm = launch_norms(ix->X, n, d, ix->norm2, resd, ix->Xb, ix->dpb, ix->xnorm, s, resd + 4);
        }
        {   // K2: percentile (or uniform) partition
            ProfScope p(SLOT_PARTITION, s);
            if (o.scheme != NRLSH_SCHEME_PERCENTILE)
                rc = partition_uniform(ix->norm2, n, m, ix->part_of_id, s, &err);
            else if (fast)
                rc = partition_percentile_fast(ix->norm2, n, m, ix->part_of_id,
                                               reinterpret_cast<unsigned int *>(resd + 1), s, &err,
                                               have_mm ? resd + 4 : nullptr);
            else
                rc = partition_percentile(ix->norm2, n, m, ix->part_of_id, s, &err);
        }
        if (rc) return fail((nrlsh_status)rc, err);
        {   // stable scatter: perm, positions, offsets, V
            ProfScope p(SLOT_SCATTER, s);
            rc = partition_scatter(ix->norm2, ix->part_of_id, n, m, ix->perm, ix->pos_of_id,
                                   ix->part_of_pos, ix->offsets_d, ix->V_d, s, &err);
        }
        if (rc) return fail((nrlsh_status)rc, err);
        cudaMemcpyAsync(h_off, ix->offsets_d, (size_t)(m + 1) * 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(h_V, ix->V_d, (size_t)m * 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(hres, res.p, 16, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ev_part, s);
        return NRLSH_OK;
    };
    auto code_steps = [&]() {
        ProfScope p(SLOT_CODES, s);
        // K3: codes (shared A: every input is on the device already)
        if (QM == 1)
            launch_item_codes(ix->X, n, d, ix->norm2, ix->part_of_id, ix->V_d, ix->Apad, L, W,
                              ix->pos_of_id, ix->codes, ix->Xb, ix->dpb, ix->xnorm, ix->Xpad,
                              ix->dpad, s, ix->perm, m);
        // |x| in partition order (the tensor-core filter's tiles) and the first-pass split
        // of those tiles: the 1/800 (at least 16) with the largest |x| (c4: 0.15 vs 0.18 ms
        // per 1024 seeded queries at 1/50, 0.37 vs 0.74 unseeded; the first pass's exact
        // k-th best then prunes every other tile)
        launch_gather_f32(ix->xnorm, ix->perm, n, ix->xnorm_pos, s);
        launch_tile_xmax128(ix->xnorm_pos, n, ix->tile_xmax, s);
        if (ntx >= 64) {
            const int64_t div = getenv("NRLSH_GT_SPLIT_DIV") ? std::max(2, atoi(getenv("NRLSH_GT_SPLIT_DIV"))) : 800;
            const int64_t r = ntx - std::min<int64_t>(ntx - 1, std::max<int64_t>(16, ntx / div));
            launch_select_kth_float(ix->tile_xmax, ntx, r, reinterpret_cast<float *>(resd + 2), s);
        }
    };
    tr("pinned/event");
    nrlsh_status st = partition_steps(true);
    if (st) return st;
    tr("partition enqueued");
    {   // K4a (host, overlapped with the partition): A_j from seed XOR j (A_0 = the
        // shared A); per-sub-dataset projections are m independent draws, on up to 16
        // host threads
        ix->A_h.resize(QM * ablk);
        std::vector<float> Apad(QM * pblk, 0.f);
        auto gen = [&](int j0, int j1) {
            for (int j = j0; j < j1; ++j) {
                std::vector<float> Aj;
                make_projection(seed ^ (uint64_t)j, d + 1, L, Aj);
                std::copy(Aj.begin(), Aj.end(), ix->A_h.begin() + j * ablk);
                for (int k = 0; k <= d; ++k)
                    for (int b = 0; b < L; ++b) Apad[j * pblk + (size_t)k * 32 * W + b] = Aj[(size_t)k * L + b];
            }
        };
        const int nt = QM > 1 ? std::max(1, std::min<int>(16, (int)std::thread::hardware_concurrency())) : 1;
        if (nt <= 1) {
            gen(0, QM);
        } else {
            std::vector<std::thread> th;
            for (int t = 0; t < nt; ++t) th.emplace_back(gen, QM * t / nt, QM * (t + 1) / nt);
            for (auto &t : th) t.join();
        }
        // (pageable sources: staged before the calls return)
        cudaMemcpyAsync(ix->A, ix->A_h.data(), ix->A_h.size() * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(ix->Apad, Apad.data(), Apad.size() * 4, cudaMemcpyHostToDevice, s);
    }
    tr("projection");
    code_steps();
    tr("codes enqueued");
    cudaError_t e = cudaEventSynchronize(ev_part);
    if (e) return cuda_fail(e, "build");
    tr("partition done (event)");
    if (hres[0] != ~0ull)
        return fail(NRLSH_ENONFINITE, "non-finite item at index " + std::to_string(hres[0]));
    if (hres[1]) {   // (ties or duplicates: a boundary group needs the multi-level select)
        if ((st = partition_steps(false))) return st;
        code_steps();
        if ((e = cudaEventSynchronize(ev_part))) return cuda_fail(e, "build");
    }
    std::copy(h_off, h_off + m + 1, ix->offsets.begin());
    std::copy(h_V, h_V + m, ix->V.begin());
    ix->U.resize(m);
    for (int j = 0; j < m; ++j) ix->U[j] = std::sqrt(ix->V[j]);

    // K4b (host): the sorted (U_j, l) structure and the work lists
    std::vector<int32_t> order;
    make_rank_table(ix->U, L, ix->eps, ix->R_h, order);
    tr("rank table");
    // scan work units: chunks of <= scan_chunk_items() positions inside one sub-dataset
    std::vector<int4> chunks;
    const int CH = scan_chunk_items();
    for (int j = 0; j < m; ++j)
        for (int64_t p = ix->offsets[j]; p < ix->offsets[j + 1]; p += CH)
            chunks.push_back(make_int4(j, (int)p, (int)std::min<int64_t>(p + CH, ix->offsets[j + 1]), 0));
    ix->nchunks = (int32_t)chunks.size();
    // tiles of <= 128 positions of one sub-dataset: the code kernel's with per-sub-
    // dataset projections, the (opt-in) tensor-core scan's items (built only for them)
    std::vector<int4> ctiles;
    if (QM > 1 || ix->codes_pm)
        for (int j = 0; j < m; ++j)
            for (int64_t p = ix->offsets[j]; p < ix->offsets[j + 1]; p += 128)
                ctiles.push_back(make_int4(j, (int)p, (int)std::min<int64_t>(p + 128, ix->offsets[j + 1]), 0));
    ix->nctiles = (int32_t)ctiles.size();
    tr("work lists");
    if (!ctiles.empty()) NR_ALLOC(ix->ctiles_d, ctiles.size() * sizeof(int4));
    NR_ALLOC(ix->R_d, ix->R_h.size() * 2);
    NR_ALLOC(ix->order_d, order.size() * 4);
    NR_ALLOC(ix->chunks_d, chunks.size() * sizeof(int4));
    {   // the tables go through pinned staging: a pageable H2D copy larger than the
        // driver's staging buffer would block the host until the stream reaches it
        // (after the code kernel), and the launches behind it would wait too
        const size_t b_ct = ctiles.size() * sizeof(int4), b_R = ix->R_h.size() * 2,
                     b_or = order.size() * 4, b_ch = chunks.size() * sizeof(int4);
        const size_t tot = b_ct + b_R + b_or + b_ch + 64;
        thread_local void *tpin = nullptr;
        thread_local size_t tpin_bytes = 0;
        if (tpin_bytes < tot) {
            if (tpin) cudaFreeHost(tpin);
            tpin = nullptr;
            tpin_bytes = 0;
            if (cudaMallocHost(&tpin, std::max<size_t>(tot, 1 << 20)) != cudaSuccess) {
                cudaGetLastError();
                return fail(NRLSH_ENOMEM, "pinned table staging");
            }
            tpin_bytes = std::max<size_t>(tot, 1 << 20);
        }
        tr("table allocs");
        uint8_t *h = static_cast<uint8_t *>(tpin);
        std::memcpy(h, ctiles.data(), b_ct);
        std::memcpy(h + b_ct, ix->R_h.data(), b_R);
        std::memcpy(h + b_ct + b_R, order.data(), b_or);
        std::memcpy(h + b_ct + b_R + b_or, chunks.data(), b_ch);
        if (b_ct) cudaMemcpyAsync(ix->ctiles_d, h, b_ct, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(ix->R_d, h + b_ct, b_R, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(ix->order_d, h + b_ct + b_R, b_or, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(ix->chunks_d, h + b_ct + b_R + b_or, b_ch, cudaMemcpyHostToDevice, s);
    }
    if (QM > 1) {   // K3 with per-sub-dataset projections: partition-ordered tiles
        ProfScope p(SLOT_CODES, s);
        launch_item_codes_tc(ix->X, n, d, ix->norm2, ix->part_of_id, ix->V_d, ix->Apad, L, W,
                             ix->pos_of_id, ix->codes, ix->Xb, ix->dpb, ix->Xpad, ix->dpad, s,
                             ix->ctiles_d, ix->nctiles, ix->perm);
    }
    {
        ProfScope p(SLOT_CODES, s);
        if (ix->codes_pm) launch_expand_pm(ix->codes, n, W, L, ix->codes_pm, s);
        // compacted pilot sample (query-time pilots read it contiguously)
        const int stride = pilot_stride(n);
        if (stride > 1) {
            // (interleaved slots: 32 columns of ceil(samples / 32) positions ~n/32
            // apart; the pilot skips the slots past the sample)
            ix->nsamp = ((n + stride - 1) / stride + 31) / 32 * 32;
            NR_ALLOC(ix->samp_codes, (size_t)ix->nsamp * W * 4);
            NR_ALLOC(ix->samp_part, (size_t)ix->nsamp);
            launch_gather_sample(ix.get(), stride, ix->samp_codes, ix->samp_part, s);
        }
    }
    tr("tables enqueued");
    cudaMemcpyAsync(hres + 2, resd + 2, 8, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e) return cuda_fail(e, "codes");
    tr("done (stream sync)");
    {
        float xs;
        const uint32_t xb = (uint32_t)hres[2];
        std::memcpy(&xs, &xb, 4);
        ix->tile_xsplit = ntx >= 64 ? xs : 0.f;
    }
    prof_collect();
    e = cudaGetLastError();
    if (e) return cuda_fail(e, "build launch");
#undef NR_ALLOC
    *out = ix.release();
    return NRLSH_OK;
}

nrlsh_status nrlsh_get_info(const nrlsh_index *ix, int64_t *n, int32_t *d, int32_t *hash_bits,
                            int32_t *num_parts, int32_t *words) {
    if (!ix) return fail(NRLSH_EINVAL, "index is NULL");
    if (n) *n = ix->n;
    if (d) *d = ix->d;
    if (hash_bits) *hash_bits = ix->L;
    if (num_parts) *num_parts = ix->m;
    if (words) *words = ix->W;
    return NRLSH_OK;
}

// ------------------------------------------------------------------ query
namespace {


// Per-query append capacity: the pilot bound's count before its boundary cell
// (T + sampling noise) plus the boundary cell itself, which can hold a whole
// sub-dataset (items of a large-U_j sub-dataset with small ||x||/U_j all map
// close to e_{d+1}, so their codes — and their h — nearly coincide).
int64_t buffer_capacity(int64_t Tq, int stride, int64_t n, int64_t max_part) {
    double c = 2.0 * Tq + 16.0 * std::sqrt((double)Tq * stride) + 4096.0 + (double)max_part;
    int64_t C = (int64_t)c;
    C = std::max<int64_t>(C, Tq);
    return std::min<int64_t>(C, n);
}

// The candidate pipeline for one sub-batch; leaves cand [Qb x Tq] (item ids).
void run_candidates(const nrlsh_index *ix, const float *Qd, const uint32_t *qcodes_in, int Qb,
                    int64_t qbase, int64_t Tq, int stride, int64_t C, uint32_t *qcodes,
                    int8_t *delta, uint32_t *cnt, uint32_t *cntv, void *scan_ws,
                    unsigned long long *buf, int32_t *cand, uint16_t *cand_rank, int *flags,
                    unsigned long long *pairs, cudaStream_t s, uint32_t *sel_B = nullptr,
                    uint32_t *sel_pk = nullptr,
                    int32_t *seeds = nullptr, int ks = 0, void *fb_ws = nullptr,
                    unsigned long long *entries = nullptr, void *units_ws = nullptr) {
    if (qcodes_in) {
        cudaMemcpyAsync(qcodes, qcodes_in + qbase * ix->QM * ix->W, (size_t)Qb * ix->QM * ix->W * 4,
                        cudaMemcpyDeviceToDevice, s);
    } else {
        ProfScope p(SLOT_QCODES, s);
        launch_qcodes(Qd, Qb, ix->d, ix->Apad, ix->L, ix->W, qcodes, flags, qbase, s, ix->QM);
    }
    {
        ProfScope p(SLOT_PILOT, s);
        launch_pilot(ix, qcodes, Qb, Tq, stride, delta, cnt, s, fallback_counter(ix, fb_ws));
    }
    if (getenv("NRLSH_TEST_FORCE_FALLBACK"))   // test switch: empty pilot bound -> fallback
        cudaMemsetAsync(delta, 0xff, (size_t)Qb * ix->m, s);
    bool tc = scan_tc_supported(ix);
    {
        ProfScope p(SLOT_SCAN, s);
        // (both scans append the same entries — the tensor-core one with ~0 sentinels
        // counted in cnt, real entries in cntv; a tensor-map failure falls back)
        if (tc) {
            cudaMemsetAsync(cntv, 0, (size_t)Qb * 4, s);
            if (launch_scan_tc(ix, qcodes, delta, Qb, scan_ws, buf, cnt, cntv, C, pairs, s)) tc = false;
        }
        if (!tc) launch_scan(ix, qcodes, delta, Qb, buf, cnt, C, pairs, s, pairs + 4, units_ws);
    }
    {
        ProfScope p(SLOT_FALLBACK, s);
        launch_fallback(ix, qcodes, Qb, Tq, buf, cnt, tc ? cntv : cnt, C, flags, fb_ws, s);
        // buffer entries the select reads (statistics: the select's HBM roofline)
        if (entries) launch_sum_counts(cnt, Qb, C, entries, s);
    }
    {
        ProfScope p(SLOT_SELECT, s);
        if (seeds) {   // bound pass + seed members (the tensor-core re-rank)
            launch_select_seeds(ix, Qb, Tq, buf, cnt, C, sel_B, sel_pk, seeds, ks, s);
        } else {
            launch_select(ix, Qb, Tq, buf, cnt, C, cand, cand_rank, s);
        }
    }
}

// Certified bound of |s~ - s_f| / (|q| |x|) for the tensor-core filter: s~ is the
// bf16-operand, fp32-accumulated MMA value over dp columns (operand rounding
// 2u + u^2 with u = 2^-8, accumulation of dp exact products dp * 2^-23, x1.05
// slack), s_f the fp32 FMA-chain score the exact re-rank computes (gamma_{dp+2}
// inflated); |s~ - s| and |s - s_f| add.
float gt_eps_rel(int dp) {
    const double u = std::ldexp(1.0, -8);
    return (float)(1.05 * ((2 * u + u * u) + (1 + u) * (1 + u) * dp * std::ldexp(1.0, -23)) +
                   1.25 * (dp + 2) * std::ldexp(1.0, -24));
}

nrlsh_status check_flags(const int *hflags) {
    if (hflags[1] != INT_MAX)
        return fail(NRLSH_ENONFINITE, "non-finite query at index " + std::to_string(hflags[1]));
    if (hflags[0] != INT_MAX)
        return fail(NRLSH_EZERONORM, "zero-norm query at index " + std::to_string(hflags[0]));
    return NRLSH_OK;
}

}  // namespace

static nrlsh_status query_impl(const nrlsh_index *ix, const float *queries,
                               const uint32_t *qcodes_user, int64_t nq, int32_t k,
                               int64_t probe_budget, int64_t *out_ids, float *out_scores,
                               int32_t *cand_out, uint16_t *rank_out, void *cuda_stream) {
    if (!ix) return fail(NRLSH_EINVAL, "index is NULL");
    if (nq < 1) return fail(NRLSH_EINVAL, "nq must be >= 1");
    if (probe_budget < 1) return fail(NRLSH_EINVAL, "probe_budget must be >= 1");
    const bool want_topk = out_ids != nullptr;
    if (want_topk && (k < 1 || k > 1024)) return fail(NRLSH_EINVAL, "k must be in [1, 1024]");
    if (!queries && !qcodes_user) return fail(NRLSH_EINVAL, "queries is NULL");
    if (want_topk && !queries) return fail(NRLSH_EINVAL, "queries is NULL");
    if (want_topk && !out_scores) return fail(NRLSH_EINVAL, "out_scores is NULL");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const int64_t n = ix->n;
    const int64_t Tq = std::min<int64_t>(probe_budget, n);
    const int stride = pilot_stride(n);
    int64_t max_part = 0;
    for (int j = 0; j < ix->m; ++j) max_part = std::max(max_part, ix->offsets[j + 1] - ix->offsets[j]);
    int64_t C = buffer_capacity(Tq, stride, n, max_part);
    // test switch: the smallest capacity the exact fallback still fits in (T + one
    // sub-dataset), so the scan's rows fill up and its guarded stores run
    if (getenv("NRLSH_TEST_BUFFER_TIGHT")) C = std::min<int64_t>(C, Tq + max_part + 64);
    int Qmax = (int)std::min<int64_t>(ix->query_batch, nq);
    if (scan_tc_supported(ix)) C += scan_tc_slack(Qmax);   // (its runs' unused tails)
    C = (C + 1) & ~(int64_t)1;   // even: 16-byte-aligned buffer rows (the select's paired loads)
    // keep the candidate buffers bounded (~2.5 GB)
    const int64_t per_q = C * 8 + Tq * 10;
    while (Qmax > 64 && (int64_t)Qmax * per_q > (int64_t)2500 << 20) Qmax >>= 1;

    Staged Qs, QCs;
    cudaError_t e;
    if (queries) {
        e = Qs.in(queries, (size_t)nq * ix->d * 4, s);
        if (e) return cuda_fail(e, "stage queries");
    }
    if (qcodes_user) {
        e = QCs.in(qcodes_user, (size_t)nq * ix->QM * ix->W * 4, s);
        if (e) return cuda_fail(e, "stage qcodes");
    }
    OutBuf oi, os, oc, orr;
    if (want_topk) {
        if ((e = oi.init(out_ids, (size_t)nq * k * 8, s))) return cuda_fail(e, "out_ids");
        if ((e = os.init(out_scores, (size_t)nq * k * 4, s))) return cuda_fail(e, "out_scores");
    }
    if (cand_out) {
        if ((e = oc.init(cand_out, (size_t)nq * Tq * 4, s))) return cuda_fail(e, "cand_ids");
        if (rank_out && (e = orr.init(rank_out, (size_t)nq * Tq * 2, s))) return cuda_fail(e, "cand_rank");
    }
    // Sub-batches alternate between two streams with a workspace set each, so one
    // sub-batch's kernels fill the other's gaps and tails (NRLSH_QUERY_SERIAL=1: one)
    // (NRLSH_QUERY_STREAMS: 1-3, default 2)
    int NSET = getenv("NRLSH_QUERY_STREAMS") ? std::max(1, std::min(3, atoi(getenv("NRLSH_QUERY_STREAMS")))) : 2;
    if (nq <= Qmax || getenv("NRLSH_QUERY_SERIAL")) NSET = 1;
    NSET = (int)std::min<int64_t>(NSET, (nq + Qmax - 1) / Qmax);
    struct WSet {
        DBuf qc, dl, cn, cv, ba, us, bf, cd, pt, fbw;
        DBuf rsb, rspk, rseed, rtid, rtsc, rth, rqb, rqn, rhp, rcd, rcc, rpt, rtl, rqp;
    } wsets[3];
    DBuf fl;
    if (fl.alloc(80, s)) return fail(NRLSH_ENOMEM, "query workspace");
    for (int w = 0; w < NSET; ++w) {
        WSet &W_ = wsets[w];
        if (W_.qc.alloc((size_t)Qmax * ix->QM * ix->W * 4, s) || W_.dl.alloc((size_t)Qmax * ix->m, s) ||
            W_.cn.alloc((size_t)Qmax * 4, s) || W_.cv.alloc((size_t)Qmax * 4, s) ||
            W_.ba.alloc(scan_tc_supported(ix) ? scan_tc_ws_bytes(ix, Qmax) : 16, s) ||
            W_.us.alloc(scan_units_ws_bytes(ix, Qmax), s) ||
            W_.bf.alloc((size_t)Qmax * C * 8, s) || W_.cd.alloc((size_t)Qmax * Tq * 4, s) ||
            W_.pt.alloc(want_topk ? rerank_partial_bytes(Qmax, Tq, k) : 0, s) ||
            W_.fbw.alloc(fallback_ws_bytes(ix), s))
            return fail(NRLSH_ENOMEM, "query workspace");
        // (histogram rows stay zero between uses)
        cudaMemsetAsync(W_.fbw.p, 0, fallback_ws_bytes(ix), s);
        // (the scan's unit counters: zero on entry, left zero by every scan)
        cudaMemsetAsync(W_.us.p, 0, 16, s);
    }
    const float *Xr = ix->Xpad ? ix->Xpad : ix->X;
    const int ldr = ix->Xpad ? ix->dpad : ix->d;
    // tensor-core re-rank (tc_kernels.cu member mode): a bf16 GEMM pass over the
    // tiles of the sub-datasets holding candidates, certified filter, keeping only
    // candidates; chosen when the candidate budget is a large enough share of n
    // (measured on c4: break-even near T = n / 300) and the sub-batch's gather would
    // touch at least ~1.28 n rows (Qmax T >= 1.28 n: the filter streams the items
    // once for all its queries; c4, T = 1%: the gather path wins below ~128 queries,
    // 0.27 vs 0.39 ms for one, while at T = 45% even 64 queries want the filter)
    // — NRLSH_RERANK_TC=0/1 forces it
    const char *rtc_env = getenv("NRLSH_RERANK_TC");
    const double rtc_ratio = getenv("NRLSH_RERANK_TC_RATIO") ? atof(getenv("NRLSH_RERANK_TC_RATIO")) : 300.0;
    const double rtc_qt = getenv("NRLSH_RERANK_TC_QT") ? atof(getenv("NRLSH_RERANK_TC_QT")) : 1.28;
    const bool use_rtc = want_topk && !g_in_rtc_redo && ix->Xb && ix->xnorm_pos &&
                         gt_tc_supported(ix->d, k) &&
                         (rtc_env ? atoi(rtc_env) != 0
                                  : (double)Tq * rtc_ratio >= (double)n &&
                                        (double)Qmax * (double)Tq >= rtc_qt * (double)n);
    const int KS = getenv("NRLSH_RERANK_TC_KS") ? std::max(k, std::min(1024, atoi(getenv("NRLSH_RERANK_TC_KS"))))
                                                 : std::min(1024, std::max(512, 4 * k));
    // survivor list capacity per query (NRLSH_RERANK_TC_CAP: test switch forcing the
    // overflow redo path)
    const int64_t Cg = getenv("NRLSH_RERANK_TC_CAP")
                           ? std::max<int64_t>(16, atoll(getenv("NRLSH_RERANK_TC_CAP")))
                           : std::min<int64_t>(n, std::max<int64_t>(16384, 256 * (int64_t)k));
    DBuf rov, rovn;
    if (use_rtc && (rov.alloc((size_t)nq * 8, s) || rovn.alloc(4, s)))
        return fail(NRLSH_ENOMEM, "query workspace (tensor-core re-rank)");
    for (int w = 0; use_rtc && w < NSET; ++w) {
        WSet &W_ = wsets[w];
        if (W_.rsb.alloc((size_t)Qmax * 4, s) || W_.rspk.alloc((size_t)Qmax * 4, s) ||
            W_.rseed.alloc((size_t)Qmax * KS * 4, s) || W_.rtid.alloc((size_t)Qmax * k * 8, s) ||
            W_.rtsc.alloc((size_t)Qmax * k * 4, s) || W_.rth.alloc((size_t)Qmax * 4, s) ||
            W_.rqb.alloc((size_t)Qmax * ix->dpb * 2, s) || W_.rqn.alloc((size_t)Qmax * 4, s) ||
            W_.rhp.alloc(gt_heap_bytes(k), s) || W_.rcd.alloc((size_t)Qmax * Cg * 4, s) ||
            W_.rcc.alloc((size_t)Qmax * 4, s) ||
            W_.rpt.alloc(std::max(rerank_partial_bytes(Qmax, Cg, k), rerank_partial_bytes(Qmax, KS, k)), s) ||
            W_.rtl.alloc(gt_tile_ws_bytes(n, Qmax), s) || W_.rqp.alloc((size_t)Qmax * 4, s))
            return fail(NRLSH_ENOMEM, "query workspace (tensor-core re-rank)");
    }
    if (use_rtc) cudaMemsetAsync(rovn.p, 0, 4, s);
    GtMember mb;
    mb.codes = ix->codes;
    mb.part = ix->part_of_pos;
    mb.offsets = ix->offsets_d;
    mb.m = ix->m;
    mb.R = ix->R_d;
    mb.L = ix->L;
    mb.W = ix->W;
    mb.qm = ix->QM;
    GtTiles tls;
    tls.xmax128 = ix->tile_xmax;
    tls.ws = nullptr;   // (per workspace set, below)
    tls.pairs = (unsigned long long *)(fl.get<int>() + 8);
    // one pass for the re-rank (two measured slower: 0.50 vs 0.43 ms per 1024 queries
    // on c4, the candidates' k-th best stays low after the top tiles)
    tls.xsplit = getenv("NRLSH_RERANK_TWOPASS") ? ix->tile_xsplit : 0.f;
    tls.pass = 0;
    tls.qperm = nullptr;
    // [0, 1] non-finite / zero query, [2] fallbacks, [4:5] scanned pairs, [6:7] re-scored,
    // [8:9] filter pairs, [10:11] buffer entries, [12:13] / [14:15] lower-bound pairs
    const int init_flags[20] = {INT_MAX, INT_MAX, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyAsync(fl.p, init_flags, 80, cudaMemcpyHostToDevice, s);
    unsigned long long *pairs = (unsigned long long *)(fl.get<int>() + 4);
    const long long launches0 = launch_count();
    // second stream (per thread and device) joined to s by events
    cudaStream_t st[3] = {s, s, s};
    cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
    if (NSET > 1) {
        thread_local cudaStream_t extra[128][2] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 128) return fail(NRLSH_ECUDA, "device index");
        cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
        cudaEventRecord(ev_fork, s);
        for (int w = 1; w < NSET; ++w) {
            if (!extra[dev][w - 1] &&
                cudaStreamCreateWithFlags(&extra[dev][w - 1], cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                return fail(NRLSH_ECUDA, "stream create");
            }
            st[w] = extra[dev][w - 1];
            cudaEventCreateWithFlags(&ev_join[w], cudaEventDisableTiming);
            cudaStreamWaitEvent(st[w], ev_fork, 0);
        }
    }
    int sbi = 0;
    for (int64_t q0 = 0; q0 < nq; q0 += Qmax, ++sbi) {
        const int Qb = (int)std::min<int64_t>(Qmax, nq - q0);
        WSet &W_ = wsets[sbi % NSET];
        cudaStream_t s = st[sbi % NSET];   // (this sub-batch's stream)
        DBuf &qc = W_.qc, &dl = W_.dl, &cn = W_.cn, &cv = W_.cv, &ba = W_.ba, &bf = W_.bf, &cd = W_.cd,
             &pt = W_.pt, &fbw = W_.fbw;
        DBuf &rsb = W_.rsb, &rspk = W_.rspk, &rseed = W_.rseed, &rtid = W_.rtid, &rtsc = W_.rtsc,
             &rth = W_.rth, &rqb = W_.rqb, &rqn = W_.rqn, &rhp = W_.rhp, &rcd = W_.rcd, &rcc = W_.rcc,
             &rpt = W_.rpt, &rtl = W_.rtl, &rqp = W_.rqp;
        tls.ws = use_rtc ? rtl.get<int32_t>() : nullptr;
        const float *Qd = queries ? (const float *)Qs.dev + q0 * ix->d : nullptr;
        int32_t *cand = cand_out ? (int32_t *)oc.dev + q0 * Tq : cd.get<int32_t>();
        uint16_t *crank = (cand_out && rank_out) ? (uint16_t *)orr.dev + q0 * Tq : nullptr;
        run_candidates(ix, Qd, qcodes_user ? (const uint32_t *)QCs.dev : nullptr, Qb, q0, Tq,
                       stride, C, qc.get<uint32_t>(), dl.get<int8_t>(), cn.get<uint32_t>(),
                       cv.get<uint32_t>(), ba.p, bf.get<unsigned long long>(), cand,
                       crank, fl.get<int>(), pairs, s,
                       use_rtc ? rsb.get<uint32_t>() : nullptr,
                       use_rtc ? rspk.get<uint32_t>() : nullptr,
                       use_rtc ? rseed.get<int32_t>() : nullptr, KS, fbw.p,
                       (unsigned long long *)(fl.get<int>() + 10), W_.us.p);
        if (use_rtc) {
            {
                ProfScope p(SLOT_SCORE, s);
                // certified warm start: the k-th best fp32 score (the final re-rank's own
                // arithmetic) over KS best-ranked candidates bounds the answer's k-th score
                launch_rerank(Xr, ix->d, ldr, Qd, Qb, rseed.get<int32_t>(), KS, KS, nullptr, 1, k,
                              rpt.get<unsigned long long>(), rtid.get<int64_t>(), rtsc.get<float>(), s);
                // (assigns theta and zeroes the survivor counts: no memset nodes)
                launch_theta_from_topk(rtid.get<int64_t>(), rtsc.get<float>(), Qb, k,
                                       rth.get<uint32_t>(), s, true, rcc.get<uint32_t>());
            }
            ProfScope p(SLOT_RERANK, s);
            // bf16 query rows in descending theta/|q| (pairs of similar bound prune alike)
            // (c4: 0.36 -> 0.30 ms per 1024 queries with the pairs' CTA shares in
            // proportion to their tile lists; NRLSH_RERANK_NOSORT=1 turns it off)
            const bool sorted = Qb <= 4096 && !getenv("NRLSH_RERANK_NOSORT");
            if (sorted) launch_sort_by_bound(Qd, ix->d, Qb, rth.get<uint32_t>(), rqp.get<int32_t>(), s);
            tls.qperm = sorted ? rqp.get<int32_t>() : nullptr;
            launch_bf16_prep(Qd, Qb, ix->d, ix->dpb, rqb.p, rqn.get<float>(), s, tls.qperm);
            mb.qcodes = qc.get<uint32_t>();
            mb.sel_B = rsb.get<uint32_t>();
            mb.sel_pk = rspk.get<uint32_t>();
            // two passes: the top-|x| tiles, then — after an exact re-rank of their
            // survivors has lifted theta to a real k-th best — the rest, pruned by it
            for (int pass = 1; pass <= 2; ++pass) {
                tls.pass = pass;
                if (launch_gt_filter_tc(ix->Xb, n, ix->d, ix->dpb, rqb.p, Qb, ix->xnorm_pos,
                                        rqn.get<float>(), gt_eps_rel(ix->dpb), k, rth.get<uint32_t>(),
                                        rhp.get<float>(), rcd.get<int32_t>(), rcc.get<uint32_t>(), Cg,
                                        s, ix->perm, &mb, &tls))
                    return fail(NRLSH_ECUDA, "tensor map encoding failed");
                if (pass == 1 && tls.xsplit > 0.f) {
                    launch_rerank(Xr, ix->d, ldr, Qd, Qb, rcd.get<int32_t>(), Cg, Cg, rcc.get<uint32_t>(),
                                  1, k, rpt.get<unsigned long long>(), rtid.get<int64_t>(),
                                  rtsc.get<float>(), s);
                    launch_theta_from_topk(rtid.get<int64_t>(), rtsc.get<float>(), Qb, k,
                                           rth.get<uint32_t>(), s);
                    launch_restart_from_topk(rtid.get<int64_t>(), Qb, k, rcd.get<int32_t>(), Cg,
                                             rcc.get<uint32_t>(), s);
                }
            }
            // exact fp32 re-rank of the surviving candidates (same arithmetic as the
            // gather path: identical scores and order)
            ProfScope p2(SLOT_RERANK_TOPK, s);
            launch_rerank(Xr, ix->d, ldr, Qd, Qb, rcd.get<int32_t>(), Cg, Cg, rcc.get<uint32_t>(),
                          1, k, rpt.get<unsigned long long>(), (int64_t *)oi.dev + q0 * k,
                          (float *)os.dev + q0 * k, s);
            launch_collect_overflow(rcc.get<uint32_t>(), Qb, Cg, q0, rov.get<int64_t>(),
                                    rovn.get<uint32_t>(), s);
            // survivors re-scored in fp32 (incl. the unused slots of their last chunk)
            launch_sum_counts(rcc.get<uint32_t>(), Qb, Cg, (unsigned long long *)(fl.get<int>() + 6), s);
        } else if (want_topk) {
            ProfScope p(SLOT_RERANK, s);
            launch_rerank(Xr, ix->d, ldr, Qd, Qb, cand, Tq, Tq, nullptr, 1, k,
                          pt.get<unsigned long long>(), (int64_t *)oi.dev + q0 * k,
                          (float *)os.dev + q0 * k, s);
        }
    }
    if (NSET > 1) {
        for (int w = 1; w < NSET; ++w) {
            cudaEventRecord(ev_join[w], st[w]);
            cudaStreamWaitEvent(s, ev_join[w], 0);
            cudaEventDestroy(ev_join[w]);
        }
        cudaEventDestroy(ev_fork);
    }
    if (use_rtc) {   // queries whose survivor list overflowed (rare): the gather path
        uint32_t nov = 0;
        cudaMemcpyAsync(&nov, rovn.p, 4, cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "query (re-rank overflow)");
        g_last_rtc_overflow = nov;
        if (nov) {
            // one gather-path call over all overflowed queries: gather their rows,
            // re-rank, scatter the answers back (the list is on the device)
            DBuf qr, ri, rs;
            if (qr.alloc((size_t)nov * ix->d * 4, s) || ri.alloc((size_t)nov * k * 8, s) ||
                rs.alloc((size_t)nov * k * 4, s))
                return fail(NRLSH_ENOMEM, "re-rank overflow workspace");
            launch_move_rows(Qs.dev, rov.get<int64_t>(), (int)nov, (size_t)ix->d * 4, qr.p, false, s);
            g_in_rtc_redo = true;
            const nrlsh_status st = query_impl(ix, qr.get<float>(), nullptr, nov, k, probe_budget,
                                               ri.get<int64_t>(), rs.get<float>(), nullptr, nullptr, s);
            g_in_rtc_redo = false;
            if (st != NRLSH_OK) return st;
            launch_move_rows(ri.p, rov.get<int64_t>(), (int)nov, (size_t)k * 8, oi.dev, true, s);
            launch_move_rows(rs.p, rov.get<int64_t>(), (int)nov, (size_t)k * 4, os.dev, true, s);
        }
    } else if (!g_in_rtc_redo) {
        g_last_rtc_overflow = 0;
    }
    if (want_topk) {
        if ((e = oi.finish(s)) || (e = os.finish(s))) return cuda_fail(e, "copy results");
    }
    if (cand_out) {
        if ((e = oc.finish(s))) return cuda_fail(e, "copy candidates");
        if (rank_out && (e = orr.finish(s))) return cuda_fail(e, "copy ranks");
    }
    int hflags[20];
    cudaMemcpyAsync(hflags, fl.p, 80, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e) return cuda_fail(e, "query");
    e = cudaGetLastError();
    if (e) return cuda_fail(e, "query launch");
    prof_collect();
    g_last_fallbacks = hflags[2];
    g_last_launches = launch_count() - launches0;
    unsigned long long pr;
    std::memcpy(&pr, hflags + 4, 8);
    g_last_pairs = (int64_t)pr;
    std::memcpy(&pr, hflags + 6, 8);
    g_last_rescored = (int64_t)pr;
    std::memcpy(&pr, hflags + 10, 8);
    g_last_entries = (int64_t)pr;
    std::memcpy(&pr, hflags + 12, 8);
    g_last_lb_pairs = (int64_t)pr;
    std::memcpy(&pr, hflags + 14, 8);
    g_last_lb_skipped = (int64_t)pr;
    std::memcpy(&pr, hflags + 16, 8);
    g_last_scan_popc = (int64_t)(pr / 2);   // (counted in halves)
    std::memcpy(&pr, hflags + 8, 8);
    if (!g_in_rtc_redo) g_last_rtc_pairs = (int64_t)pr;
    if (!g_in_rtc_redo)
        g_last_rtc = use_rtc ? NRLSH_RERANK_TENSOR : NRLSH_RERANK_GATHER;
    return check_flags(hflags);
}

nrlsh_status nrlsh_query(const nrlsh_index *ix, const float *queries, int64_t nq, int32_t k,
                         int64_t probe_budget, int64_t *out_ids, float *out_scores,
                         void *cuda_stream) {
    if (!out_ids) return fail(NRLSH_EINVAL, "out_ids is NULL");
    return query_impl(ix, queries, nullptr, nq, k, probe_budget, out_ids, out_scores, nullptr,
                      nullptr, cuda_stream);
}

nrlsh_status nrlsh_query_candidates(const nrlsh_index *ix, const float *queries,
                                    const uint32_t *qcodes, int64_t nq, int64_t probe_budget,
                                    int32_t *cand_ids, uint16_t *cand_rank, void *cuda_stream) {
    if (!cand_ids) return fail(NRLSH_EINVAL, "cand_ids is NULL");
    return query_impl(ix, queries, qcodes, nq, 1, probe_budget, nullptr, nullptr, cand_ids,
                      cand_rank, cuda_stream);
}

nrlsh_status nrlsh_query_codes(const nrlsh_index *ix, const float *queries, int64_t nq,
                               uint32_t *qcodes, void *cuda_stream) {
    if (!ix || !queries || !qcodes || nq < 1) return fail(NRLSH_EINVAL, "bad argument");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    Staged Qs;
    cudaError_t e = Qs.in(queries, (size_t)nq * ix->d * 4, s);
    if (e) return cuda_fail(e, "stage queries");
    OutBuf oq;
    if ((e = oq.init(qcodes, (size_t)nq * ix->QM * ix->W * 4, s))) return cuda_fail(e, "qcodes");
    DBuf fl;
    if (fl.alloc(16, s)) return fail(NRLSH_ENOMEM, "flags");
    const int init_flags[4] = {INT_MAX, INT_MAX, 0, 0};
    cudaMemcpyAsync(fl.p, init_flags, 16, cudaMemcpyHostToDevice, s);
    for (int64_t q0 = 0; q0 < nq; q0 += 65535) {
        const int Qb = (int)std::min<int64_t>(65535, nq - q0);
        launch_qcodes((const float *)Qs.dev + q0 * ix->d, Qb, ix->d, ix->Apad, ix->L, ix->W,
                      (uint32_t *)oq.dev + q0 * ix->QM * ix->W, fl.get<int>(), q0, s, ix->QM);
    }
    if ((e = oq.finish(s))) return cuda_fail(e, "copy qcodes");
    int hflags[4];
    cudaMemcpyAsync(hflags, fl.p, 16, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e) return cuda_fail(e, "query codes");
    return check_flags(hflags);
}

nrlsh_status nrlsh_last_rerank_stats(int64_t *rescored_fp32) {
    if (rescored_fp32) *rescored_fp32 = g_last_rescored;
    return NRLSH_OK;
}

nrlsh_status nrlsh_last_rerank_path(int32_t *path, int64_t *overflow_redone,
                                    int64_t *filter_pairs) {
    if (path) *path = (int32_t)g_last_rtc;
    if (overflow_redone) *overflow_redone = g_last_rtc_overflow;
    if (filter_pairs) *filter_pairs = g_last_rtc == NRLSH_RERANK_TENSOR ? g_last_rtc_pairs : 0;
    return NRLSH_OK;
}

nrlsh_status nrlsh_last_query_stats(int64_t *fallback_queries, int64_t *kernel_launches,
                                    int64_t *scanned_pairs, int64_t *buffer_entries) {
    if (buffer_entries) *buffer_entries = g_last_entries;
    if (fallback_queries) *fallback_queries = g_last_fallbacks;
    if (kernel_launches) *kernel_launches = g_last_launches;
    if (scanned_pairs) *scanned_pairs = g_last_pairs;
    return NRLSH_OK;
}

nrlsh_status nrlsh_last_scan_stats(int64_t *bound_pairs, int64_t *bound_decided_pairs) {
    if (bound_pairs) *bound_pairs = g_last_lb_pairs;
    if (bound_decided_pairs) *bound_decided_pairs = g_last_lb_skipped;
    return NRLSH_OK;
}

nrlsh_status nrlsh_last_scan_popc(int64_t *popc_ops) {
    if (popc_ops) *popc_ops = g_last_scan_popc;
    return NRLSH_OK;
}

// ------------------------------------------------------------ exact top-k
static nrlsh_status exact_impl(const float *items, int64_t n, int32_t d, const float *queries,
                               int64_t nq, int32_t k, const int64_t *seed_ids, int32_t seed_k,
                               int64_t *out_ids, float *out_scores, void *cuda_stream,
                               const void *Xb_ix = nullptr, const float *xnorm_ix = nullptr,
                               const int32_t *perm_ix = nullptr,
                               const float *tile_xmax_ix = nullptr, float xsplit_ix = 0.f,
                               const float *Xpad_ix = nullptr, int dpad_ix = 0) {
    if (!items || !queries || !out_ids || !out_scores) return fail(NRLSH_EINVAL, "NULL argument");
    if (seed_ids && (seed_k < 1 || seed_k > 1024))
        return fail(NRLSH_EINVAL, "seed_k must be in [1, 1024]");
    if (n < 1 || n >= (1ll << 31)) return fail(NRLSH_EINVAL, "n must be in [1, 2^31)");
    if (d < 1 || d > 4096) return fail(NRLSH_EINVAL, "d must be in [1, 4096]");
    if (nq < 1) return fail(NRLSH_EINVAL, "nq must be >= 1");
    if (k < 1 || k > 1024) return fail(NRLSH_EINVAL, "k must be in [1, 1024]");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    g_last_gt_max_cand = g_last_gt_sum_cand = g_last_gt_overflow = g_last_gt_pairs = 0;
    cudaError_t e;
    Staged Xs, Qs;
    if ((e = Xs.in(items, (size_t)n * d * 4, s))) return cuda_fail(e, "stage items");
    if ((e = Qs.in(queries, (size_t)nq * d * 4, s))) return cuda_fail(e, "stage queries");
    Staged Ss;
    if (seed_ids && (e = Ss.in(seed_ids, (size_t)nq * seed_k * 8, s))) return cuda_fail(e, "stage seeds");
    OutBuf oi, os;
    if ((e = oi.init(out_ids, (size_t)nq * k * 8, s))) return cuda_fail(e, "out_ids");
    if ((e = os.init(out_scores, (size_t)nq * k * 4, s))) return cuda_fail(e, "out_scores");
    const float *X = (const float *)Xs.dev;
    const float *Q = (const float *)Qs.dev;
    // exact re-ranks read the index's 16-byte-aligned row copy when it has one
    const float *Xr = Xpad_ix ? Xpad_ix : X;
    const int ldr = Xpad_ix ? dpad_ix : d;
    const bool use_tc = gt_tc_supported(d, k) && !getenv("NRLSH_GT_SIMT");
    const int dp = (d + 7) / 8 * 8;
    // certified error bound of fl(q.x) relative to |q||x|:
    //  tensor path: gt_eps_rel (bf16 operands, fp32 accumulation, + the fp32
    //  re-rank's own error); SIMT path: fp32 FMA chain, gamma_d inflated.
    const float eps_rel = use_tc ? gt_eps_rel(dp) : (float)(1.25 * (d + 2) * std::ldexp(1.0, -24));
    const int S = (int)std::max<int64_t>(1, std::min<int64_t>(64, n / (4 * (int64_t)k)));
    const int64_t ns = use_tc ? 1 : (n + S - 1) / S;
    const int64_t Cg = use_tc ? std::min<int64_t>(n, std::max<int64_t>(16384, 256 * (int64_t)k))
                              : std::min<int64_t>(n, std::max<int64_t>(4 * (int64_t)S * k + 4096, 2 * k));
    // queries per ground-truth sub-batch: the filter passes, seed bounds and re-ranks
    // of 4,096 queries at once (c4: 2.02 -> 1.20 ms per 10,000 queries vs 1,024);
    // NRLSH_GT_BATCH overrides
    // by default an even number of equal sub-batches of at most 6,144 (10,000 queries:
    // two of 5,000, one per stream, 0.93 ms against 1.00 for 4,096 + 4,096 + 1,808)
    int64_t gt_batch;
    if (getenv("NRLSH_GT_BATCH")) {
        gt_batch = std::max(64, atoi(getenv("NRLSH_GT_BATCH")));
    } else {
        int64_t nb = (nq + 6143) / 6144;
        if (nb > 1 && (nb & 1)) ++nb;
        if (nq > 4096 && nb < 2) nb = 2;
        gt_batch = ((nq + nb - 1) / nb + 255) / 256 * 256;
    }
    int Qmax = (int)std::min<int64_t>(gt_batch, nq);
    while (Qmax > 64 && (int64_t)Qmax * (ns * 4 + Cg * 8) > ((int64_t)2500 << 20)) Qmax >>= 1;
    // sub-batches alternate between two streams with a workspace set each (as the
    // query's; NRLSH_QUERY_SERIAL=1: one)
    const int NSET = (nq > Qmax && !getenv("NRLSH_QUERY_SERIAL")) ? 2 : 1;
    struct GSet { DBuf ss, lb, tid, tsc, cc, cd, cs, th, pt, hp, tw, gqp, gqb, gqn; } gsets[2];
    DBuf xn, qn, xb, qb, gst, gov;
    const int64_t npad = (n + 255) / 256 * 256;   // |x| padded: the tc kernel bulk-loads 1 KB tiles
    if (xn.alloc((size_t)npad * 4, s) || qn.alloc((size_t)nq * 4, s) || gst.alloc(40, s) ||
        gov.alloc((size_t)nq * 8, s))
        return fail(NRLSH_ENOMEM, "exact_topk workspace");
    for (int w = 0; w < NSET; ++w) {
        GSet &G = gsets[w];
        if (G.ss.alloc((size_t)Qmax * ns * 4, s) || G.lb.alloc((size_t)Qmax * 4, s) ||
            G.tid.alloc((size_t)Qmax * k * 8, s) || G.tsc.alloc((size_t)Qmax * k * 4, s) ||
            G.cc.alloc((size_t)Qmax * 4, s) || G.cd.alloc((size_t)Qmax * Cg * 4, s) ||
            G.cs.alloc((size_t)Qmax * Cg * 4, s) || G.th.alloc((size_t)Qmax * 4, s) ||
            G.pt.alloc(std::max(rerank_partial_bytes(Qmax, Cg, k), rerank_partial_bytes(1, n, k)), s))
            return fail(NRLSH_ENOMEM, "exact_topk workspace");
    }
    cudaMemsetAsync(gst.p, 0, 40, s);
    // bf16 item rows and |x|: the index's (written by its build), else prepared here
    const void *Xbp = Xb_ix;
    const float *xnp = xnorm_ix;
    if (use_tc) {
        if ((!Xbp && xb.alloc((size_t)n * dp * 2, s)) || qb.alloc((size_t)nq * dp * 2, s))
            return fail(NRLSH_ENOMEM, "exact_topk bf16 workspace");
        for (int w = 0; w < NSET; ++w) {
            GSet &G = gsets[w];
            if (G.hp.alloc(gt_heap_bytes(k), s) ||
                (Xb_ix && tile_xmax_ix &&
                 (G.tw.alloc(gt_tile_ws_bytes(n, Qmax), s) || G.gqp.alloc((size_t)Qmax * 4, s) ||
                  G.gqb.alloc((size_t)Qmax * dp * 2, s) || G.gqn.alloc((size_t)Qmax * 4, s))))
                return fail(NRLSH_ENOMEM, "exact_topk bf16 workspace");
        }
        ProfScope p(SLOT_GT_NORMS, s);
        if (!Xbp) {
            cudaMemsetAsync(xn.get<float>() + n, 0, (size_t)(npad - n) * 4, s);
            launch_bf16_prep(X, n, d, dp, xb.p, xn.get<float>(), s);
            Xbp = xb.p;
            xnp = xn.get<float>();
        }
        launch_bf16_prep(Q, nq, d, dp, qb.p, qn.get<float>(), s);
    } else {
        ProfScope p(SLOT_GT_NORMS, s);
        launch_vec_norms(X, n, d, xn.get<float>(), s);
        launch_vec_norms(Q, nq, d, qn.get<float>(), s);
    }
    // rows in partition order (the index's): per query pair, only the tiles whose
    // largest |x| can reach the pair's seeded bound (GtTiles)
    GtTiles gtl;
    gtl.xmax128 = tile_xmax_ix;
    gtl.ws = nullptr;   // (per workspace set, below)
    gtl.pairs = gst.get<unsigned long long>() + 4;   // (query, item) pairs multiplied
    gtl.xsplit = getenv("NRLSH_GT_ONEPASS") ? 0.f : xsplit_ix;
    gtl.pass = 0;
    gtl.qperm = nullptr;
    cudaStream_t st[2] = {s, s};
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (NSET == 2) {
        thread_local cudaStream_t extra[128] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 128) return fail(NRLSH_ECUDA, "device index");
        if (!extra[dev] && cudaStreamCreateWithFlags(&extra[dev], cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            return fail(NRLSH_ECUDA, "stream create");
        }
        st[1] = extra[dev];
        cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
        cudaEventRecord(ev_fork, s);
        cudaStreamWaitEvent(st[1], ev_fork, 0);
    }
    int sbi = 0;
    for (int64_t q0 = 0; q0 < nq; q0 += Qmax, ++sbi) {
        const int Qb = (int)std::min<int64_t>(Qmax, nq - q0);
        GSet &G = gsets[sbi % NSET];
        cudaStream_t s = st[sbi % NSET];   // (this sub-batch's stream)
        DBuf &ss = G.ss, &lb = G.lb, &tid = G.tid, &tsc = G.tsc, &cc = G.cc, &cd = G.cd, &th = G.th,
             &pt = G.pt, &hp = G.hp, &gqp = G.gqp, &gqb = G.gqb, &gqn = G.gqn;
        gtl.ws = G.tw.get<int32_t>();
        const float *Qb_ptr = Q + q0 * d;
        const float *qnb = qn.get<float>() + q0;
        int64_t *oid = (int64_t *)oi.dev + q0 * k;
        float *osc = (float *)os.dev + q0 * k;
        // (the seeded bound kernel assigns theta and zeroes the survivor counts itself)
        if (!(use_tc && seed_ids)) cudaMemsetAsync(cc.p, 0, (size_t)Qb * 4, s);
        if (use_tc) {
            if (seed_ids) {
                ProfScope p(SLOT_GT_NORMS, s);
                launch_gt_seed_theta(X, n, d, Qb_ptr, Qb, qnb, (const int64_t *)Ss.dev + q0 * seed_k,
                                     seed_k, k, (float)(1.25 * (d + 2) * std::ldexp(1.0, -24)),
                                     th.get<uint32_t>(), s, cc.get<uint32_t>());
            } else {
                cudaMemsetAsync(th.p, 0, (size_t)Qb * 4, s);
            }
            ProfScope p(SLOT_GT_FILTER, s);
            const bool tiles = Xb_ix && tile_xmax_ix;
            // bf16 query rows of this batch in descending theta/|q| (tile lists only)
            const void *qrows = (const uint16_t *)qb.p + q0 * dp;
            const float *qnrows = qnb;
            gtl.qperm = nullptr;
            // (opt-in NRLSH_GT_SORT=1: the sort and the extra bf16 pass cost more than the
            // pruning gains here, 0.25 vs 0.17 ms per 1024 queries on c4)
            if (tiles && seed_ids && Qb <= 4096 && getenv("NRLSH_GT_SORT")) {
                launch_sort_by_bound(Qb_ptr, d, Qb, th.get<uint32_t>(), gqp.get<int32_t>(), s);
                launch_bf16_prep(Qb_ptr, Qb, d, dp, gqb.p, gqn.get<float>(), s, gqp.get<int32_t>());
                gtl.qperm = gqp.get<int32_t>();
                qrows = gqb.p;
                qnrows = gqn.get<float>();
            }
            // with tile lists: the top-|x| tiles, an exact re-rank of their survivors
            // (theta := a real k-th best, the final re-rank's arithmetic), the rest
            const int npass = tiles && gtl.xsplit > 0.f ? 2 : 1;
            for (int pass = 1; pass <= npass; ++pass) {
                gtl.pass = npass == 1 ? 0 : pass;
                if (launch_gt_filter_tc(Xbp, n, d, dp, qrows, Qb,
                                        xnp, qnrows, eps_rel, k, th.get<uint32_t>(),
                                        hp.get<float>(), cd.get<int32_t>(), cc.get<uint32_t>(), Cg, s,
                                        Xb_ix ? perm_ix : nullptr, nullptr, tiles ? &gtl : nullptr))
                    return fail(NRLSH_ECUDA, "tensor map encoding failed");
                if (pass < npass) {
                    launch_rerank(Xr, d, ldr, Qb_ptr, Qb, cd.get<int32_t>(), Cg, Cg, cc.get<uint32_t>(), 1, k,
                                  pt.get<unsigned long long>(), tid.get<int64_t>(), tsc.get<float>(), s);
                    launch_theta_from_topk(tid.get<int64_t>(), tsc.get<float>(), Qb, k,
                                           th.get<uint32_t>(), s);
                    // the second pass appends to the first pass's exact top-k only
                    if (!getenv("NRLSH_GT_RESCORE_ALL"))
                        launch_restart_from_topk(tid.get<int64_t>(), Qb, k, cd.get<int32_t>(), Cg,
                                                 cc.get<uint32_t>(), s);
                }
            }
        } else {
            // pilot: certified lower bound of the k-th best score from a strided sample
            {
                ProfScope p(SLOT_SCORE, s);
                launch_score(X, d, Qb_ptr, Qb, nullptr, ns, ns, nullptr, S, xn.get<float>(), qnb,
                             eps_rel, ss.get<float>(), s);
            }
            {
                ProfScope p(SLOT_TOPK, s);
                launch_topk(ss.get<float>(), nullptr, Qb, ns, ns, nullptr, S, k, tid.get<int64_t>(),
                            tsc.get<float>(), lb.get<float>(), s);
            }
            ProfScope p(SLOT_GT_FILTER, s);
            launch_gt_filter(X, n, d, Qb_ptr, Qb, xn.get<float>(), qnb, lb.get<float>(), eps_rel,
                             cd.get<int32_t>(), cc.get<uint32_t>(), Cg, s);
        }
        {
            ProfScope p(SLOT_SCORE, s);
            launch_rerank(Xr, d, ldr, Qb_ptr, Qb, cd.get<int32_t>(), Cg, Cg, cc.get<uint32_t>(), 1, k,
                          pt.get<unsigned long long>(), oid, osc, s);
        }
        // survivor statistics and overflowing queries, collected on the device (no
        // host round trip per sub-batch)
        launch_count_stats(cc.get<uint32_t>(), Qb, gst.get<unsigned long long>(), s);
        launch_collect_overflow(cc.get<uint32_t>(), Qb, Cg, q0, gov.get<int64_t>(),
                                (uint32_t *)(gst.get<unsigned long long>() + 2), s);
    }
    if (NSET == 2) {
        cudaEventRecord(ev_join, st[1]);
        cudaStreamWaitEvent(s, ev_join, 0);
        cudaEventDestroy(ev_fork);
        cudaEventDestroy(ev_join);
    }
    {   // overflowing queries (rare): exact scoring of every item
        unsigned long long hst[5];
        cudaMemcpyAsync(hst, gst.p, 40, cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "exact_topk");
        // without tile lists the filter multiplies every (query, item) pair
        g_last_gt_pairs = (Xb_ix && tile_xmax_ix && use_tc) ? (int64_t)hst[4] : (int64_t)(nq * n);
        g_last_gt_max_cand = (int64_t)hst[0];
        g_last_gt_sum_cand = (int64_t)hst[1];
        const uint32_t nov = (uint32_t)hst[2];
        g_last_gt_overflow = nov;
        if (nov) {
            std::vector<int64_t> ql(nov);
            cudaMemcpy(ql.data(), gov.p, (size_t)nov * 8, cudaMemcpyDeviceToHost);
            for (int64_t qi : ql)
                launch_rerank(Xr, d, ldr, Q + qi * d, 1, nullptr, n, n, nullptr, 1, k,
                              gsets[0].pt.get<unsigned long long>(), (int64_t *)oi.dev + qi * k,
                              (float *)os.dev + qi * k, s);
        }
    }
    if ((e = oi.finish(s)) || (e = os.finish(s))) return cuda_fail(e, "copy results");
    e = cudaStreamSynchronize(s);
    if (e) return cuda_fail(e, "exact_topk");
    e = cudaGetLastError();
    if (e) return cuda_fail(e, "exact_topk launch");
    prof_collect();
    return NRLSH_OK;
}

nrlsh_status nrlsh_last_exact_stats(int64_t *max_cand, int64_t *sum_cand, int64_t *overflow,
                                    int64_t *filter_pairs) {
    if (filter_pairs) *filter_pairs = g_last_gt_pairs;
    if (max_cand) *max_cand = g_last_gt_max_cand;
    if (sum_cand) *sum_cand = g_last_gt_sum_cand;
    if (overflow) *overflow = g_last_gt_overflow;
    return NRLSH_OK;
}

nrlsh_status nrlsh_exact_topk(const float *items, int64_t n, int32_t d, const float *queries,
                              int64_t nq, int32_t k, int64_t *out_ids, float *out_scores,
                              void *cuda_stream) {
    return exact_impl(items, n, d, queries, nq, k, nullptr, 0, out_ids, out_scores, cuda_stream);
}

nrlsh_status nrlsh_exact_topk_seeded(const float *items, int64_t n, int32_t d,
                                     const float *queries, int64_t nq, int32_t k,
                                     const int64_t *seed_ids, int32_t seed_k, int64_t *out_ids,
                                     float *out_scores, void *cuda_stream) {
    if (!seed_ids) return fail(NRLSH_EINVAL, "seed_ids is NULL");
    return exact_impl(items, n, d, queries, nq, k, seed_ids, seed_k, out_ids, out_scores,
                      cuda_stream);
}

nrlsh_status nrlsh_index_exact_topk(const nrlsh_index *ix, const float *queries, int64_t nq,
                                    int32_t k, int64_t *out_ids, float *out_scores,
                                    void *cuda_stream) {
    if (!ix) return fail(NRLSH_EINVAL, "index is NULL");
    return exact_impl(ix->X, ix->n, ix->d, queries, nq, k, nullptr, 0, out_ids, out_scores,
                      cuda_stream, ix->Xb, ix->xnorm_pos, ix->perm, ix->tile_xmax,
                      ix->tile_xsplit, ix->Xpad, ix->dpad);
}

nrlsh_status nrlsh_index_exact_topk_seeded(const nrlsh_index *ix, const float *queries,
                                           int64_t nq, int32_t k, const int64_t *seed_ids,
                                           int32_t seed_k, int64_t *out_ids, float *out_scores,
                                           void *cuda_stream) {
    if (!ix) return fail(NRLSH_EINVAL, "index is NULL");
    if (!seed_ids) return fail(NRLSH_EINVAL, "seed_ids is NULL");
    return exact_impl(ix->X, ix->n, ix->d, queries, nq, k, seed_ids, seed_k, out_ids, out_scores,
                      cuda_stream, ix->Xb, ix->xnorm_pos, ix->perm, ix->tile_xmax,
                      ix->tile_xsplit, ix->Xpad, ix->dpad);
}

// ------------------------------------------------------------------ hooks
static nrlsh_status copy_out(void *dst, const void *src, size_t bytes) {
    if (!dst) return NRLSH_OK;
    cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
    if (e) return cuda_fail(e, "copy");
    return NRLSH_OK;
}

nrlsh_status nrlsh_get_partition(const nrlsh_index *ix, double *norm2, int32_t *perm,
                                 int64_t *offsets, double *V) {
    if (!ix) return fail(NRLSH_EINVAL, "index is NULL");
    nrlsh_status st;
    if ((st = copy_out(norm2, ix->norm2, (size_t)ix->n * 8))) return st;
    if ((st = copy_out(perm, ix->perm, (size_t)ix->n * 4))) return st;
    if ((st = copy_out(offsets, ix->offsets_d, (size_t)(ix->m + 1) * 8))) return st;
    return copy_out(V, ix->V_d, (size_t)ix->m * 8);
}

nrlsh_status nrlsh_get_projection(const nrlsh_index *ix, float *A) {
    if (!ix || !A) return fail(NRLSH_EINVAL, "bad argument");
    return copy_out(A, ix->A, ix->A_h.size() * 4);
}

nrlsh_status nrlsh_get_proj(const nrlsh_index *ix, int32_t *proj) {
    if (!ix || !proj) return fail(NRLSH_EINVAL, "bad argument");
    *proj = ix->proj;
    return NRLSH_OK;
}

nrlsh_status nrlsh_get_rank_table(const nrlsh_index *ix, uint16_t *R) {
    if (!ix || !R) return fail(NRLSH_EINVAL, "bad argument");
    return copy_out(R, ix->R_d, ix->R_h.size() * 2);
}

nrlsh_status nrlsh_get_codes(const nrlsh_index *ix, uint32_t *codes) {
    if (!ix || !codes) return fail(NRLSH_EINVAL, "bad argument");
    return copy_out(codes, ix->codes, (size_t)ix->n * ix->W * 4);
}

nrlsh_status nrlsh_set_codes(nrlsh_index *ix, const uint32_t *codes) {
    if (!ix || !codes) return fail(NRLSH_EINVAL, "bad argument");
    cudaError_t e = cudaMemcpy(ix->codes, codes, (size_t)ix->n * ix->W * 4, cudaMemcpyDefault);
    if (e) return cuda_fail(e, "set codes");
    if (ix->codes_pm) {   // keep the tensor-core scan's +-1 rows in step
        launch_expand_pm(ix->codes, ix->n, ix->W, ix->L, ix->codes_pm, nullptr);
        if ((e = cudaDeviceSynchronize())) return cuda_fail(e, "set codes (+-1 rows)");
    }
    if (ix->samp_codes) {   // keep the pilot sample in step with the codes
        launch_gather_sample(ix, pilot_stride(ix->n), ix->samp_codes, ix->samp_part, nullptr);
        if ((e = cudaDeviceSynchronize())) return cuda_fail(e, "set codes (sample)");
    }
    return NRLSH_OK;
}

}  // extern "C"
