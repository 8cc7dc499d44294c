// api.cpp -- host side of libslora: the C ABI of include/slora.h.
//
//   * Unified Paging pool bookkeeping: LIFO free stack, owner
//     table, KV handles, adapter handles, pin/evict, fragmentation report.
//   * adapter loader: pack this rank's TP shard into pinned staging,
//     H2D on the caller's stream, scatter kernel into pages.
//   * batch descriptor builder: group tokens by adapter, pack
//     (segment x projection) work into balanced units, upload.
//   * launchers of the sm_100a kernels (kernels.cu).
// Bookkeeping errors are detected before any CUDA work is enqueued and leave
// the pool unchanged.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/slora.h"
#include "slora_internal.h"

namespace slora {
int64_t launch_count();
}
using namespace slora;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static slora_status fail(slora_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}
static slora_status ok() {
    g_err.clear();
    return SLORA_OK;
}
#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return fail(SLORA_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                        __LINE__);                                                             \
    } while (0)

extern "C" const char* slora_status_string(slora_status s) {
    switch (s) {
        case SLORA_OK: return "SLORA_OK";
        case SLORA_ERR_INVALID_ARG: return "SLORA_ERR_INVALID_ARG";
        case SLORA_ERR_SHAPE: return "SLORA_ERR_SHAPE";
        case SLORA_ERR_OUT_OF_PAGES: return "SLORA_ERR_OUT_OF_PAGES";
        case SLORA_ERR_ALREADY_RESIDENT: return "SLORA_ERR_ALREADY_RESIDENT";
        case SLORA_ERR_NOT_RESIDENT: return "SLORA_ERR_NOT_RESIDENT";
        case SLORA_ERR_PINNED: return "SLORA_ERR_PINNED";
        case SLORA_ERR_NOT_PINNED: return "SLORA_ERR_NOT_PINNED";
        case SLORA_ERR_STALE_HANDLE: return "SLORA_ERR_STALE_HANDLE";
        case SLORA_ERR_FREE_PAGE_READ: return "SLORA_ERR_FREE_PAGE_READ";
        case SLORA_ERR_NONRESIDENT_ADAPTER: return "SLORA_ERR_NONRESIDENT_ADAPTER";
        case SLORA_ERR_SEGMENT_OVERLAP: return "SLORA_ERR_SEGMENT_OVERLAP";
        case SLORA_ERR_TOKEN_COUNT_NOT_ONE: return "SLORA_ERR_TOKEN_COUNT_NOT_ONE";
        case SLORA_ERR_INDIVISIBLE: return "SLORA_ERR_INDIVISIBLE";
        case SLORA_ERR_CUDA: return "SLORA_ERR_CUDA";
        case SLORA_ERR_NO_DEVICE: return "SLORA_ERR_NO_DEVICE";
    }
    return "SLORA_ERR_UNKNOWN";
}
extern "C" const char* slora_last_error(void) { return g_err.c_str(); }
extern "C" int64_t slora_launch_count(void) { return slora::launch_count(); }

// -------------------------------------------------------------------- pool
namespace {
constexpr int kNumProj = 4;
constexpr size_t kStageBytes = size_t(32) << 20;   // per staging buffer
constexpr size_t kJobBytes = size_t(64) << 10;     // job table at the head

enum Owner : uint8_t { kFree = 0, kKv = 1, kAdapter = 2 };

struct Adapter {
    int64_t id = 0;
    int32_t rank = 0, slot = -1;
    float scale = 1.f;
    bool pinned = false;
    std::vector<int32_t> pages;  // claim order: layer, proj, tensor, row, chunk
    int32_t* dev_tab = nullptr;
};

struct Kv {
    int32_t seq_len = 0;
    std::vector<std::vector<int32_t>> pages;  // [layer * 2 + kind]
};

uint64_t splitmix64(uint64_t& st) {
    st += 0x9E3779B97F4A7C15ull;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int esize_of(slora_dtype d) { return d == SLORA_F32 ? 4 : 2; }

// Kernel configuration for one (mode, K, D).  C = the smallest split (cluster
// size) whose per-CTA slices are whole 16-byte vectors and at most 4 KB (one
// warp's worth of 16-byte vectors per slice row x 8 warps), so the producer
// streams the largest slices and the most SMs stay usable (small clusters
// pack GPCs best).  SLORA_SPLIT overrides.  ns = ring slots filling smem.
KernelCfg make_kernel_cfg(int mode, int64_t K, int64_t D, int64_t P, int es, int dtype) {

    KernelCfg k;
    k.mode = mode;
    k.K = K;
    k.D = D;
    static int forced = [] {
        const char* s = getenv("SLORA_SPLIT");
        return s ? atoi(s) : 0;
    }();
    auto valid = [&](int C) {
        if (mode != kExpand && (K % C || ((K / C) * es) % 16 || (K / C) * es > 4096)) return false;
        if (mode != kExpand)
            for (int c = 0; c < C; ++c) {  // pages one CTA's K slice spans
                const int64_t k0 = c * (K / C), k1 = k0 + K / C - 1;
                if (k1 / P - k0 / P + 1 > kMaxChunks) return false;
            }
        if (mode != kShrink && (D % C || ((D / C) * es) % 16 || (D / C) * es > 4096)) return false;
        return true;
    };
    // prefer the largest split whose slices stay >= 2 KB: bulk copies of 2 KB
    // and up stream at full HBM rate (measured), and more CTAs per unit
    // spread few units over more SMs
    auto big = [&](int C) {
        return (mode == kExpand || (K / C) * es >= 2048) && (mode == kShrink || (D / C) * es >= 2048);
    };
    int C = 0;
    if (forced > 0 && forced <= 16 && valid(forced)) C = forced;
    for (int c = 16; c >= 1 && !C; --c)
        if (valid(c) && big(c)) C = c;
    for (int c = 1; c <= 16 && !C; ++c)
        if (valid(c)) C = c;
    if (!C) return k;
    k.C = C;
    const size_t budget = size_t(227) * 1024;
    const size_t base = lora_smem_bytes(mode, C, K, D, 0, es);
    const size_t per_slot = lora_smem_bytes(mode, C, K, D, 1, es) - base;
    int ns = int((budget - base) / per_slot);
    ns = std::min(ns, kMaxSlots);
    if (ns < 2) return k;
    k.ns = ns;
    k.smem = lora_smem_bytes(mode, C, K, D, ns, es);
    k.n_clusters = lora_max_clusters(mode, dtype, C, k.smem);
    k.ok = k.n_clusters > 0;
    return k;
}
}  // namespace

struct slora_pool {
    slora_pool_config cfg{};
    int64_t P = 0;          // page elements
    int es = 2;
    bool dev = false;
    std::vector<int32_t> free_stack;  // top = back
    std::vector<uint8_t> owner;
    std::unordered_map<int64_t, Adapter> adapters;
    std::vector<int64_t> slots;       // adapter id or -1
    std::unordered_map<int64_t, Kv> kv;
    int64_t kv_pages = 0, adapter_pages = 0;
    uint64_t epoch = 0;               // bumped by every eviction
    // device resources
    int32_t** slot_tab_dev = nullptr;
    void* stage_host[2] = {nullptr, nullptr};
    void* stage_dev[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    bool stage_used[2] = {false, false};
    cudaEvent_t release_ev = nullptr;
    bool release_pending = false;
    // kernel configurations: 0 fused (K=D=H), 1 shrink q/k/v (K=H),
    // 2 shrink o (K=H/N), 3 expand (D=H/N)
    KernelCfg kcfg[4];
    long long* trace_dev = nullptr;   // SLORA_TRACE=1: kernel event timestamps

    int64_t free_pages() const { return int64_t(free_stack.size()); }
    int N() const { return cfg.tp_size; }
    // (stored rows, chunks per row) of one tensor shard (reading R3/R4)
    void tensor_shape(int proj, int tensor, int rank, int& rows, int& chunks) const {
        if (proj < 3 && tensor == 0) {
            rows = rank / N();
            chunks = N();
        } else {
            rows = rank;
            chunks = 1;
        }
    }
    int64_t adapter_page_count(int rank) const { return int64_t(cfg.num_layers) * kNumProj * 2 * rank; }
};

struct slora_batch {
    slora_pool* pool = nullptr;
    bool prepared = false;
    uint64_t epoch = 0;
    int32_t T = 0, adapted = 0;
    int64_t NR = 0;
    int64_t weight_bytes_per_proj = 0;
    std::vector<DevSeg> segs;
    std::vector<const int32_t*> seg_tab;  // device page table of each segment's adapter
    std::vector<int32_t> tok_idx;
    std::vector<DevUnit> units[5];
    std::vector<DevItem> items[5];
    // LPT schedules: [kernel cfg][nproj] -> per-cluster unit lists
    std::vector<int32_t> sched_off[4][5], sched[4][5];
    // device descriptor blob
    size_t off_segs = 0, off_tok = 0, off_units[5] = {}, off_items[5] = {};
    size_t off_sched_off[4][5] = {}, off_sched[4][5] = {};
    size_t blob_cap = 0;
    void* blob_host = nullptr;
    void* blob_dev = nullptr;
    cudaEvent_t upload_ev = nullptr;
    bool upload_pending = false;
};

static slora_status check_pool(slora_pool_t p) {
    if (!p) return fail(SLORA_ERR_INVALID_ARG, "null pool");
    return SLORA_OK;
}

extern "C" slora_status slora_pool_create(const slora_pool_config* cfg, slora_pool_t* out) {
    if (!cfg || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    if (cfg->dtype != SLORA_F32 && cfg->dtype != SLORA_F16 && cfg->dtype != SLORA_BF16)
        return fail(SLORA_ERR_INVALID_ARG, "dtype");
    if (cfg->hidden < 1 || cfg->num_layers < 1 || cfg->capacity_pages < 1 || cfg->max_adapters < 1 ||
        cfg->tp_size < 1 || cfg->tp_rank < 0 || cfg->tp_rank >= cfg->tp_size)
        return fail(SLORA_ERR_INVALID_ARG, "sizes must be >= 1 and 0 <= tp_rank < tp_size");
    if (cfg->capacity_pages > INT32_MAX) return fail(SLORA_ERR_INVALID_ARG, "capacity_pages > 2^31-1");
    if (cfg->hidden % cfg->tp_size) return fail(SLORA_ERR_INDIVISIBLE, "hidden %% tp_size != 0");
    if (cfg->alloc_order != SLORA_ORDER_ASCENDING && cfg->alloc_order != SLORA_ORDER_SHUFFLE)
        return fail(SLORA_ERR_INVALID_ARG, "alloc_order");
    const int es = esize_of(cfg->dtype);
    const int64_t P = cfg->hidden / cfg->tp_size;
    if (cfg->device >= 0) {
        if (!cfg->device_buffer) return fail(SLORA_ERR_INVALID_ARG, "device pool needs device_buffer");
        if (cfg->device_buffer_bytes < cfg->capacity_pages * P * es)
            return fail(SLORA_ERR_INVALID_ARG, "device_buffer_bytes %lld < capacity*page bytes %lld",
                        (long long)cfg->device_buffer_bytes, (long long)(cfg->capacity_pages * P * es));
        if ((reinterpret_cast<uintptr_t>(cfg->device_buffer) & 15) || (P * es) % 16)
            return fail(SLORA_ERR_SHAPE, "device_buffer and page bytes must be 16-byte aligned");
    } else if (cfg->device_buffer) {
        return fail(SLORA_ERR_INVALID_ARG, "bookkeeping-only pool takes no device_buffer");
    }
    slora_pool* p = new slora_pool();
    p->cfg = *cfg;
    p->P = P;
    p->es = es;
    p->dev = cfg->device >= 0;
    const int64_t cap = cfg->capacity_pages;
    p->free_stack.resize(size_t(cap));
    for (int64_t i = 0; i < cap; ++i) p->free_stack[size_t(i)] = int32_t(cap - 1 - i);
    if (cfg->alloc_order == SLORA_ORDER_SHUFFLE) {
        uint64_t st = cfg->seed;
        for (int64_t i = cap - 1; i >= 1; --i) {
            uint64_t j = splitmix64(st) % uint64_t(i + 1);
            std::swap(p->free_stack[size_t(i)], p->free_stack[size_t(j)]);
        }
    }
    p->owner.assign(size_t(cap), kFree);
    p->slots.assign(size_t(cfg->max_adapters), -1);
    if (p->dev) {
        auto cleanup = [&](cudaError_t e, const char* what) {
            slora_status s = fail(SLORA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
            delete p;
            return s;
        };
        cudaError_t e;
        if ((e = cudaSetDevice(cfg->device))) return cleanup(e, "cudaSetDevice");
        if ((e = configure_lora_kernels(cfg->device))) return cleanup(e, "configure kernels");
        if ((e = cudaMalloc(&p->slot_tab_dev, sizeof(int32_t*) * size_t(cfg->max_adapters))))
            return cleanup(e, "cudaMalloc slot table");
        if ((e = cudaMemset(p->slot_tab_dev, 0, sizeof(int32_t*) * size_t(cfg->max_adapters))))
            return cleanup(e, "cudaMemset");
        for (int b = 0; b < 2; ++b) {
            if ((e = cudaHostAlloc(&p->stage_host[b], kStageBytes, cudaHostAllocDefault)))
                return cleanup(e, "cudaHostAlloc staging");
            if ((e = cudaMalloc(&p->stage_dev[b], kStageBytes))) return cleanup(e, "cudaMalloc staging");
            if ((e = cudaEventCreateWithFlags(&p->stage_ev[b], cudaEventDisableTiming)))
                return cleanup(e, "cudaEventCreate");
        }
        if ((e = cudaEventCreateWithFlags(&p->release_ev, cudaEventDisableTiming)))
            return cleanup(e, "cudaEventCreate");
        const int dt = cfg->dtype == SLORA_F32 ? kF32 : (cfg->dtype == SLORA_F16 ? kF16 : kBF16);
        const int64_t H = cfg->hidden;
        p->kcfg[0] = make_kernel_cfg(kFused, H, H, P, es, dt);
        p->kcfg[1] = make_kernel_cfg(kShrink, H, P, P, es, dt);
        p->kcfg[2] = make_kernel_cfg(kShrink, cfg->tp_size > 1 ? P : H, P, P, es, dt);
        p->kcfg[3] = make_kernel_cfg(kExpand, P, P, P, es, dt);
        const char* tr = getenv("SLORA_TRACE");
        if (tr && atoi(tr) == 1) {
            if ((e = cudaMalloc(&p->trace_dev, 4096 * sizeof(long long)))) return cleanup(e, "cudaMalloc trace");
            cudaMemset(p->trace_dev, 0, 4096 * sizeof(long long));
        }
        if (cfg->tp_size == 1 && !p->kcfg[0].ok) {
            slora_status s = fail(SLORA_ERR_SHAPE, "no valid MBGMV split for hidden %lld", (long long)H);
            delete p;
            return s;
        }
    }
    *out = p;
    return ok();
}

extern "C" slora_status slora_pool_destroy(slora_pool_t p) {
    if (!p) return fail(SLORA_ERR_INVALID_ARG, "null pool");
    if (p->dev) {
        cudaSetDevice(p->cfg.device);
        cudaDeviceSynchronize();
        for (auto& kvp : p->adapters)
            if (kvp.second.dev_tab) cudaFree(kvp.second.dev_tab);
        cudaFree(p->slot_tab_dev);
        for (int b = 0; b < 2; ++b) {
            cudaFreeHost(p->stage_host[b]);
            cudaFree(p->stage_dev[b]);
            cudaEventDestroy(p->stage_ev[b]);
        }
        cudaEventDestroy(p->release_ev);
    }
    delete p;
    return ok();
}

extern "C" slora_status slora_fragmentation_report(slora_pool_t p, slora_frag_report* out) {
    if (check_pool(p) || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    int64_t best = 0, run = 0;
    for (uint8_t o : p->owner) {
        if (o == kFree) {
            best = std::max(best, ++run);
        } else {
            run = 0;
        }
    }
    out->capacity_pages = p->cfg.capacity_pages;
    out->free_pages = p->free_pages();
    out->used_pages = p->cfg.capacity_pages - p->free_pages();
    out->largest_free_run = best;
    out->kv_pages = p->kv_pages;
    out->adapter_pages = p->adapter_pages;
    out->page_elems = p->P;
    out->resident_adapters = int32_t(p->adapters.size());
    return ok();
}

static void record_release(slora_pool* p, void* stream) {
    if (!p->dev) return;
    cudaEventRecord(p->release_ev, static_cast<cudaStream_t>(stream));
    p->release_pending = true;
}

// ---------------------------------------------------------------------- KV
static void kv_grow(slora_pool* p, int64_t rid, Kv& kv, int32_t n, int32_t* pages_out) {
    int64_t o = 0;
    for (int l = 0; l < p->cfg.num_layers; ++l)
        for (int kind = 0; kind < 2; ++kind)
            for (int32_t pos = 0; pos < n; ++pos) {
                int32_t pg = p->free_stack.back();
                p->free_stack.pop_back();
                p->owner[size_t(pg)] = kKv;
                kv.pages[size_t(l * 2 + kind)].push_back(pg);
                if (pages_out) pages_out[o++] = pg;
            }
    (void)rid;
    kv.seq_len += n;
    p->kv_pages += int64_t(2) * n * p->cfg.num_layers;
}

extern "C" slora_status slora_kv_alloc(slora_pool_t p, int64_t rid, int32_t n, int32_t* pages_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    if (n < 0) return fail(SLORA_ERR_INVALID_ARG, "n_tokens < 0");
    if (p->kv.count(rid)) return fail(SLORA_ERR_INVALID_ARG, "request %lld already live", (long long)rid);
    const int64_t need = int64_t(2) * n * p->cfg.num_layers;
    if (need > p->free_pages())
        return fail(SLORA_ERR_OUT_OF_PAGES, "needed=%lld free=%lld", (long long)need, (long long)p->free_pages());
    Kv kv;
    kv.pages.resize(size_t(2 * p->cfg.num_layers));
    kv_grow(p, rid, kv, n, pages_out);
    p->kv.emplace(rid, std::move(kv));
    return ok();
}

extern "C" slora_status slora_kv_append(slora_pool_t p, int64_t rid, int32_t n, int32_t* pages_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->kv.find(rid);
    if (it == p->kv.end()) return fail(SLORA_ERR_STALE_HANDLE, "request %lld not live", (long long)rid);
    if (n < 0) return fail(SLORA_ERR_INVALID_ARG, "n_tokens < 0");
    const int64_t need = int64_t(2) * n * p->cfg.num_layers;
    if (need > p->free_pages())
        return fail(SLORA_ERR_OUT_OF_PAGES, "needed=%lld free=%lld", (long long)need, (long long)p->free_pages());
    kv_grow(p, rid, it->second, n, pages_out);
    return ok();
}

extern "C" slora_status slora_kv_free(slora_pool_t p, int64_t rid, void* stream, int64_t* released_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->kv.find(rid);
    if (it == p->kv.end()) return fail(SLORA_ERR_STALE_HANDLE, "request %lld not live", (long long)rid);
    int64_t n = 0;
    for (auto& lst : it->second.pages)
        for (int32_t pg : lst) {
            p->owner[size_t(pg)] = kFree;
            p->free_stack.push_back(pg);
            ++n;
        }
    p->kv_pages -= n;
    p->kv.erase(it);
    record_release(p, stream);
    if (released_out) *released_out = n;
    return ok();
}

extern "C" slora_status slora_kv_pages(slora_pool_t p, int64_t rid, int32_t layer, int32_t kind, int32_t* out,
                                       int64_t cap, int64_t* n_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->kv.find(rid);
    if (it == p->kv.end()) return fail(SLORA_ERR_STALE_HANDLE, "request %lld not live", (long long)rid);
    if (layer < 0 || layer >= p->cfg.num_layers || kind < 0 || kind > 1)
        return fail(SLORA_ERR_INVALID_ARG, "layer/kind");
    const auto& lst = it->second.pages[size_t(layer * 2 + kind)];
    if (n_out) *n_out = int64_t(lst.size());
    if (out)
        for (int64_t i = 0; i < std::min<int64_t>(cap, int64_t(lst.size())); ++i) out[i] = lst[size_t(i)];
    return ok();
}

// ---------------------------------------------------------------- adapters
// Pack one tensor shard (dense, row-major) of this TP rank into dst.
//   A (h x r, canonical) -> q/k/v: all h rows, columns [k*r/N, (k+1)*r/N)
//                           o    : rows [k*P, (k+1)*P), all r columns
//   B (r x d, canonical) -> all r rows, columns [k*P, (k+1)*P)
static void pack_shard(const slora_pool* p, const uint8_t* A, const uint8_t* B, int proj, int tensor, int r,
                       uint8_t* dst, int& rows_out, int& cols_out) {
    const int64_t H = p->cfg.hidden, P = p->P;
    const int N = p->N(), k = p->cfg.tp_rank, es = p->es;
    if (tensor == 0) {
        if (proj < 3) {
            const int rc = r / N;
            for (int64_t row = 0; row < H; ++row)
                memcpy(dst + size_t(row * rc) * es, A + size_t(row * r + int64_t(k) * rc) * es, size_t(rc) * es);
            rows_out = int(H);
            cols_out = rc;
        } else {
            memcpy(dst, A + size_t(int64_t(k) * P * r) * es, size_t(P * r) * es);
            rows_out = int(P);
            cols_out = r;
        }
    } else {
        for (int j = 0; j < r; ++j)
            memcpy(dst + size_t(int64_t(j) * P) * es, B + size_t(int64_t(j) * H + int64_t(k) * P) * es,
                   size_t(P) * es);
        rows_out = r;
        cols_out = int(P);
    }
}

extern "C" slora_status slora_adapter_load(slora_pool_t p, int64_t id, int32_t rank, const void* host_w,
                                           float scale, void* stream, int32_t* slot_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    if (rank < 1) return fail(SLORA_ERR_INVALID_ARG, "rank < 1");
    if (rank > kRowCap) return fail(SLORA_ERR_SHAPE, "rank %d > %d (max rank of the MBGMV path)", rank, kRowCap);
    if (rank % p->N()) return fail(SLORA_ERR_INDIVISIBLE, "rank %d %% tp_size %d", rank, p->N());
    if (p->dev && !host_w) return fail(SLORA_ERR_INVALID_ARG, "host_w is NULL");
    if (!p->dev && host_w) return fail(SLORA_ERR_NO_DEVICE, "bookkeeping-only pool takes host_w = NULL");
    if (p->adapters.count(id)) return fail(SLORA_ERR_ALREADY_RESIDENT, "adapter %lld", (long long)id);
    auto sit = std::find(p->slots.begin(), p->slots.end(), int64_t(-1));
    if (sit == p->slots.end()) return fail(SLORA_ERR_OUT_OF_PAGES, "no free adapter slot");
    const int64_t need = p->adapter_page_count(rank);
    if (need > p->free_pages())
        return fail(SLORA_ERR_OUT_OF_PAGES, "needed=%lld free=%lld", (long long)need, (long long)p->free_pages());
    const int64_t H = p->cfg.hidden;
    const int es = p->es;
    const size_t tensor_max_bytes = size_t(std::max<int64_t>(H * rank, int64_t(rank) * p->P)) * es;
    if (p->dev && tensor_max_bytes + kJobBytes > kStageBytes)
        return fail(SLORA_ERR_SHAPE, "adapter tensor of %zu bytes exceeds staging", tensor_max_bytes);

    Adapter ad;
    ad.id = id;
    ad.rank = rank;
    ad.slot = int32_t(sit - p->slots.begin());
    ad.scale = scale;
    ad.pages.reserve(size_t(need));
    for (int64_t i = 0; i < need; ++i) {  // claim order: layer, proj, tensor, row, chunk
        int32_t pg = p->free_stack.back();
        p->free_stack.pop_back();
        p->owner[size_t(pg)] = kAdapter;
        ad.pages.push_back(pg);
    }
    auto rollback = [&]() {
        for (auto it = ad.pages.rbegin(); it != ad.pages.rend(); ++it) {
            p->owner[size_t(*it)] = kFree;
            p->free_stack.push_back(*it);
        }
    };

    if (p->dev) {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        cudaError_t e = cudaSetDevice(p->cfg.device);
        if (!e && p->release_pending) e = cudaStreamWaitEvent(s, p->release_ev, 0);
        if (!e) e = cudaMallocAsync(reinterpret_cast<void**>(&ad.dev_tab), sizeof(int32_t) * size_t(need), s);
        if (!e) e = cudaMemcpyAsync(ad.dev_tab, ad.pages.data(), sizeof(int32_t) * size_t(need),
                                    cudaMemcpyHostToDevice, s);
        if (!e) e = cudaMemcpyAsync(p->slot_tab_dev + ad.slot, &ad.dev_tab, sizeof(int32_t*),
                                    cudaMemcpyHostToDevice, s);
        // stream the tensors through the two staging buffers
        const uint8_t* W = static_cast<const uint8_t*>(host_w);
        const int64_t per_lp = (H * rank + int64_t(rank) * H);  // elements of A+B per (layer, proj)
        int buf = 0;
        size_t used = kJobBytes;
        std::vector<ScatterJob> jobs;
        auto flush = [&]() -> cudaError_t {
            if (jobs.empty()) return cudaSuccess;
            memcpy(p->stage_host[buf], jobs.data(), jobs.size() * sizeof(ScatterJob));
            cudaError_t e2 = cudaMemcpyAsync(p->stage_dev[buf], p->stage_host[buf], used, cudaMemcpyHostToDevice, s);
            if (!e2) e2 = launch_scatter(static_cast<uint8_t*>(p->stage_dev[buf]) + kJobBytes,
                                         static_cast<const ScatterJob*>(p->stage_dev[buf]), int(jobs.size()),
                                         p->cfg.device_buffer, p->P, es, s);
            if (!e2) e2 = cudaEventRecord(p->stage_ev[buf], s);
            p->stage_used[buf] = true;
            buf ^= 1;
            used = kJobBytes;
            jobs.clear();
            return e2;
        };
        int64_t page_cursor = 0;
        for (int l = 0; l < p->cfg.num_layers && !e; ++l)
            for (int pr = 0; pr < kNumProj && !e; ++pr) {
                const uint8_t* A = W + size_t((int64_t(l) * kNumProj + pr) * per_lp) * es;
                const uint8_t* B = A + size_t(H * rank) * es;
                for (int t = 0; t < 2 && !e; ++t) {
                    int rows_s, chunks;
                    p->tensor_shape(pr, t, rank, rows_s, chunks);
                    const size_t bytes = size_t(rows_s) * chunks * size_t(p->P) * es;
                    if (used + bytes > kStageBytes || (jobs.size() + 1) * sizeof(ScatterJob) > kJobBytes) {
                        e = flush();
                        if (e) break;
                    }
                    if (jobs.empty() && p->stage_used[buf]) {
                        e = cudaEventSynchronize(p->stage_ev[buf]);  // staging buffer free again
                        if (e) break;
                    }
                    int rows, cols;
                    pack_shard(p, A, B, pr, t, rank, static_cast<uint8_t*>(p->stage_host[buf]) + used, rows, cols);
                    ScatterJob jb;
                    jb.src_off = int64_t((used - kJobBytes) / size_t(es));
                    jb.pages = ad.dev_tab + page_cursor;
                    jb.kind = t;
                    jb.rows = rows;
                    jb.cols = cols;
                    jb.row_pages = (t == 0) ? chunks : 1;
                    jobs.push_back(jb);
                    used += bytes;
                    page_cursor += int64_t(rows_s) * chunks;
                }
            }
        if (!e) e = flush();
        if (e) {
            rollback();
            return fail(SLORA_ERR_CUDA, "adapter load: %s", cudaGetErrorString(e));
        }
    }
    p->adapter_pages += need;
    p->slots[size_t(ad.slot)] = id;
    if (slot_out) *slot_out = ad.slot;
    p->adapters.emplace(id, std::move(ad));
    return ok();
}

extern "C" slora_status slora_adapter_evict(slora_pool_t p, int64_t id, void* stream, int64_t* released_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->adapters.find(id);
    if (it == p->adapters.end()) return fail(SLORA_ERR_NOT_RESIDENT, "adapter %lld", (long long)id);
    if (it->second.pinned) return fail(SLORA_ERR_PINNED, "adapter %lld", (long long)id);
    Adapter& ad = it->second;
    for (int32_t pg : ad.pages) {
        p->owner[size_t(pg)] = kFree;
        p->free_stack.push_back(pg);
    }
    p->adapter_pages -= int64_t(ad.pages.size());
    p->slots[size_t(ad.slot)] = -1;
    if (released_out) *released_out = int64_t(ad.pages.size());
    if (p->dev && ad.dev_tab) cudaFreeAsync(ad.dev_tab, static_cast<cudaStream_t>(stream));
    record_release(p, stream);
    p->adapters.erase(it);
    ++p->epoch;
    return ok();
}

extern "C" slora_status slora_adapter_pin(slora_pool_t p, int64_t id) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->adapters.find(id);
    if (it == p->adapters.end()) return fail(SLORA_ERR_NOT_RESIDENT, "adapter %lld", (long long)id);
    it->second.pinned = true;
    return ok();
}

extern "C" slora_status slora_adapter_unpin(slora_pool_t p, int64_t id) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->adapters.find(id);
    if (it == p->adapters.end()) return fail(SLORA_ERR_NOT_RESIDENT, "adapter %lld", (long long)id);
    if (!it->second.pinned) return fail(SLORA_ERR_NOT_PINNED, "adapter %lld", (long long)id);
    it->second.pinned = false;
    return ok();
}

extern "C" slora_status slora_adapter_pages(slora_pool_t p, int64_t id, int32_t* out, int64_t cap,
                                            int64_t* n_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->adapters.find(id);
    if (it == p->adapters.end()) return fail(SLORA_ERR_NOT_RESIDENT, "adapter %lld", (long long)id);
    const auto& v = it->second.pages;
    if (n_out) *n_out = int64_t(v.size());
    if (out)
        for (int64_t i = 0; i < std::min<int64_t>(cap, int64_t(v.size())); ++i) out[i] = v[size_t(i)];
    return ok();
}

extern "C" slora_status slora_gather_pages(slora_pool_t p, const int32_t* pages, int32_t n, void* dst,
                                           void* stream) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    if (n < 0 || (n > 0 && !pages)) return fail(SLORA_ERR_INVALID_ARG, "pages");
    for (int32_t i = 0; i < n; ++i) {
        if (pages[i] < 0 || pages[i] >= p->cfg.capacity_pages)
            return fail(SLORA_ERR_INVALID_ARG, "page %d out of range", pages[i]);
        if (p->owner[size_t(pages[i])] == kFree) return fail(SLORA_ERR_FREE_PAGE_READ, "page %d is free", pages[i]);
    }
    if (!p->dev) return fail(SLORA_ERR_NO_DEVICE, "bookkeeping-only pool");
    if (n == 0) return ok();
    if (!dst) return fail(SLORA_ERR_INVALID_ARG, "dst");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t* d_pages = nullptr;
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_pages), sizeof(int32_t) * size_t(n), s));
    CUDA_TRY(cudaMemcpyAsync(d_pages, pages, sizeof(int32_t) * size_t(n), cudaMemcpyHostToDevice, s));
    CUDA_TRY(launch_gather(p->cfg.device_buffer, d_pages, n, dst, p->P, p->es, s));
    CUDA_TRY(cudaFreeAsync(d_pages, s));
    return ok();
}

// ------------------------------------------------------------------- batch
namespace {
// Items = (segment x projection x token chunk); units = items packed by
// first-fit decreasing on rank under the kernel's caps (kRowCap rows,
// kTokCap token slots, kVCap v entries, kMaxItemsPerUnit items): an r = 64
// item fills a unit alone, eight r = 8 items share one -- rank-heterogeneous
// balancing without padding to a maximum rank.
void build_units(slora_batch* b, int nproj) {
    auto& units = b->units[nproj];
    auto& items = b->items[nproj];
    units.clear();
    items.clear();
    struct It { DevItem it; int rank; };
    std::vector<It> all;
    for (int si = 0; si < int(b->segs.size()); ++si) {
        const DevSeg& s = b->segs[size_t(si)];
        // at most kItemTokCap tokens per item: a Zipf-head adapter with many
        // decode tokens is split into several items (its pages are re-read,
        // but the FMA work spreads over clusters instead of one straggler)
        const int tmax = std::max(1, std::min(std::min(kTokCap, kItemTokCap), kVCap / s.rank));
        for (int pi = 0; pi < nproj; ++pi)
            for (int t0 = 0; t0 < s.n_tok; t0 += tmax) {
                DevItem it{};
                it.tab = b->seg_tab.empty() ? nullptr : b->seg_tab[size_t(si)];
                it.vrow = s.vrow_off + int64_t(t0) * s.rank;
                it.rank = s.rank;
                it.seg = si;
                it.pi = pi;
                it.t0 = t0;
                it.nt = std::min(tmax, s.n_tok - t0);
                it.tok_off = s.tok_off + t0;
                it.scale = s.scale;
                all.push_back({it, s.rank});
            }
    }
    std::stable_sort(all.begin(), all.end(), [](const It& a, const It& c) { return a.rank > c.rank; });
    struct Bin { std::vector<DevItem> its; int rows = 0, toks = 0, v = 0; };
    std::vector<Bin> bins;
    for (const It& x : all) {
        const int r = x.rank, nt = x.it.nt;
        Bin* target = nullptr;
        for (Bin& bn : bins)
            if (bn.rows + r <= kRowCap && bn.toks + nt <= kTokCap && bn.v + nt * r <= kVCap &&
                int(bn.its.size()) < kMaxItemsPerUnit) {
                target = &bn;
                break;
            }
        if (!target) {
            bins.emplace_back();
            target = &bins.back();
        }
        DevItem it = x.it;
        it.row_off = target->rows;
        it.tok_slot = target->toks;
        it.v_off = target->v;
        target->rows += r;
        target->toks += nt;
        target->v += nt * r;
        target->its.push_back(it);
    }
    for (Bin& bn : bins) {
        DevUnit u{};
        u.item_begin = int32_t(items.size());
        u.n_items = int32_t(bn.its.size());
        u.rows = bn.rows;
        u.toks = bn.toks;
        u.ventries = bn.v;
        for (auto& it : bn.its) items.push_back(it);
        units.push_back(u);
    }
}

// LPT static schedule of units over the kernel's persistent clusters: units
// by decreasing cost, each to the least-loaded cluster.  Cost = bytes one
// cluster CTA streams for the unit + a fixed per-unit overhead.
void build_schedule(slora_batch* b, const KernelCfg& k, int es, int nproj, std::vector<int32_t>& off,
                    std::vector<int32_t>& sched) {
    off.clear();
    sched.clear();
    const auto& units = b->units[nproj];
    if (!k.ok || units.empty()) {
        off.assign(1, 0);
        return;
    }
    const int G = std::max(1, std::min<int>(k.n_clusters, int(units.size())));
    const double KSb = k.mode == kExpand ? 0.0 : double(k.K / k.C) * es;
    const double DSb = k.mode == kShrink ? 0.0 : double(k.D / k.C) * es;
    std::vector<std::pair<double, int>> cost;
    for (int u = 0; u < int(units.size()); ++u) {
        const DevUnit& U = units[size_t(u)];
        cost.push_back({U.rows * (KSb + DSb) + U.toks * KSb + 8192.0, u});
    }
    std::stable_sort(cost.begin(), cost.end(), [](auto& a, auto& c) { return a.first > c.first; });
    std::vector<double> load(size_t(G), 0.0);
    std::vector<std::vector<int32_t>> lists(static_cast<size_t>(G));
    for (auto& cu : cost) {
        size_t g = size_t(std::min_element(load.begin(), load.end()) - load.begin());
        load[g] += cu.first;
        lists[g].push_back(cu.second);
    }
    off.push_back(0);
    for (auto& l : lists) {
        for (int32_t u : l) sched.push_back(u);
        off.push_back(int32_t(sched.size()));
    }
}
}  // namespace

extern "C" slora_status slora_batch_create(slora_pool_t p, slora_batch_t* out) {
    if (check_pool(p) || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    slora_batch* b = new slora_batch();
    b->pool = p;
    if (p->dev) {
        cudaError_t e = cudaEventCreateWithFlags(&b->upload_ev, cudaEventDisableTiming);
        if (e) {
            delete b;
            return fail(SLORA_ERR_CUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
        }
    }
    *out = b;
    return ok();
}

extern "C" slora_status slora_batch_destroy(slora_batch_t b) {
    if (!b) return fail(SLORA_ERR_INVALID_ARG, "null batch");
    if (b->pool->dev) {
        if (b->upload_pending) cudaEventSynchronize(b->upload_ev);
        if (b->blob_dev) cudaFree(b->blob_dev);
        if (b->blob_host) cudaFreeHost(b->blob_host);
        cudaEventDestroy(b->upload_ev);
    }
    delete b;
    return ok();
}

extern "C" slora_status slora_batch_prepare(slora_batch_t b, const int64_t* tok_adapter, int32_t T, void* stream) {
    if (!b) return fail(SLORA_ERR_INVALID_ARG, "null batch");
    if (T < 0 || (T > 0 && !tok_adapter)) return fail(SLORA_ERR_INVALID_ARG, "token map");
    slora_pool* p = b->pool;
    for (int32_t i = 0; i < T; ++i)
        if (tok_adapter[i] != -1 && !p->adapters.count(tok_adapter[i]))
            return fail(SLORA_ERR_NONRESIDENT_ADAPTER, "token %d: adapter %lld not resident", i,
                        (long long)tok_adapter[i]);
    // group tokens by adapter, segments in order of first appearance
    std::unordered_map<int64_t, int> seg_of;
    std::vector<std::vector<int32_t>> toks;
    std::vector<int64_t> seg_ad;
    for (int32_t i = 0; i < T; ++i) {
        const int64_t a = tok_adapter[i];
        if (a == -1) continue;
        auto it = seg_of.find(a);
        int s;
        if (it == seg_of.end()) {
            s = int(toks.size());
            seg_of.emplace(a, s);
            toks.emplace_back();
            seg_ad.push_back(a);
        } else {
            s = it->second;
        }
        toks[size_t(s)].push_back(i);
    }
    b->segs.clear();
    b->seg_tab.clear();
    b->tok_idx.clear();
    b->T = T;
    b->adapted = 0;
    b->NR = 0;
    b->weight_bytes_per_proj = 0;
    for (size_t s = 0; s < toks.size(); ++s) {
        const Adapter& ad = p->adapters.at(seg_ad[s]);
        DevSeg sg{};
        sg.slot = ad.slot;
        sg.rank = ad.rank;
        sg.n_tok = int32_t(toks[s].size());
        sg.tok_off = int32_t(b->tok_idx.size());
        sg.vrow_off = b->NR;
        sg.scale = ad.scale;
        b->NR += int64_t(sg.n_tok) * ad.rank;
        b->adapted += sg.n_tok;
        b->weight_bytes_per_proj += int64_t(ad.rank) * 2 * p->P * p->es;
        for (int32_t t : toks[s]) b->tok_idx.push_back(t);
        b->segs.push_back(sg);
        b->seg_tab.push_back(ad.dev_tab);
    }
    for (int np = 1; np <= 4; ++np) build_units(b, np);
    for (int kc = 0; kc < 4; ++kc)
        for (int np = 1; np <= 4; ++np) build_schedule(b, p->kcfg[kc], p->es, np, b->sched_off[kc][np], b->sched[kc][np]);
    b->epoch = p->epoch;
    b->prepared = true;
    if (!p->dev) return ok();

    // ---- upload: [segs][tok_idx][units/items per nproj][schedules per cfg x nproj]
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t off = 0;
    b->off_segs = off;
    off = al(off + b->segs.size() * sizeof(DevSeg));
    b->off_tok = off;
    off = al(off + b->tok_idx.size() * sizeof(int32_t));
    for (int np = 1; np <= 4; ++np) {
        b->off_units[np] = off;
        off = al(off + b->units[np].size() * sizeof(DevUnit));
        b->off_items[np] = off;
        off = al(off + b->items[np].size() * sizeof(DevItem));
    }
    for (int kc = 0; kc < 4; ++kc)
        for (int np = 1; np <= 4; ++np) {
            b->off_sched_off[kc][np] = off;
            off = al(off + b->sched_off[kc][np].size() * sizeof(int32_t));
            b->off_sched[kc][np] = off;
            off = al(off + b->sched[kc][np].size() * sizeof(int32_t));
        }
    const size_t need = std::max<size_t>(off, 256);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    if (b->upload_pending) CUDA_TRY(cudaEventSynchronize(b->upload_ev));  // pinned blob free again
    if (need > b->blob_cap) {
        if (b->blob_host) CUDA_TRY(cudaFreeHost(b->blob_host));
        if (b->blob_dev) CUDA_TRY(cudaFreeAsync(b->blob_dev, s));
        b->blob_host = nullptr;
        b->blob_dev = nullptr;
        const size_t cap = need * 2;
        CUDA_TRY(cudaHostAlloc(&b->blob_host, cap, cudaHostAllocDefault));
        CUDA_TRY(cudaMallocAsync(&b->blob_dev, cap, s));
        b->blob_cap = cap;
    }
    uint8_t* h = static_cast<uint8_t*>(b->blob_host);
    auto put = [&](size_t o, const void* src, size_t n) {
        if (n) memcpy(h + o, src, n);
    };
    put(b->off_segs, b->segs.data(), b->segs.size() * sizeof(DevSeg));
    put(b->off_tok, b->tok_idx.data(), b->tok_idx.size() * sizeof(int32_t));
    for (int np = 1; np <= 4; ++np) {
        put(b->off_units[np], b->units[np].data(), b->units[np].size() * sizeof(DevUnit));
        put(b->off_items[np], b->items[np].data(), b->items[np].size() * sizeof(DevItem));
    }
    for (int kc = 0; kc < 4; ++kc)
        for (int np = 1; np <= 4; ++np) {
            put(b->off_sched_off[kc][np], b->sched_off[kc][np].data(), b->sched_off[kc][np].size() * sizeof(int32_t));
            put(b->off_sched[kc][np], b->sched[kc][np].data(), b->sched[kc][np].size() * sizeof(int32_t));
        }
    CUDA_TRY(cudaMemcpyAsync(b->blob_dev, b->blob_host, need, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaEventRecord(b->upload_ev, s));
    b->upload_pending = true;
    return ok();
}

extern "C" slora_status slora_batch_get_info(slora_batch_t b, slora_batch_info* out) {
    if (!b || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    out->T = b->T;
    out->adapted_tokens = b->adapted;
    out->segments = int32_t(b->segs.size());
    out->sum_rank_tokens = b->NR;
    out->weight_bytes_per_proj = b->weight_bytes_per_proj;
    out->mbgmm_segments = 0;
    return ok();
}

// ----------------------------------------------------------------- compute
namespace {
slora_status common_checks(slora_pool* p, slora_batch* b, int32_t layer, uint32_t mask) {
    if (!p || !b) return fail(SLORA_ERR_INVALID_ARG, "null pool/batch");
    if (b->pool != p) return fail(SLORA_ERR_INVALID_ARG, "batch belongs to another pool");
    if (!p->dev) return fail(SLORA_ERR_NO_DEVICE, "bookkeeping-only pool");
    if (!b->prepared) return fail(SLORA_ERR_INVALID_ARG, "batch not prepared");
    if (b->epoch != p->epoch) return fail(SLORA_ERR_STALE_HANDLE, "batch prepared before an eviction");
    if (layer < 0 || layer >= p->cfg.num_layers) return fail(SLORA_ERR_INVALID_ARG, "layer %d", layer);
    if (mask == 0 || mask > 0xF) return fail(SLORA_ERR_INVALID_ARG, "proj_mask 0x%x", mask);
    return SLORA_OK;
}

bool aligned16(const void* ptr, int64_t ld, int es) {
    return !(reinterpret_cast<uintptr_t>(ptr) & 15) && (ld * es) % 16 == 0;
}

void fill_common(slora_pool* p, slora_batch* b, int kc, int32_t layer, uint32_t mask, LoraParams& q) {
    memset(&q, 0, sizeof(q));
    const KernelCfg& k = p->kcfg[kc];
    q.pool = p->cfg.device_buffer;
    q.page_elems = p->P;
    q.slot_tab = p->slot_tab_dev;
    uint8_t* base = static_cast<uint8_t*>(b->blob_dev);
    q.segs = reinterpret_cast<const DevSeg*>(base + b->off_segs);
    q.tok_idx = reinterpret_cast<const int32_t*>(base + b->off_tok);
    int np = 0;
    for (int pj = 0; pj < 4; ++pj)
        if (mask & (1u << pj)) q.proj_ids[np++] = pj;
    q.nproj = np;
    q.units = reinterpret_cast<const DevUnit*>(base + b->off_units[np]);
    q.items = reinterpret_cast<const DevItem*>(base + b->off_items[np]);
    q.sched_off = reinterpret_cast<const int32_t*>(base + b->off_sched_off[kc][np]);
    q.sched = reinterpret_cast<const int32_t*>(base + b->off_sched[kc][np]);
    q.n_clusters = int32_t(b->sched_off[kc][np].size()) - 1;
    q.layer = layer;
    q.C = k.C;
    q.K = int32_t(k.K);
    q.D = int32_t(k.D);
    q.ns = k.ns;
    static const int l2pf = [] {
        const char* s = getenv("SLORA_L2PF");
        return s ? atoi(s) : 0;
    }();
    q.l2_prefetch = l2pf;
    static const int dbg = [] {
        const char* s = getenv("SLORA_DBG");
        return s ? atoi(s) : 0;
    }();
    q.dbg = dbg;
    q.NR = b->NR;
    const int N = p->N();
    for (int pj = 0; pj < 4; ++pj) {
        q.a_div[pj] = (pj < 3) ? N : 1;
        q.a_row_pages[pj] = (pj < 3) ? N : 1;
    }
}

slora_status launch(slora_pool* p, int kc, LoraParams& q, void* stream) {
    const KernelCfg& k = p->kcfg[kc];
    if (!k.ok) return fail(SLORA_ERR_SHAPE, "no valid kernel configuration for K=%lld D=%lld", (long long)k.K,
                           (long long)k.D);
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    const int dt = p->cfg.dtype == SLORA_F32 ? kF32 : (p->cfg.dtype == SLORA_F16 ? kF16 : kBF16);
    q.trace = p->trace_dev;
    CUDA_TRY(launch_lora(q, k.mode, dt, static_cast<cudaStream_t>(stream), k.smem));
    return ok();
}
}  // namespace

extern "C" slora_status slora_lora_apply(slora_pool_t p, slora_batch_t b, int32_t layer, uint32_t mask,
                                         const void* x, int64_t ldx, void* const y[4], const int64_t ldy[4],
                                         void* stream) {
    slora_status st = common_checks(p, b, layer, mask);
    if (st) return st;
    if (p->N() != 1) return fail(SLORA_ERR_INVALID_ARG, "slora_lora_apply is single-GPU; use shrink/expand under TP");
    if (b->adapted == 0) return ok();
    if (!x || !y || !ldy) return fail(SLORA_ERR_INVALID_ARG, "null x/y");
    if (!aligned16(x, ldx, p->es) || ldx < p->cfg.hidden) return fail(SLORA_ERR_SHAPE, "x alignment/stride");
    for (int pj = 0; pj < 4; ++pj)
        if (mask & (1u << pj))
            if (!y[pj] || !aligned16(y[pj], ldy[pj], p->es) || ldy[pj] < p->cfg.hidden)
                return fail(SLORA_ERR_SHAPE, "y[%d] alignment/stride", pj);
    LoraParams q;
    fill_common(p, b, 0, layer, mask, q);
    q.x = x;
    q.ldx = ldx;
    for (int pj = 0; pj < 4; ++pj) {
        q.y[pj] = y[pj];
        q.ldy[pj] = ldy[pj];
    }
    q.v_blocks = 1;
    return launch(p, 0, q, stream);
}

extern "C" slora_status slora_lora_v_elems(slora_batch_t b, uint32_t mask, int32_t div, int64_t* out) {
    if (!b || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    if (mask == 0 || mask > 0xF || div < 1) return fail(SLORA_ERR_INVALID_ARG, "mask/div");
    int np = 0;
    for (int pj = 0; pj < 4; ++pj) np += (mask >> pj) & 1;
    if (b->NR % div) return fail(SLORA_ERR_INDIVISIBLE, "NR %% div");
    *out = int64_t(np) * (b->NR / div);
    return ok();
}

extern "C" slora_status slora_lora_shrink(slora_pool_t p, slora_batch_t b, int32_t layer, uint32_t mask,
                                          const void* x, int64_t ldx, float* v, void* stream) {
    slora_status st = common_checks(p, b, layer, mask);
    if (st) return st;
    const int N = p->N();
    if (N > 1 && (mask & 0x8) && (mask & 0x7))
        return fail(SLORA_ERR_INVALID_ARG, "under TP shrink q/k/v and o in separate calls");
    if (b->adapted == 0) return ok();
    const int kc = (N > 1 && (mask & 0x8)) ? 2 : 1;
    const int64_t K = p->kcfg[kc].K;
    if (!x || !v) return fail(SLORA_ERR_INVALID_ARG, "null x/v");
    if (!aligned16(x, ldx, p->es) || ldx < K) return fail(SLORA_ERR_SHAPE, "x alignment/stride");
    LoraParams q;
    fill_common(p, b, kc, layer, mask, q);
    q.x = x;
    q.ldx = ldx;
    q.v_out = v;
    return launch(p, kc, q, stream);
}

extern "C" slora_status slora_lora_expand(slora_pool_t p, slora_batch_t b, int32_t layer, uint32_t mask,
                                          const float* v, int32_t v_blocks, void* const y[4], const int64_t ldy[4],
                                          void* stream) {
    slora_status st = common_checks(p, b, layer, mask);
    if (st) return st;
    if (v_blocks < 1) return fail(SLORA_ERR_INVALID_ARG, "v_blocks");
    if (b->adapted == 0) return ok();
    for (const DevSeg& s : b->segs)
        if (s.rank % v_blocks) return fail(SLORA_ERR_INDIVISIBLE, "rank %d %% v_blocks %d", s.rank, v_blocks);
    if (!v || !y || !ldy) return fail(SLORA_ERR_INVALID_ARG, "null v/y");
    for (int pj = 0; pj < 4; ++pj)
        if (mask & (1u << pj))
            if (!y[pj] || !aligned16(y[pj], ldy[pj], p->es) || ldy[pj] < p->P)
                return fail(SLORA_ERR_SHAPE, "y[%d] alignment/stride", pj);
    LoraParams q;
    fill_common(p, b, 3, layer, mask, q);
    q.v_in = v;
    q.v_blocks = v_blocks;
    for (int pj = 0; pj < 4; ++pj) {
        q.y[pj] = y[pj];
        q.ldy[pj] = ldy[pj];
    }
    return launch(p, 3, q, stream);
}

extern "C" slora_status slora_sync(slora_pool_t p, void* stream) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    if (!p->dev) return ok();
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    CUDA_TRY(cudaGetLastError());
    return ok();
}

extern "C" slora_status slora_debug_trace(slora_pool_t p, int64_t* out, int32_t n) {
    if (check_pool(p) || !out || n < 0) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    if (!p->trace_dev) return fail(SLORA_ERR_INVALID_ARG, "tracing is off (set SLORA_TRACE=1 before pool create)");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(out, p->trace_dev, sizeof(int64_t) * size_t(std::min(n, 4096)), cudaMemcpyDeviceToHost));
    return ok();
}
