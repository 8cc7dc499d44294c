// api.cpp -- host side of libslora: the C ABI of include/slora.h.
//
//   * Unified Paging pool bookkeeping: LIFO free stack, owner
//     table, KV handles, adapter handles, pin/evict, fragmentation report.
//   * adapter loader: a loader thread per pool packs this
//     rank's TP shard into a ring of pinned staging chunks (or reads a pinned
//     host_w directly) and streams it H2D || scatter kernel into pages on the
//     pool's copy stream, overlapping the caller's kernels (slora_adapter_prefetch).
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
#include <chrono>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/slora.h"
#include "slora_internal.h"

#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is loaded at run time (dlopen), see slora_tp_init

#include <cudaTypedefs.h>

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
        case SLORA_ERR_NCCL: return "SLORA_ERR_NCCL";
    }
    return "SLORA_ERR_UNKNOWN";
}
extern "C" const char* slora_last_error(void) { return g_err.c_str(); }
extern "C" int64_t slora_launch_count(void) { return slora::launch_count(); }

// -------------------------------------------------------------------- NCCL
// NCCL is loaded on first use with dlopen("libnccl.so.2"): in a process that
// already loaded torch's NCCL this returns that same library (one NCCL per
// process), and the C ABI works without NCCL for single-GPU use.
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    if (api.tried) return api;
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = dlerror() ? dlerror() : "dlopen libnccl.so.2 failed";
        return api;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.AllReduce &&
             api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    return api;
}
}  // namespace

// -------------------------------------------------------------------- pool
namespace {
constexpr int kNumProj = 4;       // the default projections q, k, v, o
constexpr int kMaxKc = 8;         // kernel configurations: 0-3 below, 4+ fused for other input widths
constexpr int kNpSlots = kMaxProj + 1;  // calls / headers per configuration, by projection count
constexpr size_t kStageBytes = size_t(16) << 20;   // per loader staging chunk (pinned host + device)
constexpr size_t kJobBytes = size_t(64) << 10;     // job table at the head of a chunk
constexpr int kLoadChunks = 4;                     // staging ring depth (pack || H2D || scatter)
constexpr size_t kTabBytes = size_t(1) << 20;      // pinned page-table staging per ring entry

// One adapter load in flight (slora_adapter_prefetch / slora_adapter_load).
struct LoadJob {
    int64_t id = 0;
    int32_t rank = 0;
    const uint8_t* host_w = nullptr;
    bool direct = false;            // host_w is page-locked and N == 1: H2D straight from it, no pack
    int32_t* dev_tab = nullptr;     // the adapter's device page table (claim order)
    int32_t slot = -1;
    std::vector<int32_t> pages;     // page ids in claim order (uploaded by the loader)
    cudaEvent_t ready = nullptr;    // copy stream, after the adapter's last scatter kernel
    // guarded by Loader::mu
    int state = 0;                  // 0 queued / streaming, 1 host_w consumed and all device work enqueued, 2 failed
    cudaError_t err = cudaSuccess;
    int64_t bytes = 0;              // host bytes of the shard this rank copies
};

enum Owner : uint8_t { kFree = 0, kKv = 1, kAdapter = 2 };

struct Adapter {
    int64_t id = 0;
    int32_t rank = 0, slot = -1;
    float scale = 1.f;
    bool pinned = false;
    std::vector<int32_t> pages;  // claim order: layer, proj, tensor, row, chunk
    int32_t* dev_tab = nullptr;
    std::shared_ptr<LoadJob> load;  // set while the load may still be in flight
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

// Kernel configuration for one (mode, K, D): shrink rows are whole stored A
// rows (K elements, <= one ring slot); expand pieces cover `dchunk` output
// columns (<= 256 16-byte vectors: one per consumer thread; measured: bulk
// copies of >= 2 KB stream at full rate).  ns = ring slots filling smem.
// SLORA_DCHUNK overrides the expand width.
KernelCfg make_kernel_cfg(int mode, int64_t K, int64_t D, int64_t P, int es, int dtype) {
    (void)P;
    KernelCfg k;
    k.mode = mode;
    k.K = K;
    k.D = D;
    if (mode != kExpand && (K * es + 16 > kSlotBytes || (K * es) % 16)) return k;
    static int forced = [] {
        const char* s = getenv("SLORA_DCHUNK");
        return s ? atoi(s) : 0;
    }();
    if (mode != kShrink) {
        int64_t dc = std::min<int64_t>(D, 4096 / es * 1);  // <= 4 KB per B row slice
        if (forced > 0 && D % forced == 0 && (forced * es) % 16 == 0 && forced * es <= kSlotBytes) dc = forced;
        while (dc > 1 && (D % dc || (dc * es) % 16)) --dc;
        if ((dc * es) % 16 || dc / (16 / es) > kConsumerWarps * 32) return k;
        k.dchunk = dc;
    }
    const size_t budget = size_t(226) * 1024;
    const size_t base = lora_smem_bytes(mode, K, k.dchunk, 0, es);
    int ns = int((budget - base) / lora_slot_stride(mode, K, es));
    ns = std::min(ns, kMaxSlots);
    static const int ns_cap = [] {  // experiment knob: cap the ring depth
        const char* e = getenv("SLORA_NS");
        return e ? atoi(e) : 0;
    }();
    if (ns_cap >= 2) ns = std::min(ns, ns_cap);
    if (ns < 2) return k;
    k.ns = ns;
    k.smem = lora_smem_bytes(mode, K, k.dchunk, ns, es);
    k.grid = lora_max_ctas(mode, dtype, k.smem);
    static const int grid_cap = [] {  // experiment knob: fewer persistent CTAs than SMs
        const char* e = getenv("SLORA_GRID");
        return e ? atoi(e) : 0;
    }();
    if (grid_cap > 0) k.grid = std::min(k.grid, grid_cap);
    k.ok = k.grid > 0;
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
    // adapter loader: one thread, one copy stream, a ring of staging chunks
    struct Loader {
        std::thread th;
        std::mutex mu;
        std::condition_variable cv;            // queue and job-state changes
        std::deque<std::shared_ptr<LoadJob>> q;
        bool stop = false;
        cudaStream_t stream = nullptr;
        void* host[kLoadChunks] = {};          // pinned
        void* dev[kLoadChunks] = {};
        cudaEvent_t ev[kLoadChunks] = {};      // chunk free again (its H2D and scatter done)
        void* tab_host[kLoadChunks] = {};      // pinned page-table staging (slot pointer + page ids)
        cudaEvent_t tab_ev[kLoadChunks] = {};
        bool tab_used[kLoadChunks] = {};
        int tab_next = 0;
        bool used[kLoadChunks] = {};
        int next = 0;                          // loader thread only
        slora_loader_stats stats{};            // guarded by mu
    } ld;
    // page releases (kv_free, adapter_evict) are stream-ordered: one event per
    // release, and a load waits for every release still in flight (any stream)
    std::vector<cudaEvent_t> release_evs, spare_evs;
    std::unordered_set<slora_batch*> batches;  // live batches (detached by pool_destroy)
    // kernel configurations: 0 fused (K=D=H), 1 shrink q/k/v (K=H),
    // 2 shrink o (K=H/N), 3 expand (D=H/N)
    KernelCfg kcfg[kMaxKc];  // 0 fused K=hidden (ring pipeline), 1 shrink q/k/v, 2 shrink o, 3 expand,
                             // 4.. fused for the other projection input widths (NEXT-4)
    int n_kcfg = 4;
    // LoRA'd projections (NEXT-4): count, dims, page-table layout in units of the rank
    int np = kNumProj;
    int64_t pin[kMaxProj] = {}, pout[kMaxProj] = {};
    int32_t a_units[kMaxProj] = {}, b_units[kMaxProj] = {};  // page-table entries per rank unit (A, B)
    int32_t b_row_pages[kMaxProj] = {};                      // pages per stored B row
    int32_t proj_off[kMaxProj] = {};                         // projection p's tables in a layer (units of r)
    int32_t layer_units = 0;
    bool square = true;                                      // every projection hidden -> hidden
    int fused_kc(int64_t K) const {  // the fused configuration of a call whose projections read K inputs
        for (int c = 0; c < n_kcfg; ++c)
            if ((c == 0 || c >= 4) && kcfg[c].K == K) return c;
        return -1;
    }
    long long* trace_dev = nullptr;   // SLORA_TRACE=1: kernel event timestamps
    // rotating per-launch slots: item-done counters (zeroed once; each item's
    // last expand piece re-zeroes its counter) and the fused v workspace
    int32_t* sync_dev = nullptr;
    int64_t sync_stride = 0;          // ints per slot
    void* xg_dev = nullptr;           // gathered MBGMM x rows (batch_prepare sizes it)
    size_t xg_cap = 0;
    float* ws_dev = nullptr;
    int64_t ws_stride = 0;            // floats per slot
    float* ws_slot_base = nullptr;    // slot of the call being launched
    int64_t ws_region = 0;            // floats per workspace region: ring v, warp-task v, MBGMM v (kMgVParts k-split parts)
    uint64_t launch_seq = 0;
    int sms = 148;
    // tensor parallelism (slora_tp_*): the library's NCCL communicator and fp32 exchange buffers
    ncclComm_t tp_comm = nullptr;
    float* tp_vloc = nullptr;          // q/k/v shrink output of this rank: 3 * NR / N
    float* tp_vall = nullptr;          // all-gathered q/k/v intermediate: 3 * NR
    float* tp_u = nullptr;             // o partial / all-reduced intermediate: NR
    int64_t tp_cap = 0;                // NR the buffers hold
    slora_tp_stats tp_stats{};
    // NEXT-3 device-initiated exchange (slora_tp_p2p_*): this rank's exchange region (one cudaMalloc,
    // IPC-exported) = [kLaunchSlots][N][p2p_vcap] fp32 v blocks, then [kLaunchSlots][p2p_ccap] int32
    // per-item counters (zeroed); every rank's region mapped here (peer j at p2p_base[j])
    void* p2p_local = nullptr;
    void* p2p_base[8] = {};
    bool p2p_open = false;
    int64_t p2p_vcap = 0, p2p_ccap = 0;
    int kc_tpf_qkv = -1, kc_tpf_o = -1;  // fused configurations of the device-initiated TP calls

    ~slora_pool();
    int64_t free_pages() const { return int64_t(free_stack.size()); }
    int N() const { return cfg.tp_size; }
    // (stored rows, chunks per row) of one tensor shard (reading R3/R4)
    // (stored rows, pages per row) of one tensor shard.  One GPU: A has r stored rows of
    // proj_in elements, B r rows of proj_out, each ceil(n/P) pages (reading R2, NEXT-4).
    // TP (square projections only): readings R3/R4.
    void tensor_shape(int proj, int tensor, int rank, int& rows, int& chunks) const {
        if (N() > 1) {
            rows = (proj < 3 && tensor == 0) ? rank / N() : rank;
            chunks = (proj < 3 && tensor == 0) ? N() : 1;
            return;
        }
        rows = rank;
        chunks = int(((tensor == 0 ? pin[proj] : pout[proj]) + P - 1) / P);
    }
    int64_t adapter_page_count(int rank) const { return int64_t(cfg.num_layers) * layer_units * rank; }
    // dense elements of the host tensor (A: in x r, B: r x out) of projection p
    int64_t host_elems(int proj, int tensor, int rank) const {
        return int64_t(rank) * (tensor == 0 ? pin[proj] : pout[proj]);
    }
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
    // per (kernel cfg, nproj) work descriptors, built on first use after a
    // prepare and uploaded into the batch's device arena
    struct Call {
        bool built = false;
        uint32_t mask = 0;
        std::vector<DevItem> items;
        std::vector<DevPiece> pieces;   // grouped by CTA (schedule_pieces)
        std::vector<int32_t> cta_off;   // grid + 1
        std::vector<MgUnit> mg_s, mg_e; // MBGMM shrink / expand units (fused calls with long runs)
        size_t off_items = 0, off_pieces = 0, off_cta = 0, off_mg_s = 0, off_mg_e = 0;
    } calls[kMaxKc][kNpSlots];
    // per segment: token ranges [begin, end) of the segment's token list that
    // are MBGMM runs (>= theta consecutive x rows; fused 16-bit calls only)
    std::vector<std::vector<std::pair<int32_t, int32_t>>> runs;
    int32_t n_runs = 0;
    bool mg_gather = false;    // MBGMM runs are whole segments of scattered tokens (x gathered, y via tok_idx)
    int64_t mg_units_max = 0;  // units of one 4-projection fused call (arena sizing)
    size_t off_tok = 0;
    // device arena (bump allocated per prepare) + its pinned staging mirror
    size_t arena_cap = 0, arena_used = 0;
    void* arena_host_buf[2] = {nullptr, nullptr};  // pinned mirrors, alternating per prepare (the host may
                                                     // run one step further ahead of the GPU)
    void* arena_dev = nullptr;
    size_t dirty_lo = 0, dirty_hi = 0;  // host arena bytes not yet uploaded (arena_flush)
    cudaEvent_t upload_evs[2] = {nullptr, nullptr};
    bool pending[2] = {false, false};
    int cur = 0;                          // the mirror pair this prepare writes
    // call headers at fixed device addresses ([kernel cfg][nproj]); prepare rewrites them
    CallHdr* hdr_dev = nullptr;
    CallHdr* hdr_host_buf[2] = {nullptr, nullptr};  // pinned header mirrors (with arena_host_buf)
    uint32_t used_masks[kMaxKc][kNpSlots] = {};  // call shapes launched since create: rebuilt by every prepare
    bool in_prepare = false;
    uint32_t options = 0;                 // slora_batch_set_options
};

static void batch_free_device(slora_batch* b);
static cudaError_t loader_start(slora_pool* p);
static void loader_stop(slora_pool* p);

static void tp_release(slora_pool* p) {
    if (p->tp_comm && nccl().ok) nccl().CommDestroy(p->tp_comm);
    p->tp_comm = nullptr;
}

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
    // LoRA'd projections (NEXT-4): default q,k,v,o square
    const int np = cfg->num_proj == 0 ? kNumProj : cfg->num_proj;
    if (np < 1 || np > kMaxProj) return fail(SLORA_ERR_INVALID_ARG, "num_proj %d not in 1..%d", np, kMaxProj);
    int64_t pin[kMaxProj] = {}, pout[kMaxProj] = {};
    bool square = np == kNumProj;
    for (int q = 0; q < np; ++q) {
        pin[q] = (cfg->num_proj == 0 || cfg->proj_in[q] == 0) ? cfg->hidden : cfg->proj_in[q];
        pout[q] = (cfg->num_proj == 0 || cfg->proj_out[q] == 0) ? cfg->hidden : cfg->proj_out[q];
        if (pin[q] < 1 || pout[q] < 1) return fail(SLORA_ERR_INVALID_ARG, "projection %d dims < 1", q);
        if ((pin[q] * es) % 16 || (pout[q] * es) % 16)
            return fail(SLORA_ERR_SHAPE, "projection %d dims must be multiples of 16 bytes", q);
        if ((pin[q] + P - 1) / P > kMaxChunks || (pout[q] + P - 1) / P > kMaxChunks)
            return fail(SLORA_ERR_SHAPE, "projection %d rows span more than %d pages", q, kMaxChunks);
        square = square && pin[q] == cfg->hidden && pout[q] == cfg->hidden;
    }
    if (cfg->tp_size > 1 && !square)
        return fail(SLORA_ERR_SHAPE, "tensor parallelism needs the four square projections (q,k,v,o)");
    slora_pool* p = new slora_pool();
    p->cfg = *cfg;
    p->P = P;
    p->es = es;
    p->dev = cfg->device >= 0;
    p->np = np;
    p->square = square;
    for (int q = 0; q < np; ++q) {
        p->pin[q] = pin[q];
        p->pout[q] = pout[q];
    }
    for (int q = 0; q < np; ++q) {
        int rows, ch;
        p->tensor_shape(q, 0, cfg->tp_size, rows, ch);  // rank = N: units per rank unit = rows*ch/N
        p->a_units[q] = rows * ch / cfg->tp_size;
        p->tensor_shape(q, 1, cfg->tp_size, rows, ch);
        p->b_units[q] = rows * ch / cfg->tp_size;
        p->b_row_pages[q] = ch;
        p->proj_off[q] = p->layer_units;
        p->layer_units += p->a_units[q] + p->b_units[q];
    }
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
        if ((e = configure_mbgmm_kernels())) return cleanup(e, "configure MBGMM kernels");
        if ((e = cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, cfg->device))) return cleanup(e, "SM count");
        if ((e = cudaMalloc(&p->slot_tab_dev, sizeof(int32_t*) * size_t(cfg->max_adapters))))
            return cleanup(e, "cudaMalloc slot table");
        if ((e = cudaMemset(p->slot_tab_dev, 0, sizeof(int32_t*) * size_t(cfg->max_adapters))))
            return cleanup(e, "cudaMemset");
        if ((e = loader_start(p))) return cleanup(e, "adapter loader");
        const int dt = cfg->dtype == SLORA_F32 ? kF32 : (cfg->dtype == SLORA_F16 ? kF16 : kBF16);
        const int64_t H = cfg->hidden;
        p->kcfg[0] = make_kernel_cfg(kFused, H, H, P, es, dt);
        p->kcfg[1] = make_kernel_cfg(kShrink, H, P, P, es, dt);
        p->kcfg[2] = make_kernel_cfg(kShrink, cfg->tp_size > 1 ? P : H, P, P, es, dt);
        p->kcfg[3] = make_kernel_cfg(kExpand, P, P, P, es, dt);
        for (int q = 0; q < np && cfg->tp_size == 1; ++q)  // fused configurations of the other input widths
            if (p->fused_kc(pin[q]) < 0 && p->n_kcfg < kMaxKc) p->kcfg[p->n_kcfg++] = make_kernel_cfg(kFused, pin[q], P, P, es, dt);
        if (const char* vb = getenv("SLORA_VERBOSE"); vb && atoi(vb) > 0)
            for (int c = 0; c < p->n_kcfg; ++c)
                fprintf(stderr, "slora: kcfg[%d] mode=%d K=%lld D=%lld dchunk=%lld ns=%d smem=%zu grid=%d ok=%d\n", c,
                        p->kcfg[c].mode, (long long)p->kcfg[c].K, (long long)p->kcfg[c].D,
                        (long long)p->kcfg[c].dchunk, p->kcfg[c].ns, p->kcfg[c].smem, p->kcfg[c].grid,
                        int(p->kcfg[c].ok));
        const char* tr = getenv("SLORA_TRACE");
        if (tr && atoi(tr) == 1) {
            if ((e = cudaMalloc(&p->trace_dev, 16 * kTraceSlots * sizeof(long long)))) return cleanup(e, "cudaMalloc trace");
            cudaMemset(p->trace_dev, 0, 16 * kTraceSlots * sizeof(long long));
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
        loader_stop(p);  // finishes the queued loads
        cudaDeviceSynchronize();
        for (auto& kvp : p->adapters)
            if (kvp.second.dev_tab) cudaFree(kvp.second.dev_tab);
        cudaFree(p->slot_tab_dev);
        for (cudaEvent_t ev : p->release_evs) cudaEventDestroy(ev);
        for (cudaEvent_t ev : p->spare_evs) cudaEventDestroy(ev);
        if (p->sync_dev) cudaFree(p->sync_dev);
        if (p->ws_dev) cudaFree(p->ws_dev);
        if (p->xg_dev) cudaFree(p->xg_dev);
        if (p->tp_vloc) cudaFree(p->tp_vloc);
        if (p->tp_vall) cudaFree(p->tp_vall);
        if (p->tp_u) cudaFree(p->tp_u);
        if (p->trace_dev) cudaFree(p->trace_dev);
    }
    if (p->dev) {
        for (int j = 0; j < p->N() && j < 8; ++j)
            if (p->p2p_base[j] && p->p2p_base[j] != p->p2p_local) cudaIpcCloseMemHandle(p->p2p_base[j]);
        if (p->p2p_local) cudaFree(p->p2p_local);
    }
    tp_release(p);
    for (slora_batch* b : p->batches) {  // live batches become stale handles (their device side freed here)
        if (p->dev) batch_free_device(b);
        b->pool = nullptr;
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
    cudaEvent_t ev = nullptr;
    if (!p->spare_evs.empty()) {
        ev = p->spare_evs.back();
        p->spare_evs.pop_back();
    } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaStreamSynchronize(static_cast<cudaStream_t>(stream));  // no event: make the release complete now
        return;
    }
    cudaEventRecord(ev, static_cast<cudaStream_t>(stream));
    p->release_evs.push_back(ev);
}
// make `s` wait for every page release still in flight; completed ones are recycled
static cudaError_t wait_releases(slora_pool* p, cudaStream_t s) {
    std::vector<cudaEvent_t> keep;
    for (cudaEvent_t ev : p->release_evs) {
        if (cudaEventQuery(ev) == cudaSuccess) {
            p->spare_evs.push_back(ev);
            continue;
        }
        cudaGetLastError();  // clear cudaErrorNotReady
        cudaError_t e = cudaStreamWaitEvent(s, ev, 0);
        if (e) return e;
        keep.push_back(ev);
    }
    p->release_evs.swap(keep);
    return cudaSuccess;
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
// A host copy recorded by pack_shard and run at flush time by copy_segments.
struct CopySeg {
    uint8_t* dst;
    const uint8_t* src;
    size_t bytes;
};

// Run the staging copies of one flush on several host threads (a single
// memcpy stream from pageable memory tops out near 10 GB/s, below the PCIe
// link the staged bytes then cross).  Segments are split into ~4 MB pieces.
static void copy_segments(std::vector<CopySeg>& segs) {
    std::vector<CopySeg> work;
    const size_t piece = size_t(4) << 20;
    size_t total = 0;
    for (const CopySeg& s : segs)
        for (size_t o = 0; o < s.bytes; o += piece) {
            work.push_back({s.dst + o, s.src + o, std::min(piece, s.bytes - o)});
            total += work.back().bytes;
        }
    segs.clear();
    static const int nthr = [] {
        const char* e = getenv("SLORA_LOAD_THREADS");
        const int hw = int(std::thread::hardware_concurrency());
        return e ? std::max(1, atoi(e)) : std::max(1, std::min(8, hw));
    }();
    const int nt = int(std::min<size_t>(size_t(nthr), std::max<size_t>(1, total / (size_t(2) << 20))));
    if (nt <= 1) {
        for (const CopySeg& s : work) memcpy(s.dst, s.src, s.bytes);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t)
        th.emplace_back([&work, t, nt] {
            for (size_t i = size_t(t); i < work.size(); i += size_t(nt)) memcpy(work[i].dst, work[i].src, work[i].bytes);
        });
    for (size_t i = 0; i < work.size(); i += size_t(nt)) memcpy(work[i].dst, work[i].src, work[i].bytes);
    for (auto& x : th) x.join();
}

static void pack_shard(const slora_pool* p, const uint8_t* A, const uint8_t* B, int proj, int tensor, int r,
                       uint8_t* dst, int& rows_out, int& cols_out, std::vector<CopySeg>& segs) {
    const int64_t H = p->cfg.hidden, P = p->P;
    const int N = p->N(), k = p->cfg.tp_rank, es = p->es;
    if (N == 1) {  // the dense tensor is the shard: A (proj_in x r), B (r x proj_out)
        segs.push_back({dst, tensor == 0 ? A : B, size_t(p->host_elems(proj, tensor, r)) * es});
        rows_out = int(tensor == 0 ? p->pin[proj] : r);
        cols_out = int(tensor == 0 ? r : p->pout[proj]);
        return;
    }
    if (tensor == 0) {
        if (proj < 3) {
            const int rc = r / N;
            if (N == 1)  // the whole dense A (H x r row-major) is the shard
                segs.push_back({dst, A, size_t(H * r) * es});
            else
            for (int64_t row = 0; row < H; ++row)
                memcpy(dst + size_t(row * rc) * es, A + size_t(row * r + int64_t(k) * rc) * es, size_t(rc) * es);
            rows_out = int(H);
            cols_out = rc;
        } else {
            segs.push_back({dst, A + size_t(int64_t(k) * P * r) * es, size_t(P * r) * es});
            rows_out = int(P);
            cols_out = r;
        }
    } else {
        if (N == 1)  // rows of B are whole pages: one copy
            segs.push_back({dst, B, size_t(int64_t(r) * H) * es});
        else
            for (int j = 0; j < r; ++j)
                memcpy(dst + size_t(int64_t(j) * P) * es, B + size_t(int64_t(j) * H + int64_t(k) * P) * es,
                       size_t(P) * es);
        rows_out = r;
        cols_out = int(P);
    }
}

// ---------------------------------------------------------- adapter loader
// ("prefetching ... overlapping the loading of adapters with
// the computation").  One thread per pool streams queued loads in order:
// every (layer, proj, A/B) shard of the adapter goes into the current staging
// chunk of a kLoadChunks ring; a full chunk is flushed as
//   pack (host threads, pageable host_w -> pinned chunk; skipped when host_w is
//   page-locked and N == 1: the H2D reads host_w itself)
//   -> cudaMemcpyAsync H2D -> scatter kernel (pages) -> chunk event
// on the pool's copy stream, so the pack of chunk k+1 overlaps the H2D and
// scatter of chunk k, and the caller's kernels run meanwhile.  A chunk is
// re-packed only after its event completed.
static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static cudaError_t run_load(slora_pool* p, LoadJob& jb) {
    auto& L = p->ld;
    const int64_t H = p->cfg.hidden;
    const int es = p->es;
    (void)H;
    int64_t per_layer = 0;  // host elements of one layer: A and B of every projection
    for (int pr = 0; pr < p->np; ++pr) per_layer += p->host_elems(pr, 0, jb.rank) + p->host_elems(pr, 1, jb.rank);
    size_t used = kJobBytes;
    std::vector<ScatterJob> jobs;
    std::vector<CopySeg> segs;
    cudaError_t e = cudaSuccess;
    int k = L.next;
    auto acquire = [&]() -> cudaError_t {  // chunk k's previous flush is done (host buffer reusable)
        if (!L.used[k]) return cudaSuccess;
        L.used[k] = false;
        return cudaEventSynchronize(L.ev[k]);
    };
    auto flush = [&]() -> cudaError_t {
        if (jobs.empty()) return cudaSuccess;
        uint8_t* hb = static_cast<uint8_t*>(L.host[k]);
        uint8_t* db = static_cast<uint8_t*>(L.dev[k]);
        cudaError_t e2 = cudaSuccess;
        memcpy(hb, jobs.data(), jobs.size() * sizeof(ScatterJob));
        if (jb.direct) {
            e2 = cudaMemcpyAsync(db, hb, jobs.size() * sizeof(ScatterJob), cudaMemcpyHostToDevice, L.stream);
            // consecutive shards are contiguous in host_w and in the chunk: one H2D per run
            for (size_t a = 0; a < segs.size() && !e2;) {
                size_t b2 = a + 1, n = segs[a].bytes;
                while (b2 < segs.size() && segs[b2].src == segs[a].src + n && segs[b2].dst == segs[a].dst + n)
                    n += segs[b2++].bytes;
                e2 = cudaMemcpyAsync(db + (segs[a].dst - hb), segs[a].src, n, cudaMemcpyHostToDevice, L.stream);
                a = b2;
            }
            segs.clear();
        } else {
            copy_segments(segs);
            e2 = cudaMemcpyAsync(db, hb, used, cudaMemcpyHostToDevice, L.stream);
        }
        if (!e2) e2 = launch_scatter(db + kJobBytes, reinterpret_cast<const ScatterJob*>(db), int(jobs.size()),
                                     p->cfg.device_buffer, p->P, es, L.stream);
        if (!e2) e2 = cudaEventRecord(L.ev[k], L.stream);
        L.used[k] = true;
        k = (k + 1) % kLoadChunks;
        used = kJobBytes;
        jobs.clear();
        return e2;
    };
    {  // page table, then the slot's table pointer, from pinned staging (never a pageable copy:
       // that would drain the copy stream)
        const int tk = L.tab_next;
        L.tab_next = (tk + 1) % kLoadChunks;
        if (L.tab_used[tk] && (e = cudaEventSynchronize(L.tab_ev[tk]))) return e;
        uint8_t* th = static_cast<uint8_t*>(L.tab_host[tk]);
        memcpy(th, &jb.dev_tab, sizeof(int32_t*));
        memcpy(th + 16, jb.pages.data(), jb.pages.size() * sizeof(int32_t));
        e = cudaMemcpyAsync(jb.dev_tab, th + 16, jb.pages.size() * sizeof(int32_t), cudaMemcpyHostToDevice, L.stream);
        if (!e) e = cudaMemcpyAsync(p->slot_tab_dev + jb.slot, th, sizeof(int32_t*), cudaMemcpyHostToDevice, L.stream);
        if (!e) e = cudaEventRecord(L.tab_ev[tk], L.stream);
        L.tab_used[tk] = true;
        if (e) return e;
    }
    int64_t page_cursor = 0;
    for (int l = 0; l < p->cfg.num_layers && !e; ++l) {
        const uint8_t* A = jb.host_w + size_t(int64_t(l) * per_layer) * es;
        for (int pr = 0; pr < p->np && !e; ++pr) {
            const uint8_t* B = A + size_t(p->host_elems(pr, 0, jb.rank)) * es;
            const uint8_t* An = B + size_t(p->host_elems(pr, 1, jb.rank)) * es;  // the next projection's A
            for (int t = 0; t < 2 && !e; ++t) {
                int rows_s, chunks;
                p->tensor_shape(pr, t, jb.rank, rows_s, chunks);
                // staging bytes of this rank's shard (dense; = host bytes / N)
                const size_t bytes = size_t(p->host_elems(pr, t, jb.rank) / p->N()) * es;
                if (used + bytes > kStageBytes || (jobs.size() + 1) * sizeof(ScatterJob) > kJobBytes) {
                    if ((e = flush())) break;
                }
                if (jobs.empty() && (e = acquire())) break;
                int rows, cols;
                pack_shard(p, A, B, pr, t, jb.rank, static_cast<uint8_t*>(L.host[k]) + used, rows, cols, segs);
                ScatterJob sj;
                sj.src_off = int64_t((used - kJobBytes) / size_t(es));
                sj.pages = jb.dev_tab + page_cursor;
                sj.kind = t;
                sj.rows = rows;
                sj.cols = cols;
                sj.row_pages = chunks;
                jobs.push_back(sj);
                used += (bytes + 15) & ~size_t(15);
                jb.bytes += int64_t(bytes);
                page_cursor += int64_t(rows_s) * chunks;
            }
            A = An;
        }
    }
    if (!e) e = flush();
    // host_w is consumed once its last chunk is packed (or, read directly, once its H2D completed)
    if (!e && jb.direct) e = cudaEventSynchronize(L.ev[(k + kLoadChunks - 1) % kLoadChunks]);
    if (!e) e = cudaEventRecord(jb.ready, L.stream);
    L.next = k;
    return e;
}

static void loader_main(slora_pool* p) {
    auto& L = p->ld;
    cudaSetDevice(p->cfg.device);
    for (;;) {
        std::shared_ptr<LoadJob> jb;
        {
            std::unique_lock<std::mutex> lk(L.mu);
            L.cv.wait(lk, [&] { return L.stop || !L.q.empty(); });
            if (L.q.empty()) return;  // stop requested, queue drained
            jb = L.q.front();
        }
        const double t0 = now_s();
        cudaError_t e = run_load(p, *jb);
        const double t1 = now_s();
        {
            std::lock_guard<std::mutex> lk(L.mu);
            jb->err = e;
            jb->state = e ? 2 : 1;
            L.q.pop_front();
            L.stats.loads += 1;
            L.stats.bytes += jb->bytes;
            L.stats.direct_loads += jb->direct ? 1 : 0;
            L.stats.busy_s += t1 - t0;
        }
        L.cv.notify_all();
    }
}

static cudaError_t loader_start(slora_pool* p) {
    auto& L = p->ld;
    // the copy stream runs at the lowest priority: the LoRA kernels' CTAs go first
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaError_t e = cudaStreamCreateWithPriority(&L.stream, cudaStreamNonBlocking, least);
    for (int k = 0; k < kLoadChunks && !e; ++k) {
        if (!e) e = cudaHostAlloc(&L.host[k], kStageBytes, cudaHostAllocDefault);
        if (!e) e = cudaMalloc(&L.dev[k], kStageBytes);
        if (!e) e = cudaEventCreateWithFlags(&L.ev[k], cudaEventDisableTiming);
        if (!e) e = cudaHostAlloc(&L.tab_host[k], kTabBytes, cudaHostAllocDefault);
        if (!e) e = cudaEventCreateWithFlags(&L.tab_ev[k], cudaEventDisableTiming);
    }
    if (e) return e;
    L.th = std::thread(loader_main, p);
    return cudaSuccess;
}

static void loader_stop(slora_pool* p) {
    auto& L = p->ld;
    if (L.th.joinable()) {
        {
            std::lock_guard<std::mutex> lk(L.mu);
            L.stop = true;
        }
        L.cv.notify_all();
        L.th.join();
    }
    if (L.stream) cudaStreamSynchronize(L.stream);
    for (int k = 0; k < kLoadChunks; ++k) {
        if (L.host[k]) cudaFreeHost(L.host[k]);
        if (L.dev[k]) cudaFree(L.dev[k]);
        if (L.ev[k]) cudaEventDestroy(L.ev[k]);
        if (L.tab_host[k]) cudaFreeHost(L.tab_host[k]);
        if (L.tab_ev[k]) cudaEventDestroy(L.tab_ev[k]);
        L.host[k] = L.dev[k] = L.tab_host[k] = nullptr;
        L.ev[k] = L.tab_ev[k] = nullptr;
    }
    if (L.stream) cudaStreamDestroy(L.stream);
    L.stream = nullptr;
}

slora_pool::~slora_pool() { loader_stop(this); }

// Block until the adapter's load reached `state` >= want (1: host_w consumed and
// all its device work enqueued); surfaces a failed load.
static slora_status load_wait_host(slora_pool* p, Adapter& ad) {
    if (!ad.load) return SLORA_OK;
    auto& L = p->ld;
    std::unique_lock<std::mutex> lk(L.mu);
    L.cv.wait(lk, [&] { return ad.load->state != 0; });
    if (ad.load->state == 2)
        return fail(SLORA_ERR_CUDA, "adapter %lld load: %s", (long long)ad.id, cudaGetErrorString(ad.load->err));
    return SLORA_OK;
}
// Make `stream` wait for the adapter's load (stream-ordered); drop the job once complete.
static slora_status load_fence(slora_pool* p, Adapter& ad, cudaStream_t stream) {
    if (!ad.load) return SLORA_OK;
    if (slora_status st = load_wait_host(p, ad)) return st;
    if (cudaEventQuery(ad.load->ready) == cudaSuccess) {
        cudaEventDestroy(ad.load->ready);
        ad.load.reset();
        return SLORA_OK;
    }
    cudaGetLastError();  // cudaErrorNotReady
    if (cudaError_t e = cudaStreamWaitEvent(stream, ad.load->ready, 0))
        return fail(SLORA_ERR_CUDA, "adapter load fence: %s", cudaGetErrorString(e));
    return SLORA_OK;
}

// Claim pages and slot (synchronous, leaves the pool unchanged on error), upload
// the page table on the copy stream and queue the data load.
static slora_status adapter_begin(slora_pool* p, int64_t id, int32_t rank, const void* host_w, float scale,
                                  int32_t* slot_out) {
    if (rank < 1) return fail(SLORA_ERR_INVALID_ARG, "rank < 1");
    if (rank > kMaxRank) return fail(SLORA_ERR_SHAPE, "rank %d > %d (max rank of the MBGMV path)", rank, kMaxRank);
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
    size_t tensor_max_bytes = 0;
    for (int pr = 0; pr < p->np; ++pr)
        for (int t = 0; t < 2; ++t) tensor_max_bytes = std::max(tensor_max_bytes, size_t(p->host_elems(pr, t, rank)) * es);
    (void)H;
    if (p->dev && tensor_max_bytes + kJobBytes > kStageBytes)
        return fail(SLORA_ERR_SHAPE, "adapter tensor of %zu bytes exceeds staging", tensor_max_bytes);
    if (p->dev && size_t(need) * sizeof(int32_t) + 16 > kTabBytes)
        return fail(SLORA_ERR_SHAPE, "adapter page table of %lld pages exceeds staging", (long long)need);

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
    if (p->dev) {
        auto& L = p->ld;
        auto jb = std::make_shared<LoadJob>();
        jb->id = id;
        jb->rank = rank;
        jb->host_w = static_cast<const uint8_t*>(host_w);
        cudaPointerAttributes at{};
        if (p->N() == 1 && cudaPointerGetAttributes(&at, host_w) == cudaSuccess && at.type == cudaMemoryTypeHost)
            jb->direct = true;  // page-locked: no pack, the H2D reads host_w
        cudaGetLastError();
        cudaError_t e = cudaSetDevice(p->cfg.device);
        // page reuse fence, taken now: released pages may still be read by queued kernels
        if (!e) e = wait_releases(p, L.stream);
        if (!e) e = cudaEventCreateWithFlags(&jb->ready, cudaEventDisableTiming);
        if (!e) e = cudaMallocAsync(reinterpret_cast<void**>(&ad.dev_tab), sizeof(int32_t) * size_t(need), L.stream);
        if (e) {
            if (jb->ready) cudaEventDestroy(jb->ready);
            if (ad.dev_tab) cudaFree(ad.dev_tab);
            for (auto it = ad.pages.rbegin(); it != ad.pages.rend(); ++it) {
                p->owner[size_t(*it)] = kFree;
                p->free_stack.push_back(*it);
            }
            return fail(SLORA_ERR_CUDA, "adapter load: %s", cudaGetErrorString(e));
        }
        jb->dev_tab = ad.dev_tab;
        jb->slot = ad.slot;
        jb->pages = ad.pages;  // the loader uploads the page table (pinned copy) ahead of the data
        ad.load = jb;
        {
            std::lock_guard<std::mutex> lk(L.mu);
            L.q.push_back(jb);
        }
        L.cv.notify_all();
    }
    p->adapter_pages += need;
    p->slots[size_t(ad.slot)] = id;
    if (slot_out) *slot_out = ad.slot;
    p->adapters.emplace(id, std::move(ad));
    return SLORA_OK;
}

extern "C" slora_status slora_adapter_prefetch(slora_pool_t p, int64_t id, int32_t rank, const void* host_w,
                                               float scale, int32_t* slot_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    if (slora_status st = adapter_begin(p, id, rank, host_w, scale, slot_out)) return st;
    return ok();
}

extern "C" slora_status slora_adapter_load(slora_pool_t p, int64_t id, int32_t rank, const void* host_w,
                                           float scale, void* stream, int32_t* slot_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    if (slora_status st = adapter_begin(p, id, rank, host_w, scale, slot_out)) return st;
    if (!p->dev) return ok();
    // host_w is free on return; completion is stream-ordered on `stream`
    Adapter& ad = p->adapters.at(id);
    if (slora_status st = load_fence(p, ad, static_cast<cudaStream_t>(stream))) return st;
    return ok();
}

extern "C" slora_status slora_adapter_wait(slora_pool_t p, int64_t id) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->adapters.find(id);
    if (it == p->adapters.end()) return fail(SLORA_ERR_NOT_RESIDENT, "adapter %lld", (long long)id);
    Adapter& ad = it->second;
    if (!ad.load) return ok();
    if (slora_status st = load_wait_host(p, ad)) return st;
    if (cudaError_t e = cudaEventSynchronize(ad.load->ready))
        return fail(SLORA_ERR_CUDA, "adapter %lld load: %s", (long long)id, cudaGetErrorString(e));
    cudaEventDestroy(ad.load->ready);
    ad.load.reset();
    return ok();
}

extern "C" slora_status slora_adapter_query(slora_pool_t p, int64_t id, int32_t* loading) {
    if (check_pool(p) || !loading) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    auto it = p->adapters.find(id);
    if (it == p->adapters.end()) return fail(SLORA_ERR_NOT_RESIDENT, "adapter %lld", (long long)id);
    Adapter& ad = it->second;
    *loading = 0;
    if (!ad.load) return ok();
    int st;
    {
        std::lock_guard<std::mutex> lk(p->ld.mu);
        st = ad.load->state;
    }
    if (st == 2) return fail(SLORA_ERR_CUDA, "adapter %lld load: %s", (long long)id, cudaGetErrorString(ad.load->err));
    if (st == 1 && cudaEventQuery(ad.load->ready) == cudaSuccess) {
        cudaEventDestroy(ad.load->ready);
        ad.load.reset();
        return ok();
    }
    cudaGetLastError();
    *loading = 1;
    return ok();
}

extern "C" slora_status slora_loader_get_stats(slora_pool_t p, slora_loader_stats* out) {
    if (check_pool(p) || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    std::lock_guard<std::mutex> lk(p->ld.mu);
    *out = p->ld.stats;
    out->queued = int64_t(p->ld.q.size());
    return ok();
}

extern "C" slora_status slora_adapter_evict(slora_pool_t p, int64_t id, void* stream, int64_t* released_out) {
    if (check_pool(p)) return SLORA_ERR_INVALID_ARG;
    auto it = p->adapters.find(id);
    if (it == p->adapters.end()) return fail(SLORA_ERR_NOT_RESIDENT, "adapter %lld", (long long)id);
    if (it->second.pinned) return fail(SLORA_ERR_PINNED, "adapter %lld", (long long)id);
    Adapter& ad = it->second;
    // a load still in flight: its scatters must land before the pages can be reused
    if (load_fence(p, ad, static_cast<cudaStream_t>(stream)) != SLORA_OK) {
        // the load failed: nothing of it may still be writing once the copy stream drained; the
        // adapter is released all the same (otherwise it could never leave the pool)
        cudaStreamSynchronize(p->ld.stream);
        cudaGetLastError();
    }
    if (ad.load) cudaEventDestroy(ad.load->ready);  // still pending: destruction is deferred by CUDA
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
extern "C" slora_status slora_batch_create(slora_pool_t p, slora_batch_t* out) {
    if (check_pool(p) || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    slora_batch* b = new slora_batch();
    b->pool = p;
    p->batches.insert(b);
    if (p->dev) {
        cudaError_t e = cudaEventCreateWithFlags(&b->upload_evs[0], cudaEventDisableTiming);
        if (!e) e = cudaEventCreateWithFlags(&b->upload_evs[1], cudaEventDisableTiming);
        if (!e) e = cudaMalloc(&b->hdr_dev, sizeof(CallHdr) * kMaxKc * kNpSlots);
        if (!e) e = cudaMemset(b->hdr_dev, 0, sizeof(CallHdr) * kMaxKc * kNpSlots);
        for (int i = 0; i < 2 && !e; ++i)
            e = cudaHostAlloc(&b->hdr_host_buf[i], sizeof(CallHdr) * kMaxKc * kNpSlots, cudaHostAllocDefault);
        if (e) {
            if (b->hdr_dev) cudaFree(b->hdr_dev);
            p->batches.erase(b);
            delete b;
            return fail(SLORA_ERR_CUDA, "batch create: %s", cudaGetErrorString(e));
        }
        for (int i = 0; i < 2; ++i) memset(b->hdr_host_buf[i], 0, sizeof(CallHdr) * kMaxKc * kNpSlots);
    }
    *out = b;
    return ok();
}

static void batch_free_device(slora_batch* b) {
    for (int i = 0; i < 2; ++i) {
        if (b->pending[i]) cudaEventSynchronize(b->upload_evs[i]);
        if (b->arena_host_buf[i]) cudaFreeHost(b->arena_host_buf[i]);
        if (b->hdr_host_buf[i]) cudaFreeHost(b->hdr_host_buf[i]);
        if (b->upload_evs[i]) cudaEventDestroy(b->upload_evs[i]);
        b->arena_host_buf[i] = nullptr;
        b->hdr_host_buf[i] = nullptr;
        b->upload_evs[i] = nullptr;
        b->pending[i] = false;
    }
    if (b->arena_dev) cudaFree(b->arena_dev);
    if (b->hdr_dev) cudaFree(b->hdr_dev);
    b->hdr_dev = nullptr;
    b->arena_dev = nullptr;
}

extern "C" slora_status slora_batch_destroy(slora_batch_t b) {
    if (!b) return fail(SLORA_ERR_INVALID_ARG, "null batch");
    if (!b->pool) {  // its pool was destroyed first: the device side is already freed
        delete b;
        return ok();
    }
    b->pool->batches.erase(b);
    if (b->pool->dev) batch_free_device(b);
    delete b;
    return ok();
}

namespace {
// Copy `n` bytes into the batch's pinned arena and enqueue their H2D copy into
// the device arena; returns the device offset.  The arena is bump-allocated
// per prepare and sized by prepare (grown there, never mid-batch).
// Bump-allocate n bytes of the batch arena and fill its pinned mirror; the
// device copy happens in arena_flush (one H2D per prepare).
size_t arena_put(slora_batch* b, const void* src, size_t n, cudaStream_t, cudaError_t& err) {
    const size_t off = b->arena_used;
    const size_t n_al = (n + 255) & ~size_t(255);
    if (off + n_al > b->arena_cap) {
        err = cudaErrorMemoryAllocation;
        return 0;
    }
    if (n) {
        memcpy(static_cast<uint8_t*>(b->arena_host_buf[b->cur]) + off, src, n);
        if (b->dirty_hi == b->dirty_lo) b->dirty_lo = off;
        b->dirty_hi = off + n;
    }
    b->arena_used = off + n_al;
    return off;
}

// Point the header of call (kc, np) at its descriptors in the arena.
void set_hdr(slora_pool* p, slora_batch* b, int kc, int np) {
    const slora_batch::Call& call = b->calls[kc][np];
    uint8_t* base = static_cast<uint8_t*>(b->arena_dev);
    CallHdr& h = b->hdr_host_buf[b->cur][kc * kNpSlots + np];
    h.tok_idx = reinterpret_cast<const int32_t*>(base + b->off_tok);
    h.items = reinterpret_cast<const DevItem*>(base + call.off_items);
    h.pieces = reinterpret_cast<const DevPiece*>(base + call.off_pieces);
    h.cta_off = reinterpret_cast<const int32_t*>(base + call.off_cta);
    h.sync = p->sync_dev;
    h.sync_stride = p->sync_stride;
    h.ws = p->ws_dev;
    h.ws_stride = p->ws_stride;
    h.NR = b->NR;
    h.n_items = int32_t(call.items.size());
    h.n_pieces = int32_t(call.pieces.size());
}

// Upload the arena bytes written since the last flush and the call headers:
// two H2D copies on the prepare's stream.
cudaError_t arena_flush(slora_batch* b, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (b->dirty_hi > b->dirty_lo)
        e = cudaMemcpyAsync(static_cast<uint8_t*>(b->arena_dev) + b->dirty_lo,
                            static_cast<uint8_t*>(b->arena_host_buf[b->cur]) + b->dirty_lo, b->dirty_hi - b->dirty_lo,
                            cudaMemcpyHostToDevice, s);
    b->dirty_lo = b->dirty_hi = 0;
    if (!e) e = cudaMemcpyAsync(b->hdr_dev, b->hdr_host_buf[b->cur], sizeof(CallHdr) * kMaxKc * kNpSlots,
                                cudaMemcpyHostToDevice, s);
    if (!e) e = cudaEventRecord(b->upload_evs[b->cur], s);
    b->pending[b->cur] = true;
    return e;
}

// Static schedule: LPT (largest first onto the least-loaded CTA) over the
// pieces' streamed bytes, shrink pieces first, then expand pieces on top of
// the shrink loads; each CTA's list keeps shrink before expand (the kernel's
// deadlock-freedom argument, kernels.cu header).  The per-piece constant
// stands for the fixed cost of a piece (barriers, v exchange).
void schedule_pieces(const std::vector<DevPiece>& in, const std::vector<int64_t>& cost, int grid,
                     std::vector<DevPiece>& out, std::vector<int32_t>& cta_off,
                     const std::vector<int32_t>* prio = nullptr) {
    grid = std::max(1, grid);
    std::vector<std::vector<int32_t>> lists(static_cast<size_t>(grid));
    std::vector<int64_t> load(static_cast<size_t>(grid), 0);
    using HE = std::pair<int64_t, int32_t>;  // (load, cta), min-heap
    std::priority_queue<HE, std::vector<HE>, std::greater<HE>> heap;
    for (int c = 0; c < grid; ++c) heap.push({0, c});
    for (int kind = kPieceS; kind <= kPieceE; ++kind) {
        std::vector<int32_t> idx;
        for (int32_t i = 0; i < int32_t(in.size()); ++i)
            if (in[size_t(i)].kind == kind) idx.push_back(i);
        // largest first; equal costs (most shrink pieces: 8 full A rows) by priority: the pieces of
        // the items whose expand pieces are largest first, so that their v is ready earliest
        std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t c) {
            if (cost[size_t(a)] != cost[size_t(c)]) return cost[size_t(a)] > cost[size_t(c)];
            return prio && (*prio)[size_t(a)] > (*prio)[size_t(c)];
        });
        for (int32_t i : idx) {
            HE h = heap.top();
            heap.pop();
            lists[size_t(h.second)].push_back(i);
            h.first += cost[size_t(i)];
            heap.push(h);
        }
    }
    out.clear();
    cta_off.assign(size_t(grid) + 1, 0);
    for (int c = 0; c < grid; ++c) {
        cta_off[size_t(c)] = int32_t(out.size());
        for (int32_t i : lists[size_t(c)]) out.push_back(in[size_t(i)]);
    }
    cta_off[size_t(grid)] = int32_t(out.size());
}

// Items = (segment x projection of the call x token chunk of <= kItemTokCap
// tokens); pieces: each item's stored A rows in groups of kShrinkRows (shrink,
// full K), and its output columns in chunks of kc.dchunk (expand), scheduled
// onto the kernel's persistent CTAs by schedule_pieces.
void build_call(slora_batch* b, const KernelCfg& k, int N, int nproj, uint32_t mask, slora_batch::Call& call,
                bool allow_mbgmm = true) {
    call.items.clear();
    call.pieces.clear();
    const slora_pool* pl = b->pool;
    int proj_ids[kMaxProj], np = 0;
    for (int pj = 0; pj < pl->np; ++pj)
        if (mask & (1u << pj)) proj_ids[np++] = pj;
    (void)nproj;
    const int es = pl->es;
    const int64_t P = pl->P;
    // B-row width of projection pj in this call: its output width (TP: this rank's H/N slice)
    auto proj_D = [&](int pj) -> int64_t { return N > 1 ? P : (k.mode == kShrink ? 0 : pl->pout[pj]); };
    bool all_square = true;  // MBGMM serves square projections only
    for (int i = 0; i < np; ++i)
        all_square = all_square && pl->pin[proj_ids[i]] == pl->cfg.hidden && pl->pout[proj_ids[i]] == pl->cfg.hidden;
    // expand column chunk per item (SLORA_HIRANK_SPLIT=r: items of rank >= r get
    // half-width chunks; off by default: measured slower on C2, 1.45-1.52 vs 1.42 ms)
    static const int hirank = [] {
        const char* e = getenv("SLORA_HIRANK_SPLIT");
        return e ? atoi(e) : 0;
    }();
    // Single-projection (o) calls: items of rank >= 64 get half-width expand
    // pieces, whose rank-64 pieces are otherwise the launch's stragglers
    // (measured on C2 decode with the rank-ordered schedule: o launch 14.06 us
    // at threshold 32, 13.56 at 64, 13.60 off; SLORA_O_HIRANK=r to move it, 0 = off)
    static const int o_hirank = [] {
        const char* e = getenv("SLORA_O_HIRANK");
        return e ? atoi(e) : 64;
    }();
    auto item_dchunk = [&](int rank) -> int64_t {  // divides the page (k.dchunk | P): pieces never straddle a page
        const int64_t half = k.dchunk / 2;
        if (hirank > 0 && rank >= hirank && half > 0 && P % half == 0 && (half * es) % 16 == 0) return half;
        if (o_hirank > 0 && np == 1 && rank >= o_hirank && half > 0 && P % half == 0 && (half * es) % 16 == 0)
            return half;
        return k.dchunk;
    };
    // expand pieces of one item: page by page over [0, D), chunks of dch within each page
    auto for_expand_chunks = [&](int64_t D, int64_t dch, auto&& fn) {
        if (dch <= 0) return;  // no expand configuration (bookkeeping pools)
        for (int64_t p0 = 0; p0 < D; p0 += P)
            for (int64_t c0 = p0; c0 < std::min(D, p0 + P); c0 += dch) fn(c0, std::min(dch, std::min(D, p0 + P) - c0));
    };
    auto item_n_ep = [&](int rank, int pj) -> int64_t {
        if (k.mode == kShrink || k.dchunk <= 0) return 0;
        int64_t n = 0;
        for_expand_chunks(proj_D(pj), item_dchunk(rank), [&](int64_t, int64_t) { ++n; });
        return n;
    };
    // stored A rows per shrink piece: 16 for calls of several projections, 8 for single-projection
    // (o) calls (measured on C2 decode with the rank-ordered schedule: q/k/v launch 22.80 -> 21.50 us
    // with 16 rows, o launch 13.57 -> 14.07 us: its shorter chain wants more, smaller pieces)
    static const int srows_multi = [] {
        const char* e = getenv("SLORA_SHRINK_ROWS_MULTI");
        return e ? std::max(1, std::min(kShrinkRows, atoi(e))) : std::min(kShrinkRows, 16);
    }();
    static const int srows_single = [] {
        const char* e = getenv("SLORA_SHRINK_ROWS_SINGLE");
        return e ? std::max(1, std::min(kShrinkRows, atoi(e))) : std::min(kShrinkRows, 8);
    }();
    const int srows = np == 1 ? srows_single : srows_multi;
    // (the MBGMM kernels index the default q,k,v,o page-table layout: square pools only)
    const bool use_runs = allow_mbgmm && k.mode == kFused && b->n_runs > 0 && all_square && pl->square;
    call.mg_s.clear();
    call.mg_e.clear();
    for (int si = 0; si < int(b->segs.size()); ++si) {
        const DevSeg& s = b->segs[size_t(si)];
        // MBGMV token ranges: the segment minus its MBGMM runs
        std::vector<std::pair<int32_t, int32_t>> ranges;
        int32_t cur = 0;
        if (use_runs)
            for (const auto& rn : b->runs[size_t(si)]) {
                if (rn.first > cur) ranges.push_back({cur, rn.first});
                cur = rn.second;
            }
        if (cur < s.n_tok) ranges.push_back({cur, s.n_tok});
        for (int pi = 0; pi < np; ++pi) {
            const int proj = proj_ids[pi];
            const int div = (k.mode == kExpand) ? 1 : ((proj < 3) ? N : 1);
            const int ra = s.rank / div;
            for (const auto& rg : ranges)
                for (int t0 = rg.first; t0 < rg.second; t0 += kItemTokCap) {
                    DevItem it{};
                    it.tab = b->seg_tab.empty() ? nullptr : b->seg_tab[size_t(si)];
                    it.vrow = s.vrow_off + int64_t(t0) * s.rank;
                    it.rank = s.rank;
                    it.seg = si;
                    it.pi = pi;
                    it.t0 = t0;
                    it.nt = std::min(kItemTokCap, rg.second - t0);
                    it.tok_off = s.tok_off + t0;
                    it.scale = s.scale;
                    it.n_sp = (k.mode == kExpand) ? 0 : (ra + srows - 1) / srows;
                    it.n_ep = int32_t(item_n_ep(s.rank, proj));
                    call.items.push_back(it);
                }
            if (!use_runs) continue;
            for (const auto& rn : b->runs[size_t(si)])
                for (int t0 = rn.first; t0 < rn.second; t0 += kMgTileTok) {
                    MgUnit u{};
                    u.tab = b->seg_tab.empty() ? nullptr : b->seg_tab[size_t(si)];
                    u.vbase = int64_t(pi) * b->NR + s.vrow_off + int64_t(t0) * s.rank;
                    u.pi = pi;
                    u.rank = s.rank;
                    // x-map row of the tile's first token: its x row, or (gathered) its tok_idx position
                    u.row0 = b->mg_gather ? s.tok_off + t0 : b->tok_idx[size_t(s.tok_off + t0)];
                    u.nt = std::min(kMgTileTok, rn.second - t0);
                    u.scale = s.scale;
                    const bool whole = mbgmm_shrink_whole_rank();
                    const int srows = whole ? s.rank : mbgmm_rows(k.K);  // A rows per shrink unit
                    const int split = mbgmm_split(k.K);
                    for (int r0 = 0; r0 < s.rank; r0 += srows)
                        for (int ks = 0; ks < split; ++ks) {  // k-split parts (the expand adds them in order)
                            u.a = r0;
                            u.b = std::min(srows, s.rank - r0);
                            u.pad = ks;
                            call.mg_s.push_back(u);
                        }
                    u.pad = 0;
                    const int ecols = mbgmm_expand_cols(s.rank);
                    for (int64_t c0 = 0; c0 < k.D; c0 += ecols) {
                        u.a = int32_t(c0);
                        u.b = int32_t(std::min<int64_t>(ecols, k.D - c0));
                        call.mg_e.push_back(u);
                    }
                }
        }
    }
    std::vector<DevPiece> pieces;
    std::vector<int64_t> cost;
    std::vector<int32_t> prio;  // tie-break among equal-cost pieces: the item's rank (see schedule_pieces)
    static const int64_t kPieceOverhead = [] {  // bytes-equivalent fixed cost of a piece (LPT weight)
        const char* e = getenv("SLORA_PIECE_OVH");
        return e ? int64_t(atoll(e)) : int64_t(4096);
    }();
    static const bool by_rank = [] {
        const char* e = getenv("SLORA_SCHED_PRIO");
        return !(e && atoi(e) == 0);
    }();
    for (int32_t ii = 0; ii < int32_t(call.items.size()); ++ii) {
        const DevItem& it = call.items[size_t(ii)];
        const int proj = proj_ids[it.pi];
        const int ra = it.rank / ((k.mode == kExpand) ? 1 : ((proj < 3) ? N : 1));
        if (k.mode != kExpand)
            for (int r0 = 0; r0 < ra; r0 += srows) {
                const int nr = std::min(srows, ra - r0);
                pieces.push_back({kPieceS, ii, r0, nr});
                cost.push_back(int64_t(nr) * k.K * es + kPieceOverhead);
                prio.push_back(by_rank ? it.rank : 0);
            }
        if (k.mode != kShrink)
            for_expand_chunks(proj_D(proj), item_dchunk(it.rank), [&](int64_t c0, int64_t dc) {
                pieces.push_back({kPieceE, ii, int32_t(c0), int32_t(dc)});
                cost.push_back(int64_t(it.rank) * dc * es + kPieceOverhead);
                prio.push_back(by_rank ? it.rank : 0);
            });
    }
    schedule_pieces(pieces, cost, k.grid, call.pieces, call.cta_off, &prio);
}
slora_status ensure_call(slora_pool* p, slora_batch* b, int kc, uint32_t mask, void* stream);

// The single-GPU fused call's configuration: the ring-pipeline MBGMV kernel (kcfg[0]).
int fused_kc(const slora_pool* p, int) { return p->fused_kc(p->cfg.hidden); }
}  // namespace

extern "C" slora_status slora_batch_prepare(slora_batch_t b, const int64_t* tok_adapter, int32_t T, void* stream) {
    if (!b) return fail(SLORA_ERR_INVALID_ARG, "null batch");
    if (!b->pool) return fail(SLORA_ERR_STALE_HANDLE, "the batch's pool was destroyed");
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
    // adapters still loading (slora_adapter_prefetch): the batch's stream waits for them
    for (int64_t a : seg_ad)
        if (slora_status st = load_fence(p, p->adapters.at(a), static_cast<cudaStream_t>(stream))) return st;
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
    // MBGMM runs: >= theta consecutive x rows of one adapter (fused, 16-bit, one GPU)
    b->runs.assign(b->segs.size(), {});
    b->n_runs = 0;
    b->mg_units_max = 0;
    {
        static const int theta = [] {
            const char* e = getenv("SLORA_MBGMM_MIN");
            return e ? atoi(e) : kMgDefaultTheta;
        }();
        const int mg_rows = mbgmm_rows(p->cfg.hidden);
        const int mg_split = mbgmm_split(p->cfg.hidden);
        const bool ok_shape = !(b->options & SLORA_BATCH_MBGMV_ONLY) && p->square && p->cfg.dtype != SLORA_F32 && p->N() == 1 &&
                              theta > 0 && p->cfg.hidden % 64 == 0 &&
                              p->cfg.hidden % kMgCols % 64 == 0 && mbgmm_smem(false, p->cfg.hidden, 0) <= 227 * 1024 &&
                              (p->cfg.hidden / 64) % mg_split == 0;
        for (size_t si = 0; ok_shape && si < b->segs.size(); ++si) {
            const DevSeg& sg = b->segs[si];
            int32_t t = 0;
            while (t < sg.n_tok) {
                int32_t e2 = t + 1;
                while (e2 < sg.n_tok && b->tok_idx[size_t(sg.tok_off + e2)] == b->tok_idx[size_t(sg.tok_off + e2 - 1)] + 1)
                    ++e2;
                if (e2 - t >= theta) {
                    b->runs[si].push_back({t, e2});
                    ++b->n_runs;
                    const int64_t tiles = (e2 - t + kMgTileTok - 1) / kMgTileTok;
                    b->mg_units_max += 4 * tiles * (mg_split * ((sg.rank + mg_rows - 1) / mg_rows) +
                                                    (p->cfg.hidden + kMgCols / 2 - 1) / (kMgCols / 2));
                }
                t = e2;
            }
        }
        // Gathered mode (reading R9: dispatch by segment token count, not by phase):
        // a batch with no consecutive runs (decode: every request contributes one
        // token) whose segments still hold >= theta_g tokens of one adapter sends
        // those whole segments to MBGMM; their x rows are gathered into a
        // contiguous workspace per call and y is written through tok_idx.
        static const int theta_g = [] {
            const char* e = getenv("SLORA_MBGMM_GATHER_MIN");
            return e ? atoi(e) : 4;  // measured on C4: 32 -> 16.2, 16 -> 13.0, 8 -> 12.2, 4 -> 10.2 ms/step (off: 18.0)
        }();
        // ... and only for rank >= 32: a rank-8 segment never pays for the gather
        // and the two extra launches (measured on C1, all rank 8: 0.71 -> 2.45
        // ms/step when its Zipf-head segments were gathered)
        static const int rank_g = [] {
            const char* e = getenv("SLORA_MBGMM_GATHER_RANK");
            return e ? atoi(e) : 32;
        }();
        // ... and only when those segments hold at least half of the adapted
        // tokens: the gather and the two MBGMM launches run before the call's
        // MBGMV launch, so one large segment in a decode batch does not pay
        // (measured on C3, one 18-token rank-64 segment of 64: 2.14 -> 4.07 ms)
        int64_t gather_tok = 0;
        for (const DevSeg& sg : b->segs)
            if (sg.n_tok >= theta_g && sg.rank >= rank_g) gather_tok += sg.n_tok;
        b->mg_gather = false;
        if (ok_shape && b->n_runs == 0 && theta_g > 0 && 2 * gather_tok >= b->adapted)
            for (size_t si = 0; si < b->segs.size(); ++si) {
                const DevSeg& sg = b->segs[si];
                if (sg.n_tok < theta_g || sg.rank < rank_g) continue;
                b->runs[si].push_back({0, sg.n_tok});
                ++b->n_runs;
                b->mg_gather = true;
                const int64_t tiles = (sg.n_tok + kMgTileTok - 1) / kMgTileTok;
                b->mg_units_max += 4 * tiles * (mg_split * ((sg.rank + mg_rows - 1) / mg_rows) +
                                                (p->cfg.hidden + kMgCols / 2 - 1) / (kMgCols / 2));
            }
    }
    for (auto& row : b->calls)
        for (auto& c : row) c.built = false;
    b->epoch = p->epoch;
    b->prepared = true;
    if (!p->dev) {
        // bookkeeping pools still build the descriptors (tested on CPU)
        for (int np = 1; np <= 4; ++np) build_call(b, p->kcfg[0], p->N(), np, (1u << np) - 1, b->calls[0][np]);
        return ok();
    }
    // ---- device arena: tok_idx now, call descriptors on first use.  Sized
    // for every call this prepare can see (items <= segs*4*chunks).
    int64_t chunks = 0;
    for (const DevSeg& s : b->segs) chunks += (s.n_tok + kItemTokCap - 1) / kItemTokCap;
    const int64_t max_items = std::max(kNumProj, p->np) * chunks;
    // ring kernel: <= ceil(r/8) shrink pieces + D/(dchunk/2) expand pieces per item
    const int64_t dmin = std::max<int64_t>(1, p->kcfg[0].dchunk / 2);
    int64_t max_out = p->cfg.hidden, max_in = p->cfg.hidden;
    for (int q = 0; q < p->np; ++q) {
        max_out = std::max(max_out, p->pout[q]);
        max_in = std::max(max_in, p->pin[q]);
    }
    (void)max_in;
    const int64_t max_pieces_per_item =
        kMaxRank /* shrink pieces: at most one per rank row */ + (max_out + dmin - 1) / dmin + (max_out + p->P - 1) / p->P;
    int n_shapes = 6;  // eager shapes + those launched since create (rebuilt below)
    for (auto& row : b->used_masks)
        for (uint32_t m : row) n_shapes += m ? 1 : 0;
    const size_t need = 256 + size_t(T) * 4 + size_t(n_shapes) * (1024 + 4 * 1024 + size_t(b->mg_units_max) * sizeof(MgUnit) +
                                                   size_t(max_items) * sizeof(DevItem) +
                                                   size_t(max_items * max_pieces_per_item) * sizeof(DevPiece));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    // the mirror pair of two prepares ago: free once its uploads completed (the host runs up to one
    // step ahead of the GPU without waiting)
    b->cur ^= 1;
    if (b->pending[b->cur]) CUDA_TRY(cudaEventSynchronize(b->upload_evs[b->cur]));
    b->pending[b->cur] = false;
    if (need > b->arena_cap) {
        for (int i = 0; i < 2; ++i) {
            if (b->pending[i]) CUDA_TRY(cudaEventSynchronize(b->upload_evs[i]));
            b->pending[i] = false;
            if (b->arena_host_buf[i]) CUDA_TRY(cudaFreeHost(b->arena_host_buf[i]));
            b->arena_host_buf[i] = nullptr;
        }
        if (b->arena_dev) CUDA_TRY(cudaFreeAsync(b->arena_dev, s));
        b->arena_dev = nullptr;
        const size_t cap = need + need / 4;  // sized from this batch's call shapes; grows at a later prepare
        for (int i = 0; i < 2; ++i) CUDA_TRY(cudaHostAlloc(&b->arena_host_buf[i], cap, cudaHostAllocDefault));
        CUDA_TRY(cudaMallocAsync(&b->arena_dev, cap, s));
        b->arena_cap = cap;
    }
    b->arena_used = 0;
    b->dirty_lo = b->dirty_hi = 0;
    b->in_prepare = true;
    struct PrepGuard {
        slora_batch* b;
        ~PrepGuard() { b->in_prepare = false; }
    } prep_guard{b};
    cudaError_t e = cudaSuccess;
    b->off_tok = arena_put(b, b->tok_idx.data(), b->tok_idx.size() * sizeof(int32_t), s, e);
    if (e) return fail(SLORA_ERR_CUDA, "batch upload: %s", cudaGetErrorString(e));
    // per-launch sync slots and fused workspace, sized for this batch
    const int64_t sync_need = 2 + max_items + 32;
    // workspace slot = three regions of ws_need floats: the ring kernel's v,
    // the warp-task kernel's v (readiness flags, kept "empty" between
    // launches) and MBGMM's v
    const int64_t ws_need = std::max(kNumProj, p->np) * b->NR + 64;
    if (sync_need > p->sync_stride) {
        if (p->sync_dev) CUDA_TRY(cudaFreeAsync(p->sync_dev, s));
        const int64_t st = sync_need * 2;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p->sync_dev), sizeof(int32_t) * st * kLaunchSlots, s));
        CUDA_TRY(cudaMemsetAsync(p->sync_dev, 0, sizeof(int32_t) * st * kLaunchSlots, s));
        p->sync_stride = st;
    }
    if (b->mg_gather) {  // gathered MBGMM rows: all adapted tokens in tok_idx order
        const size_t xg_need = size_t(b->adapted) * size_t(p->cfg.hidden) * size_t(p->es);
        if (xg_need > p->xg_cap) {
            if (p->xg_dev) CUDA_TRY(cudaFreeAsync(p->xg_dev, s));
            CUDA_TRY(cudaMallocAsync(&p->xg_dev, xg_need, s));
            p->xg_cap = xg_need;
        }
    }
    if (ws_need > p->ws_stride) {
        if (p->ws_dev) CUDA_TRY(cudaFreeAsync(p->ws_dev, s));
        const int64_t st = ws_need * (2 + kMgVParts);
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p->ws_dev), sizeof(float) * st * kLaunchSlots, s));
        CUDA_TRY(cudaMemsetAsync(p->ws_dev, 0xFF, sizeof(float) * st * kLaunchSlots, s));
        p->ws_stride = st;
        p->ws_region = ws_need;
    }
    // tensor-parallel exchange buffers (slora_tp_*): 3*NR/N, 3*NR and NR fp32
    if (p->tp_comm && b->NR > p->tp_cap) {
        const int64_t cap = b->NR * 2;
        for (float** buf : {&p->tp_vloc, &p->tp_vall, &p->tp_u})
            if (*buf) CUDA_TRY(cudaFreeAsync(*buf, s));
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p->tp_vloc), sizeof(float) * size_t(3 * cap), s));
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p->tp_vall), sizeof(float) * size_t(3 * cap), s));
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p->tp_u), sizeof(float) * size_t(cap), s));
        p->tp_cap = cap;
    }
    // eager descriptors for the usual calls (q/k/v together, o alone)
    slora_status st2 = SLORA_OK;
    if (b->adapted > 0) {
        if (p->N() == 1) {
            if (!st2) st2 = ensure_call(p, b, fused_kc(p, 3), 0x7, stream);
            if (!st2) st2 = ensure_call(p, b, fused_kc(p, 1), 0x8, stream);
        }
        // split (TP) calls: eagerly whenever they can run, so that a CUDA graph
        // of slora_tp_lora_* captures kernel launches and NCCL calls only
        if (p->N() > 1 || p->tp_comm) {
            const int kc_o = p->N() > 1 ? 2 : 1;  // the o shrink's configuration (slora_lora_shrink)
            if (!st2 && p->kcfg[1].ok) st2 = ensure_call(p, b, 1, 0x7, stream);
            if (!st2 && p->kcfg[kc_o].ok) st2 = ensure_call(p, b, kc_o, 0x8, stream);
            if (!st2 && p->kcfg[3].ok) st2 = ensure_call(p, b, 3, 0x7, stream);
            if (!st2 && p->kcfg[3].ok) st2 = ensure_call(p, b, 3, 0x8, stream);
        }
    }
    if (!st2 && p->p2p_open && b->adapted > 0) {  // device-initiated TP calls (slora_tp_fused_*)
        st2 = ensure_call(p, b, p->kc_tpf_qkv, 0x7, stream);
        if (!st2) st2 = ensure_call(p, b, p->kc_tpf_o, 0x8, stream);
    }
    // every call shape launched since the batch was created is rebuilt too, and all headers
    // are uploaded with the descriptors in one flush: a CUDA graph that captured those
    // launches replays the new batch (MBGMV path; see slora_batch_get_info().graph_ok)
    for (int kc = 0; kc < p->n_kcfg && !st2; ++kc)
        for (int np = 1; np <= kMaxProj && !st2; ++np)
            if (b->used_masks[kc][np] && p->kcfg[kc].ok) st2 = ensure_call(p, b, kc, b->used_masks[kc][np], stream);
    b->in_prepare = false;
    if (st2) return st2;
    if (cudaError_t e = arena_flush(b, s)) return fail(SLORA_ERR_CUDA, "batch upload: %s", cudaGetErrorString(e));
    return ok();
}

extern "C" slora_status slora_batch_set_options(slora_batch_t b, uint32_t flags) {
    if (!b) return fail(SLORA_ERR_INVALID_ARG, "null batch");
    if (flags & ~uint32_t(SLORA_BATCH_MBGMV_ONLY)) return fail(SLORA_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
    b->options = flags;
    return ok();
}

extern "C" slora_status slora_batch_get_info(slora_batch_t b, slora_batch_info* out) {
    if (!b || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    out->T = b->T;
    out->adapted_tokens = b->adapted;
    out->segments = int32_t(b->segs.size());
    out->sum_rank_tokens = b->NR;
    out->weight_bytes_per_proj = b->weight_bytes_per_proj;
    out->mbgmm_segments = b->n_runs;
    return ok();
}

// ----------------------------------------------------------------- compute
namespace {
slora_status common_checks(slora_pool* p, slora_batch* b, int32_t layer, uint32_t mask) {
    if (!p || !b) return fail(SLORA_ERR_INVALID_ARG, "null pool/batch");
    if (!b->pool) return fail(SLORA_ERR_STALE_HANDLE, "the batch's pool was destroyed");
    if (b->pool != p) return fail(SLORA_ERR_INVALID_ARG, "batch belongs to another pool");
    if (!p->dev) return fail(SLORA_ERR_NO_DEVICE, "bookkeeping-only pool");
    if (!b->prepared) return fail(SLORA_ERR_INVALID_ARG, "batch not prepared");
    if (b->epoch != p->epoch) return fail(SLORA_ERR_STALE_HANDLE, "batch prepared before an eviction");
    if (layer < 0 || layer >= p->cfg.num_layers) return fail(SLORA_ERR_INVALID_ARG, "layer %d", layer);
    if (mask == 0 || (mask >> p->np)) return fail(SLORA_ERR_INVALID_ARG, "proj_mask 0x%x (%d projections)", mask, p->np);
    int64_t K = -1;  // the projections of one call read the same x
    for (int pj = 0; pj < p->np; ++pj)
        if (mask & (1u << pj)) {
            if (K >= 0 && p->pin[pj] != K)
                return fail(SLORA_ERR_SHAPE, "proj_mask 0x%x mixes input widths (%lld, %lld)", mask, (long long)K,
                            (long long)p->pin[pj]);
            K = p->pin[pj];
        }
    return SLORA_OK;
}

int popcount_mask(uint32_t mask) {
    int n = 0;
    for (int pj = 0; pj < kMaxProj; ++pj) n += (mask >> pj) & 1;
    return n;
}
// input width of a call's projections (common_checks makes them agree)
int64_t mask_in(const slora_pool* p, uint32_t mask) {
    for (int pj = 0; pj < p->np; ++pj)
        if (mask & (1u << pj)) return p->pin[pj];
    return p->cfg.hidden;
}

bool aligned16(const void* ptr, int64_t ld, int es) {
    return !(reinterpret_cast<uintptr_t>(ptr) & 15) && (ld * es) % 16 == 0;
}

// Build + upload the (kernel cfg, mask) call descriptor if this prepare has not
// yet (prepare builds the usual q/k/v and o calls eagerly so that a captured
// CUDA graph of the layer sequence contains kernel launches only).
slora_status ensure_call(slora_pool* p, slora_batch* b, int kc, uint32_t mask, void* stream) {
    const int np = popcount_mask(mask);
    slora_batch::Call& call = b->calls[kc][np];
    if (call.built && call.mask == mask) return SLORA_OK;
    if (!p->kcfg[kc].ok) return fail(SLORA_ERR_SHAPE, "no valid kernel configuration");
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (p->dev && cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cap) == cudaSuccess &&
        cap != cudaStreamCaptureStatusNone)
        return fail(SLORA_ERR_INVALID_ARG, "call descriptor (kernel cfg %d, mask 0x%x) not built by the last prepare: "
                    "a CUDA graph may only capture calls whose descriptors exist (run the call once eagerly "
                    "after prepare, or use the calls prepare builds)", kc, mask);
    // the device-initiated TP calls are one MBGMV kernel each: every segment on MBGMV
    build_call(b, p->kcfg[kc], p->N(), np, mask, call, kc != p->kc_tpf_qkv && kc != p->kc_tpf_o);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    call.off_items = arena_put(b, call.items.data(), call.items.size() * sizeof(DevItem), s, e);
    if (!e) call.off_pieces = arena_put(b, call.pieces.data(), call.pieces.size() * sizeof(DevPiece), s, e);
    if (!e) call.off_cta = arena_put(b, call.cta_off.data(), call.cta_off.size() * sizeof(int32_t), s, e);
    if (!e) call.off_mg_s = arena_put(b, call.mg_s.data(), call.mg_s.size() * sizeof(MgUnit), s, e);
    if (!e) call.off_mg_e = arena_put(b, call.mg_e.data(), call.mg_e.size() * sizeof(MgUnit), s, e);
    if (e) return fail(SLORA_ERR_CUDA, "call descriptor upload: %s", cudaGetErrorString(e));
    call.built = true;
    call.mask = mask;
    if (p->dev) {
        if (!b->in_prepare && b->pending[b->cur]) cudaEventSynchronize(b->upload_evs[b->cur]);  // mirror free
        set_hdr(p, b, kc, np);
        if (!b->in_prepare) {  // built lazily by a call: upload now (prepare flushes once at its end)
            if ((e = arena_flush(b, s))) return fail(SLORA_ERR_CUDA, "call descriptor upload: %s", cudaGetErrorString(e));
        }
    }
    return SLORA_OK;
}

// Resolve (building + uploading on first use) the call descriptor and fill the
// launch parameters common to all modes.
slora_status prepare_call(slora_pool* p, slora_batch* b, int kc, int32_t layer, uint32_t mask, void* stream,
                          LoraParams& q) {
    const KernelCfg& k = p->kcfg[kc];
    if (!k.ok) return fail(SLORA_ERR_SHAPE, "no valid kernel configuration for K=%lld D=%lld", (long long)k.K,
                           (long long)k.D);
    memset(&q, 0, sizeof(q));
    int np = 0;
    for (int pj = 0; pj < p->np; ++pj)
        if (mask & (1u << pj)) q.proj_ids[np++] = pj;
    q.nproj = np;
    // descriptors depend on the mask only through np and which projections
    // are q/k/v vs o (the stored-row divisor under TP); key by (kc, np) and
    // rebuild when the o-ness of the mask differs
    slora_batch::Call& call = b->calls[kc][np];
    slora_status cs = ensure_call(p, b, kc, mask, stream);
    if (cs) return cs;
    (void)call;
    b->used_masks[kc][np] = mask;
    q.pool = p->cfg.device_buffer;
    q.page_elems = p->P;
    q.hdr = b->hdr_dev + (kc * kNpSlots + np);
    const uint64_t slot = p->launch_seq++ % kLaunchSlots;
    q.slot = int32_t(slot);
    q.layer = layer;
    q.K = int32_t(k.K);
    q.D = int32_t(k.D);
    q.ns = k.ns;
    static const int dbg = [] {
        const char* e = getenv("SLORA_DBG");
        return e ? atoi(e) : 0;
    }();
    q.dbg = dbg;
    const int N = p->N();
    q.layer_units = p->layer_units;
    for (int pj = 0; pj < p->np; ++pj) {
        int rows, ch;
        p->tensor_shape(pj, 0, N, rows, ch);
        q.a_div[pj] = (N > 1 && pj < 3) ? N : 1;
        q.a_row_pages[pj] = ch;
        q.a_units[pj] = p->a_units[pj];
        q.b_row_pages[pj] = p->b_row_pages[pj];
        q.proj_off[pj] = p->proj_off[pj];
    }
    p->ws_slot_base = p->ws_dev + int64_t(slot) * p->ws_stride;  // MBGMM's regions of the slot (host-baked)
    q.trace = p->trace_dev;
    return SLORA_OK;
}

slora_status launch(slora_pool* p, int kc, LoraParams& q, void* stream) {
    const KernelCfg& k = p->kcfg[kc];
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    const int dt = p->cfg.dtype == SLORA_F32 ? kF32 : (p->cfg.dtype == SLORA_F16 ? kF16 : kBF16);
    CUDA_TRY(launch_lora(q, k.mode, dt, k.grid, static_cast<cudaStream_t>(stream), k.smem));
    return ok();
}
}  // namespace

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// The two MBGMM launches of a fused call with long runs (shrink into the
// call's workspace, then expand into y); the MBGMV launch for the remaining
// tokens follows on the same stream.
slora_status launch_mbgmm_pair(slora_pool* p, slora_batch* b, const slora_batch::Call& call, const LoraParams& q,
                               const void* x, int64_t ldx, void* stream) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return fail(SLORA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    MgParams m;
    memset(&m, 0, sizeof(m));
    const int64_t H = p->cfg.hidden;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint8_t* base = static_cast<uint8_t*>(b->arena_dev);
    const int32_t* tok_dev = reinterpret_cast<const int32_t*>(base + b->off_tok);
    if (b->mg_gather) {  // x rows of the batch in tok_idx order -> the contiguous workspace
        CUDA_TRY(launch_gather_rows(x, ldx, tok_dev, b->adapted, p->xg_dev, H, p->es, s));
        x = p->xg_dev;
        ldx = H;
    }
    const cuuint64_t dims[2] = {cuuint64_t(H), cuuint64_t(b->mg_gather ? b->adapted : b->T)};
    const cuuint64_t strides[1] = {cuuint64_t(ldx) * cuuint64_t(p->es)};
    const cuuint32_t box[2] = {64, cuuint32_t(kMgTileTok)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&m.xmap, p->cfg.dtype == SLORA_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                      2, const_cast<void*>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SLORA_ERR_CUDA, "cuTensorMapEncodeTiled: %d", int(cr));
    m.pool = p->cfg.device_buffer;
    m.yrow = b->mg_gather ? tok_dev : nullptr;
    m.page_elems = p->P;
    m.v = p->ws_slot_base + 2 * p->ws_region;  // the slot's MBGMM regions (see slora_batch_prepare)
    m.ksplit = mbgmm_split(H);
    m.srows = mbgmm_rows(H);
    m.vpart = p->ws_region;
    for (int pj = 0; pj < 4; ++pj) {
        m.y[pj] = q.y[pj];
        m.ldy[pj] = q.ldy[pj];
        m.proj_ids[pj] = q.proj_ids[pj];
    }
    m.layer = q.layer;
    m.K = int32_t(H);
    size_t esmem = 0;
    for (const MgUnit& u : call.mg_e) esmem = std::max(esmem, mbgmm_smem(true, 0, u.rank));
    const int dt = p->cfg.dtype == SLORA_F16 ? kF16 : kBF16;
    m.units = reinterpret_cast<const MgUnit*>(base + call.off_mg_s);
    CUDA_TRY(launch_mbgmm(m, false, dt, int(call.mg_s.size()), mbgmm_smem(false, H, 0), s, true));
    m.units = reinterpret_cast<const MgUnit*>(base + call.off_mg_e);
    CUDA_TRY(launch_mbgmm(m, true, dt, int(call.mg_e.size()), esmem, s, true));
    return SLORA_OK;
}
}  // namespace

extern "C" slora_status slora_lora_apply(slora_pool_t p, slora_batch_t b, int32_t layer, uint32_t mask,
                                         const void* x, int64_t ldx, void* const y[SLORA_MAX_PROJ], const int64_t ldy[SLORA_MAX_PROJ],
                                         void* stream) {
    slora_status st = common_checks(p, b, layer, mask);
    if (st) return st;
    if (p->N() != 1) return fail(SLORA_ERR_INVALID_ARG, "slora_lora_apply is single-GPU; use shrink/expand under TP");
    if (b->adapted == 0) return ok();
    if (!x || !y || !ldy) return fail(SLORA_ERR_INVALID_ARG, "null x/y");
    const int64_t K = mask_in(p, mask);
    if (!aligned16(x, ldx, p->es) || ldx < K) return fail(SLORA_ERR_SHAPE, "x alignment/stride");
    for (int pj = 0; pj < p->np; ++pj)
        if (mask & (1u << pj))
            if (!y[pj] || !aligned16(y[pj], ldy[pj], p->es) || ldy[pj] < p->pout[pj])
                return fail(SLORA_ERR_SHAPE, "y[%d] alignment/stride", pj);
    const int kc = p->fused_kc(K);
    if (kc < 0) return fail(SLORA_ERR_SHAPE, "no fused kernel configuration for input width %lld", (long long)K);
    LoraParams q;
    st = prepare_call(p, b, kc, layer, mask, stream, q);
    if (st) return st;
    q.x = x;
    q.ldx = ldx;
    for (int pj = 0; pj < p->np; ++pj) {
        q.y[pj] = y[pj];
        q.ldy[pj] = ldy[pj];
    }
    q.v_blocks = 1;
    const slora_batch::Call& call = b->calls[kc][q.nproj];
    if (!call.mg_s.empty()) {
        st = launch_mbgmm_pair(p, b, call, q, x, ldx, stream);
        if (st) return st;
        // every token went to MBGMM: no MBGMV launch (a batch with MBGMM segments is outside the
        // replay-across-batches guarantee anyway, see slora_batch_set_options)
        if (call.pieces.empty()) return ok();
    }
    return launch(p, kc, q, stream);
}

extern "C" slora_status slora_lora_apply_many(slora_pool_t p, slora_batch_t b, const slora_call* calls,
                                              int32_t n_calls, void* stream, int32_t* failed_out) {
    if (failed_out) *failed_out = -1;
    if (n_calls < 0 || (n_calls > 0 && !calls)) return fail(SLORA_ERR_INVALID_ARG, "calls");
    for (int32_t i = 0; i < n_calls; ++i) {
        const slora_call& c = calls[i];
        if (slora_status st = slora_lora_apply(p, b, c.layer, c.proj_mask, c.x, c.ldx, c.y, c.ldy, stream)) {
            if (failed_out) *failed_out = i;
            return st;
        }
    }
    return ok();
}

extern "C" slora_status slora_lora_v_elems(slora_batch_t b, uint32_t mask, int32_t div, int64_t* out) {
    if (!b || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    if (mask == 0 || (mask >> kMaxProj) || div < 1) return fail(SLORA_ERR_INVALID_ARG, "mask/div");
    const int np = popcount_mask(mask);
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
    if (N == 1 && mask_in(p, mask) != K)
        return fail(SLORA_ERR_SHAPE, "split shrink serves input width %lld only", (long long)K);
    if (!x || !v) return fail(SLORA_ERR_INVALID_ARG, "null x/v");
    if (!aligned16(x, ldx, p->es) || ldx < K) return fail(SLORA_ERR_SHAPE, "x alignment/stride");
    LoraParams q;
    st = prepare_call(p, b, kc, layer, mask, stream, q);
    if (st) return st;
    q.x = x;
    q.ldx = ldx;
    q.v = v;
    return launch(p, kc, q, stream);
}

extern "C" slora_status slora_lora_expand(slora_pool_t p, slora_batch_t b, int32_t layer, uint32_t mask,
                                          const float* v, int32_t v_blocks, void* const y[SLORA_MAX_PROJ], const int64_t ldy[SLORA_MAX_PROJ],
                                          void* stream) {
    slora_status st = common_checks(p, b, layer, mask);
    if (st) return st;
    if (v_blocks < 1) return fail(SLORA_ERR_INVALID_ARG, "v_blocks");
    if (b->adapted == 0) return ok();
    for (const DevSeg& s : b->segs)
        if (s.rank % v_blocks) return fail(SLORA_ERR_INDIVISIBLE, "rank %d %% v_blocks %d", s.rank, v_blocks);
    if (!v || !y || !ldy) return fail(SLORA_ERR_INVALID_ARG, "null v/y");
    for (int pj = 0; pj < p->np; ++pj)
        if (mask & (1u << pj))
            if (!y[pj] || !aligned16(y[pj], ldy[pj], p->es) || ldy[pj] < (p->N() > 1 ? p->P : p->pout[pj]))
                return fail(SLORA_ERR_SHAPE, "y[%d] alignment/stride", pj);
    LoraParams q;
    st = prepare_call(p, b, 3, layer, mask, stream, q);
    if (st) return st;
    q.v_in = v;
    q.v_blocks = v_blocks;
    for (int pj = 0; pj < p->np; ++pj) {
        q.y[pj] = y[pj];
        q.ldy[pj] = ldy[pj];
    }
    return launch(p, 3, q, stream);
}

// ---------------------------------------------------------- a6/a8: TP
extern "C" slora_status slora_tp_unique_id(void* id_out) {
    if (!id_out) return fail(SLORA_ERR_INVALID_ARG, "null id_out");
    static_assert(sizeof(ncclUniqueId) == SLORA_TP_ID_BYTES, "ncclUniqueId size");
    NcclApi& n = nccl();
    if (!n.ok) return fail(SLORA_ERR_NCCL, "NCCL unavailable: %s", n.why.c_str());
    ncclUniqueId id;
    const ncclResult_t r = n.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(SLORA_ERR_NCCL, "ncclGetUniqueId: %s", n.GetErrorString(r));
    memcpy(id_out, &id, sizeof(id));
    return ok();
}

extern "C" slora_status slora_tp_init(slora_pool_t p, const void* id, int32_t rank, int32_t size) {
    if (check_pool(p) || !id) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    if (!p->dev) return fail(SLORA_ERR_NO_DEVICE, "bookkeeping-only pool");
    if (size != p->cfg.tp_size || rank != p->cfg.tp_rank)
        return fail(SLORA_ERR_INVALID_ARG, "rank/size %d/%d differ from the pool's tp_rank/tp_size %d/%d", rank, size,
                    p->cfg.tp_rank, p->cfg.tp_size);
    if (p->tp_comm) return fail(SLORA_ERR_INVALID_ARG, "communicator already initialized");
    NcclApi& n = nccl();
    if (!n.ok) return fail(SLORA_ERR_NCCL, "NCCL unavailable: %s", n.why.c_str());
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    const ncclResult_t r = n.CommInitRank(&p->tp_comm, size, uid, rank);
    if (r != ncclSuccess) {
        p->tp_comm = nullptr;
        return fail(SLORA_ERR_NCCL, "ncclCommInitRank: %s", n.GetErrorString(r));
    }
    return ok();
}

namespace {
slora_status tp_checks(slora_pool* p, slora_batch* b) {
    if (!p || !b) return fail(SLORA_ERR_INVALID_ARG, "null pool/batch");
    if (!p->tp_comm) return fail(SLORA_ERR_INVALID_ARG, "no communicator: call slora_tp_init first");
    if (b->adapted > 0 && b->NR > p->tp_cap)
        return fail(SLORA_ERR_SHAPE, "exchange buffers hold NR=%lld < %lld: prepare the batch after slora_tp_init",
                    (long long)p->tp_cap, (long long)b->NR);
    return SLORA_OK;
}
}  // namespace

extern "C" slora_status slora_tp_lora_qkv(slora_pool_t p, slora_batch_t b, int32_t layer, const void* x,
                                          int64_t ldx, void* const y[3], const int64_t ldy[3], void* stream) {
    slora_status st = tp_checks(p, b);
    if (st) return st;
    if (b->adapted == 0) return ok();
    if (!y || !ldy) return fail(SLORA_ERR_INVALID_ARG, "null y");
    const int N = p->N();
    int64_t n_loc = 0;
    if ((st = slora_lora_v_elems(b, 0x7, N, &n_loc))) return st;
    if ((st = slora_lora_shrink(p, b, layer, 0x7, x, ldx, p->tp_vloc, stream))) return st;
    NcclApi& n = nccl();
    const ncclResult_t r = n.AllGather(p->tp_vloc, p->tp_vall, size_t(n_loc), ncclFloat, p->tp_comm,
                                       static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return fail(SLORA_ERR_NCCL, "ncclAllGather: %s", n.GetErrorString(r));
    p->tp_stats.allgather_calls += 1;
    p->tp_stats.allgather_send_elems += int64_t(N - 1) * n_loc;  // this rank's shard to each of N-1 peers
    p->tp_stats.allgather_recv_elems += int64_t(N - 1) * n_loc;
    void* ys[4] = {y[0], y[1], y[2], nullptr};
    const int64_t lds[4] = {ldy[0], ldy[1], ldy[2], 0};
    return slora_lora_expand(p, b, layer, 0x7, p->tp_vall, N, ys, lds, stream);
}

extern "C" slora_status slora_tp_lora_o(slora_pool_t p, slora_batch_t b, int32_t layer, const void* z, int64_t ldz,
                                        void* base_partial, int64_t ld_base, void* stream) {
    slora_status st = tp_checks(p, b);
    if (st) return st;
    if (b->adapted == 0) return ok();
    if (!base_partial || ld_base < p->cfg.hidden) return fail(SLORA_ERR_INVALID_ARG, "base partial / stride");
    const int N = p->N();
    int64_t n_u = 0;
    if ((st = slora_lora_v_elems(b, 0x8, 1, &n_u))) return st;
    if ((st = slora_lora_shrink(p, b, layer, 0x8, z, ldz, p->tp_u, stream))) return st;
    NcclApi& n = nccl();
    const ncclResult_t r = n.AllReduce(p->tp_u, p->tp_u, size_t(n_u), ncclFloat, ncclSum, p->tp_comm,
                                       static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return fail(SLORA_ERR_NCCL, "ncclAllReduce: %s", n.GetErrorString(r));
    p->tp_stats.allreduce_calls += 1;
    p->tp_stats.allreduce_count += n_u;
    p->tp_stats.allreduce_send_elems += 2 * int64_t(N - 1) * n_u / N;  // ring: reduce-scatter + all-gather
    // fold (reading R13): the expand writes column slice k of the base partial sum
    void* ys[4] = {nullptr, nullptr, nullptr,
                   static_cast<uint8_t*>(base_partial) + size_t(int64_t(p->cfg.tp_rank) * p->P) * p->es};
    const int64_t lds[4] = {0, 0, 0, ld_base};
    return slora_lora_expand(p, b, layer, 0x8, p->tp_u, 1, ys, lds, stream);
}

// ------------------------------------------- NEXT-3: device-initiated TP exchange
namespace {
constexpr int64_t kP2PVcap = int64_t(3) * 65536;  // floats per rank block: 3 NR/N (q/k/v) or NR (o) <= this
constexpr int64_t kP2PCcap = 65536;                 // per-item counters per launch slot
size_t p2p_bytes(int N) {
    return sizeof(float) * size_t(kLaunchSlots) * size_t(N) * size_t(kP2PVcap) +
           sizeof(int32_t) * size_t(kLaunchSlots) * size_t(kP2PCcap);
}
}  // namespace

extern "C" slora_status slora_tp_p2p_export(slora_pool_t p, void* handle_out) {
    if (check_pool(p) || !handle_out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    if (!p->dev) return fail(SLORA_ERR_NO_DEVICE, "bookkeeping-only pool");
    const int N = p->N();
    if (N > 8) return fail(SLORA_ERR_SHAPE, "tp_size %d > 8", N);
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    if (!p->p2p_local) {
        CUDA_TRY(cudaMalloc(&p->p2p_local, p2p_bytes(N)));
        CUDA_TRY(cudaMemset(p->p2p_local, 0, p2p_bytes(N)));
        CUDA_TRY(cudaDeviceSynchronize());
        p->p2p_vcap = kP2PVcap;
        p->p2p_ccap = kP2PCcap;
        // fused configurations: q/k/v (K = hidden: stored A rows span N pages; B rows of H/N) and o (K = H/N)
        const int dt = p->cfg.dtype == SLORA_F32 ? kF32 : (p->cfg.dtype == SLORA_F16 ? kF16 : kBF16);
        if (p->n_kcfg + 2 > kMaxKc) return fail(SLORA_ERR_SHAPE, "no kernel configuration slot left");
        p->kc_tpf_qkv = p->n_kcfg;
        p->kcfg[p->n_kcfg++] = make_kernel_cfg(kFused, p->cfg.hidden, p->P, p->P, p->es, dt);
        p->kc_tpf_o = p->n_kcfg;
        p->kcfg[p->n_kcfg++] = make_kernel_cfg(kFused, p->P, p->P, p->P, p->es, dt);
    }
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, p->p2p_local));
    static_assert(sizeof(cudaIpcMemHandle_t) <= SLORA_TP_P2P_HANDLE_BYTES, "IPC handle size");
    memset(handle_out, 0, SLORA_TP_P2P_HANDLE_BYTES);
    memcpy(handle_out, &h, sizeof(h));
    return ok();
}

extern "C" slora_status slora_tp_p2p_open(slora_pool_t p, const void* handles) {
    if (check_pool(p) || !handles) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    if (!p->p2p_local) return fail(SLORA_ERR_INVALID_ARG, "call slora_tp_p2p_export first");
    if (p->p2p_open) return fail(SLORA_ERR_INVALID_ARG, "already open");
    const int N = p->N(), k = p->cfg.tp_rank;
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    for (int j = 0; j < N; ++j) {
        if (j == k) {
            p->p2p_base[j] = p->p2p_local;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, static_cast<const uint8_t*>(handles) + size_t(j) * SLORA_TP_P2P_HANDLE_BYTES, sizeof(h));
        cudaError_t e = cudaIpcOpenMemHandle(&p->p2p_base[j], h, cudaIpcMemLazyEnablePeerAccess);
        if (e) {
            for (int i = 0; i < j; ++i)
                if (i != k && p->p2p_base[i]) cudaIpcCloseMemHandle(p->p2p_base[i]);
            for (auto& b : p->p2p_base) b = nullptr;
            return fail(SLORA_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", j, cudaGetErrorString(e));
        }
    }
    p->p2p_open = true;
    return ok();
}

namespace {
// Fill the device-initiated TP fields of a prepared call: this launch slot's block of every rank.
slora_status p2p_params(slora_pool* p, slora_batch* b, uint32_t mask, LoraParams& q) {
    const int N = p->N();
    const int64_t need = (mask == 0x8) ? b->NR : 3 * (b->NR / N);
    if (need > p->p2p_vcap) return fail(SLORA_ERR_SHAPE, "exchange block holds %lld < %lld floats",
                                        (long long)p->p2p_vcap, (long long)need);
    if (int64_t(b->calls[mask == 0x8 ? p->kc_tpf_o : p->kc_tpf_qkv][mask == 0x8 ? 1 : 3].items.size()) > p->p2p_ccap)
        return fail(SLORA_ERR_SHAPE, "more items than exchange counters");
    const int64_t vslot = int64_t(q.slot) * N * p->p2p_vcap;
    const int64_t cslot = int64_t(q.slot) * p->p2p_ccap;
    const int64_t voff_ctr = int64_t(kLaunchSlots) * N * p->p2p_vcap;  // floats before the counters
    for (int j = 0; j < N; ++j) {
        float* vb = static_cast<float*>(p->p2p_base[j]);
        q.peer_v[j] = vb + vslot;
        q.peer_ctr[j] = reinterpret_cast<int32_t*>(vb + voff_ctr) + cslot;
    }
    q.n_peers = N;
    q.peer_rank = p->cfg.tp_rank;
    q.peer_block = p->p2p_vcap;
    q.v_sum_blocks = mask == 0x8 ? 1 : 0;
    return SLORA_OK;
}

slora_status p2p_checks(slora_pool* p, slora_batch* b) {
    if (!p || !b) return fail(SLORA_ERR_INVALID_ARG, "null pool/batch");
    if (!p->p2p_open) return fail(SLORA_ERR_INVALID_ARG, "call slora_tp_p2p_export / _open first");
    return SLORA_OK;
}
}  // namespace

extern "C" slora_status slora_tp_fused_qkv(slora_pool_t p, slora_batch_t b, int32_t layer, const void* x,
                                           int64_t ldx, void* const y[3], const int64_t ldy[3], void* stream) {
    slora_status st = p2p_checks(p, b);
    if (!st) st = common_checks(p, b, layer, 0x7);
    if (st) return st;
    if (b->adapted == 0) return ok();
    if (!x || !y || !ldy || !aligned16(x, ldx, p->es) || ldx < p->cfg.hidden)
        return fail(SLORA_ERR_SHAPE, "x alignment/stride");
    for (int pj = 0; pj < 3; ++pj)
        if (!y[pj] || !aligned16(y[pj], ldy[pj], p->es) || ldy[pj] < p->P)
            return fail(SLORA_ERR_SHAPE, "y[%d] alignment/stride", pj);
    LoraParams q;
    if ((st = prepare_call(p, b, p->kc_tpf_qkv, layer, 0x7, stream, q))) return st;
    if ((st = p2p_params(p, b, 0x7, q))) return st;
    q.x = x;
    q.ldx = ldx;
    for (int pj = 0; pj < 3; ++pj) {
        q.y[pj] = y[pj];
        q.ldy[pj] = ldy[pj];
    }
    const KernelCfg& k = p->kcfg[p->kc_tpf_qkv];
    const int dt = p->cfg.dtype == SLORA_F32 ? kF32 : (p->cfg.dtype == SLORA_F16 ? kF16 : kBF16);
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    CUDA_TRY(launch_lora(q, kTPFused, dt, k.grid, static_cast<cudaStream_t>(stream), k.smem));
    return ok();
}

extern "C" slora_status slora_tp_fused_o(slora_pool_t p, slora_batch_t b, int32_t layer, const void* z, int64_t ldz,
                                         void* base_partial, int64_t ld_base, void* stream) {
    slora_status st = p2p_checks(p, b);
    if (!st) st = common_checks(p, b, layer, 0x8);
    if (st) return st;
    if (b->adapted == 0) return ok();
    if (!z || !aligned16(z, ldz, p->es) || ldz < p->P) return fail(SLORA_ERR_SHAPE, "z alignment/stride");
    if (!base_partial || ld_base < p->cfg.hidden || !aligned16(base_partial, ld_base, p->es))
        return fail(SLORA_ERR_INVALID_ARG, "base partial / stride");
    LoraParams q;
    if ((st = prepare_call(p, b, p->kc_tpf_o, layer, 0x8, stream, q))) return st;
    if ((st = p2p_params(p, b, 0x8, q))) return st;
    q.x = z;
    q.ldx = ldz;
    // fold (reading R13): the expand writes column slice k of the base partial sum
    q.y[3] = static_cast<uint8_t*>(base_partial) + size_t(int64_t(p->cfg.tp_rank) * p->P) * p->es;
    q.ldy[3] = ld_base;
    const KernelCfg& k = p->kcfg[p->kc_tpf_o];
    const int dt = p->cfg.dtype == SLORA_F32 ? kF32 : (p->cfg.dtype == SLORA_F16 ? kF16 : kBF16);
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    CUDA_TRY(launch_lora(q, kTPFused, dt, k.grid, static_cast<cudaStream_t>(stream), k.smem));
    return ok();
}

extern "C" slora_status slora_tp_get_stats(slora_pool_t p, slora_tp_stats* out) {
    if (check_pool(p) || !out) return fail(SLORA_ERR_INVALID_ARG, "null argument");
    *out = p->tp_stats;
    return ok();
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
    CUDA_TRY(cudaMemcpy(out, p->trace_dev, sizeof(int64_t) * size_t(std::min(n, 16 * kTraceSlots)), cudaMemcpyDeviceToHost));
    return ok();
}
