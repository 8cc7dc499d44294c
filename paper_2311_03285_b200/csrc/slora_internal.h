// Internal types shared by the host side (api.cpp) and the kernels
// (kernels.cu) of libslora.  Not part of the C ABI (include/slora.h).
#pragma once
#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

namespace slora {

// ---------------------------------------------------------------- batch ---
// One segment = the tokens of one adapter in a batch (the kernels
// "gather adapter weights with different ranks from the memory pool").
struct DevSeg {
    int32_t slot;      // adapter slot
    int32_t rank;      // r (full, unsharded rank)
    int32_t n_tok;     // tokens of this adapter in the batch
    int32_t tok_off;   // first entry in tok_idx
    int64_t vrow_off;  // sum over earlier segments of n_tok * rank
    float scale;       // per-adapter scale (reading R6)
    int32_t pad;
};
static_assert(sizeof(DevSeg) == 32, "DevSeg layout");

// A work item = (segment, projection of the call, token chunk of <=
// kItemTokCap tokens).  Self-contained: the kernel resolves it with one load.
struct DevItem {
    const int32_t* tab;  // the adapter's device page table (layer/proj offset added in-kernel)
    int64_t vrow;      // v row offset of the chunk: segment vrow_off + t0 * rank
    int32_t rank;
    int32_t pi;        // index of the projection in the call's mask order
    int32_t t0, nt;    // token chunk [t0, t0+nt) of the segment
    int32_t tok_off;   // index in tok_idx of the chunk's first token
    int32_t n_sp;      // number of shrink pieces of this item (fused dependency count)
    float scale;
    int32_t seg;
    int32_t n_ep;      // number of expand pieces of this item (fused: the last one resets the counter)
    int32_t pad[3];
};
static_assert(sizeof(DevItem) == 64, "DevItem layout");

// A piece = the unit of scheduling.  kind 0 (shrink): rows [a, a+b) of the
// item's stored A rows, full K.  kind 1 (expand): all B rows, output columns
// [a, a+b).  The host assigns pieces to the persistent CTAs (LPT on bytes,
// api.cpp schedule_pieces); every CTA runs all its shrink pieces before any
// expand piece, so an expand piece only ever waits on shrink pieces, which
// never wait (no deadlock with all CTAs resident).
struct DevPiece {
    int32_t kind, item, a, b;
};
static_assert(sizeof(DevPiece) == 16, "DevPiece layout");

#ifndef SLORA_ITEM_TOK
#define SLORA_ITEM_TOK 2
#endif
// tokens per item (larger segments are chunked).  Measured on C2 decode
// (profiles/knob_sweep_r01.txt): 4 -> 1.403, 3 -> 1.311, 2 -> 1.249,
// 1 -> 1.346 ms/step; 2 halves the x buffers (ring depth 4 -> 5 slots) and
// the Zipf-head items, whose expand pieces were the stragglers.
constexpr int kItemTokCap = SLORA_ITEM_TOK;
constexpr int kMaxRank = 64;     // max rank of the MBGMV path
constexpr int kMaxProj = 8;      // LoRA'd projections per layer (q,k,v,o by default; NEXT-4: + MLP)
#ifndef SLORA_SHRINK_ROWS
#define SLORA_SHRINK_ROWS 16
#endif
constexpr int kShrinkRows = SLORA_SHRINK_ROWS;  // max A rows per shrink piece (the host picks <= this per call)
constexpr int kConsumerWarps = 8;
// warp roles: 0-7 consumers, then streamer 0, resolver, streamer 1, expand-v
// prefetcher, shrink publisher, streamers 2.. (bulk-copy issue costs ~90 ns
// per copy per warp, measured: more issuers stream 4 KB row slices faster)
#ifndef SLORA_STREAMERS
#define SLORA_STREAMERS 2
#endif
constexpr int kStreamers = SLORA_STREAMERS;
constexpr int kWarpStreamer0 = kConsumerWarps, kWarpResolver = kConsumerWarps + 1,
              kWarpStreamer1 = kConsumerWarps + 2, kWarpPrefetch = kConsumerWarps + 3,
              kWarpPublish = kConsumerWarps + 4, kWarpStreamerX = kConsumerWarps + 5;
constexpr int kWarpsEnd = kConsumerWarps + 3 + kStreamers;  // one past the last streamer
constexpr int kThreads = kWarpsEnd * 32;
// streamer index of a warp (-1: not a streamer)
inline __host__ __device__ int streamer_id(int warp) {
    return warp == kWarpStreamer0 ? 0
           : warp == kWarpStreamer1 ? 1
           : (warp >= kWarpStreamerX && warp < kWarpsEnd ? 2 + warp - kWarpStreamerX : -1);
}
constexpr int kMaxChunks = 8;    // pages one stored A row spans (TP q/k/v: N)
constexpr int kSlotBytes = 32 * 1024;  // ring slot
constexpr int kMaxSlots = 16;
constexpr int kMeta = 4;         // resolved-piece ring (resolver runs up to kMeta-1 pieces ahead)
constexpr int kLaunchSlots = 8;
constexpr int kTraceSlots = 1024;  // debug trace: globaltimer events per traced CTA (16 CTAs)  // rotating per-launch counter/workspace slots

enum Mode : int { kFused = 0, kShrink = 1, kExpand = 2, kTPFused = 3 };
enum DType : int { kF32 = 0, kF16 = 1, kBF16 = 2 };
enum PieceKind : int { kPieceS = 0, kPieceE = 1, kPieceStop = 2 };

// The batch-dependent part of a call, at a FIXED device address per (batch,
// call shape): slora_batch_prepare rewrites it (one H2D with the descriptor
// upload), so a CUDA graph of the MBGMV launches stays valid while the batch
// changes every iteration (iteration-level batching).
struct CallHdr {
    const int32_t* tok_idx;
    const DevItem* items;
    const DevPiece* pieces;       // grouped by CTA: CTA b runs pieces [cta_off[b], cta_off[b+1])
    const int32_t* cta_off;       // grid + 1 entries
    int32_t* sync;                // kLaunchSlots slots of sync_stride per-item done counters (self-resetting)
    float* ws;                    // kLaunchSlots slots of ws_stride floats: the fused call's v workspace
    int64_t sync_stride, ws_stride;
    int64_t NR;                   // sum over adapted tokens of rank
    int32_t n_items, n_pieces;
};
static_assert(sizeof(CallHdr) == 80, "CallHdr layout");

struct LoraParams {
    const void* pool;             // page buffer
    int64_t page_elems;           // P
    const CallHdr* hdr;           // the call's descriptor header (batch_prepare rewrites it)
    int32_t slot;                 // rotating launch slot: sync counters / workspace of this launch
    int32_t nproj;
    int32_t proj_ids[kMaxProj];
    int32_t layer;
    int32_t K, D;                 // stored A-row length (the call's input width), config B width
    int32_t a_div[kMaxProj];      // A rank columns stored = r / a_div[p]
    int32_t a_row_pages[kMaxProj];  // pages per stored A row
    int32_t b_row_pages[kMaxProj];  // pages per stored B row (NEXT-4: d_out > page)
    int32_t proj_off[kMaxProj];   // projection p's page tables within a layer, in units of the rank:
    int32_t layer_units;          //   tab(layer, p) = adapter table + r * (layer * layer_units + proj_off[p]);
                                  //   A entries [0, r*a_row_pages*stored/r), B after them (r x b_row_pages)
    int32_t a_units[kMaxProj];    // A entries per rank unit (B starts at r * a_units[p])
    int32_t ns;                   // ring slots
    int32_t dbg;                  // debug: bit0 skip shrink math, bit1 skip expand math
    const void* x;
    int64_t ldx;
    void* y[kMaxProj];
    int64_t ldy[kMaxProj];
    long long* trace;             // debug: per-CTA event timestamps (nullptr = off)
    float* v;                     // shrink output (split mode; C-ABI v layout, div as stored); fused: nullptr
    const float* v_in;            // expand input
    int32_t v_blocks;
    // kTPFused (NEXT-3, device-initiated TP exchange): every rank's exchange region is mapped into
    // every process (CUDA IPC over NVLink); this launch's slot of each region:
    float* peer_v[8];             //   v blocks [rank][proj][seg][token][r/div] of peer j (j = 0..N-1)
    int32_t* peer_ctr[8];         //   per-item done counters of peer j
    int32_t n_peers;              //   N
    int32_t peer_rank;            //   this rank k: its shrink writes block k of every peer
    int64_t peer_block;           //   floats per block (nproj * NR / div)
    int32_t v_sum_blocks;         //   1: the expand sums the N blocks (o: all-reduce); 0: gathers them (q/k/v)
};

// Per-launch kernel configuration (chosen on the host, see api.cpp).
struct KernelCfg {
    int mode = 0;
    int ns = 0;
    int64_t K = 0, D = 0;
    int64_t dchunk = 0;           // expand piece width (elements)
    size_t smem = 0;
    int grid = 0;                 // persistent CTAs
    bool ok = false;
};

// smem bytes for a launch (host and device agree via smem_layout in kernels.cu)
size_t lora_smem_bytes(int mode, int64_t K, int64_t dchunk, int ns, int esize);
size_t lora_slot_stride(int mode, int64_t K, int esize);  // ring slot stride (bytes)
int lora_max_ctas(int mode, int dtype, size_t smem);
cudaError_t launch_lora(const LoraParams& p, int mode, int dtype, int grid, cudaStream_t s, size_t smem);
cudaError_t configure_lora_kernels(int device);
// ------------------------------------------------------------------ MBGMM
// Long prefill runs (>= theta consecutive x rows of one adapter) go to the
// tensor-core MBGMM kernels (mbgmm.cu); units are built on the host.
constexpr int kMgTileTok = 64;   // tokens per tile (4 mma m-tiles)
#ifndef SLORA_MG_ROWS
#define SLORA_MG_ROWS 16
#endif
constexpr int kMgRows = SLORA_MG_ROWS;  // stored A rows per shrink unit
#ifndef SLORA_MG_COLS
#define SLORA_MG_COLS 1024
#endif
constexpr int kMgCols = SLORA_MG_COLS;  // output columns per expand unit (rank <= 32; half above)
// expand slab width: B slab of r x cols 16-bit <= 64 KB (two CTAs per SM)
inline int mbgmm_expand_cols(int rank) { return rank <= 32 ? kMgCols : kMgCols / 2; }
constexpr int kMgDefaultTheta = 32;  // run length from which MBGMM is used (SLORA_MBGMM_MIN)
struct MgUnit {
    const int32_t* tab;  // adapter page table
    int64_t vbase;       // v index of (tile token 0, rank row 0)
    int32_t pi;          // projection index in the call's mask order
    int32_t rank;
    int32_t row0;        // x / y row of the tile's first token (the run's rows are consecutive)
    int32_t nt;          // tokens in the tile (<= kMgTileTok)
    int32_t a, b;        // shrink: first A row, rows; expand: first column, columns
    float scale;
    int32_t pad;         // tcgen05 shrink: k-split part
};
static_assert(sizeof(MgUnit) == 48, "MgUnit layout");
struct alignas(64) MgParams {
    CUtensorMap xmap;    // x as a 2-D tensor [rows T][K], 64x64 boxes, 128-byte swizzle
    const void* pool;
    int64_t page_elems;
    const MgUnit* units;
    float* v;            // the call's fp32 workspace (MBGMV layout)
    void* y[kMaxProj];
    int64_t ldy[kMaxProj];
    int32_t proj_ids[kMaxProj];
    int32_t layer, K;
    int32_t ksplit;      // shrink k-split parts (unit.pad = part); the expand sums them in order
    int32_t srows;       // mma.sync shrink: stored A rows per unit (smem layout; <= 32)
    int64_t vpart;       // floats between the parts' v regions
    const int32_t* yrow; // gathered mode: y row of x-map row i (the batch's tok_idx); nullptr: row i
};
#ifndef SLORA_MG_KSPLIT
#define SLORA_MG_KSPLIT 2
#endif
constexpr int kMgKsplit = SLORA_MG_KSPLIT;  // tcgen05 shrink: K parts per (tile, projection)
constexpr int kMgVParts = 8;                // MBGMM v workspace regions (k-split parts), >= kMgKsplit
static_assert(kMgKsplit <= kMgVParts, "MBGMM v parts");
int mbgmm_split(int64_t K);      // K parts of the MBGMM shrink (tcgen05: kMgKsplit; mma.sync: SLORA_MG_SPLIT, default 1)
size_t mbgmm_smem(bool expand, int64_t K, int rmax);
int mbgmm_rows(int64_t K);       // stored A rows per mma.sync shrink unit (32, 16 or 8: the tallest whose K part fits)
cudaError_t launch_gather_rows(const void* x, int64_t ldx, const int32_t* idx, int n, void* out, int64_t K, int es,
                               cudaStream_t s);
bool mbgmm_shrink_whole_rank();  // tcgen05 shrink: one unit per (tile, projection) covering all r A rows
cudaError_t configure_mbgmm_kernels();
cudaError_t launch_mbgmm(const MgParams& p, bool expand, int dtype, int n_units, size_t smem, cudaStream_t s, bool pdl);

// Adapter scatter: jobs describe how rows of a packed staging buffer land in
// pages (see api.cpp pack_shard).
struct ScatterJob {
    int64_t src_off;    // element offset of the dense shard in staging
    const int32_t* pages; // device page list for this tensor (rows*chunks)
    int32_t kind;       // 0 = A shard (Krows x rcols row-major, stored transposed)
                        // 1 = B shard (rows x P row-major)
    int32_t rows;       // A: Krows (input rows of the shard); B: rank rows
    int32_t cols;       // A: stored rank columns; B: P
    int32_t row_pages;  // pages per stored row: A ceil(Krows / P) (TP q/k/v: N), B ceil(cols / P)
};
cudaError_t launch_scatter(const void* staging, const ScatterJob* jobs_dev, int n_jobs, void* pool,
                           int64_t page_elems, int esize, cudaStream_t s);
cudaError_t launch_gather(const void* pool, const int32_t* pages_dev, int n, void* dst,
                          int64_t page_elems, int esize, cudaStream_t s);

void count_launch();

}  // namespace slora
