// Internal types shared by the host side (api.cpp) and the kernels
// (kernels.cu) of libslora.  Not part of the C ABI (include/slora.h).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace slora {

// ---------------------------------------------------------------- batch ---
// One segment = the tokens of one adapter in a batch (the kernels
// "gather adapter weights with different ranks from the memory pool").
struct DevSeg {
    int32_t slot;      // adapter slot -> slot_tab[slot] = its device page table
    int32_t rank;      // r (full, unsharded rank)
    int32_t n_tok;     // tokens of this adapter in the batch
    int32_t tok_off;   // first entry in tok_idx
    int64_t vrow_off;  // sum over earlier segments of n_tok * rank
    float scale;       // per-adapter scale (reading R6)
    int32_t pad;
};
static_assert(sizeof(DevSeg) == 32, "DevSeg layout");

// A work item = (segment, projection index within the call's mask, token
// chunk).  Items are packed into units of balanced size; one cluster of C
// CTAs processes one unit, CTA c owning the c-th 1/C slice of the K (shrink)
// and D (expand) dimensions.
struct DevItem {
    int32_t seg;
    int32_t pi;        // index of the projection in the call's mask order
    int32_t t0, nt;    // token chunk [t0, t0+nt) of the segment
    int32_t row_off;   // first smem row of this item (full-rank units)
    int32_t tok_slot;  // first x row slot in smem
    int32_t v_off;     // first v entry (full-rank units) within the unit
    int32_t pad;
};
static_assert(sizeof(DevItem) == 32, "DevItem layout");

struct DevUnit {
    int32_t item_begin, n_items;
    int32_t rows, toks, ventries;  // totals (full-rank units)
    int32_t pad[3];
};
static_assert(sizeof(DevUnit) == 32, "DevUnit layout");

constexpr int kMaxItemsPerUnit = 16;
constexpr int kThreads = 256;

enum Mode : int { kFused = 0, kShrink = 1, kExpand = 2 };
enum DType : int { kF32 = 0, kF16 = 1, kBF16 = 2 };

struct LoraParams {
    const void* pool;             // page buffer
    int64_t page_elems;           // P
    const int32_t* const* slot_tab;
    const DevSeg* segs;
    const int32_t* tok_idx;
    const DevUnit* units;
    const DevItem* items;
    int32_t n_units;
    int32_t nproj;
    int32_t proj_ids[4];
    int32_t layer;
    int32_t C;                    // K/D split (cluster size for fused/shrink)
    int32_t K, D;                 // A-row length, B-row length (elements)
    int32_t a_div[4];             // A rank columns stored = r / a_div[p]
    int32_t a_row_pages[4];       // pages per stored A row
    int32_t rcap, tcap, vcap;     // smem capacities (rows, x rows, v entries)
    const void* x;
    int64_t ldx;
    void* y[4];
    int64_t ldy[4];
    float* v_out;
    const float* v_in;
    int32_t v_blocks;
    int64_t NR;                   // sum over adapted tokens of rank
};

// launchers (kernels.cu); return cudaError_t of the launch
cudaError_t launch_lora(const LoraParams& p, int mode, int dtype, cudaStream_t s, size_t smem);
size_t lora_smem_bytes(const LoraParams& p, int mode, int esize);
cudaError_t configure_lora_kernels(int device);

// Adapter scatter: jobs describe how rows of a packed staging buffer land in
// pages (see api.cpp pack_shard).
struct ScatterJob {
    int64_t src_off;    // element offset of the dense shard in staging
    const int32_t* pages; // device page list for this tensor (rows*chunks)
    int32_t kind;       // 0 = A shard (Krows x rcols row-major, stored transposed)
                        // 1 = B shard (rows x P row-major)
    int32_t rows;       // A: Krows (input rows of the shard); B: rank rows
    int32_t cols;       // A: stored rank columns; B: P
    int32_t row_pages;  // A: pages per stored row (Krows / P); B: 1
};
cudaError_t launch_scatter(const void* staging, const ScatterJob* jobs_dev, int n_jobs, void* pool,
                           int64_t page_elems, int esize, cudaStream_t s);
cudaError_t launch_gather(const void* pool, const int32_t* pages_dev, int n, void* dst,
                          int64_t page_elems, int esize, cudaStream_t s);

void count_launch();

}  // namespace slora
