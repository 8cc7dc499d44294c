/*
 * slora.h -- C ABI of the B200-native S-LoRA hot path (arXiv 2311.03285):
 * heterogeneous batched LoRA over Unified Paging.
 *
 * P:L = PAPER.md line L (the paper's text; citations are documentation).
 * S:L = SPEC.md line L (interface / error names only).
 *
 * Conventions (every function):
 *   - returns slora_status; SLORA_OK == 0.  On error nothing was enqueued and
 *     the pool's bookkeeping is unchanged; slora_last_error() returns a
 *     thread-local one-line detail ("needed=64 free=5").
 *   - asynchronous CUDA faults surface as SLORA_ERR_CUDA on a later call or on
 *     slora_sync().
 *   - `stream` arguments are cudaStream_t passed as void* (0 = legacy default
 *     stream).  No call synchronizes the device on the hot path.
 *   - a pool (and every batch made from it) is externally serialized: one
 *     thread at a time.
 *   - ownership: the pool owns its metadata, its pinned staging and its
 *     device page tables; the pool's page buffer, x, y and v are caller-owned
 *     device memory that must outlive the calls using them.
 *   - no C++ type, exception or torch type crosses this boundary.
 *
 * Data layout in HBM
 *   pool buffer: capacity_pages pages of page_elems = hidden / tp_size
 *     elements of `dtype` each; page p starts at byte p * page_elems * esize.
 *     KV pages and adapter pages are interleaved.
 *   adapter tensors (reading R1): A (h x r) is stored TRANSPOSED -- one page
 *     row per rank column j (its h input elements); B (r x d) one page row per
 *     rank row.  "a LoRA weight tensor of rank R takes up R pages".
 *   under N-way tensor parallelism (reading R3/R4) the pool on
 *   rank k holds only k's shards, each still r pages of H/N elements:
 *     q,k,v: A1 column shard (rank columns k*r/N..), each column of length h
 *            spans N pages; B1 column shard (output columns k*d/N..).
 *     o    : A2 row shard (input rows k*d/N..), B2 column shard (k*h/N..).
 */
#ifndef SLORA_H
#define SLORA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct slora_pool* slora_pool_t;   /* opaque, owned by the library */
typedef struct slora_batch* slora_batch_t; /* opaque, owned by the library */

typedef enum { SLORA_F32 = 0, SLORA_F16 = 1, SLORA_BF16 = 2 } slora_dtype;

/* Which free page is handed out (reading R10): LIFO free stack that pops
 * 0,1,2,... initially, or a splitmix64-seeded Fisher-Yates shuffle of it
 * (for i = cap-1..1: j = splitmix64() % (i+1); swap).  Frees push in release
 * order. */
typedef enum { SLORA_ORDER_ASCENDING = 0, SLORA_ORDER_SHUFFLE = 1 } slora_alloc_order;

typedef enum {
    SLORA_OK = 0,
    SLORA_ERR_INVALID_ARG = 1,
    SLORA_ERR_SHAPE = 2,              /* shape error                         */
    SLORA_ERR_OUT_OF_PAGES = 3,       /* InsufficientPages(needed, free)    */
    SLORA_ERR_ALREADY_RESIDENT = 4,
    SLORA_ERR_NOT_RESIDENT = 5,
    SLORA_ERR_PINNED = 6,             /* PinnedEviction                     */
    SLORA_ERR_NOT_PINNED = 7,
    SLORA_ERR_STALE_HANDLE = 8,       /* double free / use of a freed handle / a
                                         batch prepared before an eviction */
    SLORA_ERR_FREE_PAGE_READ = 9,
    SLORA_ERR_NONRESIDENT_ADAPTER = 10, /* batch names an adapter not loaded */
    SLORA_ERR_SEGMENT_OVERLAP = 11,   /* reserved; segments are derived here */
    SLORA_ERR_TOKEN_COUNT_NOT_ONE = 12, /* decode-only call on a multi-token segment */
    SLORA_ERR_INDIVISIBLE = 13,       /* IndivisibleDimension               */
    SLORA_ERR_CUDA = 14,
    SLORA_ERR_NO_DEVICE = 15,         /* device call on a bookkeeping-only pool     */
    SLORA_ERR_NCCL = 16               /* NCCL missing, or an NCCL call failed       */
} slora_status;

const char* slora_status_string(slora_status s);
const char* slora_last_error(void);

/* ------------------------------------------------------------------ a1 ---
 * Pool create ("allocate a large buffer statically ... each page
 * corresponding to a vector of H").  The buffer is caller-owned (torch).
 * device = -1 makes a bookkeeping-only pool (no CUDA calls; device_buffer must
 * be NULL and adapter loads take host_w = NULL): used by CPU tests. */
typedef struct {
    int32_t device;             /* CUDA ordinal, or -1 = bookkeeping only      */
    slora_dtype dtype;
    int64_t hidden;             /* H; d = h = H for q/k/v/o (reading R2)       */
    int32_t num_layers;         /* L                                          */
    int32_t tp_size;            /* N >= 1; N | hidden                         */
    int32_t tp_rank;            /* 0 <= k < N                                 */
    int64_t capacity_pages;     /* >= 1                                       */
    void* device_buffer;        /* >= capacity_pages*page_elems*esize bytes, 16B aligned */
    int64_t device_buffer_bytes;
    int32_t max_adapters;       /* adapter slots (resident adapters), >= 1    */
    slora_alloc_order alloc_order;
    uint64_t seed;              /* for SLORA_ORDER_SHUFFLE                    */
    /* NEXT-4 (P:321-327 uses the MLP as its example): the LoRA'd
     * projections of a layer and their shapes.  num_proj = 0 means the four
     * square attention projections q,k,v,o.  Projection p maps
     * proj_in[p] inputs to proj_out[p] outputs (0 = hidden), e.g. Llama-7B
     * MLP gate/up 4096 -> 11008, down 11008 -> 4096, or GQA k/v 4096 -> 1024.
     * A stored row of n elements spans ceil(n / page_elems) pages, the last
     * one partly used (reading R2): per adapter and layer, projection p takes
     * r * (ceil(proj_in[p]/P) + ceil(proj_out[p]/P)) pages.  Non-square
     * projections need tp_size == 1; every dim is a multiple of 16 bytes of
     * the dtype and spans <= 8 pages; a fused call's input width must fit
     * one 32 KB ring slot (proj_in * esize + 16 <= 32768: 16376 for
     * fp16/bf16, 8188 for fp32), else the call fails with SHAPE; the host
     * buffer of slora_adapter_load
     * holds, per layer and projection p in order, A (proj_in x r) then B
     * (r x proj_out), row-major. */
    int32_t num_proj;           /* 1..8, or 0 = 4 (q,k,v,o)                    */
    int64_t proj_in[8];
    int64_t proj_out[8];
} slora_pool_config;
#define SLORA_MAX_PROJ 8

slora_status slora_pool_create(const slora_pool_config* cfg, slora_pool_t* out);
slora_status slora_pool_destroy(slora_pool_t pool); /* synchronizes the device */

typedef struct {
    int64_t capacity_pages, used_pages, free_pages;
    int64_t largest_free_run;   /* longest run of consecutive free page ids    */
    int64_t kv_pages, adapter_pages;
    int64_t page_elems;         /* hidden / tp_size                           */
    int32_t resident_adapters;
} slora_frag_report;

/* S:161-163 fragmentation_report. */
slora_status slora_fragmentation_report(slora_pool_t pool, slora_frag_report* out);

/* ------------------------------------------------------------------ a2 ---
 * Adapter load, host -> pool pages ("fetch ... the LoRA adapters needed
 * for the currently running batch").  Pages needed: L * 4 * 2 * rank
 * (every tensor shard takes `rank` pages, see the layout note above).
 *   host_w: the FULL (unsharded) adapter, dtype of the pool, canonical layout:
 *     for layer l in 0..L-1, for proj p in (q,k,v,o): A (h x r, row-major)
 *     then B (r x d, row-major); h = d = hidden.  The library packs its TP
 *     shard into its own pinned staging, copies it H2D and scatters it into
 *     pages (the loader pipeline of slora_adapter_prefetch below), and makes
 *     `stream` wait for it; host_w may be reused as soon as the call returns.
 *     Must be NULL for a bookkeeping-only pool, non-NULL otherwise.
 *   scale: multiplies this adapter's delta (reading R6; 1.0 = the paper).
 *   Errors: INVALID_ARG (rank < 1, bad pointer), INDIVISIBLE (N does not
 *     divide rank), ALREADY_RESIDENT, OUT_OF_PAGES (pages or slots).
 *   Pages are claimed in pop order layer, proj, tensor (A then B), row, chunk.
 *   The load waits (stream-ordered) for the last page release. */
slora_status slora_adapter_load(slora_pool_t pool, int64_t adapter_id, int32_t rank,
                                const void* host_w, float scale, void* stream,
                                int32_t* slot_out);
/* Release an adapter's pages (errors NOT_RESIDENT, PINNED).  The release is
 * stream-ordered: a later load waits for `stream`'s queued work.  Batches
 * prepared before the eviction become STALE_HANDLE. */
slora_status slora_adapter_evict(slora_pool_t pool, int64_t adapter_id, void* stream,
                                 int64_t* released_out);
/* NEXT-1: asynchronous adapter load ("prefetch": the adapters a
 * coming batch needs are fetched while the current batch computes).
 *   Pages and slot are claimed synchronously, with the same checks and errors
 *   as slora_adapter_load (the pool is unchanged on error); the call then
 *   returns and the pool's loader thread streams the data: every tensor shard
 *   is packed into a ring of kLoadChunks pinned staging chunks (16 MB) --
 *   skipped when host_w is page-locked (cudaHostAlloc / cudaHostRegister) and
 *   tp_size == 1: the H2D then reads host_w itself -- and each chunk is copied
 *   H2D and scattered into pages on the pool's own copy stream, so the pack of
 *   chunk k+1, the H2D of chunk k and the caller's kernels overlap.
 *   Page reuse is fenced: the copy stream first waits (cudaStreamWaitEvent,
 *   taken at this call) for every page release still in flight.
 *   Ownership: host_w must stay valid and unchanged until slora_adapter_wait
 *   returns, or slora_adapter_query reports loading == 0.
 *   The adapter may be named in a batch at once: slora_batch_prepare makes
 *   its stream wait for the load (stream-ordered; the host blocks only until
 *   the loader has enqueued the adapter's last chunk).  Evicting a loading
 *   adapter fences its load the same way.  A failed copy surfaces as CUDA on
 *   wait / query / prepare / evict.  slora_adapter_load is prefetch + that
 *   fence on its stream (host_w free on return). */
slora_status slora_adapter_prefetch(slora_pool_t pool, int64_t adapter_id, int32_t rank,
                                    const void* host_w, float scale, int32_t* slot_out);
/* Block until the adapter's load completed on the device (NOT_RESIDENT, CUDA). */
slora_status slora_adapter_wait(slora_pool_t pool, int64_t adapter_id);
/* loading_out = 1 while the adapter's load is in flight, else 0. */
slora_status slora_adapter_query(slora_pool_t pool, int64_t adapter_id, int32_t* loading_out);
typedef struct {
    int64_t loads;          /* loads the loader thread finished                        */
    int64_t direct_loads;   /* of which read a page-locked host_w directly (no pack)   */
    int64_t bytes;          /* host bytes of this rank's shards streamed               */
    double busy_s;          /* loader-thread wall time spent streaming (host side)     */
    int64_t queued;         /* loads waiting or in progress now                        */
} slora_loader_stats;
slora_status slora_loader_get_stats(slora_pool_t pool, slora_loader_stats* out);
slora_status slora_adapter_pin(slora_pool_t pool, int64_t adapter_id);   /* NOT_RESIDENT */
slora_status slora_adapter_unpin(slora_pool_t pool, int64_t adapter_id); /* NOT_RESIDENT, NOT_PINNED */
/* The adapter's page ids in claim order (n_out = count; copies min(cap, n)). */
slora_status slora_adapter_pages(slora_pool_t pool, int64_t adapter_id, int32_t* out,
                                 int64_t cap, int64_t* n_out);

/* ------------------------------------------------------------------ a3 ---
 * KV cache bookkeeping: K and V of a request are two
 * (S, H) tensors per layer (reading R11) -> 2 * S * L pages, claimed in order
 * layer, kind (K=0, V=1), position.  pages_out (nullable) receives them.
 * Errors: INVALID_ARG (n < 0, request already live), OUT_OF_PAGES;
 * append/free/pages of a request that is not live: STALE_HANDLE. */
slora_status slora_kv_alloc(slora_pool_t pool, int64_t request_id, int32_t n_tokens,
                            int32_t* pages_out);
slora_status slora_kv_append(slora_pool_t pool, int64_t request_id, int32_t n_tokens,
                             int32_t* pages_out);
slora_status slora_kv_free(slora_pool_t pool, int64_t request_id, void* stream,
                           int64_t* released_out);
slora_status slora_kv_pages(slora_pool_t pool, int64_t request_id, int32_t layer, int32_t kind,
                            int32_t* out, int64_t cap, int64_t* n_out);

/* Copy page rows to dst (n x page_elems, device) -- the SPEC gather op
 * (S:157-160), for tests.  FREE_PAGE_READ if a page is free. */
slora_status slora_gather_pages(slora_pool_t pool, const int32_t* pages_host, int32_t n,
                                void* dst_device, void* stream);

/* ------------------------------------------------------------------ a4 ---
 * Batch descriptor.  token_adapter_host[i] = adapter id of token i or -1
 * (no adapter: its y rows are never written, reading R7).  prepare groups
 * tokens by adapter into segments (each adapter's weights are read once per
 * call, reading R8), attaches ranks and page tables, packs (segment x
 * projection) work into balanced units (no padding to a max rank), chooses
 * MBGMV or MBGMM per segment by token count (reading R9) and uploads the
 * descriptor on `stream`.  Errors: NONRESIDENT_ADAPTER.  The descriptor is
 * valid until the next prepare of the same batch or an eviction. */
slora_status slora_batch_create(slora_pool_t pool, slora_batch_t* out);
slora_status slora_batch_destroy(slora_batch_t batch);
slora_status slora_batch_prepare(slora_batch_t batch, const int64_t* token_adapter_host, int32_t T,
                                 void* stream);
/* CUDA-graph replay across batches (the batch changes every
 * iteration).  The MBGMV launches read their descriptors through a header at
 * a fixed device address per (batch, call shape); prepare rewrites every
 * header (one H2D with the descriptors, on its stream) and rebuilds every
 * call shape launched on this batch since it was created.  So a graph that
 * captured fused / split calls of this batch handle replays, after each
 * prepare, the NEW batch -- provided each prepared batch has
 * mbgmm_segments == 0 (MBGMM launch counts are batch-dependent and baked
 * into a graph); SLORA_BATCH_MBGMV_ONLY guarantees it (every segment on the
 * MBGMV path).  Under TP the NCCL element counts are baked as well: replay
 * only batches of the same sum of ranks. */
enum { SLORA_BATCH_MBGMV_ONLY = 1 };
slora_status slora_batch_set_options(slora_batch_t batch, uint32_t flags);

typedef struct {
    int32_t T;                 /* tokens in the batch                         */
    int32_t adapted_tokens;    /* tokens with an adapter                      */
    int32_t segments;          /* distinct adapters in the batch              */
    int64_t sum_rank_tokens;   /* NR = sum over adapted tokens of its rank    */
    int64_t weight_bytes_per_proj; /* sum over segments of this rank's shard bytes of A and B */
    int32_t mbgmm_segments;    /* segments routed to the tensor-core kernel   */
} slora_batch_info;
slora_status slora_batch_get_info(slora_batch_t batch, slora_batch_info* out);

/* ---------------------------------------------------------------- a5+a7 --
 * Fused shrink -> expand on one GPU (Eq. lora_factored P:121 per token; the
 * rank-r intermediate stays on chip):
 *   for every projection p in proj_mask (bit p: 0=q 1=k 2=v 3=o by default;
 *   projection p of the pool's proj_in/proj_out list otherwise) and every
 *   adapted token i with adapter a:
 *     y_p[i, :] = round( y_p[i, :] + scale_a * (x[i, :] A_{a,layer,p}) B_{a,layer,p} )
 *   x: T x proj_in (the projections of one call share their input width),
 *   row stride ldx elements; y[p]: T x proj_out[p], stride ldy[p] (y and ldy
 *   are indexed by projection id; only the mask's entries are read);
 *   pool dtype; 16-byte aligned rows.  fp32 accumulation; one rounding.
 *   Only for tp_size == 1 (else INVALID_ARG).
 *   Segments are served by MBGMV, or -- consecutive runs of >= 32 tokens of
 *   one adapter, or (decode batches) segments of >= 4 scattered tokens of
 *   rank >= 32 holding at least half of the adapted tokens -- by the MBGMM
 *   tensor-core pair (reading R9); all intermediates (v, gathered
 *   x rows) live in pool-owned workspaces sized by slora_batch_prepare and
 *   are used in stream order. */
slora_status slora_lora_apply(slora_pool_t pool, slora_batch_t batch, int32_t layer,
                              uint32_t proj_mask, const void* x, int64_t ldx,
                              void* const y[SLORA_MAX_PROJ], const int64_t ldy[SLORA_MAX_PROJ], void* stream);

/* Many fused calls in one enqueue (the host cost of a decode step: one ABI
 * crossing instead of one per call).  calls[i] is slora_lora_apply's argument
 * list; the calls are enqueued in order on `stream`.  Stops at the first
 * failing call (its index in *failed_out when non-NULL; -1 on success): the
 * calls before it are enqueued. */
typedef struct {
    int32_t layer;
    uint32_t proj_mask;
    const void* x;
    int64_t ldx;
    void* y[SLORA_MAX_PROJ];
    int64_t ldy[SLORA_MAX_PROJ];
} slora_call;
slora_status slora_lora_apply_many(slora_pool_t pool, slora_batch_t batch, const slora_call* calls,
                                   int32_t n_calls, void* stream, int32_t* failed_out);

/* Split form (for tensor parallelism).
 * shrink: v = x A_shard in fp32.  For projection p, the stored A shard has
 *   r/div rank columns, div = tp_size for q,k,v and 1 for o (and 1 when
 *   tp_size == 1); x has the shard's input width (hidden for q,k,v;
 *   hidden/tp_size for o under TP).  v layout (fp32, dense):
 *     [proj in mask order][segment][token][r/div]
 *   with slora_lora_v_elems(batch, mask, div) elements in total.
 * expand: y_p[i, :] += scale_a * v_i B_shard, y width hidden/tp_size.
 *   v is read as v_blocks equal blocks laid out back to back, block b holding
 *   rank columns [b*r/v_blocks, (b+1)*r/v_blocks) in the shrink layout above
 *   (v_blocks = tp_size after the q/k/v all-gather, 1 after the o
 *   all-reduce or on one GPU). */
slora_status slora_lora_v_elems(slora_batch_t batch, uint32_t proj_mask, int32_t div,
                                int64_t* out);
slora_status slora_lora_shrink(slora_pool_t pool, slora_batch_t batch, int32_t layer,
                               uint32_t proj_mask, const void* x, int64_t ldx, float* v,
                               void* stream);
slora_status slora_lora_expand(slora_pool_t pool, slora_batch_t batch, int32_t layer,
                               uint32_t proj_mask, const float* v, int32_t v_blocks,
                               void* const y[SLORA_MAX_PROJ], const int64_t ldy[SLORA_MAX_PROJ], void* stream);

/* ---------------------------------------------------------------- a6/a8 --
 * Tensor-parallel LoRA (Fig. lora_tp; readings R3/R4/R13/R14):
 * N ranks, one process per GPU, each with a pool created with tp_size = N and
 * its own tp_rank.  The library owns an NCCL communicator (NCCL is loaded at
 * run time with dlopen("libnccl.so.2"), so a process that already loaded
 * torch's NCCL shares it) and carries the two exchange steps between its
 * shrink and expand kernels, on the caller's stream, capturable in a CUDA
 * graph.  The exchanged intermediate is fp32.
 *
 * slora_tp_unique_id: ncclGetUniqueId into id_out (SLORA_TP_ID_BYTES bytes).
 *   Rank 0 calls it; the bytes reach the other ranks by any channel (e.g. a
 *   torch.distributed broadcast).
 * slora_tp_init: ncclCommInitRank(size, id, rank) on the pool's device.
 *   rank/size must equal the pool's tp_rank/tp_size; size 1 is allowed (the
 *   collectives become one-rank NCCL calls).  Errors: INVALID_ARG, NO_DEVICE,
 *   NCCL.  The communicator lives until slora_pool_destroy.
 *   The exchange buffers (fp32, library-owned) are sized by every later
 *   slora_batch_prepare: prepare after init.
 * slora_tp_lora_qkv (the q/k/v projections as "W1"): for p in q,k,v
 *     v_k   = x A1_{k,p}                 (fp32, T x r/N per token, shrink)
 *     v     = all_gather_k(v_k)          ONE ncclAllGather of the three
 *                                        projections' shards (reading R14)
 *     y_p  += scale * v B1_{k,p}         (expand; y_p is this rank's T x H/N
 *                                        column shard of the q/k/v output)
 *   x: T x H (replicated), stride ldx; y[0..2]: T x H/N, strides ldy[0..2].
 * slora_tp_lora_o (the o projection as "W2", reading R13):
 *     u_k   = z_k A2_k                   (fp32 partial over this rank's H/N
 *                                        input rows, shrink)
 *     u     = all_reduce_sum(u_k)        ncclAllReduce
 *     base[:, k*H/N:(k+1)*H/N] += scale * u B2_k
 *   z: this rank's T x H/N slice of the attention output (stride ldz);
 *   base: this rank's T x H partial sum of the base o projection (stride
 *   ld_base).  The LoRA output is folded into column slice k, so the base
 *   layer's own all-reduce (the caller's) then carries base + LoRA.
 * Both: errors INVALID_ARG (no communicator, tp_size mismatch), SHAPE
 *   (exchange buffers smaller than the batch: prepare after init), CUDA, NCCL.
 * slora_tp_get_stats: per-device element counts taken from the count
 *   arguments passed to NCCL, with the ring schedule's per-device volumes
 *   (all-gather: (N-1) * sendcount sent; all-reduce: 2(N-1)/N * count sent),
 *   which equal P:337's 3(N-1)*NR/N and 2(N-1)*NR/N per layer. */
#define SLORA_TP_ID_BYTES 128
typedef struct {
    int64_t allgather_calls;
    int64_t allgather_send_elems;  /* per device, fp32 elements */
    int64_t allgather_recv_elems;
    int64_t allreduce_calls;
    int64_t allreduce_count;       /* sum of the count arguments */
    int64_t allreduce_send_elems;  /* per device, ring schedule: 2(N-1)/N * count */
} slora_tp_stats;
slora_status slora_tp_unique_id(void* id_out);
slora_status slora_tp_init(slora_pool_t pool, const void* id, int32_t rank, int32_t size);
slora_status slora_tp_lora_qkv(slora_pool_t pool, slora_batch_t batch, int32_t layer, const void* x,
                               int64_t ldx, void* const y[3], const int64_t ldy[3], void* stream);
slora_status slora_tp_lora_o(slora_pool_t pool, slora_batch_t batch, int32_t layer, const void* z,
                             int64_t ldz, void* base_partial, int64_t ld_base, void* stream);

/* NEXT-3: device-initiated TP exchange fused into ONE kernel per call
 * ("enhanced fused kernels").  Instead of shrink ->
 * NCCL -> expand, the shrink pieces of rank k store their v entries straight
 * into block k of EVERY rank's exchange region (NVLink peer stores through
 * CUDA IPC mappings) and release a per-item counter on every rank
 * (system-scope red.release); an expand piece waits until its item's counter
 * shows all N ranks' shrink pieces, then reads the N blocks -- gathered for
 * q/k/v (the all-gather of P:323), summed in rank order for o (the
 * all-reduce of P:324, deterministic) -- and expands into y as
 * slora_tp_lora_qkv / _o do (same arguments, same results).
 * slora_tp_p2p_export: allocates this rank's exchange region (kLaunchSlots x
 *   N x 196608 fp32 + counters) and writes its CUDA IPC handle into
 *   handle_out (SLORA_TP_P2P_HANDLE_BYTES).  slora_tp_p2p_open: handles =
 *   the N ranks' handles in rank order (the caller all-gathers them, e.g.
 *   with torch.distributed); maps every peer region (lazy peer access).
 *   After open, slora_batch_prepare builds the fused calls' descriptors
 *   eagerly.  Requirements: all N ranks launch the same calls in the same
 *   order (an expand waits for the other ranks' shrink pieces of the same
 *   launch); every rank's GPU runs its whole grid at once.  Errors:
 *   INVALID_ARG (not exported / opened), SHAPE (NR beyond the exchange
 *   capacity), CUDA.  Unmeasured beyond one GPU in this repository: with
 *   N = 1 it is tested bit-exact against the NCCL path. */
#define SLORA_TP_P2P_HANDLE_BYTES 64
slora_status slora_tp_p2p_export(slora_pool_t pool, void* handle_out);
slora_status slora_tp_p2p_open(slora_pool_t pool, const void* handles);
slora_status slora_tp_fused_qkv(slora_pool_t pool, slora_batch_t batch, int32_t layer, const void* x,
                                int64_t ldx, void* const y[3], const int64_t ldy[3], void* stream);
slora_status slora_tp_fused_o(slora_pool_t pool, slora_batch_t batch, int32_t layer, const void* z,
                              int64_t ldz, void* base_partial, int64_t ld_base, void* stream);
slora_status slora_tp_get_stats(slora_pool_t pool, slora_tp_stats* out);

/* Wait for `stream` and surface any deferred CUDA error. */
slora_status slora_sync(slora_pool_t pool, void* stream);

/* Debug: when the environment variable SLORA_TRACE=1 is set at pool creation,
 * the next kernel launches record per-CTA event timestamps (ns, %globaltimer)
 * for CTAs 0..15, 1024 slots each.  Copies min(n, 16384) values to out_host
 * (synchronizes the device); INVALID_ARG when tracing is off. */
slora_status slora_debug_trace(slora_pool_t pool, int64_t* out_host, int32_t n);

/* Number of this library's kernel launches so far (for bench accounting). */
int64_t slora_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SLORA_H */
