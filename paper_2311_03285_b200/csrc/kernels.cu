// kernels.cu -- sm_100a kernels of the S-LoRA hot path.
//
// mbgmv_kernel<T, MODE>: MBGMV gather-shrink-expand over Unified Paging
//   (Sec. 5.3; Eq. lora_factored).
//
//   Persistent (one CTA per SM), warp-specialized, statically scheduled.
//   The host cuts every (segment x projection x token chunk) item into
//     shrink pieces  -- a group of kShrinkRows stored A rows over the full K:
//                       v_j = <x_t, A_j> for the item's tokens (complete dot
//                       products, no partial sums), and
//     expand pieces  -- all r B rows over one chunk of output columns:
//                       y_t[cols] += scale * sum_j v_j B_j[cols].
//   and assigns them to CTAs (LPT on bytes, api.cpp); each CTA runs its
//   shrink pieces before its expand pieces, and an expand piece waits
//   (per-item done counter, acquire) for its item's shrink pieces, which
//   never wait themselves (no deadlock with all CTAs resident).  In the fused
//   mode the rank-r intermediate goes through a small per-launch workspace
//   (<= nproj*NR fp32, a few KB, written and read within microseconds: it
//   lives in L2, never streamed through HBM like the weights).  The counters
//   reset themselves (the item's last expand piece), so a launch needs no
//   teardown and no host memset.
//
//   warp 9 (resolver): loads the CTA's piece list + items (one per lane) and
//     resolves each piece's page ids from the adapter page table, up to
//     kMeta-1 pieces ahead of the consumers.
//   warps 8, 10 (streamers): stream the piece's pages (whole 8 KB A rows; 4 KB B
//     row slices) and x rows into an mbarrier ring with cp.async.bulk (TMA
//     engine, SASS UBLKCP); weights of the first piece are fetched before
//     griddepcontrol.wait (programmatic dependent launch), activations after.
//   warps 0-7 (consumers): shrink -- one A row per warp, mixed-precision
//     FHFMA dot products (fp16/bf16 x fp16/bf16 -> fp32), warp-shuffle
//     reduction; expand -- each thread owns a 16-byte column vector, fp32
//     axpys over the B rows, y read once and written once (one rounding).
//   Reduction orders depend only on (K, dtype): bit-identical results under
//   any page placement, batch permutation or schedule.
//
// MODE kShrink (TP): shrink pieces only; v written in the C-ABI layout.
// MODE kExpand (TP): expand pieces only; v read from v_in (v_blocks blocks).
//
// scatter_kernel: adapter load, staging -> pages (A transposed).
// gather_kernel:  test-only page gather.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "slora_internal.h"

namespace slora {

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// mbarrier wait.  SLORA_WAIT_MODE 0: try_wait (hardware-chosen suspend),
// 1: try_wait with a suspend-time hint, 2: test_wait spin.
#ifndef SLORA_WAIT_MODE
#define SLORA_WAIT_MODE 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if SLORA_WAIT_MODE == 1
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(1000000)
        : "memory");
#elif SLORA_WAIT_MODE == 2
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
// Back-off wait for the helper warps (streamers, resolver, prefetcher,
// publisher): polls with test_wait and sleeps in between, so that idle
// helpers do not flood the CTA's barrier unit with probes while the
// consumers' own waits need it (measured: polling helpers slowed every
// consumer barrier operation ~10x).
#ifndef SLORA_HELPER_SLEEP_NS
#define SLORA_HELPER_SLEEP_NS 32  // measured: 128 -> 1.241, 32 -> 1.227 ms per C2 step
#endif
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#if SLORA_HELPER_SLEEP_NS > 0
    while (!mbar_test(bar, parity)) __nanosleep(SLORA_HELPER_SLEEP_NS);
#else
    mbar_wait(bar, parity);
#endif
}
// 1-D bulk copy global -> own shared memory on the TMA engine (SASS UBLKCP),
// completing `bytes` of transaction count on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// system scope (peer GPUs over NVLink: kTPFused)
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add_sys(int* p, int v) {
    asm volatile("red.release.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(ev)                                                                                  \
    do {                                                                                           \
        if (p.trace && blockIdx.x < 16 && (ev) < kTraceSlots) p.trace[blockIdx.x * kTraceSlots + (ev)] = gtimer(); \
    } while (0)

// ---------------------------------------------------- element conversions
template <typename T> struct Vec;
template <> struct Vec<float> {
    static constexpr int VE = 4;
    __device__ static void to_f32(const uint4& u, float* f) {
        f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
        f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
    }
    __device__ static uint4 from_f32(const float* f) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                          __float_as_uint(f[3]));
    }
};
template <> struct Vec<__half> {
    static constexpr int VE = 8;
    __device__ static void to_f32(const uint4& u, float* f) {
        const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 t = __half22float2(h[i]);
            f[2 * i] = t.x; f[2 * i + 1] = t.y;
        }
    }
    __device__ static uint4 from_f32(const float* f) {
        uint4 u;
        __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
        return u;
    }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int VE = 8;
    __device__ static void to_f32(const uint4& u, float* f) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 t = __bfloat1622float2(h[i]);
            f[2 * i] = t.x; f[2 * i + 1] = t.y;
        }
    }
    __device__ static uint4 from_f32(const float* f) {
        uint4 u;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
        return u;
    }
};

// Mixed-precision FMA: f16/bf16 x f16/bf16 + f32 -> f32 in ONE instruction
// (SASS FHFMA, with .H1 operand selects for the upper halves): the product
// of two 16-bit floats is exact in fp32, so this equals convert + fmaf.
__device__ __forceinline__ float fma16(uint32_t a, uint32_t b, float c, __half*) {
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"((unsigned short)a), "h"((unsigned short)b));
    return c;
}
__device__ __forceinline__ float fma16(uint32_t a, uint32_t b, float c, __nv_bfloat16*) {
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(c) : "h"((unsigned short)a), "h"((unsigned short)b));
    return c;
}
// acc0/acc1 += <a, x> over one 16-byte vector (two interleaved chains)
template <typename T>
__device__ __forceinline__ void dot16(const uint4& a, const uint4& x, float& acc0, float& acc1) {
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        acc0 = fma16(aw[i] & 0xffffu, xw[i] & 0xffffu, acc0, (T*)nullptr);
        acc1 = fma16(aw[i] >> 16, xw[i] >> 16, acc1, (T*)nullptr);
    }
}
template <>
__device__ __forceinline__ void dot16<float>(const uint4& a, const uint4& x, float& acc0, float& acc1) {
    acc0 = fmaf(__uint_as_float(a.x), __uint_as_float(x.x), acc0);
    acc1 = fmaf(__uint_as_float(a.y), __uint_as_float(x.y), acc1);
    acc0 = fmaf(__uint_as_float(a.z), __uint_as_float(x.z), acc0);
    acc1 = fmaf(__uint_as_float(a.w), __uint_as_float(x.w), acc1);
}

// ------------------------------------------------------------ smem layout
constexpr int kMaxPiecePages = kMaxRank > kShrinkRows * kMaxChunks ? kMaxRank : kShrinkRows * kMaxChunks;
struct PieceMeta {
    int32_t kind, item, nt, r, ra, row0, nrows, dcol0, dcols, doff, proj, arp, n_sp, n_ep;
    float scale;
    int32_t pi;                   // projection index in the call's mask order
    int64_t vbase;                // v index of (token 0, rank row 0) of this item
    int64_t vrow;                 // the item's v row offset (full rank units)
    int32_t tok[kItemTokCap];
    int32_t pages[kMaxPiecePages];
};

struct SmemLayout {
    size_t bars, meta, pubq, vbuf, red, xrows, ring, total;
};
constexpr int kPub = 4;        // shrink-done queue (consumers -> publisher warp)
constexpr int kNumBars = 2 * kMaxSlots + 4 + 2 * kMeta + 4 + 2 * kPub;
constexpr int kRedFloats = kConsumerWarps * kShrinkRows * kItemTokCap;  // per buffer
__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }
// Shrink rows sit in a slot at a stride of (row bytes + 16) and the slot
// stride is offset by 16 B per row of the previous slot (mod 128), so that 8
// consecutive A rows -- the 8 row addresses of an ldmatrix -- hit 8 distinct
// 16-byte bank groups (conflict-free tensor-core operand loads).
__host__ __device__ inline int shrink_rows_per_slot(int64_t K, int es) {
    return int((kSlotBytes + 128) / (K * es + 16));  // rows * (K*es + 16) <= kSlotBytes + 128 < slot_stride
}
// expand rows (B row slices of rowb bytes) also sit at a 16-byte stagger
__host__ __device__ inline int expand_rows_per_slot(uint32_t rowb) {  // a multiple of 4 (unrolled axpys) when >= 4
    const int n = int((kSlotBytes + 128) / (rowb + 16));
    return n >= 4 ? (n & ~3) : n;
}
// x row buffers: two (the next shrink piece's x loads while this one
// computes) unless the rows are wide (16 KB: one, to keep the ring deep)
#ifndef SLORA_XBUF
#define SLORA_XBUF 2
#endif
__host__ __device__ inline int x_buffers(int64_t K, int es) { return K * es <= 8192 ? SLORA_XBUF : 1; }
__host__ __device__ inline size_t slot_stride(int mode, int64_t K, int es) {
    const int rps = mode == kExpand ? 0 : shrink_rows_per_slot(K, es);
    return size_t(kSlotBytes) + 256 + size_t((16 * rps) & 127);
}
__host__ __device__ inline SmemLayout smem_layout(int mode, int64_t K, int64_t dchunk, int ns, int es) {
    (void)dchunk;
    SmemLayout L{};
    size_t off = 0;
    L.bars = off;
    off = al128(off + sizeof(uint64_t) * kNumBars);
    L.meta = off;
    off = al128(off + kMeta * sizeof(PieceMeta));
    L.pubq = off;
    off = al128(off + kPub * sizeof(int32_t) + 64);  // + 16 zero bytes at +64 (padding-row ldmatrix source)
    L.vbuf = off;
    off = al128(off + (mode != kShrink ? size_t(2) * kItemTokCap * kMaxRank * 4 : 0));
    L.red = off;
    off = al128(off + (mode != kExpand ? size_t(2) * kRedFloats * 4 : 0));
    L.xrows = off;
    off = al128(off + (mode != kExpand ? size_t(x_buffers(K, es)) * kItemTokCap * (K * es + 16) : 0));  // x rows, staggered
    L.ring = off;
    off = al128(off + size_t(ns) * slot_stride(mode, K, es));
    L.total = off;
    return L;
}
size_t lora_smem_bytes(int mode, int64_t K, int64_t dchunk, int ns, int esize) {
    return smem_layout(mode, K, dchunk, ns, esize).total;
}
size_t lora_slot_stride(int mode, int64_t K, int esize) { return slot_stride(mode, K, esize); }

struct Ring {
    int slot = 0;
    uint32_t lap = 0;
    __device__ __forceinline__ void advance(int ns) {
        if (++slot == ns) { slot = 0; ++lap; }
    }
};

// Sum VV (power of two) per-lane values across the warp by transposition:
// VV-1 + 5-log2(VV) shuffles instead of 5*VV.  On return lane l holds the
// warp total of value index (l >> (5 - LOG2VV)) & (VV - 1); the lanes whose
// low 5-LOG2VV bits are zero are the writers.  Fixed order (deterministic).
template <int VV, int LOG2VV>
__device__ __forceinline__ float xreduce(float (&v)[VV], int lane) {
#pragma unroll
    for (int step = 0; step < LOG2VV; ++step) {
        const int o = 16 >> step;
        const int half = VV >> (step + 1);
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
            const float send = up ? v[j] : v[j + half];
            const float keep = up ? v[j + half] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    float s = v[0];
#pragma unroll
    for (int o = 16 >> LOG2VV; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// Shrink of one piece, K-split across the consumer warps: warp w owns the
// 16-byte vectors [w*sl, (w+1)*sl) of every stored A row (sl = nvec/8; XV =
// ceil(sl/32) per lane), holds the matching slice of the item's x rows in
// registers (read from smem once per piece; the x buffer is released at
// once), takes the slot's rows two at a time (all loads first), and reduces
// the 2*NT partial dot products of a row pair across lanes by transposition;
// the 8 warps' partials meet in smem (red) and each v entry is written once,
// complete.  Warps do equal work per slot.
template <typename T, int NT, int XV>
__device__ __forceinline__ void shrink_piece(const LoraParams& p, const PieceMeta& M, const unsigned char* ring,
                                             size_t SS, const uint4* xs, int nvec, uint32_t srow, int rps_s,
                                             uint64_t* full, uint64_t* empty, Ring& rg, int ns, uint64_t* xempty,
                                             float* red, float* vout, int warp, int lane, int i) {
    constexpr int NTP = NT == 3 ? 4 : NT;
    constexpr int VV = 2 * NTP;
    constexpr int LOG2VV = VV == 2 ? 1 : (VV == 4 ? 2 : 3);
    const int sl = (nvec + kConsumerWarps - 1) / kConsumerWarps;
    const int v0 = warp * sl, v1 = min(nvec, v0 + sl);
    uint4 xv[NT][XV];
    int li[XV];
#pragma unroll
    for (int k = 0; k < XV; ++k) {
        const int idx = v0 + lane + 32 * k;
        li[k] = min(idx, nvec - 1);  // clamped: x is zero there, so the product vanishes
#pragma unroll
        for (int t = 0; t < NT; ++t) xv[t][k] = idx < v1 ? xs[t * int(srow / 16) + idx] : make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(xempty);  // x slice in registers: buffer free for the next shrink piece
    const bool math = !(p.dbg & 1);
    const int nrows = M.nrows;
    const int nslots = (nrows + rps_s - 1) / rps_s;
    const int wsh = 5 - LOG2VV;
    const int vidx = (lane >> wsh) & (VV - 1);
    const bool writer = (lane & ((1 << wsh) - 1)) == 0;
    const int rsel = vidx / NTP, tw = vidx % NTP;
    // slot by slot (no runtime divisions in the loop); within a slot, rows
    // RQ at a time: all loads first, independent row-pair reductions
    // (RQ = 2 for the widest rows: registers)
    constexpr int RQ = XV >= 4 ? 2 : 4;
    for (int k = 0, rbase = 0; k < nslots; ++k, rbase += rps_s) {
        mbar_wait(&full[rg.slot], rg.lap & 1);
        if (k == 0 && warp == 0 && lane == 0 && i < 48) TRACE(304 + i);
        const int nrow = min(rps_s, nrows - rbase);
        if (math) {
            const unsigned char* sb = ring + size_t(rg.slot) * SS;
            for (int q0 = 0; q0 < nrow; q0 += RQ) {
                uint4 av[RQ][XV];
#pragma unroll
                for (int j = 0; j < RQ; ++j) {
                    const uint4* rp = reinterpret_cast<const uint4*>(sb + size_t(min(q0 + j, nrow - 1)) * srow);
#pragma unroll
                    for (int kk = 0; kk < XV; ++kk) av[j][kk] = rp[li[kk]];
                }
#pragma unroll
                for (int h = 0; h < RQ / 2; ++h) {
                    float c0[VV], c1[VV];
#pragma unroll
                    for (int j = 0; j < VV; ++j) c0[j] = c1[j] = 0.f;
#pragma unroll
                    for (int kk = 0; kk < XV; ++kk)
#pragma unroll
                        for (int t = 0; t < NT; ++t) {
                            dot16<T>(av[2 * h][kk], xv[t][kk], c0[t], c1[t]);
                            dot16<T>(av[2 * h + 1][kk], xv[t][kk], c0[NTP + t], c1[NTP + t]);
                        }
#pragma unroll
                    for (int j = 0; j < VV; ++j) c0[j] += c1[j];
                    const float sum = xreduce<VV, LOG2VV>(c0, lane);
                    const int q = q0 + 2 * h + rsel;
                    if (writer && tw < NT && q < nrow)
                        red[(warp * kShrinkRows + rbase + q) * kItemTokCap + tw] = sum;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rg.slot]);
        rg.advance(ns);
    }
    if (warp == 0 && lane == 0 && i < 48) TRACE(352 + i);
    consumer_sync();  // all warps' partials of the piece are in red
    if (warp == 0 && lane == 0 && i < 48) TRACE(400 + i);
    const int tid = warp * 32 + lane;
    if (tid < M.nrows * NT && math) {
        const int q = tid / NT, t = tid % NT;
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) s += red[(w * kShrinkRows + q) * kItemTokCap + t];
        const int64_t vi = M.vbase + int64_t(t) * M.ra + M.row0 + q;
        if (p.n_peers == 0) {
            vout[vi] = s;
        } else {  // kTPFused: block k of every rank's exchange region (NVLink peer stores)
            for (int j = 0; j < p.n_peers; ++j) p.peer_v[j][int64_t(p.peer_rank) * p.peer_block + vi] = s;
        }
    }
}

// ------------------------------------------------ tensor-core shrink (HMMA)
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
#ifndef SLORA_SHRINK_NACC
#define SLORA_SHRINK_NACC 4
#endif
template <typename T> struct MmaOp {  // fp32: never used (no TF32 for fp32 inputs)
    __device__ static void run(float (&)[4], uint32_t, uint32_t, uint32_t, uint32_t) {}
};
template <> struct MmaOp<__half> {
    __device__ static void run(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
    }
};
template <> struct MmaOp<__nv_bfloat16> {
    __device__ static void run(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
    }
};

// Shrink of one piece on the tensor cores (fp16/bf16): D[token][row] over
// the warp's K-slice with mma.m16n8k16 (M = tokens, rows 8-15 of A are the
// zero register; N = 8 stored A rows; K = 16), fragments loaded with ldmatrix
// from the staggered x rows and A rows (conflict-free).  Rows go 8 at a time
// (the slots holding them are waited for, then released); the 8 warps'
// partials meet in smem (red) as on the CUDA-core path.  Exact products,
// fp32 accumulation in a fixed order (deterministic).  Requires K % 256 == 0
// and a power-of-two rows-per-slot.
template <typename T>
__device__ __forceinline__ void shrink_piece_mma(const LoraParams& p, const PieceMeta& M, const unsigned char* ring,
                                                 size_t SS, const unsigned char* xs, uint32_t zero16, int K,
                                                 uint32_t srow, int lg_rps, uint64_t* full, uint64_t* empty, Ring& rg,
                                                 int ns, uint64_t* xempty, float* red, float* vout, int warp,
                                                 int lane, int i) {
    constexpr int ES = sizeof(T);
    const int kslice = K / kConsumerWarps;  // elements of K per warp (multiple of 16)
    const int k0w = warp * kslice;
    const int mi = lane >> 3, rr = lane & 7;  // ldmatrix: this lane addresses row rr of matrix mi
    const int g = lane >> 2, c = lane & 3;    // mma fragment coordinates
    const int nt = M.nt, nrows = M.nrows;
    // x operand rows: tokens >= nt read 16 zero bytes (and do not advance)
    const bool xreal = rr < nt;
    const uint32_t xbase = xreal ? smem_u32(xs) + uint32_t(rr) * srow + uint32_t(k0w + mi * 8) * ES : zero16;
    const uint32_t xadv = xreal ? 32u * ES : 0u;  // two k-steps per ldmatrix.x4
    const bool math = !(p.dbg & 1);
    const int rps = 1 << lg_rps;
    const int nslots = (nrows + rps - 1) >> lg_rps;
    const int s0 = rg.slot;
    const uint32_t l0 = rg.lap;
    const uint32_t ring_u32 = smem_u32(ring);
    int waited = 0, released = 0;
    bool xfree = false;
    for (int gb = 0; gb < nrows; gb += 8) {
        const int ge = min(gb + 8, nrows);
        const int need = (ge - 1) >> lg_rps;  // last slot this group reads
        for (; waited <= need; ++waited) {
            int a = s0 + waited;  // a piece may span more than one lap of the ring (16 rows of 16 KB)
            uint32_t lap = l0;
            while (a >= ns) { a -= ns; ++lap; }
            mbar_wait(&full[a], lap & 1);
            if (warp == 0 && lane == 0) {
                const int sq = int(lap) * ns + a;
                if (sq < 240) TRACE(512 + sq);
            }
        }
        if (gb == 0 && warp == 0 && lane == 0 && i < 48) TRACE(304 + i);
        if (math) {
            // A-row operand: this lane addresses stored row min(gb + rr, ge - 1) (padding rows repeat a real
            // row; their columns of D are discarded)
            const int row = min(gb + rr, ge - 1);
            int a = s0 + (row >> lg_rps);
            while (a >= ns) a -= ns;
            const uint32_t bbase = ring_u32 + uint32_t(a) * uint32_t(SS) + uint32_t(row & (rps - 1)) * srow +
                                   uint32_t(k0w + mi * 8) * ES;
            const int npair = kslice >> 5;  // k-step pairs
#if SLORA_SHRINK_NACC == 1
            float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
            for (int kp = 0; kp < npair; ++kp) {
                uint32_t xa0, xa1, xa2, xa3, b0, b1, b2, b3;
                ldsm_x4(xbase + uint32_t(kp) * xadv, xa0, xa1, xa2, xa3);
                ldsm_x4(bbase + uint32_t(kp) * (32u * ES), b0, b1, b2, b3);
                MmaOp<T>::run(d, xa0, xa1, b0, b1);
                MmaOp<T>::run(d, xa2, xa3, b2, b3);
            }
#else
            // four independent accumulators (k-steps 4q .. 4q+3): the MMA
            // dependency chain is npair/2 deep instead of 2*npair; combined in
            // a fixed order at the end (deterministic)
            float da[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) da[u][0] = da[u][1] = da[u][2] = da[u][3] = 0.f;
            int kp = 0;
#pragma unroll 2
            for (; kp + 1 < npair; kp += 2) {
                uint32_t xa[2][4], bb[2][4];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    ldsm_x4(xbase + uint32_t(kp + u) * xadv, xa[u][0], xa[u][1], xa[u][2], xa[u][3]);
                    ldsm_x4(bbase + uint32_t(kp + u) * (32u * ES), bb[u][0], bb[u][1], bb[u][2], bb[u][3]);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    MmaOp<T>::run(da[2 * u], xa[u][0], xa[u][1], bb[u][0], bb[u][1]);
                    MmaOp<T>::run(da[2 * u + 1], xa[u][2], xa[u][3], bb[u][2], bb[u][3]);
                }
            }
            if (kp < npair) {
                uint32_t xa0, xa1, xa2, xa3, b0, b1, b2, b3;
                ldsm_x4(xbase + uint32_t(kp) * xadv, xa0, xa1, xa2, xa3);
                ldsm_x4(bbase + uint32_t(kp) * (32u * ES), b0, b1, b2, b3);
                MmaOp<T>::run(da[0], xa0, xa1, b0, b1);
                MmaOp<T>::run(da[1], xa2, xa3, b2, b3);
            }
            float d[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) d[e] = (da[0][e] + da[1][e]) + (da[2][e] + da[3][e]);
#endif
            // d0, d1: token g, rows gb + 2c, gb + 2c + 1 (d2, d3: tokens g + 8, zero)
            if (g < nt) {
                if (gb + 2 * c < nrows) red[(warp * kShrinkRows + gb + 2 * c) * kItemTokCap + g] = d[0];
                if (gb + 2 * c + 1 < nrows) red[(warp * kShrinkRows + gb + 2 * c + 1) * kItemTokCap + g] = d[1];
            }
        }
        if (ge >= nrows && !xfree) {  // the last group: x rows no longer needed
            __syncwarp();
            if (lane == 0) mbar_arrive(xempty);
            xfree = true;
        }
        // release the slots wholly consumed by this group
        const int fin = (ge >= nrows) ? nslots : (ge >> lg_rps);
        __syncwarp();
        for (; released < fin; ++released) {
            int a = s0 + released;
            while (a >= ns) a -= ns;
            if (lane == 0) mbar_arrive(&empty[a]);
        }
    }
    for (int j = 0; j < nslots; ++j) rg.advance(ns);
    if (warp == 0 && lane == 0 && i < 48) TRACE(352 + i);
    consumer_sync();  // all warps' partials of the piece are in red
    if (warp == 0 && lane == 0 && i < 48) TRACE(400 + i);
    const int tid = warp * 32 + lane;
    if (tid < nrows * nt && math) {
        const int q = tid / nt, t = tid % nt;
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) sum += red[(w * kShrinkRows + q) * kItemTokCap + t];
        const int64_t vi = M.vbase + int64_t(t) * M.ra + M.row0 + q;
        if (p.n_peers == 0) {
            vout[vi] = sum;
        } else {  // kTPFused: block k of every rank's exchange region (NVLink peer stores)
            for (int j = 0; j < p.n_peers; ++j) p.peer_v[j][int64_t(p.peer_rank) * p.peer_block + vi] = sum;
        }
    }
}

// Expand of one piece on the tensor cores (fp16/bf16): D[col][token] =
// B^T v^T with mma.m16n8k16 (M = 16 output columns, A operand = B rows read
// transposed by ldmatrix.trans from the staggered slot rows; N = 8 tokens,
// B operand = v split into a 16-bit high and low part (two MMAs: v = hi + lo
// to ~2^-22, so the expand keeps fp32-grade accuracy); K = 16 rank rows,
// i.e. two slots of 8 rows).  The warp owns M.dcols/8 columns (m-tiles of
// 16); D stays in registers over the whole piece and is added once into y
// (y = y + scale*D, one rounding).  Requires dcols % 128 == 0, r % 8 == 0,
// 8 rows per slot.
template <typename T> struct MmaFull;
template <> struct MmaFull<__half> {
    __device__ static void run(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                               uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    __device__ static uint32_t pack(float lo, float hi) {
        __half2 h = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static float2 unpack(uint32_t u) { return __half22float2(*reinterpret_cast<__half2*>(&u)); }
};
template <> struct MmaFull<__nv_bfloat16> {
    __device__ static void run(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                               uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    __device__ static uint32_t pack(float lo, float hi) {
        __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static float2 unpack(uint32_t u) { return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u)); }
};
template <> struct MmaFull<float> {  // never used (fp32 keeps the CUDA-core expand)
    __device__ static void run(float*, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t) {}
    __device__ static uint32_t pack(float, float) { return 0; }
    __device__ static float2 unpack(uint32_t) { return make_float2(0.f, 0.f); }
};
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

constexpr int kMaxMT = 16;  // m-tiles (16 columns) per warp: dcols <= 2048
template <typename T>
__device__ __forceinline__ void expand_piece_mma(const LoraParams& p, const PieceMeta& M, const unsigned char* ring,
                                                 size_t SS, uint32_t erow, uint64_t* full, uint64_t* empty, Ring& rg,
                                                 int ns, const float* vbuf, int warp, int lane, int i) {
    using MF = MmaFull<T>;
    constexpr int ES = sizeof(T);
    const int r = M.r, nt = M.nt;
    const int g = lane >> 2, c = lane & 3;
    const int mi = lane >> 3, rr = lane & 7;
    const int nks = (r + 15) >> 4;  // k-steps of 16 rank rows (<= 4)
    const bool math = !(p.dbg & 2);
    // v operand (col layout, k = rank row, n = token), per k-step: b0b1 = v[tok g][16ks + 2c .. +1],
    // b2b3 = v[tok g][16ks + 8 + 2c .. +1]; split v = hi + lo
    auto vfrag = [&](int ks, int h, uint32_t& hi, uint32_t& lo) {
        const int j = 16 * ks + 8 * h + 2 * c;
        const float v0 = (g < nt && j < r) ? vbuf[g * r + j] : 0.f;
        const float v1 = (g < nt && j + 1 < r) ? vbuf[g * r + j + 1] : 0.f;
        hi = MF::pack(v0, v1);
        const float2 hf = MF::unpack(hi);
        lo = MF::pack(v0 - hf.x, v1 - hf.y);
    };
    const int mt = M.dcols >> 7;  // m-tiles per warp (dcols / 8 warps / 16)
    const int col0 = warp * (mt << 4);
    {  // pull this warp's y segments (nt rows x mt*32 bytes) into L1 now; the epilogue then hits L1
        const int lines = (mt * 16 * ES + 127) >> 7;
        const int t = lane / lines, l = lane % lines;
        if (t < nt && math)
            prefetch_l1(reinterpret_cast<const T*>(p.y[M.proj]) + int64_t(M.tok[t]) * p.ldy[M.proj] + M.dcol0 + col0 +
                        l * (128 / ES));
    }
    float d[kMaxMT][4];
#pragma unroll
    for (int m = 0; m < kMaxMT; ++m) d[m][0] = d[m][1] = d[m][2] = d[m][3] = 0.f;
    const uint32_t ring_u32 = smem_u32(ring);
    // this lane's ldmatrix row: k-row (mi >= 2 ? 8 : 0) + rr of the k-step, column half (mi & 1)
    const int krow = ((mi >> 1) << 3) + rr;
    const uint32_t coff = uint32_t(col0 + ((mi & 1) << 3)) * ES;
    for (int ks = 0; ks < nks; ++ks) {
        // the k-step's rows 16ks..16ks+15 are the next two slots (the second only if r > 16ks + 8)
        const bool two = r > 16 * ks + 8;
        const int sa = rg.slot;
        const uint32_t la = rg.lap;
        int sb = sa + 1;
        uint32_t lb = la;
        if (sb == ns) { sb = 0; ++lb; }
        mbar_wait(&full[sa], la & 1);
        if (two) mbar_wait(&full[sb], lb & 1);
        if (math) {
            uint32_t h0, h1, l0, l1;
            vfrag(ks, 0, h0, l0);
            vfrag(ks, 1, h1, l1);
            // rows 8-15 of a half k-step (r % 16 == 8) re-read rows 0-7 (finite); their v is zero
            const int srow_slot = (krow >= 8 && two) ? sb : sa;
            const uint32_t base = ring_u32 + uint32_t(srow_slot) * uint32_t(SS) + uint32_t(krow & 7) * erow + coff;
#pragma unroll
            for (int m = 0; m < kMaxMT; ++m) {
                if (m < mt) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_t(base + uint32_t(m) * (16u * ES), a0, a1, a2, a3);
                    MF::run(d[m], a0, a1, a2, a3, h0, h1);
                    MF::run(d[m], a0, a1, a2, a3, l0, l1);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[sa]);
            if (two) mbar_arrive(&empty[sb]);
        }
        rg.advance(ns);
        if (two) rg.advance(ns);
    }
    if (warp == 0 && lane == 0 && i < 48) TRACE(352 + i);
    if (!math) return;
    // y[tok][dcol0 + col] += scale * D: d0 (col g, tok 2c), d1 (col g, tok 2c+1), d2/d3 (col g+8)
    T* y = reinterpret_cast<T*>(p.y[M.proj]);
    const int64_t ldy = p.ldy[M.proj];
    const float sc = M.scale;
    // all of a token's y loads first, then the stores (no load waits behind a store)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int t = 2 * c + h;
        if (t < nt) {
            T* yr = y + int64_t(M.tok[t]) * ldy + M.dcol0 + col0 + g;
#pragma unroll
            for (int m0 = 0; m0 < kMaxMT; m0 += 4) {
                if (m0 < mt) {
                    T yv[4][2];
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (m0 + m < mt) {
                            yv[m][0] = yr[(m0 + m) * 16];
                            yv[m][1] = yr[(m0 + m) * 16 + 8];
                        }
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (m0 + m < mt) {
                            yr[(m0 + m) * 16] = T(float(yv[m][0]) + sc * d[m0 + m][h]);
                            yr[(m0 + m) * 16 + 8] = T(float(yv[m][1]) + sc * d[m0 + m][2 + h]);
                        }
                }
            }
        }
    }
}

// Expand of one piece (all B rows of the item over this piece's columns)
// for NT tokens: y_t += scale * v_t B over this thread's 16-byte column
// vector; walks ring slots every `rps` rows.
template <typename T, int NT>
__device__ __forceinline__ void expand_piece(const LoraParams& p, const PieceMeta& M, const unsigned char* ring, size_t SS,
                                             uint32_t rowb, int rps, uint64_t* full, uint64_t* empty, Ring& rg,
                                             int ns, const float* vbuf, bool active, int cv, int lane, int tg,
                                             int ntg) {
    using V = Vec<T>;
    constexpr int VE = V::VE;
    uint32_t own = 0;  // tokens of this piece owned by this thread: t % ntg == tg
    if (active)
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if ((t & (ntg - 1)) == tg) own |= 1u << t;
    active = own != 0;
    float acc[NT][VE];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < VE; ++e) acc[t][e] = 0.f;
    T* y = reinterpret_cast<T*>(p.y[M.proj]);
    const int64_t ldy = p.ldy[M.proj];
    const int64_t col = int64_t(M.dcol0) + int64_t(cv) * VE;
    // y prefetched into registers (hidden behind the row loop) for small
    // token counts; larger counts load it after the loop (register budget)
    constexpr bool kPrefetchY = NT <= 2;
    uint4 yv[kPrefetchY ? NT : 1];
    if (kPrefetchY && active) {
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if (own >> t & 1u)
                yv[kPrefetchY ? t : 0] = *reinterpret_cast<const uint4*>(y + int64_t(M.tok[t]) * ldy + col);
    } else if (active) {  // larger token counts: into L1 (registers are short), read after the rows
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if ((own >> t & 1u) && (cv & 7) == 0) prefetch_l1(y + int64_t(M.tok[t]) * ldy + col);
    }
    const int r = M.r;
    const uint32_t rowv = (rowb + 16) / 16;  // 16-byte vectors per (staggered) row slice
    for (int j0 = 0; j0 < r; j0 += rps) {
        if (j0 > 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[rg.slot]);
            rg.advance(ns);
        }
        mbar_wait(&full[rg.slot], rg.lap & 1);
        if (threadIdx.x == 0) {
            const int sq = int(rg.lap) * ns + rg.slot;
            if (sq < 240) TRACE(512 + sq);
        }
        if (active) {
            const uint4* sl = reinterpret_cast<const uint4*>(ring + size_t(rg.slot) * SS) + cv;
            const int nrow = min(rps, r - j0);
            if ((nrow & 3) == 0) {  // the usual case (ranks are multiples of 4): 4 rows at a time, loads first
                for (int q0 = 0; q0 < nrow; q0 += 4) {
                    uint4 bv[4];
                    float vv[4][NT];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        bv[q] = sl[(q0 + q) * rowv];
#pragma unroll
                        for (int t = 0; t < NT; ++t)  // tokens this thread does not own: v = 0 (branch-free FMAs)
                            vv[q][t] = (own >> t & 1u) ? vbuf[t * r + j0 + q0 + q] : 0.f;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        float b[VE];
                        V::to_f32(bv[q], b);
#pragma unroll
                        for (int t = 0; t < NT; ++t)
#pragma unroll
                            for (int e = 0; e < VE; ++e) acc[t][e] = fmaf(vv[q][t], b[e], acc[t][e]);
                    }
                }
            } else {
                for (int q = 0; q < nrow; ++q) {
                    float b[VE];
                    V::to_f32(sl[q * rowv], b);
                    const float* vc = vbuf + j0 + q;
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        if (own >> t & 1u) {
                            const float vj = vc[t * r];
#pragma unroll
                            for (int e = 0; e < VE; ++e) acc[t][e] = fmaf(vj, b[e], acc[t][e]);
                        }
                    }
                }
            }
        }
    }
    __syncwarp();  // release the piece's last slot
    if (lane == 0) mbar_arrive(&empty[rg.slot]);
    rg.advance(ns);
    if (active) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (!(own >> t & 1u)) continue;
            float yf[VE];
            uint4* yp = reinterpret_cast<uint4*>(y + int64_t(M.tok[t]) * ldy + col);
            V::to_f32(kPrefetchY ? yv[kPrefetchY ? t : 0] : *yp, yf);
#pragma unroll
            for (int e = 0; e < VE; ++e) yf[e] = yf[e] + M.scale * acc[t][e];
            *yp = V::from_f32(yf);
        }
    }
}

// ------------------------------------------------------------ the kernel
template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads, 1) mbgmv_kernel(const __grid_constant__ LoraParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    using V = Vec<T>;
    constexpr int VE = V::VE;
    constexpr int ES = sizeof(T);
    const int64_t K = p.K;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const SmemLayout L = smem_layout(MODE, K, 0, p.ns, ES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + kMaxSlots;
    uint64_t* xfull = empty + kMaxSlots;  // [2] x rows of the CTA's shrink pieces, alternating
    uint64_t* xempty = xfull + 2;
    uint64_t* mfull = xempty + 2;         // [kMeta] resolved piece published
    uint64_t* mempty = mfull + kMeta;     // [kMeta] piece retired by every role
    uint64_t* vfull = mempty + kMeta;     // [2] expand v rows staged (prefetcher -> consumers)
    uint64_t* vempty = vfull + 2;
    uint64_t* pfull = vempty + 2;         // [kPub] shrink piece done (consumers -> publisher)
    uint64_t* pempty = pfull + kPub;
    PieceMeta* meta = reinterpret_cast<PieceMeta*>(smem + L.meta);
    int32_t* pubq = reinterpret_cast<int32_t*>(smem + L.pubq);
    float* vbuf = reinterpret_cast<float*>(smem + L.vbuf);  // [2][kItemTokCap * kMaxRank]
    float* red = reinterpret_cast<float*>(smem + L.red);    // [2][kRedFloats]
    T* xrows = reinterpret_cast<T*>(smem + L.xrows);        // [2][kItemTokCap][K]
    unsigned char* ring = smem + L.ring;                    // [ns][kSlotBytes]
    const int ns = p.ns;
    const uint32_t arow_bytes = uint32_t(K * ES);            // shrink row (full K)
    const uint32_t srow = arow_bytes + 16;                    // its smem stride (staggered; x rows too)
    const int rps_s = shrink_rows_per_slot(K, ES);            // shrink rows per slot
    const size_t SS = slot_stride(MODE, K, ES);               // ring slot stride
    const int nxb = x_buffers(K, ES);                         // x row buffers
    constexpr int kRoles = kConsumerWarps + kStreamers + 1;  // mempty arrivals: consumers, streamers, prefetcher

    if (tid == 0) TRACE(0);
    if (tid == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xfull[b], 1);
            mbar_init(&xempty[b], kConsumerWarps);
            mbar_init(&vfull[b], 1);
            mbar_init(&vempty[b], kConsumerWarps);
        }
        for (int b = 0; b < kMeta; ++b) {
            mbar_init(&mfull[b], 1);
            mbar_init(&mempty[b], kRoles);
        }
        for (int b = 0; b < kPub; ++b) {
            mbar_init(&pfull[b], kConsumerWarps);
            mbar_init(&pempty[b], 1);
        }
        *reinterpret_cast<uint4*>(smem + L.pubq + 64) = make_uint4(0, 0, 0, 0);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_trigger();  // the next launch may start its prologue
    const T* pool = reinterpret_cast<const T*>(p.pool);
    const int64_t P = p.page_elems;
    // the call's descriptors (prepare rewrites the header; written before this grid by a memcpy)
    const CallHdr& H = *p.hdr;
    int32_t* const sync = MODE == kTPFused ? p.peer_ctr[p.peer_rank] : H.sync + int64_t(p.slot) * H.sync_stride;
    float* const vout = MODE == kFused ? H.ws + int64_t(p.slot) * H.ws_stride : p.v;
    const int64_t NR = H.NR;

    if (warp == kWarpResolver) {
        // ============================ resolver ============================
        // This CTA's pieces (host schedule) are loaded 32 at a time, one per
        // lane, with their items; each piece then needs one dependent load
        // (its page ids), kMeta-1 pieces ahead of the consumers.
        const int pb = H.cta_off[blockIdx.x], pe = H.cta_off[blockIdx.x + 1];
        int i = 0;
        for (int base = pb; base < pe; base += 32) {
            const int cnt = min(32, pe - base);
            DevPiece pcl{};
            DevItem itl{};
            if (lane < cnt) {
                pcl = H.pieces[base + lane];
                itl = H.items[pcl.item];
            }
            for (int q = 0; q < cnt; ++q, ++i) {
                const int m = i & (kMeta - 1);
                if (i >= kMeta) mbar_wait_sleep(&mempty[m], ((i / kMeta) - 1) & 1);
                PieceMeta& M = meta[m];
                const int kind = __shfl_sync(0xffffffffu, pcl.kind, q);
                const int pa = __shfl_sync(0xffffffffu, pcl.a, q);
                const int pbn = __shfl_sync(0xffffffffu, pcl.b, q);
                const int rank = __shfl_sync(0xffffffffu, itl.rank, q);
                const int pi = __shfl_sync(0xffffffffu, itl.pi, q);
                const int nt = __shfl_sync(0xffffffffu, itl.nt, q);
                const int tok_off = __shfl_sync(0xffffffffu, itl.tok_off, q);
                const int32_t* itab = reinterpret_cast<const int32_t*>(
                    __shfl_sync(0xffffffffu, (unsigned long long)reinterpret_cast<uintptr_t>(itl.tab), q));
                const int proj = p.proj_ids[pi];
                const int div = (MODE == kExpand) ? 1 : p.a_div[proj];
                const int arp = (MODE == kExpand) ? 1 : p.a_row_pages[proj];
                // the adapter's tables of (layer, proj): A entries (stored rows x arp), then B (r x brp)
                const int32_t* tab = itab + int64_t(rank) * (int64_t(p.layer) * p.layer_units + p.proj_off[proj]);
                int doff = 0;
                if (lane < nt) M.tok[lane] = H.tok_idx[tok_off + lane];
                if (kind == kPieceS) {
                    for (int w = lane; w < pbn * arp; w += 32) M.pages[w] = tab[pa * arp + w];
                } else {  // B rows' pages of the piece's page column (its columns never straddle a page)
                    const int brp = p.b_row_pages[proj];
                    const int c = int(pa / P);
                    doff = pa - int(c * P);
                    const int32_t* tb = tab + int64_t(rank) * p.a_units[proj] + c;
                    for (int w = lane; w < rank; w += 32) M.pages[w] = tb[w * brp];
                }
                if (lane == q) {
                    M.kind = kind;
                    M.item = pcl.item;
                    M.nt = nt;
                    M.r = rank;
                    M.ra = rank / div;
                    M.proj = proj;
                    M.arp = arp;
                    M.n_sp = itl.n_sp;
                    M.n_ep = itl.n_ep;
                    M.scale = itl.scale;
                    M.vbase = int64_t(pi) * (NR / div) + itl.vrow / div;
                    M.pi = pi;
                    M.vrow = itl.vrow;
                    M.row0 = M.dcol0 = pa;
                    M.nrows = M.dcols = pbn;
                    M.doff = doff;
                }
                __syncwarp();
                if (lane == 0 && i < 48) TRACE(16 + i);
                if (lane == 0 && i < 48 && p.trace && blockIdx.x < 16)  // piece code: kind, tokens, rows / rank
                    p.trace[blockIdx.x * kTraceSlots + 208 + i] = kind * 1000000 + nt * 100000 + (kind == kPieceS ? pbn : rank);
                if (lane == 0) mbar_arrive(&mfull[m]);
            }
        }
        const int m = i & (kMeta - 1);
        if (i >= kMeta) mbar_wait_sleep(&mempty[m], ((i / kMeta) - 1) & 1);
        if (lane == 0) {
            meta[m].kind = kPieceStop;
            mbar_arrive(&mfull[m]);
        }
    } else if (streamer_id(warp) >= 0) {
        // ============================ streamers ===========================
        // kStreamers warps issue ring slots round robin (bulk-copy issue costs ~90 ns
        // per copy per warp, measured; two issuers double the rate).
        // Adapter pages are written only by the loader's scatter kernel, which
        // never triggers its dependents early, so the first piece's pages are
        // streamed before griddepcontrol.wait; x, y and v only after it.
        const int sid = streamer_id(warp);
        Ring rg;
        uint32_t seq = 0;  // slot sequence number (shared numbering, both warps)
        bool waited = false;
        int xs = 0;        // shrink pieces seen (x buffer = xs & 1)
        for (int i = 0;; ++i) {
            const int m = i & (kMeta - 1);
            mbar_wait_sleep(&mfull[m], (i / kMeta) & 1);
            const PieceMeta& M = meta[m];
            if (M.kind == kPieceStop) break;
            const bool S = M.kind == kPieceS;
            const int R = S ? M.nrows : M.r;
            const uint32_t rowb = S ? arow_bytes : uint32_t(M.dcols * ES);
            const int rps = S ? rps_s : expand_rows_per_slot(rowb);
            auto issue_slot = [&](int base) {
                const bool mine = (seq++ % uint32_t(kStreamers)) == uint32_t(sid);
                if (!mine) {
                    rg.advance(ns);
                    return;
                }
                const int nrow = min(rps, R - base);
                mbar_wait_sleep(&empty[rg.slot], (rg.lap & 1) ^ 1);
                if (p.dbg & 4) {  // debug: no data movement (consumer-only throughput)
                    if (lane == 0) {
                        const int sq = int(rg.lap) * ns + rg.slot;
                        if (sq < 240) TRACE(768 + sq);
                    }
                    if (lane == 0) mbar_arrive(&full[rg.slot]);
                    rg.advance(ns);
                    return;
                }
                if (lane == 0) {
                    const int sq = int(rg.lap) * ns + rg.slot;
                    if (sq < 240) TRACE(768 + sq);
                }
                if (lane == 0) mbar_arrive_expect_tx(&full[rg.slot], uint32_t(nrow) * rowb);
                __syncwarp();
                unsigned char* sbase = ring + size_t(rg.slot) * SS;
                if (S) {
                    // row q: K elements over arp pages of P (TP q/k/v rows span N pages)
                    const int nc = nrow * M.arp;
                    const int sp = (p.dbg & 8) ? 2 : 1;  // debug: split each page copy in two
                    for (int w = lane; w < nc * sp; w += 32) {
                        const int ww = w / sp, h = w % sp;
                        const int q = ww / M.arp, ch = ww % M.arp;
                        const int64_t k0 = int64_t(ch) * P;
                        const int64_t len = min(P, K - k0) / sp;
                        bulk_g2s(sbase + size_t(q) * srow + (k0 + h * len) * ES,
                                 pool + int64_t(M.pages[(base + q) * M.arp + ch]) * P + h * len, uint32_t(len * ES),
                                 &full[rg.slot]);
                    }
                } else {
                    for (int q = lane; q < nrow; q += 32)
                        bulk_g2s(sbase + size_t(q) * (rowb + 16), pool + int64_t(M.pages[base + q]) * P + M.doff, rowb,
                                 &full[rg.slot]);
                }
                rg.advance(ns);
            };
            int pre = 0;  // slots issued before the PDL wait (first piece only)
            if (!waited) {
                for (int base = 0; base < R && pre < ns; base += rps, ++pre) issue_slot(base);
                pdl_wait();
                waited = true;
            }
            if (S) {  // x rows of the item's tokens
                const int xb = xs % nxb;
                if (sid == 0) {
                    if (xs >= nxb) mbar_wait_sleep(&xempty[xb], ((xs / nxb) - 1) & 1);
                    const bool xcopy = !(p.dbg & (4 | 16));  // debug bit 16: no x rows
                    if (lane == 0) mbar_arrive_expect_tx(&xfull[xb], xcopy ? uint32_t(M.nt) * arow_bytes : 0u);
                    __syncwarp();
                    if (lane < M.nt && xcopy) {
                        const T* x = reinterpret_cast<const T*>(p.x);
                        bulk_g2s(reinterpret_cast<unsigned char*>(xrows) + (size_t(xb) * kItemTokCap + lane) * srow,
                                 x + int64_t(M.tok[lane]) * p.ldx,
                                 arow_bytes, &xfull[xb]);
                    }
                }
                ++xs;
            }
            for (int base = pre * rps; base < R; base += rps) issue_slot(base);
            if (lane == 0 && i < 48) TRACE(160 + i);
            __syncwarp();
            if (lane == 0) mbar_arrive(&mempty[m]);
        }
    } else if (warp == kWarpPrefetch) {
        // ======================= expand-v prefetcher ======================
        // Stages each expand piece's v rows (after its item's shrink pieces
        // are published, fused mode) into vbuf while the consumers still work
        // on earlier pieces.
        int es = 0;
        for (int i = 0;; ++i) {
            const int m = i & (kMeta - 1);
            mbar_wait_sleep(&mfull[m], (i / kMeta) & 1);
            const PieceMeta& M = meta[m];
            if (M.kind == kPieceStop) break;
            if (M.kind == kPieceE) {
                const int eb = es & 1;
                if (es >= 2) mbar_wait_sleep(&vempty[eb], ((es >> 1) - 1) & 1);
                float* vb = vbuf + eb * (kItemTokCap * kMaxRank);
                if (es == 0) pdl_wait();
                if (MODE == kTPFused) {
                    // every rank's shrink pieces of this item (N x n_sp, peer stores + system-scope
                    // releases), then v: the N rank blocks gathered (q/k/v: all-gather) or summed in
                    // rank order (o: all-reduce, deterministic)
                    const int want = p.n_peers * M.n_sp;
                    if (lane == 0) {
                        const long long t_end = gtimer() + 4000000000LL;
                        while (ld_acquire_sys(&sync[M.item]) < want) {
                            __nanosleep(32);
                            if (gtimer() > t_end) {
                                printf("slora: TP expand piece of item %d waited > 4 s for the ranks' shrink pieces\n",
                                       M.item);
                                __trap();
                            }
                        }
                    }
                    __syncwarp();
                    const float* vloc = p.peer_v[p.peer_rank];
                    if (p.v_sum_blocks) {
                        for (int e = lane; e < M.nt * M.r; e += 32) {
                            float a = 0.f;
                            for (int j = 0; j < p.n_peers; ++j) a += __ldcv(vloc + int64_t(j) * p.peer_block + M.vbase + e);
                            vb[e] = a;
                        }
                    } else {
                        const int vbk = p.n_peers, rb = M.r / vbk;
                        const int64_t base = int64_t(M.pi) * (NR / vbk) + M.vrow / vbk;
                        for (int e = lane; e < M.nt * M.r; e += 32) {
                            const int t = e / M.r, j = e % M.r;
                            vb[e] = __ldcv(vloc + int64_t(j / rb) * p.peer_block + base + int64_t(t) * rb + j % rb);
                        }
                    }
                    __syncwarp();
                    if (lane == 0 && atomicAdd(&sync[M.item], 1) == want + M.n_ep - 1) atomicExch(&sync[M.item], 0);
                } else if (MODE == kFused) {
                    if (lane == 0) {
                        // bounded: an expand piece waits for shrink pieces of other CTAs, which
                        // must all be resident (grid <= co-resident CTAs, api.cpp).  If the device
                        // cannot hold them (e.g. SMs taken by MPS / green contexts), fail the
                        // launch after ~4 s instead of hanging (surfaces as SLORA_ERR_CUDA).
                        const long long t_end = gtimer() + 4000000000LL;
                        // a tight acquire-poll (measured: with a 32 ns nanosleep per probe the
                        // C2 layer took 18.90 instead of 18.74 us per launch)
                        while (ld_acquire(&sync[M.item]) < M.n_sp) {
                            if (gtimer() > t_end) {
                                printf("slora: expand piece of item %d waited > 4 s for its shrink pieces: "
                                       "not all CTAs are resident\n", M.item);
                                __trap();
                            }
                        }
                    }
                    __syncwarp();
                    for (int e = lane; e < M.nt * M.r; e += 32) vb[e] = __ldcg(vout + M.vbase + e);
                    __syncwarp();
                    // the item's last expand piece to read v resets its counter for
                    // the launch slot's next use (which starts after this grid ends)
                    if (lane == 0 && atomicAdd(&sync[M.item], 1) == M.n_sp + M.n_ep - 1)
                        atomicExch(&sync[M.item], 0);
                } else {  // v from v_in: block layout of slora_lora_expand
                    const int vbk = p.v_blocks, rb = M.r / vbk;
                    const int64_t stride = int64_t(p.nproj) * (NR / vbk);
                    const int64_t base = int64_t(M.pi) * (NR / vbk) + M.vrow / vbk;
                    for (int e = lane; e < M.nt * M.r; e += 32) {
                        const int t = e / M.r, j = e % M.r;
                        vb[e] = p.v_in[int64_t(j / rb) * stride + base + int64_t(t) * rb + j % rb];
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&vfull[eb]);
                ++es;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&mempty[m]);
        }
    } else if (warp == kWarpPublish) {
        // ========================== publisher =============================
        // Releases each finished shrink piece to the item's expand pieces
        // (red.release.gpu; cumulative over the consumers' v stores observed
        // through the mbarrier), off the consumers' critical path.
        for (int s = 0; MODE == kFused || MODE == kTPFused; ++s) {
            const int b = s & (kPub - 1);
            mbar_wait(&pfull[b], (s / kPub) & 1);  // try_wait, no back-off: the release is on the
            const int item = pubq[b];                 // cross-CTA critical path (measured, see the poll)
            __syncwarp();
            if (lane == 0) mbar_arrive(&pempty[b]);
            if (item < 0) break;
            if (MODE == kFused) {
                if (lane == 0) red_release_add(&sync[item], 1);
            } else if (lane < p.n_peers) {  // kTPFused: the item's counter on every rank
                __threadfence_system();      // the consumers' peer v stores (observed via the mbarrier)
                red_release_add_sys(p.peer_ctr[lane] + item, 1);
            }
        }
    } else {
        // ============================ consumers ===========================
        Ring rg;
        const int nvec = int(arow_bytes / 16);
        // tensor-core shrink for 16-bit types when the shapes allow (fp32 keeps
        // the CUDA-core path: no TF32); SLORA_DBG bit 32 forces CUDA cores
        int lg_rps = 0;
        while ((2 << lg_rps) <= rps_s) ++lg_rps;
        const bool use_mma = ES == 2 && (K % 256) == 0 && (1 << lg_rps) == rps_s && (8 >> lg_rps) <= ns &&
                             !(p.dbg & 32);
        const uint32_t zero16 = smem_u32(smem + L.pubq + 64);
        int xs = 0, es = 0, ps = 0;
        auto publish = [&](int item) {  // hand a finished shrink piece (or the stop mark) to the publisher
            const int b = ps & (kPub - 1);
            if (ps >= kPub) mbar_wait(&pempty[b], ((ps / kPub) - 1) & 1);
            if (tid == 0) pubq[b] = item;
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[b]);
            ++ps;
        };
        for (int i = 0;; ++i) {
            const int m = i & (kMeta - 1);
            mbar_wait(&mfull[m], (i / kMeta) & 1);
            const PieceMeta& M = meta[m];
            if (M.kind == kPieceStop) break;
            if (tid == 0 && i < 48) TRACE(64 + i);
            if (M.kind == kPieceS) {
                // ------------------------------ shrink ------------------------------
                const int xb = xs % nxb;
                mbar_wait(&xfull[xb], (xs / nxb) & 1);
                if (tid == 0 && i < 48) TRACE(256 + i);
                const uint4* xsm = reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned char*>(xrows) +
                                                                  size_t(xb) * kItemTokCap * srow);
                float* rd = red + (xs & 1) * kRedFloats;
                const int xvn = ((nvec + kConsumerWarps - 1) / kConsumerWarps + 31) / 32;
                if (use_mma) {
                    shrink_piece_mma<T>(p, M, ring, SS, reinterpret_cast<const unsigned char*>(xsm), zero16, int(K),
                                        srow, lg_rps, full, empty, rg, ns, &xempty[xb], rd, vout, warp, lane, i);
                } else
                switch (M.nt * 16 + (xvn <= 1 ? 1 : (xvn == 2 ? 2 : (xvn <= 4 ? 4 : 8)))) {
#define SLORA_SHRINK_CASE(N, X)                                                                                  \
    case N * 16 + X:                                                                                           \
        shrink_piece<T, N, X>(p, M, ring, SS, xsm, nvec, srow, rps_s, full, empty, rg, ns, &xempty[xb], rd,      \
                              vout, warp, lane, i);                                                             \
        break;
#ifdef SLORA_FEW_VARIANTS
                    SLORA_SHRINK_CASE(1, 2)
#else
                    // only the token counts an item can have (NT <= kItemTokCap)
                    SLORA_SHRINK_CASE(1, 1) SLORA_SHRINK_CASE(1, 2) SLORA_SHRINK_CASE(1, 4) SLORA_SHRINK_CASE(1, 8)
#if SLORA_ITEM_TOK >= 2
                    SLORA_SHRINK_CASE(2, 1) SLORA_SHRINK_CASE(2, 2) SLORA_SHRINK_CASE(2, 4) SLORA_SHRINK_CASE(2, 8)
#endif
#if SLORA_ITEM_TOK >= 3
                    SLORA_SHRINK_CASE(3, 1) SLORA_SHRINK_CASE(3, 2) SLORA_SHRINK_CASE(3, 4)
#endif
#if SLORA_ITEM_TOK >= 4
                    SLORA_SHRINK_CASE(4, 1) SLORA_SHRINK_CASE(4, 2) SLORA_SHRINK_CASE(4, 4)
#endif
#endif
#undef SLORA_SHRINK_CASE
                    default: break;
                }
                ++xs;
                if (MODE == kFused || MODE == kTPFused) publish(M.item);
            } else {
                // ------------------------------ expand ------------------------------
                const int eb = es & 1;
                mbar_wait(&vfull[eb], (es >> 1) & 1);
                if (tid == 0 && i < 48) TRACE(256 + i);
                const float* vb = vbuf + eb * (kItemTokCap * kMaxRank);
                const uint32_t rowb = uint32_t(M.dcols * ES);
                const int rps = expand_rows_per_slot(rowb);
                const int cvs = M.dcols / VE;
                const int nwc = max(1, (cvs + 31) / 32);
                int ntg = 1;
                while (ntg * 2 * nwc <= kConsumerWarps) ntg *= 2;
                const int wc = warp % nwc, tg = warp / nwc;
                const int cv = wc * 32 + lane;
                const bool active = cv < cvs && tg < ntg && !(p.dbg & 2);
                // tensor-core expand: opt-in (SLORA_DBG bit 128).  Measured slower than the CUDA-core axpys
                // at decode token counts, and using it for some items only would make a token's rounding
                // depend on how its segment is chunked (breaks the batch-permutation bit-identity).
                const bool use_emma = ES == 2 && (p.dbg & 128) && (M.dcols & 127) == 0 && (M.dcols >> 7) <= kMaxMT &&
                                      (M.r & 7) == 0 && M.r <= 64 && expand_rows_per_slot(rowb) == 8;
                if (use_emma)
                    expand_piece_mma<T>(p, M, ring, SS, rowb + 16, full, empty, rg, ns, vb, warp, lane, i);
                else
                switch (M.nt) {
#define SLORA_EXPAND_CASE(N)                                                                                   \
    case N:                                                                                                    \
        expand_piece<T, N>(p, M, ring, SS, rowb, rps, full, empty, rg, ns, vb, active, cv, lane, tg, ntg); \
        break;
#ifdef SLORA_FEW_VARIANTS
                    SLORA_EXPAND_CASE(1)
#else
                    SLORA_EXPAND_CASE(1)
#if SLORA_ITEM_TOK >= 2
                    SLORA_EXPAND_CASE(2)
#endif
#if SLORA_ITEM_TOK >= 3
                    SLORA_EXPAND_CASE(3)
#endif
#if SLORA_ITEM_TOK >= 4
                    SLORA_EXPAND_CASE(4)
#endif
#endif
#undef SLORA_EXPAND_CASE
                    default: break;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&vempty[eb]);
                ++es;
            }
            __syncwarp();
            if (tid == 0 && i < 48) TRACE(112 + i);
            if (lane == 0) mbar_arrive(&mempty[m]);
        }
        if (MODE == kFused || MODE == kTPFused) publish(-1);
    }
    if (tid == 0) TRACE(2);
}

static bool pdl_enabled() {
    static const bool on = [] {
        const char* s = getenv("SLORA_PDL");
        return !(s && atoi(s) == 0);
    }();
    return on;
}

template <typename T, int MODE>
static void* kernel_ptr() {
    return reinterpret_cast<void*>(&mbgmv_kernel<T, MODE>);
}
static void* kernel_for(int mode, int dtype) {
    switch (dtype * 4 + mode) {
        case 0: return kernel_ptr<float, kFused>();
        case 1: return kernel_ptr<float, kShrink>();
        case 2: return kernel_ptr<float, kExpand>();
        case 3: return kernel_ptr<float, kTPFused>();
        case 4: return kernel_ptr<__half, kFused>();
        case 5: return kernel_ptr<__half, kShrink>();
        case 6: return kernel_ptr<__half, kExpand>();
        case 7: return kernel_ptr<__half, kTPFused>();
        case 8: return kernel_ptr<__nv_bfloat16, kFused>();
        case 9: return kernel_ptr<__nv_bfloat16, kShrink>();
        case 10: return kernel_ptr<__nv_bfloat16, kExpand>();
        default: return kernel_ptr<__nv_bfloat16, kTPFused>();
    }
}

template <typename T, int MODE>
static cudaError_t launch_t(const LoraParams& p, int grid, cudaStream_t s, size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (pdl_enabled()) {  // programmatic dependent launch: prologue overlaps the previous kernel
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    count_launch();
    return cudaLaunchKernelEx(&cfg, mbgmv_kernel<T, MODE>, p);
}

template <typename T>
static cudaError_t launch_mode(const LoraParams& p, int mode, int grid, cudaStream_t s, size_t smem) {
    switch (mode) {
        case kFused: return launch_t<T, kFused>(p, grid, s, smem);
        case kShrink: return launch_t<T, kShrink>(p, grid, s, smem);
        case kTPFused: return launch_t<T, kTPFused>(p, grid, s, smem);
        default: return launch_t<T, kExpand>(p, grid, s, smem);
    }
}

cudaError_t launch_lora(const LoraParams& p, int mode, int dtype, int grid, cudaStream_t s, size_t smem) {
    if (grid == 0) return cudaSuccess;  // empty calls still launch: a captured graph may replay a later batch
    switch (dtype) {
        case kF32: return launch_mode<float>(p, mode, grid, s, smem);
        case kF16: return launch_mode<__half>(p, mode, grid, s, smem);
        default: return launch_mode<__nv_bfloat16>(p, mode, grid, s, smem);
    }
}

int lora_max_ctas(int mode, int dtype, size_t smem) {
    void* k = kernel_for(mode, dtype);
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kThreads, smem) != cudaSuccess) return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return blocks * sms;
}

cudaError_t configure_lora_kernels(int /*device*/) {
    const int max_smem = 226 * 1024;  // 227 KB opt-in minus the kernel's static smem
    for (int dt = 0; dt < 3; ++dt)
        for (int m = 0; m < 4; ++m) {
            cudaError_t e = cudaFuncSetAttribute(kernel_for(m, dt), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 max_smem);
            if (e) return e;
        }
    return cudaSuccess;
}

// ------------------------------------------------------------- adapter load
// One CTA per (job, row-block).  A jobs: thread k copies input row k of the
// dense shard (its stored rank columns) into position k of each column page
// -> reads and writes are both coalesced across threads.  B jobs: plain row
// copies.
// It runs beside the LoRA kernels while adapters load (slora_adapter_prefetch), so its CTAs are
// small and short-lived: <= 32 registers x 256 threads (they fit on an SM next to a persistent
// LoRA CTA) and one (job, part) each.
template <typename T>
__global__ void __launch_bounds__(256, 8) scatter_kernel(const T* __restrict__ staging,
                                                         const ScatterJob* __restrict__ jobs, int n_jobs, T* pool,
                                                         int64_t P) {
    constexpr int VE = 16 / int(sizeof(T));
    {
        const int q = blockIdx.y;
        const ScatterJob jb = jobs[q];
        const T* src = staging + jb.src_off;
        if (jb.kind == 0) {
            // A: input row k (cols stored rank columns, contiguous) -> position k%P of column page j
            const bool vec = (jb.cols % VE) == 0 && (jb.src_off % VE) == 0;
            for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < jb.rows;
                 k += int64_t(gridDim.x) * blockDim.x) {
                const int64_t chunk = k / P, off = k % P;
                const T* row = src + k * jb.cols;
                if (vec) {
                    for (int j0 = 0; j0 < jb.cols; j0 += VE) {
                        const uint4 u = *reinterpret_cast<const uint4*>(row + j0);
                        const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
                        for (int t = 0; t < VE; ++t)
                            pool[int64_t(jb.pages[(j0 + t) * jb.row_pages + chunk]) * P + off] = e[t];
                    }
                } else {
                    for (int j = 0; j < jb.cols; ++j)
                        pool[int64_t(jb.pages[j * jb.row_pages + chunk]) * P + off] = row[j];
                }
            }
        } else {
            // B: row j (cols elements) -> its row_pages pages (element e: page e / P, offset e % P),
            // 16-byte vectors (a vector never straddles a page: P % VE == 0)
            const int64_t nv = jb.cols / VE;
            const bool vec = (jb.cols % VE) == 0 && (jb.src_off % VE) == 0 && (P % VE) == 0;
            if (vec) {
                for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < int64_t(jb.rows) * nv;
                     i += int64_t(gridDim.x) * blockDim.x) {
                    const int64_t j = i / nv, e = (i % nv) * VE;
                    *reinterpret_cast<uint4*>(pool + int64_t(jb.pages[j * jb.row_pages + e / P]) * P + e % P) =
                        reinterpret_cast<const uint4*>(src + j * jb.cols)[e / VE];
                }
            } else {
                const int64_t n = int64_t(jb.rows) * jb.cols;
                for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
                     i += int64_t(gridDim.x) * blockDim.x) {
                    const int64_t j = i / jb.cols, e = i % jb.cols;
                    pool[int64_t(jb.pages[j * jb.row_pages + e / P]) * P + e % P] = src[i];
                }
            }
        }
    }
}

cudaError_t launch_scatter(const void* staging, const ScatterJob* jobs_dev, int n_jobs, void* pool,
                           int64_t page_elems, int esize, cudaStream_t s) {
    if (n_jobs == 0) return cudaSuccess;
    const dim3 grid(4, unsigned(n_jobs));
    count_launch();
    if (esize == 4)
        scatter_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(staging), jobs_dev, n_jobs,
                                                      static_cast<uint32_t*>(pool), page_elems);
    else
        scatter_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(staging), jobs_dev, n_jobs,
                                                      static_cast<uint16_t*>(pool), page_elems);
    return cudaGetLastError();
}

__global__ void gather_kernel(const uint8_t* __restrict__ pool, const int32_t* __restrict__ pages, uint8_t* dst,
                              int64_t row_bytes) {
    const int64_t i = blockIdx.x;
    const uint8_t* src = pool + int64_t(pages[i]) * row_bytes;
    for (int64_t b = threadIdx.x; b < row_bytes; b += blockDim.x) dst[i * row_bytes + b] = src[b];
}

cudaError_t launch_gather(const void* pool, const int32_t* pages_dev, int n, void* dst, int64_t page_elems,
                          int esize, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    count_launch();
    gather_kernel<<<n, 256, 0, s>>>(static_cast<const uint8_t*>(pool), pages_dev, static_cast<uint8_t*>(dst),
                                    page_elems * esize);
    return cudaGetLastError();
}

}  // namespace slora
