// kernels.cu -- sm_100a kernels of the S-LoRA hot path.
//
// mbgmv_kernel<T, MODE>: MBGMV gather-shrink-expand over Unified Paging
//   (Sec. 5.3; Eq. lora_factored).
//
//   Persistent, warp-specialized, one thread-block cluster of C CTAs per
//   schedule lane.  CTA c of a cluster owns the c-th 1/C slice of the hidden
//   dimension (K for the shrink, D for the expand).  Each cluster walks its
//   LPT-balanced list of work units (host-built, api.cpp).
//
//   producer warp (warp 8): resolves the unit's items -> adapter page tables,
//     then streams every page slice the unit needs -- x rows into a
//     double-buffered unit stage, A rows and then B rows into a ring of
//     kRowsPerSlot-row slots -- with cp.async.bulk (TMA engine), completion
//     tracked by mbarrier transaction counts.  It runs ahead of the
//     consumers by the ring depth, across unit boundaries, so the next unit's
//     pages are in flight while the current one is expanded.
//   consumer warps (0..7):
//     shrink: one A page-slice row per warp, fp32 dot products with the
//       unit's x rows (16-byte smem vectors, warp-shuffle reductions); each
//       partial v entry is pushed straight into slot [c] of every cluster
//       CTA's exchange buffer (st.shared::cluster), then one remote mbarrier
//       arrive per peer.  Every CTA sums the C partials in the fixed order
//       c = 0..C-1 -> identical v on all CTAs; the rank-r intermediate never
//       leaves distributed shared memory.
//     expand: each thread owns 8 output columns (one 16-byte vector) of a
//       subset of the unit's tokens and accumulates v_j * B_j over the B rows
//       in fp32 registers; y is prefetched into registers at the start and
//       written back once (one rounding).
//   Reduction order depends only on (K, C): results are bit-identical under
//   any page placement, batch permutation or schedule.
//
// MODE kShrink (TP): no expand; v written to global in the C-ABI layout.
// MODE kExpand (TP): no shrink; v read from global (v_blocks rank blocks).
//
// scatter_kernel: adapter load, staging -> pages (A transposed).
// gather_kernel:  test-only page gather.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
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
// arrive on the barrier at the same smem offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
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
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_dsmem(const float* local, uint32_t rank, float v) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(local)), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}
__device__ __forceinline__ uint4 ld_global_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(ev)                                                                       \
    do {                                                                                \
        if (p.trace && blockIdx.x < 16 && (ev) < 256) p.trace[blockIdx.x * 256 + (ev)] = gtimer(); \
    } while (0)
#define TRACE_SLOT(base, seq)              \
    do {                                   \
        if ((seq) < 64) TRACE((base) + (seq)); \
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

// ------------------------------------------------------------ smem layout
struct ItemMeta {
    const int32_t* tab;  // page table of (adapter, layer, proj): A rows then B rows
    int32_t rowA, ra;    // first A row in the unit stream, stored A rows (r / a_div)
    int32_t rowB, r;     // first B row, B rows (= rank)
    int32_t ts, nt;      // token slots
    int32_t v_off;       // first v entry (local units: r/a_div per token in shrink modes)
    int32_t vf_off;      // first v entry in full-rank units (expand)
    int32_t proj, arp;   // projection id, pages per stored A row
    float scale;
    int32_t pi;          // projection index in the call's mask order
    int64_t vrow;        // v row offset (segment vrow_off + t0 * rank)
};
struct UnitMeta {
    int32_t n_items, RA, RB, toks, E, EF, pad0, pad1;
    int32_t tok[kTokCap];        // token row of each slot
    int32_t tok_item[kTokCap];   // item of each slot
    ItemMeta it[kMaxItemsPerUnit];
    int32_t pa[kRowCap][kMaxChunks];  // pages of this CTA's K slice of each A row
    int32_t pb[kRowCap];              // page of each B row
    uint8_t rowA_item[kRowCap];
    uint8_t rowB_item[kRowCap];
};

struct SmemLayout {
    size_t bars, meta, xbuf, vfull, xrows, ring, total, row_bytes;
};
__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }
__host__ __device__ inline SmemLayout smem_layout(int mode, int C, int64_t K, int64_t D, int ns, int es) {
    SmemLayout L{};
    const size_t KS = size_t(K / C), DS = size_t(D / C);
    size_t rb = 0;
    if (mode != kExpand) rb = KS * es;
    if (mode != kShrink && DS * es > rb) rb = DS * es;
    L.row_bytes = (rb + 15) & ~size_t(15);
    size_t off = 0;
    L.bars = off;
    off = al128(off + sizeof(uint64_t) * (2 * kMaxSlots + 8));
    L.meta = off;
    off = al128(off + 2 * sizeof(UnitMeta));
    L.xbuf = off;
    off = al128(off + (mode != kExpand ? size_t(2) * C * kVCap * 4 : 0));
    L.vfull = off;
    off = al128(off + size_t(kVCap) * 4);
    L.xrows = off;
    off = al128(off + (mode != kExpand ? size_t(2) * kTokCap * KS * es : 0));
    L.ring = off;
    off = al128(off + size_t(ns) * kRowsPerSlot * L.row_bytes);
    L.total = off;
    return L;
}
size_t lora_smem_bytes(int mode, int C, int64_t K, int64_t D, int ns, int esize) {
    return smem_layout(mode, C, K, D, ns, esize).total;
}

// ------------------------------------------------------ v4 building blocks
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

// async remote store: value into CTA `rank`'s smem at the address of `local`,
// completing 4 bytes of transaction count on that CTA's barrier `bar`.
__device__ __forceinline__ void st_async_f32(const float* local, const uint64_t* bar, uint32_t rank, float v) {
    uint32_t a, b;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(local)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(a),
                 "r"(__float_as_uint(v)), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct Ring {
    int slot = 0;
    uint32_t lap = 0;
    __device__ __forceinline__ void advance(int ns) {
        if (++slot == ns) { slot = 0; ++lap; }
    }
};

// Shrink of one stored A row slice for NT tokens: v_t = <A_j, x_t> over the
// CTA's K slice; partials pushed to slot [c] of every cluster CTA.
template <typename T, int NT>
__device__ __forceinline__ void shrink_row(const uint4* arow, const T* xr, int64_t KS, int nvec, const ItemMeta& it,
                                           int j, float* xb, uint64_t* xbar, int C, int c, int lane) {
    float a0[NT], a1[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) a0[t] = a1[t] = 0.f;
    const uint4* xv = reinterpret_cast<const uint4*>(xr + size_t(it.ts) * KS);
    const int xstride = int(KS * sizeof(T) / 16);
    for (int q = lane; q < nvec; q += 32) {
        const uint4 a = arow[q];
#pragma unroll
        for (int t = 0; t < NT; ++t) dot16<T>(a, xv[t * xstride + q], a0[t], a1[t]);
    }
    float out[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        float s = a0[t] + a1[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        out[t] = s;
    }
    for (int w = lane; w < NT * C; w += 32) {
        const int t = w / C, cc = w % C;
        float s = 0.f;
#pragma unroll
        for (int tt = 0; tt < NT; ++tt)
            if (tt == t) s = out[tt];
        st_async_f32(xb + size_t(c) * kVCap + it.v_off + t * it.ra + j, xbar, uint32_t(cc), s);
    }
}

// Expand of one item (all its B rows) for NT tokens: y_t += scale * v_t B over
// this thread's 16-byte column vector; walks ring slots at 8-row boundaries.
template <typename T, int NT>
__device__ __forceinline__ void expand_item(const LoraParams& p, const UnitMeta& M, const ItemMeta& it,
                                            const unsigned char* ring, size_t rowb, uint64_t* full, uint64_t* empty,
                                            Ring& rg, int ns, int& row, const float* vfull, bool active, int cv,
                                            int64_t cDS, int lane, int tg, int ntg) {
    using V = Vec<T>;
    constexpr int VE = V::VE;
    // tokens of this item owned by this thread: t % ntg == tg (ntg power of 2)
    uint32_t own = 0;
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
    T* y = reinterpret_cast<T*>(p.y[it.proj]);
    const int64_t ldy = p.ldy[it.proj];
    // y is prefetched into registers for small token counts (hidden behind the
    // row loop); larger items load it after the loop to stay within registers
    constexpr bool kPrefetchY = NT <= 4;
    uint4 yv[kPrefetchY ? NT : 1];
    if (kPrefetchY && active) {
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if (own >> t & 1u)
                yv[kPrefetchY ? t : 0] =
                    *reinterpret_cast<const uint4*>(y + int64_t(M.tok[it.ts + t]) * ldy + cDS + int64_t(cv) * VE);
    }
    for (int j = 0; j < it.r; ++j, ++row) {
        if ((row & (kRowsPerSlot - 1)) == 0) {
            if (row > 0) {
                __syncwarp();
                if (threadIdx.x == 0) TRACE_SLOT(192, int(rg.lap) * ns + rg.slot);
                if (lane == 0) mbar_arrive(&empty[rg.slot]);
                rg.advance(ns);
            }
            mbar_wait(&full[rg.slot], rg.lap & 1);
            if (threadIdx.x == 0) TRACE_SLOT(128, int(rg.lap) * ns + rg.slot);
        }
        if (active) {
            float b[VE];
            V::to_f32(reinterpret_cast<const uint4*>(ring + (size_t(rg.slot) * kRowsPerSlot +
                                                            (row & (kRowsPerSlot - 1))) * rowb)[cv], b);
            const float* vc = vfull + it.vf_off + j;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (own >> t & 1u) {
                    const float vj = vc[t * it.r];
#pragma unroll
                    for (int e = 0; e < VE; ++e) acc[t][e] = fmaf(vj, b[e], acc[t][e]);
                }
            }
        }
    }
    if (active) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (!(own >> t & 1u)) continue;
            float yf[VE];
            uint4* yp = reinterpret_cast<uint4*>(y + int64_t(M.tok[it.ts + t]) * ldy + cDS + int64_t(cv) * VE);
            V::to_f32(kPrefetchY ? yv[kPrefetchY ? t : 0] : *yp, yf);
#pragma unroll
            for (int e = 0; e < VE; ++e) yf[e] = yf[e] + it.scale * acc[t][e];
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
    const int C = p.C;
    const int cl = int(blockIdx.x) / C;
    const int c = (MODE == kExpand) ? int(blockIdx.x % C) : int(cluster_ctarank());
    const int64_t KS = p.K / C, DS = p.D / C;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const SmemLayout L = smem_layout(MODE, C, p.K, p.D, p.ns, ES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + kMaxSlots;
    uint64_t* xfull = empty + kMaxSlots;
    uint64_t* xempty = xfull + 2;
    uint64_t* exch = xempty + 2;
    uint64_t* mfull = exch + 2;
    UnitMeta* meta = reinterpret_cast<UnitMeta*>(smem + L.meta);
    float* xbuf = reinterpret_cast<float*>(smem + L.xbuf);  // [2][C][kVCap]
    float* vfull = reinterpret_cast<float*>(smem + L.vfull);
    T* xrows = reinterpret_cast<T*>(smem + L.xrows);        // [2][kTokCap][KS]
    unsigned char* ring = smem + L.ring;                     // [ns][kRowsPerSlot][row_bytes]
    const int ns = p.ns;
    const size_t rowb = L.row_bytes;

    if (tid == 0) TRACE(0);
    if (tid == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xfull[b], 1);
            mbar_init(&xempty[b], kConsumerWarps);
            mbar_init(&exch[b], 1);
            mbar_init(&mfull[b], 1);
        }
        fence_mbar_init();
    }
    if (MODE == kExpand) __syncthreads();
    else cluster_sync_all();  // peers push into our smem / arrive on our barriers
    pdl_trigger();            // the next launch may start its prologue
    if (tid == 0) TRACE(1);

    const int u_beg = p.sched_off[cl], u_end = p.sched_off[cl + 1];
    const T* pool = reinterpret_cast<const T*>(p.pool);
    const int64_t P = p.page_elems;

    if (warp == kConsumerWarps + 1) {
        // ============================ resolver ============================
        // Resolves unit i (items -> segments -> adapter page tables -> the
        // page ids of every row slice this CTA will stream) one unit ahead of
        // the streamer.  Reads only the batch descriptor and page tables, so
        // under PDL it overlaps the previous launch.
        for (int i = 0; u_beg + i < u_end; ++i) {
            const int ub = i & 1;
            if (i >= 2) mbar_wait(&xempty[ub], ((i >> 1) - 1) & 1);
            UnitMeta& M = meta[ub];
            const DevUnit U = p.units[p.sched[u_beg + i]];
            int ra = 0, rr = 0, ve = 0, vf = 0;
            ItemMeta im{};
            if (lane < U.n_items) {
                const DevItem it = p.items[U.item_begin + lane];
                const int proj = p.proj_ids[it.pi];
                const int div = (MODE == kExpand) ? 1 : p.a_div[proj];
                im.tab = it.tab + int64_t((p.layer * 4 + proj) * 2) * it.rank;
                im.ra = it.rank / div;
                im.r = it.rank;
                im.ts = it.tok_slot;
                im.nt = it.nt;
                im.v_off = it.v_off / div;
                im.vf_off = it.v_off;
                im.proj = proj;
                im.arp = p.a_row_pages[proj];
                im.scale = it.scale;
                im.pi = it.pi;
                im.vrow = it.vrow;
                ra = im.ra;
                rr = im.r;
                ve = im.nt * im.ra;
                vf = im.nt * im.r;
                for (int t = 0; t < it.nt; ++t) {
                    M.tok[it.tok_slot + t] = p.tok_idx[it.tok_off + t];
                    M.tok_item[it.tok_slot + t] = lane;
                }
            }
            int pa = ra, pb = rr;  // inclusive prefix sums over items -> row offsets
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int xa = __shfl_up_sync(0xffffffffu, pa, o);
                const int xb = __shfl_up_sync(0xffffffffu, pb, o);
                if (lane >= o) { pa += xa; pb += xb; }
            }
            if (lane < U.n_items) {
                im.rowA = pa - ra;
                im.rowB = pb - rr;
                M.it[lane] = im;
                for (int j = 0; j < ra; ++j) M.rowA_item[im.rowA + j] = uint8_t(lane);
                for (int j = 0; j < rr; ++j) M.rowB_item[im.rowB + j] = uint8_t(lane);
            }
            int tot_ve = ve, tot_vf = vf;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                tot_ve += __shfl_xor_sync(0xffffffffu, tot_ve, o);
                tot_vf += __shfl_xor_sync(0xffffffffu, tot_vf, o);
            }
            const int RA = __shfl_sync(0xffffffffu, pa, 31);
            const int RB = __shfl_sync(0xffffffffu, pb, 31);
            if (lane == 0) {
                M.n_items = U.n_items;
                M.RA = RA;
                M.RB = RB;
                M.toks = U.toks;
                M.E = tot_ve;
                M.EF = tot_vf;
            }
            __syncwarp();
            if (MODE != kExpand) {
                for (int q = lane; q < RA; q += 32) {
                    const ItemMeta& it = M.it[M.rowA_item[q]];
                    const int j = q - it.rowA;
                    const int64_t k0 = int64_t(c) * KS;
                    const int ch0 = int(k0 / P), ch1 = int((k0 + KS - 1) / P);
                    for (int ch = ch0; ch <= ch1; ++ch) M.pa[q][ch - ch0] = it.tab[j * it.arp + ch];
                }
            }
            if (MODE != kShrink) {
                for (int q = lane; q < RB; q += 32) {
                    const ItemMeta& it = M.it[M.rowB_item[q]];
                    M.pb[q] = it.tab[it.r + (q - it.rowB)];
                }
            }
            __syncwarp();
            if (lane == 0 && i < 4) TRACE(2 + i * 8);
            if (lane == 0) mbar_arrive(&mfull[ub]);
            // Pull the unit's pages into L2 ahead of the streamer: whole pages,
            // each CTA of the cluster taking every C-th row, so the ring's bulk
            // copies hit L2 (more bytes in flight than shared memory holds).
            if (p.l2_prefetch) {
                const uint32_t page_bytes = uint32_t(P * ES);
                if (MODE != kExpand)
                    for (int q = c + lane * C; q < M.RA; q += 32 * C) {
                        const ItemMeta& it = M.it[M.rowA_item[q]];
                        const int j = q - it.rowA;
                        for (int ch = 0; ch < it.arp; ++ch)
                            prefetch_l2(pool + int64_t(it.tab[j * it.arp + ch]) * P, page_bytes);
                    }
                if (MODE != kShrink)
                    for (int q = c + lane * C; q < M.RB; q += 32 * C)
                        prefetch_l2(pool + int64_t(M.pb[q]) * P, page_bytes);
            }
        }
    } else if (warp == kConsumerWarps) {
        // ============================ streamer ============================
        // Adapter pages are written only by the loader's scatter kernel, which
        // never triggers its dependents early, so pages may be streamed before
        // griddepcontrol.wait; x and y (and v) are touched only after it.
        Ring rg;
        bool waited = false;
        for (int i = 0; u_beg + i < u_end; ++i) {
            const int ub = i & 1;
            mbar_wait(&mfull[ub], (i >> 1) & 1);
            if (lane == 0 && i < 4) TRACE(3 + i * 8);
            const UnitMeta& M = meta[ub];
            const int RA = M.RA, RB = M.RB, toks = M.toks;
            auto issue_slot = [&](int phase, int base) {
                const int R = phase == 0 ? RA : RB;
                const uint32_t row_bytes = uint32_t((phase == 0 ? KS : DS) * ES);
                const int nrow = min(kRowsPerSlot, R - base);
                mbar_wait(&empty[rg.slot], (rg.lap & 1) ^ 1);
                if (lane == 0) mbar_arrive_expect_tx(&full[rg.slot], uint32_t(nrow) * row_bytes);
                __syncwarp();
                if (lane < nrow) {
                    const int row = base + lane;
                    unsigned char* dst = ring + (size_t(rg.slot) * kRowsPerSlot + lane) * rowb;
                    if (phase == 0) {
                        int64_t k = int64_t(c) * KS;
                        const int64_t kend = k + KS;
                        int ch = 0;
                        while (k < kend) {  // a slice may span pages (TP q/k/v rows)
                            const int32_t page = M.pa[row][ch++];
                            const int64_t len = min(P - k % P, kend - k);
                            bulk_g2s(dst, pool + int64_t(page) * P + k % P, uint32_t(len * ES), &full[rg.slot]);
                            dst += len * ES;
                            k += len;
                        }
                    } else {
                        bulk_g2s(dst, pool + int64_t(M.pb[row]) * P + int64_t(c) * DS, row_bytes, &full[rg.slot]);
                    }
                }
                if (lane == 0) TRACE_SLOT(64, int(rg.lap) * ns + rg.slot);
                rg.advance(ns);
            };
            const int first_phase = MODE == kExpand ? 1 : 0;
            int pre = 0;  // slots of the first phase issued before the PDL wait
            if (!waited) {
                const int R0 = first_phase == 0 ? RA : RB;
                for (int base = 0; base < R0 && pre < ns; base += kRowsPerSlot, ++pre) issue_slot(first_phase, base);
                pdl_wait();
                waited = true;
            }
            if (MODE != kExpand) {  // x rows of the unit; the same arrive publishes the meta
                if (lane == 0) mbar_arrive_expect_tx(&xfull[ub], uint32_t(toks * KS * ES));
                __syncwarp();
                if (lane < toks) {
                    const T* x = reinterpret_cast<const T*>(p.x);
                    bulk_g2s(xrows + (size_t(ub) * kTokCap + lane) * KS, x + int64_t(M.tok[lane]) * p.ldx + c * KS,
                             uint32_t(KS * ES), &xfull[ub]);
                }
            } else {
                if (lane == 0) mbar_arrive(&xfull[ub]);
            }
            for (int phase = first_phase; phase < 2; ++phase) {  // A rows (K slice c), then B rows (D slice c)
                if (phase == 1 && MODE == kShrink) continue;
                const int R = phase == 0 ? RA : RB;
                for (int base = (phase == first_phase ? pre : 0) * kRowsPerSlot; base < R; base += kRowsPerSlot)
                    issue_slot(phase, base);
            }
            if (lane == 0 && i < 4) TRACE(4 + i * 8);
        }
    } else {
        // ============================ consumers ===========================
        Ring rg;
        const int nvec_k = int(KS * ES / 16);
        // expand: nwc warps cover the D slice's 16-byte column vectors; the
        // remaining warps split the item's tokens (token t -> group t % ntg)
        const int cvs = int(DS / VE);
        const int nwc = max(1, (cvs + 31) / 32);
        int ntg = 1;
        while (ntg * 2 * nwc <= kConsumerWarps) ntg *= 2;
        const int wc = warp % nwc, tg = warp / nwc;
        const int cv = wc * 32 + lane;
        const bool active = cv < cvs && tg < ntg;
        for (int i = 0; u_beg + i < u_end; ++i) {
            const int ub = i & 1;
            mbar_wait(&xfull[ub], (i >> 1) & 1);
            if (tid == 0 && i < 4) TRACE(5 + i * 8);
            const UnitMeta& M = meta[ub];
            if (MODE != kExpand) {
                // ------------------------------ shrink ------------------------------
                float* xb = xbuf + size_t(ub) * C * kVCap;
                if (tid == 0) mbar_arrive_expect_tx(&exch[ub], (p.dbg & 1) ? 0u : uint32_t(C * M.E * 4));
                const T* xr = xrows + size_t(ub) * kTokCap * KS;
                for (int base = 0; base < M.RA; base += kRowsPerSlot) {
                    mbar_wait(&full[rg.slot], rg.lap & 1);
                    if (tid == 0) TRACE_SLOT(128, int(rg.lap) * ns + rg.slot);
                    const int row = base + warp;
                    if (row < M.RA && !(p.dbg & 1)) {
                        const ItemMeta& it = M.it[M.rowA_item[row]];
                        const int j = row - it.rowA;
                        const uint4* arow =
                            reinterpret_cast<const uint4*>(ring + (size_t(rg.slot) * kRowsPerSlot + warp) * rowb);
                        switch (it.nt) {
#define SLORA_SHRINK_CASE(N) \
    case N: shrink_row<T, N>(arow, xr, KS, nvec_k, it, j, xb, &exch[ub], C, c, lane); break;
                            SLORA_SHRINK_CASE(1) SLORA_SHRINK_CASE(2) SLORA_SHRINK_CASE(3) SLORA_SHRINK_CASE(4)
                            SLORA_SHRINK_CASE(5) SLORA_SHRINK_CASE(6) SLORA_SHRINK_CASE(7) SLORA_SHRINK_CASE(8)
#undef SLORA_SHRINK_CASE
                            default: break;
                        }
                    }
                    __syncwarp();
                    if (tid == 0) TRACE_SLOT(192, int(rg.lap) * ns + rg.slot);
                    if (lane == 0) mbar_arrive(&empty[rg.slot]);
                    rg.advance(ns);
                }
                if (tid == 0 && i < 4) TRACE(6 + i * 8);
                mbar_wait(&exch[ub], (i >> 1) & 1);  // all C partials landed (st.async complete_tx)
                if (tid == 0 && i < 4) TRACE(7 + i * 8);
                for (int e = tid; e < M.E; e += kConsumerWarps * 32) {
                    float s = 0.f;
                    for (int cc = 0; cc < C; ++cc) s += xb[size_t(cc) * kVCap + e];  // fixed order
                    if (MODE == kFused) {
                        vfull[e] = s;
                    } else if (e % C == c) {
                        // global v layout: [proj idx][segment][token][r/div]
                        int ii = 0;
                        while (ii + 1 < M.n_items && M.it[ii + 1].v_off <= e) ++ii;
                        const ItemMeta& it = M.it[ii];
                        const int div = it.r / it.ra;
                        const int64_t base = int64_t(it.pi) * (p.NR / div) + it.vrow / div;
                        p.v_out[base + (e - it.v_off)] = s;
                    }
                }
                consumer_sync();
            } else {
                // v from global: block layout of slora_lora_expand
                const int vb = p.v_blocks;
                const int64_t stride = int64_t(p.nproj) * (p.NR / vb);
                for (int e = tid; e < M.EF; e += kConsumerWarps * 32) {
                    int ii = 0;
                    while (ii + 1 < M.n_items && M.it[ii + 1].vf_off <= e) ++ii;
                    const ItemMeta& it = M.it[ii];
                    const int r = it.r, rb = r / vb;
                    const int le = e - it.vf_off, t = le / r, j = le % r;
                    const int64_t base = int64_t(it.pi) * (p.NR / vb) + it.vrow / vb;
                    vfull[e] = p.v_in[int64_t(j / rb) * stride + base + int64_t(t) * rb + (j % rb)];
                }
                consumer_sync();
            }
            if (MODE != kShrink) {
                // ------------------------------ expand ------------------------------
                int row = 0;
                const int64_t cDS = int64_t(c) * DS;
                for (int ii = 0; ii < M.n_items; ++ii) {
                    const ItemMeta& it = M.it[ii];
                    switch (it.nt) {
#define SLORA_EXPAND_CASE(N)                                                                              \
    case N:                                                                                               \
        expand_item<T, N>(p, M, it, ring, rowb, full, empty, rg, ns, row, vfull, active && !(p.dbg & 2), cv, cDS, \
                          lane, tg, ntg);                                                                   \
        break;
                        SLORA_EXPAND_CASE(1) SLORA_EXPAND_CASE(2) SLORA_EXPAND_CASE(3) SLORA_EXPAND_CASE(4)
                        SLORA_EXPAND_CASE(5) SLORA_EXPAND_CASE(6) SLORA_EXPAND_CASE(7) SLORA_EXPAND_CASE(8)
#undef SLORA_EXPAND_CASE
                        default: break;
                    }
                }
                if (row > 0) {  // release the unit's last B slot
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[rg.slot]);
                    rg.advance(ns);
                }
            }
            if (tid == 0 && i < 4) TRACE(8 + i * 8);
            __syncwarp();
            if (lane == 0) mbar_arrive(&xempty[ub]);
        }
    }
    if (tid == 0) TRACE(40);
    if (MODE != kExpand) cluster_sync_all();  // no CTA leaves while peers may touch its smem
    if (tid == 0) TRACE(41);
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
    switch (dtype * 3 + mode) {
        case 0: return kernel_ptr<float, kFused>();
        case 1: return kernel_ptr<float, kShrink>();
        case 2: return kernel_ptr<float, kExpand>();
        case 3: return kernel_ptr<__half, kFused>();
        case 4: return kernel_ptr<__half, kShrink>();
        case 5: return kernel_ptr<__half, kExpand>();
        case 6: return kernel_ptr<__nv_bfloat16, kFused>();
        case 7: return kernel_ptr<__nv_bfloat16, kShrink>();
        default: return kernel_ptr<__nv_bfloat16, kExpand>();
    }
}

template <typename T, int MODE>
static cudaError_t launch_t(const LoraParams& p, cudaStream_t s, size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(p.n_clusters) * unsigned(p.C));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (MODE != kExpand) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = unsigned(p.C);
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
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
static cudaError_t launch_mode(const LoraParams& p, int mode, cudaStream_t s, size_t smem) {
    switch (mode) {
        case kFused: return launch_t<T, kFused>(p, s, smem);
        case kShrink: return launch_t<T, kShrink>(p, s, smem);
        default: return launch_t<T, kExpand>(p, s, smem);
    }
}

cudaError_t launch_lora(const LoraParams& p, int mode, int dtype, cudaStream_t s, size_t smem) {
    if (p.n_clusters == 0) return cudaSuccess;
    switch (dtype) {
        case kF32: return launch_mode<float>(p, mode, s, smem);
        case kF16: return launch_mode<__half>(p, mode, s, smem);
        default: return launch_mode<__nv_bfloat16>(p, mode, s, smem);
    }
}

int lora_max_clusters(int mode, int dtype, int C, size_t smem) {
    void* k = kernel_for(mode, dtype);
    if (mode == kExpand) {
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kThreads, smem) != cudaSuccess) return 0;
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return blocks * sms / C;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(C));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) return 0;
    return n;
}

cudaError_t configure_lora_kernels(int /*device*/) {
    const int max_smem = 227 * 1024;
    for (int dt = 0; dt < 3; ++dt)
        for (int m = 0; m < 3; ++m) {
            void* k = kernel_for(m, dt);
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
            if (e) return e;
            if (m != kExpand) {
                e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                if (e) return e;
            }
        }
    return cudaSuccess;
}

// ------------------------------------------------------------- adapter load
// One CTA per (job, row-block).  A jobs: thread k copies input row k of the
// dense shard (its stored rank columns) into position k of each column page
// -> reads and writes are both coalesced across threads.  B jobs: plain row
// copies.
template <typename T>
__global__ void scatter_kernel(const T* __restrict__ staging, const ScatterJob* __restrict__ jobs, T* pool,
                               int64_t P) {
    const ScatterJob jb = jobs[blockIdx.y];
    const T* src = staging + jb.src_off;
    if (jb.kind == 0) {
        for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < jb.rows;
             k += int64_t(gridDim.x) * blockDim.x) {
            const int64_t chunk = k / P, off = k % P;
            for (int j = 0; j < jb.cols; ++j) {
                const int32_t page = jb.pages[j * jb.row_pages + chunk];
                pool[page * P + off] = src[k * jb.cols + j];
            }
        }
    } else {
        const int64_t n = int64_t(jb.rows) * jb.cols;
        for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
            const int64_t j = i / jb.cols, e = i % jb.cols;
            pool[int64_t(jb.pages[j]) * P + e] = src[i];
        }
    }
}

cudaError_t launch_scatter(const void* staging, const ScatterJob* jobs_dev, int n_jobs, void* pool,
                           int64_t page_elems, int esize, cudaStream_t s) {
    if (n_jobs == 0) return cudaSuccess;
    dim3 grid(8, unsigned(n_jobs));
    count_launch();
    if (esize == 4)
        scatter_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(staging), jobs_dev,
                                                      static_cast<uint32_t*>(pool), page_elems);
    else
        scatter_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(staging), jobs_dev,
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
