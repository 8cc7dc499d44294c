// mbgmm.cu -- tensor-core kernels for long prefill runs (MBGMM, PAPER.md
// Sec. 5.3: "for the prefill stage ... MBGMM").
//
// A *run* is a maximal range of >= theta consecutive x rows (tokens) that use
// the same adapter (a prefill request's tokens).  Its LoRA delta is a small
// GEMM pair, y[n x d] += scale * (x[n x h] A[h x r]) B[r x d], so the weights
// are read once per 64-token tile instead of once per token chunk.  Two
// launches per call (before the MBGMV launch for the remaining tokens):
//
//  mbgmm_shrink_kernel<T>: one CTA per (run tile of <= 64 tokens, projection,
//    group of <= 16 stored A rows).  The 16 A page rows (8 KB each at h=4096)
//    are bulk-copied into smem once, at a 16-byte stagger; x streams through a
//    4-stage ring of 64x64 tiles loaded by TMA (2-D tensor map, 128-byte
//    swizzle).  4 consumer warps, one 16-token m-tile each, run
//    mma.m16n8k16 (M = tokens, N = 8 A rows, K = 16) with ldmatrix operand
//    loads (conflict-free: swizzle for x, stagger for A).  v (fp32) goes to
//    the call's workspace in the MBGMV layout.
//  mbgmm_expand_kernel<T>: one CTA per (run tile, projection, slab of <= 1024
//    output columns).  The slab's r B row slices (2 KB each) are bulk-copied
//    into smem (staggered); the tile's v is split into a 16-bit high and low
//    part (v = hi + lo to ~2^-22) in smem; mma.m16n8k16 (M = tokens, N = 8
//    columns, K = 16 rank rows, B operand via ldmatrix.trans), two MMAs per
//    step (hi, lo); y = y + scale * D, rounded once.
//
// Both accumulate in fp32 in a fixed order (deterministic).  fp16/bf16 only
// (fp32 batches stay on MBGMV: no TF32 for fp32 inputs).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "slora_internal.h"

namespace slora {
namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b))
        : "memory");
}
// 2-D TMA tile load (tensor map in kernel parameter space)
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void grid_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void ldm4(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}
__device__ __forceinline__ void ldm4t(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <typename T> struct Mma;
template <> struct Mma<__half> {
    __device__ static void run(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    __device__ static uint16_t bits(float v) { return __half_as_ushort(__float2half_rn(v)); }
    __device__ static float val(uint16_t b) { return __half2float(__ushort_as_half(b)); }
    __device__ static uint32_t pack2(float lo, float hi) {
        __half2 h = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static float2 unpack2(uint32_t u) { return __half22float2(*reinterpret_cast<__half2*>(&u)); }
};
template <> struct Mma<__nv_bfloat16> {
    __device__ static void run(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    __device__ static uint16_t bits(float v) { return __bfloat16_as_ushort(__float2bfloat16_rn(v)); }
    __device__ static float val(uint16_t b) { return __bfloat162float(__ushort_as_bfloat16(b)); }
    __device__ static uint32_t pack2(float lo, float hi) {
        __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static float2 unpack2(uint32_t u) { return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u)); }
};

constexpr int kMgConsumers = 4;                        // 4 x 16-token m-tiles
constexpr int kMgThreads = (kMgConsumers + 1) * 32;    // + producer warp
#ifndef SLORA_MG_XSTAGES
#define SLORA_MG_XSTAGES 12
#endif
constexpr int kXStages = SLORA_MG_XSTAGES;  // 96 KB of x in flight per CTA (measured: 4 stages -9%, 8 -> 12 +1.5% on C2-mixed)
constexpr int kXTileBytes = kMgTileTok * 64 * 2;       // 64 tokens x 64 elements (8 KB)
constexpr int kMgMaxRows = 32;                          // stored A rows per shrink unit, at most

__host__ __device__ inline size_t al(size_t x, size_t a) { return (x + a - 1) & ~(a - 1); }

// shrink smem: [bars][A rows R x (Kp*2+16)][x ring of 8 KB stages, 1 KB aligned]: a unit holds R
// stored A rows over Kp = K / split columns (its K part), with as many x stages as fit (<= kXStages).
// The host picks (split, R) per hidden size (mg_plan): the x tile streams through the SM once per
// R A rows, so fewer, taller units move less x; splitting K makes room for taller units.
__host__ __device__ inline size_t mg_shrink_base(int64_t Kp, int rows) {
    return al(256 + size_t(rows) * (Kp * 2 + 16), 1024) + 1024;
}
__host__ __device__ inline int mg_xstages_rows(int64_t Kp, int rows) {
    const size_t base = mg_shrink_base(Kp, rows), lim = size_t(227) * 1024;
    const int st = base >= lim ? 0 : int((lim - base) / kXTileBytes);
    return st < kXStages ? st : kXStages;
}
// the tallest unit (32, 16 or 8 A rows) that leaves room for >= 8 x stages
__host__ __device__ inline int mg_rows_kp(int64_t Kp) {
    for (int r = kMgMaxRows; r > 8; r /= 2)
        if (mg_xstages_rows(Kp, r) >= 8) return r;
    return 8;
}
__host__ __device__ inline size_t mg_shrink_smem_kp(int64_t Kp, int rows) {
    return mg_shrink_base(Kp, rows) + size_t(mg_xstages_rows(Kp, rows)) * kXTileBytes;
}
// expand smem: [bars][B slab r x (nc*2+16)][v hi, lo: 64 x (rp+8) 16-bit each]; the host
// sizes slabs (mbgmm_expand_cols) so that two CTAs fit on an SM (one loads while one computes)
// [y staging: one 16-row x 64-column tile per consumer warp, rows kYs 16-bit elements apart]
constexpr int kYs = 72;  // 144-byte rows: the accumulator-layout accesses hit 32 distinct banks
__host__ __device__ inline size_t mg_expand_smem_unit(int r, int nc) {
    const int rp = (r + 15) & ~15;
    return 256 + size_t(r) * (size_t(nc) * 2 + 16) + 2 * size_t(kMgTileTok) * (rp + 8) * 2 +
           size_t(kMgConsumers) * 16 * kYs * 2 + 128;
}

// NG = 16-row groups per unit (1: <= 16 A rows, 2: <= 32)
template <typename T, int NG>
__global__ void __launch_bounds__(kMgThreads, 1) mbgmm_shrink_kernel(const __grid_constant__ MgParams p) {
    using O = Mma<T>;
    constexpr int ES = 2;
    extern __shared__ __align__(1024) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const MgUnit u = p.units[blockIdx.x];
    const int Kp = p.K / p.ksplit;                  // this unit's part of K (u.pad = part)
    const int kb0 = u.pad * (Kp / 64);              // its first 64-column x block
    const uint32_t arow = uint32_t(Kp) * ES + 16;  // staggered A row stride
    uint64_t* abar = reinterpret_cast<uint64_t*>(sm);
    uint64_t* xfull = abar + 1;
    uint64_t* xempty = xfull + kXStages;
    unsigned char* arows = sm + 256;
    unsigned char* xring = sm + al(256 + size_t(p.srows) * arow, 1024);
    // the dynamic smem base is 1 KB aligned only up to the driver's guarantee: align the ring explicitly
    xring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(xring) + 1023) & ~uintptr_t(1023));
    const int nrows = u.b;
    const int nkc = Kp / 64;
    const int xst = mg_xstages_rows(Kp, p.srows);  // x ring stages
    if (tid == 0) {
        bar_init(abar, 1);
        for (int s = 0; s < xst; ++s) {
            bar_init(&xfull[s], 1);
            bar_init(&xempty[s], kMgConsumers);
        }
        bar_fence_init();
    }
    __syncthreads();
    grid_trigger();
    if (warp == kMgConsumers) {
        // ---- producer: the group's A rows (pages: loader-written, safe before the PDL wait), then x tiles
        const int proj = p.proj_ids[u.pi];
        const int32_t* tab = u.tab + int64_t((p.layer * 4 + proj) * 2) * u.rank;  // [A rows][B rows]
        if (lane == 0) bar_expect(abar, uint32_t(nrows) * uint32_t(Kp) * ES);
        __syncwarp();
        if (lane < nrows)
            copy_g2s(arows + size_t(lane) * arow,
                     static_cast<const T*>(p.pool) + int64_t(tab[u.a + lane]) * p.page_elems + int64_t(kb0) * 64,
                     uint32_t(Kp) * ES, abar);
        grid_wait();
        if (lane == 0)
            for (int kc = 0; kc < nkc; ++kc) {
                const int s = kc % xst;
                if (kc >= xst) bar_wait(&xempty[s], ((kc / xst) - 1) & 1);
                bar_expect(&xfull[s], kXTileBytes);
                tma_2d(xring + size_t(s) * kXTileBytes, &p.xmap, (kb0 + kc) * 64, u.row0, &xfull[s]);
            }
        return;
    }
    // ---- consumers: warp w = tokens 16w..16w+15
    const int mi = lane >> 3, rr = lane & 7, g = lane >> 2, c = lane & 3;
    const int xrow = warp * 16 + ((mi & 1) << 3) + rr;      // A-operand (x) row of this lane's ldmatrix
    const int achk = mi >> 1;                               // its 16-byte chunk within the k-step
    uint32_t bbase[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) {
        // B-operand (A row) of this lane in 16-row group q; padding rows repeat a real one
        const int brow = min(16 * q + ((mi >> 1) << 3) + rr, nrows - 1);
        bbase[q] = su32(arows) + uint32_t(brow) * arow + uint32_t((mi & 1) << 4);
    }
    const uint32_t xbase = su32(xring) + uint32_t(xrow) * 128u;
    float d[2 * NG][4] = {};
    bar_wait(abar, 0);
    for (int kc = 0; kc < nkc; ++kc) {
        const int s = kc % xst;
        bar_wait(&xfull[s], (kc / xst) & 1);
        const uint32_t xs = xbase + uint32_t(s) * kXTileBytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t a[4];
            const int chunk = 2 * kk + achk;  // 128-byte swizzle: 16-byte chunk j of row r sits at j ^ (r & 7)
            ldm4(xs + uint32_t((chunk ^ (xrow & 7)) << 4), a);
#pragma unroll
            for (int q = 0; q < NG; ++q) {
                uint32_t b[4];
                ldm4(bbase[q] + uint32_t(kc * 64 + kk * 16) * ES, b);
                O::run(d[2 * q], a, b[0], b[1]);
                O::run(d[2 * q + 1], a, b[2], b[3]);
            }
        }
        __syncwarp();
        if (lane == 0) bar_arrive(&xempty[s]);
    }
    // d[n][0..1]: token 16w+g, A rows 8n+2c, 8n+2c+1; d[n][2..3]: token 16w+g+8
    float* vout = p.v + int64_t(u.pad) * p.vpart;
#pragma unroll
    for (int n = 0; n < 2 * NG; ++n)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = warp * 16 + g + 8 * h;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = 8 * n + 2 * c + e;
                if (t < u.nt && row < nrows) vout[u.vbase + int64_t(t) * u.rank + u.a + row] = d[n][2 * h + e];
            }
        }
}

template <typename T>
__global__ void __launch_bounds__(kMgThreads, 2) mbgmm_expand_kernel(const __grid_constant__ MgParams p) {
    using O = Mma<T>;
    constexpr int ES = 2;
    extern __shared__ __align__(1024) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const MgUnit u = p.units[blockIdx.x];
    const int r = u.rank, nc = u.b;
    const int rp = (r + 15) & ~15;                 // rank padded to whole k-steps
    const uint32_t brow = uint32_t(nc) * ES + 16;  // staggered B row-slice stride
    const int vst = rp + 8;                        // v tile row stride (16-bit elements)
    uint64_t* bbar = reinterpret_cast<uint64_t*>(sm);
    unsigned char* slab = sm + 256;
    uint16_t* vhi = reinterpret_cast<uint16_t*>(sm + 256 + size_t(r) * brow);
    uint16_t* vlo = vhi + kMgTileTok * vst;
    if (tid == 0) {
        bar_init(bbar, 1);
        bar_fence_init();
    }
    __syncthreads();
    grid_trigger();
    if (warp == kMgConsumers) {
        const int proj = p.proj_ids[u.pi];
        const int32_t* tab = u.tab + int64_t((p.layer * 4 + proj) * 2) * r + r;  // B rows
        if (lane == 0) bar_expect(bbar, uint32_t(r) * uint32_t(nc) * ES);
        __syncwarp();
        for (int j = lane; j < r; j += 32)
            copy_g2s(slab + size_t(j) * brow, static_cast<const T*>(p.pool) + int64_t(tab[j]) * p.page_elems + u.a,
                     uint32_t(nc) * ES, bbar);
        return;
    }
    grid_wait();  // v (previous kernel) and y are read below
    // v tile -> smem, split into hi + lo (zero beyond the tile's tokens and the rank)
    // (eight independent loads in flight per thread, then the conversions: a serial
    // load -> store loop waits one L2 round trip per element)
    // the k-split parts are summed part by part with kU loads in flight per round (a per-element
    // loop over the parts waited one L2 round trip per part and element batch)
#ifndef SLORA_MG_VU
#define SLORA_MG_VU 8
#endif
    constexpr int kU = SLORA_MG_VU;
    const int nel = kMgTileTok * rp;
    for (int e0 = tid; e0 < nel; e0 += kU * kMgConsumers * 32) {
        float val[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) val[q] = 0.f;
        if (e0 < u.nt * rp)
            for (int ks = 0; ks < p.ksplit; ++ks) {
                const float* vp = p.v + ks * p.vpart + u.vbase;
                float tmp[kU];
#pragma unroll
                for (int q = 0; q < kU; ++q) {
                    const int e = e0 + q * kMgConsumers * 32;
                    const int t = e / rp, j = e % rp;
                    tmp[q] = (e < nel && t < u.nt && j < r) ? __ldcg(vp + int64_t(t) * r + j) : 0.f;
                }
#pragma unroll
                for (int q = 0; q < kU; ++q) val[q] += tmp[q];  // parts added in order (deterministic)
            }
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const int e = e0 + q * kMgConsumers * 32;
            if (e < nel) {
                const int t = e / rp, j = e % rp;
                const uint16_t hb = O::bits(val[q]);
                vhi[t * vst + j] = hb;
                vlo[t * vst + j] = O::bits(val[q] - O::val(hb));
            }
        }
    }
    named_sync(1, kMgConsumers * 32);
    bar_wait(bbar, 0);
    const int mi = lane >> 3, rr = lane & 7, g = lane >> 2, c = lane & 3;
    // warps -> (16-token m-tile, column group): a tile of <= 16 / <= 32 tokens (gathered decode
    // segments) gives each m-tile 4 / 2 warps that split the slab's 64-column sub-chunks, so all
    // four warps keep y loads in flight instead of idling on empty m-tiles
#ifndef SLORA_MG_NO_WSPLIT
    const int wpm = u.nt <= 16 ? 4 : (u.nt <= 32 ? 2 : 1);
#else
    const int wpm = 1;
#endif
    const int mt = warp / wpm, cg = warp % wpm;
    // A operand (v): row = token 16mt + (mi&1)*8 + rr, k chunk (mi>>1)*8
    const int arow_ = mt * 16 + ((mi & 1) << 3) + rr;
    const uint32_t ahi = su32(vhi) + uint32_t(arow_ * vst + ((mi >> 1) << 3)) * ES;
    const uint32_t alo = su32(vlo) + uint32_t(arow_ * vst + ((mi >> 1) << 3)) * ES;
    T* y = reinterpret_cast<T*>(p.y[p.proj_ids[u.pi]]);
    const int64_t ldy = p.ldy[p.proj_ids[u.pi]];
    const int t0 = mt * 16 + g, t1 = t0 + 8;
    // gathered mode (segments of scattered tokens): x-map row i is token p.yrow[i]
    const int64_t yr0 = t0 < u.nt ? (p.yrow ? p.yrow[u.row0 + t0] : u.row0 + t0) : 0;
    const int64_t yr1 = t1 < u.nt ? (p.yrow ? p.yrow[u.row0 + t1] : u.row0 + t1) : 0;
    T* y0 = y + yr0 * ldy + u.a;
    T* y1 = y + yr1 * ldy + u.a;
    const int sc0 = cg * 64, scs = wpm * 64;  // this warp's first sub-chunk and its stride
#ifndef SLORA_MG_NO_YPF
    // the warp's y row lines into L2 now (one 128-byte line per prefetch, lanes c == 0 of each row
    // pair): the sub-chunk loads below then wait for L2, not HBM
    if (c == 0) {
        for (int sc = sc0; sc < nc; sc += scs)
            for (int l = sc * ES; l < (sc + 64) * ES && l < nc * ES; l += 128) {
                if (t0 < u.nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(y0) + l));
                if (t1 < u.nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(y1) + l));
            }
    }
#endif
    if (mt * 16 >= u.nt) return;  // (wpm = 1: an m-tile past the tile's tokens)
    // y moves through a warp-private smem tile in whole 128-byte rows (coalesced 16-byte vectors:
    // lane = row 4i + lane/8, 16-byte chunk lane%8), one 64-column sub-chunk ahead in registers;
    // the accumulator-layout read-modify-write happens in smem; each y element is read and
    // written once
    uint16_t* ys = vlo + kMgTileTok * vst + warp * 16 * kYs;
    const int vr = lane >> 3, vc = (lane & 7) * 8;
    T* yrow4[4];
    bool live[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int t = mt * 16 + 4 * i + vr;
        live[i] = t < u.nt;
        yrow4[i] = y + (live[i] ? (p.yrow ? p.yrow[u.row0 + t] : u.row0 + t) : 0) * ldy + u.a + vc;
    }
    uint4 yn[4];
    auto load_y = [&](int sc) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (live[i]) yn[i] = *reinterpret_cast<const uint4*>(yrow4[i] + sc);
    };
    if (sc0 < nc) load_y(sc0);
    for (int sc = sc0; sc < nc; sc += scs) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(ys + (4 * i + vr) * kYs + vc) = yn[i];
        if (sc + scs < nc) load_y(sc + scs);
        float d[8][4] = {};
        for (int k = 0; k < rp; k += 16) {
            uint32_t ah[4], alw[4];
            ldm4(ahi + uint32_t(k) * ES, ah);
            ldm4(alo + uint32_t(k) * ES, alw);
            // B operand (B rows, k = rank row, n = column) through ldmatrix.trans: matrices
            // (rows k..k+7 | k+8..k+15) x (cols n..n+7 | n+8..n+15); rows >= r repeat row r-1 (v is 0 there)
            const int krow = min(k + ((mi & 1) << 3) + rr, r - 1);
#pragma unroll
            for (int n2 = 0; n2 < 4; ++n2) {
                uint32_t b[4];
                ldm4t(su32(slab) + uint32_t(krow) * brow + uint32_t(sc + n2 * 16 + ((mi >> 1) << 3)) * ES, b);
                O::run(d[2 * n2], ah, b[0], b[1]);
                O::run(d[2 * n2 + 1], ah, b[2], b[3]);
#ifndef SLORA_MG_NO_LO
                O::run(d[2 * n2], alw, b[0], b[1]);
                O::run(d[2 * n2 + 1], alw, b[2], b[3]);
#endif
            }
        }
        __syncwarp();
        // y += scale * D: d[n][0..1] row g, columns 8n + 2c (+1); d[n][2..3] row g + 8
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t* e = reinterpret_cast<uint32_t*>(ys + (g + 8 * h) * kYs + 8 * n + 2 * c);
                const float2 f = O::unpack2(*e);
                *e = O::pack2(f.x + u.scale * d[n][2 * h], f.y + u.scale * d[n][2 * h + 1]);
            }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (live[i])
                *reinterpret_cast<uint4*>(yrow4[i] + sc) = *reinterpret_cast<const uint4*>(ys + (4 * i + vr) * kYs + vc);
        __syncwarp();
    }
}


// ------------------------------------------------------------------ tcgen05
// mbgmm_shrink_tc_kernel<T>: one CTA per (run tile of <= 64 tokens,
// projection, quarter of K) computes the tile's shrink on the 5th-generation tensor
// cores: D[token][j] (fp32, TMEM) = sum_k x[token][k] A_j[k] for all r stored
// A rows at once (N = r rounded up to 16), so x streams through the SM once
// per tile instead of once per group of A rows.  Per 64-wide k-block:
//   * the x tile arrives by TMA (2-D tensor map, SWIZZLE_128B = the canonical
//     K-major layout the tensor core reads), 8 stages of 64 rows x 128 B;
//     the MMA uses M = 128 (the smallest single-CTA shape with a plain
//     lane = row accumulator layout): stages are 8 KB apart, so operand rows
//     64..127 are the next stage's tile and only feed accumulator rows that
//     are never read back;
//   * the A k-block (N rows x 128 B, gathered from N pool pages) is copied by
//     two loader warps with cp.async (16 B per lane) straight into the
//     canonical layout -- row n at (n/8)*1024 + (n%8)*128, 16-byte chunk c at
//     (c ^ n%8)*16 -- rows >= r zero-filled; each loader makes its copies
//     visible to the async proxy (fence.proxy.async) before arriving on the
//     stage's barrier;
//   * one thread issues 4 tcgen05.mma.cta_group::1.kind::f16 (K = 16 each,
//     descriptors advanced 32 B inside the swizzle atom) into 4 independent
//     TMEM accumulators (k-step j -> accumulator j: short dependency chains),
//     then tcgen05.commit frees the stage.
// Epilogue: warps 0-1 (TMEM lanes 0-63 = the tile's tokens) load the 4
// accumulators (tcgen05.ld.32x32b.x16), add them in a fixed order
// ((d0 + d1) + (d2 + d3): deterministic) and write the part's partial v; the
// expand kernel adds the kMgKsplit parts in order.
constexpr int kTcThreads = 192;  // warps 0-1 epilogue, 2 TMEM + x producer, 3 MMA issuer, 4-5 A loaders
#ifndef SLORA_TC_STAGES
#define SLORA_TC_STAGES 6  // 6 x 16 KB: two CTAs per SM
#endif
constexpr int kTcStages = SLORA_TC_STAGES;
constexpr int kTcXStage = kXTileBytes;  // 8 KB (see above: M = 128 windows overlap the next stage)
constexpr int kTcAStage = 64 * 128;     // N <= 64 rows x 128 B
constexpr int kTcLoaders = 64;
constexpr int kTcAhead = 4;             // A stages a loader keeps in flight before publishing

__host__ __device__ inline size_t mg_shrink_tc_smem(int64_t) {
    return 1024 + 1024 + size_t(kTcStages) * (kTcXStage + kTcAStage) + kTcXStage;
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    // start address >> 4 (bits 0-13), LBO 1 (unused for swizzled K-major), SBO = 1024 B >> 4 (bits 32-45),
    // version 1 (bit 46), layout SWIZZLE_128B = 2 (bits 61-63)
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) |
           (uint64_t(2) << 61);
}
template <typename T> struct TcFmt;
template <> struct TcFmt<__half> { static constexpr uint32_t v = 0; };
template <> struct TcFmt<__nv_bfloat16> { static constexpr uint32_t v = 1; };

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&d)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
          "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(taddr));
}

template <typename T>
__global__ void __launch_bounds__(kTcThreads, 2) mbgmm_shrink_tc_kernel(const __grid_constant__ MgParams p) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const MgUnit u = p.units[blockIdx.x];
    const int K = p.K;
    const int nkc = K / 64 / p.ksplit;  // k-blocks of this unit's part of K
    const int kb0 = u.pad * nkc;        // its first k-block
    float* vout = p.v + u.pad * p.vpart;
    const int r = u.rank;
    const int npad = (r + 15) & ~15;  // MMA N
    uint64_t* xfull = reinterpret_cast<uint64_t*>(sm);
    uint64_t* afull = xfull + kTcStages;
    uint64_t* sempty = afull + kTcStages;
    uint64_t* done = sempty + kTcStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    unsigned char* aring = sm + 1024;                               // kTcStages x 8 KB (1 KB-aligned atoms)
    unsigned char* xring = aring + size_t(kTcStages) * kTcAStage;   // kTcStages x 8 KB + 8 KB pad
    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            bar_init(&xfull[s], 1);
            bar_init(&afull[s], kTcLoaders);
            bar_init(&sempty[s], 1);
        }
        bar_init(done, 1);
        bar_fence_init();
    }
    if (warp == 2) {  // TMEM: 4 accumulators x 64 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    grid_trigger();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
    if (warp >= 4) {
        // ---- A loaders: thread i copies chunk (i & 7) of rows (i >> 3) + 8 m (pages: loader-written,
        // safe before the PDL wait)
        const int i = tid - 128, c = i & 7, n0 = i >> 3;
        const int proj = p.proj_ids[u.pi];
        const int32_t* tab = u.tab + int64_t((p.layer * 4 + proj) * 2) * r;
        const T* pool = static_cast<const T*>(p.pool);
        const T* src[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int n = n0 + 8 * m;
            src[m] = pool + int64_t(tab[min(n, r - 1)]) * p.page_elems + c * 8;
        }
        const uint32_t abase = su32(aring) + uint32_t(n0 & 7) * 128u + uint32_t((c ^ (n0 & 7)) << 4);
        for (int kc = 0; kc < nkc; ++kc) {
            const int s = kc % kTcStages;
            if (kc >= kTcStages) bar_wait(&sempty[s], ((kc / kTcStages) - 1) & 1);
            const uint32_t dst = abase + uint32_t(s) * kTcAStage;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int n = n0 + 8 * m;
                if (n < npad)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + uint32_t(m) * 1024u),
                                 "l"(src[m] + int64_t(kb0 + kc) * 64), "r"(n < r ? 16 : 0)
                                 : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            if (kc >= kTcAhead) {  // publish the stage issued kTcAhead k-blocks ago
                asm volatile("cp.async.wait_group %0;" ::"n"(kTcAhead) : "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bar_arrive(&afull[(kc - kTcAhead) % kTcStages]);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int kc = max(0, nkc - kTcAhead); kc < nkc; ++kc) bar_arrive(&afull[kc % kTcStages]);
    } else if (tid == 64) {
        // ---- x producer (after the PDL wait: x is the previous launch's output)
        grid_wait();
        for (int kc = 0; kc < nkc; ++kc) {
            const int s = kc % kTcStages;
            if (kc >= kTcStages) bar_wait(&sempty[s], ((kc / kTcStages) - 1) & 1);
            bar_expect(&xfull[s], kXTileBytes);
            tma_2d(xring + size_t(s) * kTcXStage, &p.xmap, (kb0 + kc) * 64, u.row0, &xfull[s]);
        }
    } else if (tid == 96) {
        // ---- MMA issuer (one thread)
        const uint32_t idesc = (1u << 4) | (TcFmt<T>::v << 7) | (TcFmt<T>::v << 10) | (uint32_t(npad >> 3) << 17) |
                               ((128u >> 4) << 24);
        const uint32_t xb = su32(xring), ab = su32(aring);
        for (int kc = 0; kc < nkc; ++kc) {
            const int s = kc % kTcStages;
            const uint32_t ph = (kc / kTcStages) & 1;
            bar_wait(&xfull[s], ph);
            bar_wait(&afull[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // k-step k (32 B inside the 128-byte swizzle atom) -> accumulator k
                const uint64_t da = umma_desc_sw128(xb + uint32_t(s) * kTcXStage + uint32_t(k) * 32u);
                const uint64_t db = umma_desc_sw128(ab + uint32_t(s) * kTcAStage + uint32_t(k) * 32u);
                const uint32_t acc = kc > 0 ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + uint32_t(k) * 64u),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(&sempty[s]))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(done))
                     : "memory");
    } else if (warp < 2) {
        // ---- epilogue: TMEM lanes 0-63 = the tile's tokens
        bar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int t = warp * 32 + lane;
        const uint32_t lrow = uint32_t(warp * 32) << 16;
        for (int j0 = 0; j0 < npad; j0 += 16) {
            uint32_t d0[16], d1[16], d2[16], d3[16];
            tmem_ld16(tmem + lrow + 0 * 64 + uint32_t(j0), d0);
            tmem_ld16(tmem + lrow + 1 * 64 + uint32_t(j0), d1);
            tmem_ld16(tmem + lrow + 2 * 64 + uint32_t(j0), d2);
            tmem_ld16(tmem + lrow + 3 * 64 + uint32_t(j0), d3);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (t < u.nt)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j0 + j < r)
                        vout[u.vbase + int64_t(t) * r + j0 + j] =
                            (__uint_as_float(d0[j]) + __uint_as_float(d1[j])) +
                            (__uint_as_float(d2[j]) + __uint_as_float(d3[j]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

template <typename T>
cudaError_t launch_kernel(void (*k)(MgParams), const MgParams& p, int grid, size_t smem, cudaStream_t s, bool pdl,
                          int threads = kMgThreads) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    count_launch();
    return cudaLaunchKernelEx(&cfg, k, p);
}

}  // namespace

// SLORA_MBGMM_TC=1 selects the tcgen05 shrink.  Off by default: measured on
// C2-mixed (tools/layer_micro.py) it is bit-exact but slower than the
// mma.sync shrink at these shapes (<= 64-token tiles, N = r <= 64): 92-99 vs
// 84 us per layer launch.
static bool use_tc();
bool mbgmm_shrink_whole_rank() { return use_tc(); }
static bool use_tc() {
    static const bool on = [] {
        const char* e = getenv("SLORA_MBGMM_TC");
        return e && atoi(e) == 1;
    }();
    return on;
}

// (split, rows) of the mma.sync shrink for hidden size K: SLORA_MG_SPLIT (K parts) and
// SLORA_MG_SROWS (A rows per unit, <= 32) override the defaults
int mbgmm_split(int64_t K) {
    if (use_tc()) return kMgKsplit;
    static const int env = [] {
        const char* e = getenv("SLORA_MG_SPLIT");
        return e ? atoi(e) : 0;
    }();
    // default: K parts of 4096 columns at K >= 8192 (16-row units, x streamed four times per
    // rank-64 tile instead of eight: C4 60.6 -> 50.6 us per launch with 2048-column parts and
    // 32-row units at first; after the expand's v-part and y changes, 4096-column parts are
    // 2% faster: 43.7 -> 42.7), whole K below (K = 4096 on C2-mixed: split 2 / 4 measured
    // 6% / 26% slower, its long runs already fill the GPU)
    int sp = env > 0 ? env : (K >= 8192 ? int(K / 4096) : 1);
    while (sp > 1 && ((K / 64) % sp != 0 || sp > kMgVParts)) sp /= 2;
    return sp;
}
int mbgmm_rows(int64_t K) {
    static const int env = [] {
        const char* e = getenv("SLORA_MG_SROWS");
        return e ? atoi(e) : 0;
    }();
    const int64_t Kp = K / mbgmm_split(K);
    const int auto_rows = mg_rows_kp(Kp);
    if (env == 8 || env == 16 || env == 32)
        return mg_xstages_rows(Kp, env) >= 2 ? env : auto_rows;
    return auto_rows;
}

// Gathered MBGMM input: out row i = x row idx[i] (K elements, 16-byte vectors).
// Launched without PDL: it reads x, which the previous kernel may write.
// blockIdx.y splits a row into parts so that every SM has rows to move (a 256-row batch of 16 KB
// rows is otherwise 256 CTAs, each latency-bound on its own row)
__global__ void gather_rows_kernel(const uint4* __restrict__ x, int64_t ldx16, const int32_t* __restrict__ idx, int n,
                                   uint4* __restrict__ out, int64_t k16) {
    const int64_t part = (k16 + gridDim.y - 1) / gridDim.y;
    const int64_t c0 = int64_t(blockIdx.y) * part, c1 = c0 + part < k16 ? c0 + part : k16;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const uint4* src = x + int64_t(__ldg(idx + i)) * ldx16;
        uint4* dst = out + int64_t(i) * k16;
        for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) dst[c] = __ldcs(src + c);
    }
}
cudaError_t launch_gather_rows(const void* x, int64_t ldx, const int32_t* idx, int n, void* out, int64_t K, int es,
                               cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    count_launch();
    const int64_t k16 = K * es / 16;
    const int parts = int(std::max<int64_t>(1, std::min<int64_t>((148 * 8 + n - 1) / n, k16 / 256)));
    gather_rows_kernel<<<dim3(unsigned(std::min(n, 148 * 8)), unsigned(parts)), 256, 0, s>>>(
        static_cast<const uint4*>(x), ldx * es / 16, idx, n, static_cast<uint4*>(out), k16);
    return cudaGetLastError();
}

size_t mbgmm_smem(bool expand, int64_t K, int rmax) {
    return expand ? mg_expand_smem_unit(rmax, mbgmm_expand_cols(rmax))
                  : (use_tc() ? mg_shrink_tc_smem(K) : mg_shrink_smem_kp(K / mbgmm_split(K), mbgmm_rows(K)));
}

cudaError_t configure_mbgmm_kernels() {
    const int lim = 227 * 1024;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(mbgmm_shrink_kernel<__half, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim))) return e;
    if ((e = cudaFuncSetAttribute(mbgmm_shrink_kernel<__nv_bfloat16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim)))
        return e;
    if ((e = cudaFuncSetAttribute(mbgmm_shrink_kernel<__half, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim))) return e;
    if ((e = cudaFuncSetAttribute(mbgmm_shrink_kernel<__nv_bfloat16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim)))
        return e;
    if ((e = cudaFuncSetAttribute(mbgmm_shrink_tc_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim)))
        return e;
    if ((e = cudaFuncSetAttribute(mbgmm_shrink_tc_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lim)))
        return e;
    if ((e = cudaFuncSetAttribute(mbgmm_expand_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim))) return e;
    if ((e = cudaFuncSetAttribute(mbgmm_expand_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim)))
        return e;
    // two expand CTAs per SM: all of the unified L1/shared capacity as shared memory
    if ((e = cudaFuncSetAttribute(mbgmm_expand_kernel<__half>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)))
        return e;
    return cudaFuncSetAttribute(mbgmm_expand_kernel<__nv_bfloat16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

cudaError_t launch_mbgmm(const MgParams& p, bool expand, int dtype, int n_units, size_t smem, cudaStream_t s,
                         bool pdl) {
    if (n_units == 0) return cudaSuccess;
    if (!expand && use_tc())
        return dtype == kF16 ? launch_kernel<__half>(mbgmm_shrink_tc_kernel<__half>, p, n_units, smem, s, pdl, kTcThreads)
                             : launch_kernel<__nv_bfloat16>(mbgmm_shrink_tc_kernel<__nv_bfloat16>, p, n_units, smem, s,
                                                            pdl, kTcThreads);
    if (expand)
        return dtype == kF16 ? launch_kernel<__half>(mbgmm_expand_kernel<__half>, p, n_units, smem, s, pdl)
                             : launch_kernel<__nv_bfloat16>(mbgmm_expand_kernel<__nv_bfloat16>, p, n_units, smem, s, pdl);
    if (p.srows > 16)
        return dtype == kF16 ? launch_kernel<__half>(mbgmm_shrink_kernel<__half, 2>, p, n_units, smem, s, pdl)
                             : launch_kernel<__nv_bfloat16>(mbgmm_shrink_kernel<__nv_bfloat16, 2>, p, n_units, smem, s, pdl);
    return dtype == kF16 ? launch_kernel<__half>(mbgmm_shrink_kernel<__half, 1>, p, n_units, smem, s, pdl)
                         : launch_kernel<__nv_bfloat16>(mbgmm_shrink_kernel<__nv_bfloat16, 1>, p, n_units, smem, s, pdl);
}

}  // namespace slora
