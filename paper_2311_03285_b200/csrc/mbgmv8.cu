// mbgmv8.cu -- MBGMV gather-shrink-expand, warp-task form (sm_100a).
//
// PAPER.md Sec. 5.3, Eq. lora_factored: for every token
// i of adapter a, v_i = x_i A_a (shrink) and y_i += scale_a v_i B_a (expand),
// with the rows of A (stored transposed, reading R1) and B living in pool
// pages reached through the adapter's page table.
//
// Why this form.  The ring-pipelined kernel (kernels.cu, mbgmv_kernel) moves
// data with TMA into a shared ring and hands every piece through resolver /
// streamer / publisher warps; measured on C2 decode, its control chain alone
// (no data, no math: SLORA_DBG=7) costs 12 us per launch -- as much as the
// whole launch's HBM time.  Here there are no helper warps and no ring:
//
//   * one persistent CTA per SM, kW8 warps; every warp takes the next task of
//     its CTA's list (host LPT schedule, api.cpp) from a shared-memory ticket;
//   * every warp streams its tasks as a sequence of 8 KB chunks through its
//     own two-chunk shared-memory buffer with cp.async (LDGSTS, 16 B per lane,
//     L1 bypassed): chunk n+1 -- of this task or the next one -- is in flight
//     while chunk n is consumed, and each lane only ever reads back the 16 B
//     vectors it copied itself, so no barrier is involved at all (kW8 x 16 KB
//     in flight per SM without spending registers on it);
//   * a shrink task is ONE stored A row (K elements over `arp` pages, 8 KB
//     per chunk): dot products with the item's x rows (L1-resident: all warps
//     of the item read the same rows) by mixed-precision FMAs, a butterfly
//     reduction (fixed order), then lane 0 writes v and releases the item's
//     counter (red.release.gpu);
//   * an expand task is all r B rows of one item over a column chunk, in
//     passes of 32 lanes x 16 B columns and chunks of kRBX rows: the weights
//     stream before the item's counter is even checked (they do not depend on
//     v), v is staged in a per-warp shared buffer, each lane owns one 16-byte
//     column vector for every token (fp32 accumulators), and y is read once
//     and written once (one rounding).  The item's last expand task resets
//     the counter.
//
// Deadlock freedom: every CTA list holds all its shrink tasks before any
// expand task and tickets are taken in list order, so a warp blocked on an
// expand task only waits for shrink tasks that are already taken (shrink tasks
// never wait); all CTAs are co-resident (grid = #SMs, one CTA each).
// Determinism: every v entry is one warp's fixed-order sum, every y column one
// lane's fixed-order sum: results are bit-identical under page placement,
// batch permutation and schedule.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "slora_internal.h"

namespace slora {
namespace v8 {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_relaxed_u32(const float* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(float* p, float v) {
    asm volatile("st.relaxed.gpu.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

template <typename T> struct Cvt;
template <> struct Cvt<float> {
    static constexpr int VE = 4;
    __device__ static void to_f32(const uint4& u, float* f) {
        f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
        f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
    }
    __device__ static uint4 from_f32(const float* f) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
    }
    // acc0/acc1 += <a, x> over one 16-byte vector
    __device__ static void dot(const uint4& a, const uint4& x, float& acc0, float& acc1) {
        acc0 = fmaf(__uint_as_float(a.x), __uint_as_float(x.x), acc0);
        acc1 = fmaf(__uint_as_float(a.y), __uint_as_float(x.y), acc1);
        acc0 = fmaf(__uint_as_float(a.z), __uint_as_float(x.z), acc0);
        acc1 = fmaf(__uint_as_float(a.w), __uint_as_float(x.w), acc1);
    }
};
// f16/bf16: the product of two 16-bit floats is exact in fp32, so the mixed
// FMA (one SASS FHFMA) equals convert + fmaf
__device__ __forceinline__ float fma_mixed(uint32_t a, uint32_t b, float c, __half*) {
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"((unsigned short)a), "h"((unsigned short)b));
    return c;
}
__device__ __forceinline__ float fma_mixed(uint32_t a, uint32_t b, float c, __nv_bfloat16*) {
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(c) : "h"((unsigned short)a), "h"((unsigned short)b));
    return c;
}
template <typename H> struct Cvt16 {
    static constexpr int VE = 8;
    __device__ static void dot(const uint4& a, const uint4& x, float& acc0, float& acc1) {
        const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc0 = fma_mixed(aw[i] & 0xffffu, xw[i] & 0xffffu, acc0, (H*)nullptr);
            acc1 = fma_mixed(aw[i] >> 16, xw[i] >> 16, acc1, (H*)nullptr);
        }
    }
};
template <> struct Cvt<__half> : Cvt16<__half> {
    __device__ static void to_f32(const uint4& u, float* f) {
        const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 t = __half22float2(h[i]);
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
template <> struct Cvt<__nv_bfloat16> : Cvt16<__nv_bfloat16> {
    __device__ static void to_f32(const uint4& u, float* f) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 t = __bfloat1622float2(h[i]);
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

// A resolved task (warp-uniform fields; `tok`, `pg0`, `pg1` lane-distributed).
struct Task {
    int kind;          // kPieceS, kPieceE, kPieceStop
    int item, nt, r, ra, proj, pi, arp, n_sp, n_ep, a, b;
    int nchunks;       // 8 KB chunks of the task
    float scale;
    int64_t vbase, vrow;
    int tok;           // lane t < nt: token (x / y row) t of the item
    int pg0, pg1;      // shrink: lane c < arp: page of chunk c of the row; expand: pages of B rows lane, lane + 32
};

#ifndef SLORA_W8_CHUNK
#define SLORA_W8_CHUNK 8192
#endif
constexpr int kChunkVec = SLORA_W8_CHUNK / 16;  // 16-byte vectors per chunk (8 KB: 16 per lane)
constexpr int kRBX = SLORA_W8_CHUNK / 512;      // B rows per expand chunk (rows x 32 lanes x 16 B)
#ifndef SLORA_W8_XSLOT
#define SLORA_W8_XSLOT 0  // 1: token 0's x slice rides in the chunk slot (measured: no gain on C2)
#endif
// shrink chunk: kSV vectors of the A row (+ with XSLOT the same kSV vectors of x, token 0)
constexpr int kSV = SLORA_W8_XSLOT ? kChunkVec / 2 : kChunkVec;
constexpr uint32_t kVEmpty = 0xFFFFFFFFu;  // fused workspace: entry not yet written (see stage_v)

__device__ __forceinline__ DevTask8 load_desc(const LoraParams& p, int idx, int end) {
    if (idx >= end) {
        DevTask8 d{};
        d.kind = kPieceStop;
        return d;
    }
    return p.tasks[idx];
}

// Resolve a task descriptor: its token rows and page ids (one dependent hop
// through the adapter's page table, issued two tasks before they are used).
template <int MODE>
__device__ __forceinline__ Task resolve(const LoraParams& p, const DevTask8& d, int lane, int KV, int PV) {
    Task t;
    t.kind = d.kind;
    t.nchunks = 0;
    if (d.kind == kPieceStop) return t;
    t.item = d.item;
    t.a = d.a;
    t.b = d.b;
    t.nt = d.nt;
    t.r = d.rank;
    t.pi = d.pi;
    t.proj = p.proj_ids[d.pi];
    const int div = (MODE == kExpand) ? 1 : p.a_div[t.proj];
    t.arp = (MODE == kExpand) ? 1 : p.a_row_pages[t.proj];
    t.ra = d.rank / div;
    t.n_sp = d.n_sp;
    t.n_ep = d.n_ep;
    t.scale = d.scale;
    t.vrow = d.vrow;
    t.vbase = int64_t(d.pi) * (p.NR / div) + d.vrow / div;
    const int32_t* tab = d.tab + int64_t((p.layer * 4 + t.proj) * 2) * d.rank;
    t.tok = lane < d.nt ? p.tok_idx[d.tok_off + lane] : 0;
    if (t.kind == kPieceS) {
        t.pg0 = lane < t.arp ? tab[d.a * t.arp + lane] : 0;
        t.pg1 = 0;
        t.nchunks = (KV + kSV - 1) / kSV;
    } else {
        t.pg0 = lane < d.rank ? tab[d.rank + lane] : 0;
        t.pg1 = lane + 32 < d.rank ? tab[d.rank + lane + 32] : 0;
        t.nchunks = ((d.b + PV - 1) / PV) * ((d.rank + kRBX - 1) / kRBX);  // passes x row batches
    }
    return t;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy global -> shared (LDGSTS, L1 bypassed); n = 0 zero-fills
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Issue chunk `ci` of task c into the warp buffer at `dst` (this lane's 16 of
// the chunk's 512 vectors).  Shrink: vectors [512 ci, 512 ci + 512) of the
// stored A row.  Expand: pass ci / nb (32 x VE columns), rows kRBX (ci % nb)..
// The fields of a task that issuing its chunks needs (passed by value: the
// tasks stay in registers).
struct IssueRef {
    int kind, arp, r, a, b, pg0, pg1, nt, tok;
};
__device__ __forceinline__ IssueRef iref(const Task& t) {
    return {t.kind, t.arp, t.r, t.a, t.b, t.pg0, t.pg1, t.nt, t.tok};
}

template <typename T>
__device__ __noinline__ void issue_chunk(const LoraParams& p, IssueRef c, int ci, uint32_t dst, int lane, int KV,
                                         int PV, bool with_x) {
    constexpr int VE = Cvt<T>::VE;
    const T* pool = reinterpret_cast<const T*>(p.pool);
    const int64_t P = p.page_elems;
    if (c.kind == kPieceS) {
        const int base = ci * kSV;
        if (c.arp == 1) {
            const T* row = pool + int64_t(__shfl_sync(0xffffffffu, c.pg0, 0)) * P;
#pragma unroll
            for (int k = 0; k < kSV / 32; ++k) {
                const int vi = base + lane + 32 * k;
                cp16(dst + uint32_t(lane + 32 * k) * 16u, row + int64_t(min(vi, KV - 1)) * VE, vi < KV);
            }
        } else {  // TP q/k/v: a stored row spans arp pages of P elements
#pragma unroll
            for (int k = 0; k < kSV / 32; ++k) {
                const int vi = base + lane + 32 * k;
                const int64_t e = int64_t(min(vi, KV - 1)) * VE;
                const int ch = int(e / P);
                const int pg = __shfl_sync(0xffffffffu, c.pg0, ch);
                cp16(dst + uint32_t(lane + 32 * k) * 16u, pool + int64_t(pg) * P + (e - int64_t(ch) * P), vi < KV);
            }
        }
        if (SLORA_W8_XSLOT && with_x) {  // token 0's x slice rides along (only after the PDL wait: x is the previous launch's output)
            const T* xr = reinterpret_cast<const T*>(p.x) + int64_t(__shfl_sync(0xffffffffu, c.tok, 0)) * p.ldx;
#pragma unroll
            for (int k = 0; k < kSV / 32; ++k) {
                const int vi = base + lane + 32 * k;
                cp16(dst + uint32_t(kSV + lane + 32 * k) * 16u, xr + int64_t(min(vi, KV - 1)) * VE, vi < KV);
            }
        }
    } else {
        const int nb = (c.r + kRBX - 1) / kRBX;
        const int pass = ci / nb, j0 = (ci - pass * nb) * kRBX;
        const int64_t col = int64_t(c.a) + int64_t(pass) * PV + int64_t(lane) * VE;
        const bool active = col < int64_t(c.a) + c.b;
#pragma unroll
        for (int q = 0; q < kRBX; ++q) {
            const int j = j0 + q;
            const int pg = __shfl_sync(0xffffffffu, j < 32 ? c.pg0 : c.pg1, j & 31);
            cp16(dst + uint32_t(q * 32 + lane) * 16u, pool + int64_t(pg) * P + (active ? col : 0),
                 active && j < c.r);
        }
    }
}

// Dot products of one chunk for the item's tokens (token loop unrolled to
// the cap with a guard, one code path for every token count: the kernel
// stays small enough for the instruction cache).
template <typename T>
__device__ __forceinline__ void shrink_chunk(const LoraParams& p, const Task& c, int ci, const uint4* buf, int lane,
                                             int KV, bool x_in_slot, float (&acc)[kItemTokCap][2]) {
    const T* x = reinterpret_cast<const T*>(p.x);
    const int base = ci * kSV;
#pragma unroll
    for (int t = 0; t < kItemTokCap; ++t) {
        const int tok = __shfl_sync(0xffffffffu, c.tok, t);
        if (t < c.nt) {
            // vectors past the row end hold zero-filled A (cp.async src-size
            // 0), so they add exact zeros against a clamped x vector
            uint4 xv[kSV / 32];
            if (SLORA_W8_XSLOT && t == 0 && x_in_slot) {
#pragma unroll
                for (int k = 0; k < kSV / 32; ++k) xv[k] = buf[kSV + lane + 32 * k];
            } else {
                const uint4* xr = reinterpret_cast<const uint4*>(x + int64_t(tok) * p.ldx);
#pragma unroll
                for (int k = 0; k < kSV / 32; ++k) xv[k] = __ldg(xr + min(base + lane + 32 * k, KV - 1));
            }
#pragma unroll
            for (int k = 0; k < kSV / 32; ++k) Cvt<T>::dot(buf[lane + 32 * k], xv[k], acc[t][0], acc[t][1]);
        }
    }
}

template <int MODE>
__device__ __forceinline__ void shrink_finish(const LoraParams& p, const Task& c, int lane,
                                              float (&acc)[kItemTokCap][2]) {
    float s[kItemTokCap];
#pragma unroll
    for (int t = 0; t < kItemTokCap; ++t) s[t] = acc[t][0] + acc[t][1];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int t = 0; t < kItemTokCap; ++t) s[t] += __shfl_xor_sync(0xffffffffu, s[t], o);
    if (lane == 0) {
#pragma unroll
        for (int t = 0; t < kItemTokCap; ++t)
            if (t < c.nt) st_relaxed(p.v + c.vbase + int64_t(t) * c.ra + c.a, s[t]);
    }
}

// v of the item into the warp's stage.  Fused: the workspace entries are the
// readiness flags themselves -- every entry holds kVEmpty (an fp32 NaN bit
// pattern no arithmetic result or 16-bit input can produce) until its shrink
// warp stores the dot product, so an expand task polls exactly the entries it
// needs and no release fence / counter sits on the shrink path.  The item's
// last expand task (relaxed counter) puts the entries back to kVEmpty for the
// workspace slot's next launch.
template <int MODE>
__device__ __forceinline__ void stage_v(const LoraParams& p, const Task& c, float* vs, int lane) {
    const int r = c.r;
    if (MODE == kFused) {
        const int n = c.nt * r;
        float* v = p.v + c.vbase;
        for (int e = lane; e < n; e += 32) {
            uint32_t u = ld_relaxed_u32(v + e);
            for (int spin = 0; u == kVEmpty && spin < (1 << 24); ++spin) {  // bounded: never hang the GPU
                __nanosleep(32);
                u = ld_relaxed_u32(v + e);
            }
            vs[e] = __uint_as_float(u);
        }
        __syncwarp();
        int last = 0;
        if (lane == 0) last = atomicAdd(&p.sync[c.item], 1) == c.n_ep - 1;
        if (__shfl_sync(0xffffffffu, last, 0)) {
            for (int e = lane; e < n; e += 32) st_relaxed(v + e, __uint_as_float(kVEmpty));
            if (lane == 0) atomicExch(&p.sync[c.item], 0);
        }
    } else {  // v from v_in: block layout of slora_lora_expand
        const int vbk = p.v_blocks, rb = r / vbk;
        const int64_t stride = int64_t(p.nproj) * (p.NR / vbk);
        const int64_t base = int64_t(c.pi) * (p.NR / vbk) + c.vrow / vbk;
        for (int e = lane; e < c.nt * r; e += 32) {
            const int t = e / r, j = e % r;
            vs[e] = p.v_in[int64_t(j / rb) * stride + base + int64_t(t) * rb + j % rb];
        }
    }
    __syncwarp();
}

// One expand chunk: rows j0 .. j0 + kRBX of pass `pass`; the pass's y update
// after its last row batch.  Tokens beyond nt multiply v = 0 (never written).
template <typename T>
__device__ __forceinline__ void expand_chunk(const LoraParams& p, const Task& c, int ci, const uint4* buf,
                                             const float* vs, int lane, int PV,
                                             float (&acc)[kItemTokCap][Cvt<T>::VE]) {
    using C = Cvt<T>;
    constexpr int VE = C::VE;
    const int r = c.r, nt = c.nt;
    const int nb = (r + kRBX - 1) / kRBX;
    const int pass = ci / nb, bi = ci - pass * nb, j0 = bi * kRBX;
    if (bi == 0)
#pragma unroll
        for (int t = 0; t < kItemTokCap; ++t)
#pragma unroll
            for (int e = 0; e < VE; ++e) acc[t][e] = 0.f;
    const int nrow = min(kRBX, r - j0);
#pragma unroll 2
    for (int q = 0; q < nrow; ++q) {
        float b[VE];
        C::to_f32(buf[q * 32 + lane], b);
#pragma unroll
        for (int t = 0; t < kItemTokCap; ++t) {
            const float vj = t < nt ? vs[t * r + j0 + q] : 0.f;
#pragma unroll
            for (int e = 0; e < VE; ++e) acc[t][e] = fmaf(vj, b[e], acc[t][e]);
        }
    }
    if (bi == nb - 1) {
        const int64_t col = int64_t(c.a) + int64_t(pass) * PV + int64_t(lane) * VE;
        int tk[kItemTokCap];
#pragma unroll
        for (int t = 0; t < kItemTokCap; ++t) tk[t] = __shfl_sync(0xffffffffu, c.tok, t);
        if (col < int64_t(c.a) + c.b) {
            T* y = reinterpret_cast<T*>(p.y[c.proj]);
            const int64_t ldy = p.ldy[c.proj];
            uint4 yv[kItemTokCap];
#pragma unroll
            for (int t = 0; t < kItemTokCap; ++t)
                if (t < nt) yv[t] = *reinterpret_cast<const uint4*>(y + int64_t(tk[t]) * ldy + col);
#pragma unroll
            for (int t = 0; t < kItemTokCap; ++t)
                if (t < nt) {
                    float yf[VE];
                    C::to_f32(yv[t], yf);
#pragma unroll
                    for (int e = 0; e < VE; ++e) yf[e] = yf[e] + c.scale * acc[t][e];
                    *reinterpret_cast<uint4*>(y + int64_t(tk[t]) * ldy + col) = C::from_f32(yf);
                }
        }
    }
}

#ifndef SLORA_W8_SLOTS
#define SLORA_W8_SLOTS 3
#endif
constexpr int kNSlot = SLORA_W8_SLOTS;               // 8 KB chunk slots per warp (kNSlot - 1 in flight ahead)
constexpr int kWarpBufBytes = kNSlot * kChunkVec * 16;
constexpr int kVStageFloats = kItemTokCap * kMaxRank;

template <typename T, int MODE>
__global__ void __launch_bounds__(kW8 * 32, 1) mbgmv8_kernel(const __grid_constant__ LoraParams p) {
    extern __shared__ __align__(128) unsigned char smem8[];
    __shared__ int ticket;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbuf = smem8 + size_t(warp) * kWarpBufBytes;
    float* vs = reinterpret_cast<float*>(smem8 + size_t(kW8) * kWarpBufBytes) + warp * kVStageFloats;
    if (threadIdx.x == 0) ticket = 0;
    __syncthreads();
    pdl_trigger();  // the next launch may start its prologue
    const int pb = p.cta_off[blockIdx.x], pe = p.cta_off[blockIdx.x + 1];
    auto grab = [&]() {
        int t = 0;
        if (lane == 0) t = atomicAdd(&ticket, 1);
        return pb + __shfl_sync(0xffffffffu, t, 0);
    };
    constexpr int ES = sizeof(T);
    constexpr int PV = 32 * Cvt<T>::VE;  // columns per expand pass
    const int KV = int(int64_t(p.K) * ES / 16);  // 16-byte vectors per stored A row
    const uint32_t b0 = smem_addr(wbuf);
    // task pipeline: cur (being consumed), nxt and nx2 resolved (page ids in
    // flight), d3 = the descriptor after them (in flight).  Chunks are issued
    // kNSlot - 1 ahead of the one being consumed, across task boundaries.
    const DevTask8 d0 = load_desc(p, grab(), pe), d1 = load_desc(p, grab(), pe), d2 = load_desc(p, grab(), pe);
    DevTask8 d3 = load_desc(p, grab(), pe);
    Task cur = resolve<MODE>(p, d0, lane, KV, PV);
    if (cur.kind == kPieceStop) return;
    Task nxt = resolve<MODE>(p, d1, lane, KV, PV);
    Task nx2 = resolve<MODE>(p, d2, lane, KV, PV);
    int iss_t = 0, iss_c = 0;  // next chunk to issue: task (0 cur, 1 nxt, 2 nx2), chunk
    int seq_i = 0, seq_c = 0;  // chunks issued / consumed (slot = seq % kNSlot)
    auto issue_next = [&]() {
        if (iss_t <= 2) {
            // branches, not selects: a select would wait for nx2's page ids,
            // which are still in flight
            int kind, nch;
            if (iss_t == 0) { kind = cur.kind; nch = cur.nchunks; }
            else if (iss_t == 1) { kind = nxt.kind; nch = nxt.nchunks; }
            else { kind = nx2.kind; nch = nx2.nchunks; }
            if (kind != kPieceStop) {
                const uint32_t dst = b0 + uint32_t(seq_i % kNSlot) * uint32_t(kChunkVec * 16);
                const bool wx = seq_i >= kNSlot - 1;  // chunks issued before the PDL wait carry no x
                if (iss_t == 0) issue_chunk<T>(p, iref(cur), iss_c, dst, lane, KV, PV, wx);
                else if (iss_t == 1) issue_chunk<T>(p, iref(nxt), iss_c, dst, lane, KV, PV, wx);
                else issue_chunk<T>(p, iref(nx2), iss_c, dst, lane, KV, PV, wx);
                ++seq_i;
                if (++iss_c == nch) {
                    ++iss_t;
                    iss_c = 0;
                }
            }
        }
        cp_commit();  // (possibly empty) group: keeps the wait_group count uniform
    };
    for (int k = 0; k < kNSlot - 1; ++k) issue_next();  // weights: before the PDL wait
    pdl_wait();  // x, y (and the workspace state) of the previous launch
    float sacc[kItemTokCap][2];
    float eacc[kItemTokCap][Cvt<T>::VE];
    int ci = 0;
    bool staged = false;
    // debug trace (SLORA_TRACE=1): per traced CTA and warp, up to 10 tasks x
    // (start, first chunk landed, computed, finished, next resolved, code)
    long long* tr = (p.trace && blockIdx.x < 16 && warp < 16) ? p.trace + blockIdx.x * kTraceSlots + warp * 64 : nullptr;
    int ntask = 0;
    auto gt = []() {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    };
    if (tr && lane == 0) tr[0] = tr[1] = gt();
    for (;;) {
        const bool last = ci + 1 == cur.nchunks;
        issue_next();
        asm volatile("cp.async.wait_group %0;" ::"n"(kNSlot - 1) : "memory");  // chunk seq_c landed (this lane's part)
        const uint4* cb = reinterpret_cast<const uint4*>(wbuf + size_t(seq_c % kNSlot) * (kChunkVec * 16));
        const bool x_in_slot = seq_c >= kNSlot - 1;
        ++seq_c;
        if (tr && lane == 0 && ci == 0 && ntask < 10) tr[1 + 6 * ntask + 1] = gt();  // first chunk landed
        if (cur.kind == kPieceS) {
            if (ci == 0)
#pragma unroll
                for (int t = 0; t < kItemTokCap; ++t) sacc[t][0] = sacc[t][1] = 0.f;
            shrink_chunk<T>(p, cur, ci, cb, lane, KV, x_in_slot, sacc);
            if (tr && lane == 0 && last && ntask < 10) tr[1 + 6 * ntask + 2] = gt();  // computed
            if (last) shrink_finish<MODE>(p, cur, lane, sacc);
        } else {
            if (!staged) {
                stage_v<MODE>(p, cur, vs, lane);
                staged = true;
            }
            expand_chunk<T>(p, cur, ci, cb, vs, lane, PV, eacc);
        }
        if (!last) {
            ++ci;
            continue;
        }
        if (tr && lane == 0 && ntask < 10) {
            tr[1 + 6 * ntask + 3] = gt();  // finished
            tr[1 + 6 * ntask + 5] = cur.kind * 1000000 + cur.nt * 100000 + cur.r;
        }
        __syncwarp();  // the v stage is rewritten by the next expand task
        if (nxt.kind == kPieceStop) break;
        cur = nxt;
        nxt = nx2;
        nx2 = resolve<MODE>(p, d3, lane, KV, PV);
        d3 = load_desc(p, grab(), pe);
        --iss_t;
        ci = 0;
        staged = false;
        if (tr && lane == 0 && ntask < 10) tr[1 + 6 * ntask + 4] = gt();  // next resolved
        ++ntask;
        if (tr && lane == 0 && ntask < 10) tr[1 + 6 * ntask] = gt();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

static bool pdl_on() {
    static const bool on = [] {
        const char* s = getenv("SLORA_PDL");
        return !(s && atoi(s) == 0);
    }();
    return on;
}

template <typename T, int MODE>
static cudaError_t launch_t(const LoraParams& p, int grid, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kW8 * 32);
    cfg.dynamicSmemBytes = lora8_smem_bytes();
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (pdl_on()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    count_launch();
    return cudaLaunchKernelEx(&cfg, mbgmv8_kernel<T, MODE>, p);
}

template <typename T, int MODE>
static cudaError_t configure_t() {
    return cudaFuncSetAttribute(mbgmv8_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(lora8_smem_bytes()));
}

}  // namespace v8

size_t lora8_smem_bytes() { return size_t(kW8) * (v8::kWarpBufBytes + v8::kVStageFloats * 4); }

cudaError_t configure_lora8_kernels() {
    using namespace v8;
    cudaError_t e;
    if ((e = configure_t<float, kFused>())) return e;
    if ((e = configure_t<float, kShrink>())) return e;
    if ((e = configure_t<float, kExpand>())) return e;
    if ((e = configure_t<__half, kFused>())) return e;
    if ((e = configure_t<__half, kShrink>())) return e;
    if ((e = configure_t<__half, kExpand>())) return e;
    if ((e = configure_t<__nv_bfloat16, kFused>())) return e;
    if ((e = configure_t<__nv_bfloat16, kShrink>())) return e;
    return configure_t<__nv_bfloat16, kExpand>();
}

cudaError_t launch_lora8(const LoraParams& p, int mode, int dtype, int grid, cudaStream_t s) {
    using namespace v8;
    switch (dtype * 3 + mode) {
        case 0: return launch_t<float, kFused>(p, grid, s);
        case 1: return launch_t<float, kShrink>(p, grid, s);
        case 2: return launch_t<float, kExpand>(p, grid, s);
        case 3: return launch_t<__half, kFused>(p, grid, s);
        case 4: return launch_t<__half, kShrink>(p, grid, s);
        case 5: return launch_t<__half, kExpand>(p, grid, s);
        case 6: return launch_t<__nv_bfloat16, kFused>(p, grid, s);
        case 7: return launch_t<__nv_bfloat16, kShrink>(p, grid, s);
        default: return launch_t<__nv_bfloat16, kExpand>(p, grid, s);
    }
}

}  // namespace slora
