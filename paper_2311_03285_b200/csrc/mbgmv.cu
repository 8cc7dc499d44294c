// mbgmv.cu -- the fused single-GPU MBGMV of the S-LoRA hot path on sm_100a:
// heterogeneous batched LoRA, y_i += scale_a * (x_i A_a) B_a, over adapter
// rows gathered from Unified Paging pages (Sec. 5.3, P:279-289;
// Eq. lora_factored; reading R1: page j of A holds column j of A).
//
// Decomposition.  The host (api.cpp plan_group_call) cuts the batch into
// items = (adapter segment, projection, chunk of <= 8 tokens) and assigns
// them (LPT on streamed bytes) to G groups of C consecutive CTAs of one
// persistent grid.  All C CTAs of a group walk the same item list; CTA c
//   shrink:   reads the K-slice c (Kc = K/C elements) of each of the item's r
//             stored A rows and computes partial dot products with the same
//             slice of the tokens' x rows (mma.sync m16n8k16: M = tokens,
//             N = 8 A rows, K = 16, fp32 accumulate);
//   exchange: writes its partial (nt x r fp32) to a small L2 workspace and
//             releases the item's arrival counter; the exchange warp of every
//             CTA of the group waits for the C arrivals and sums the C
//             partials in a fixed order -> v (complete, fp32) in shared memory;
//   expand:   reads the output-column slice c (Dc = D/C) of the item's r B
//             rows and writes y[tok][slice] = y + scale * sum_j v_j B_j
//             (mma.sync m16n8k8: M = 16 output columns (B^T through
//             ldmatrix.trans), N = tokens, K = 8 rank rows; v enters as a
//             16-bit hi + lo pair, so the products keep ~fp32 accuracy; fp32
//             accumulate, one rounding into y).
// fp32 inputs never use tensor cores (no TF32, reading R5): the fp32 shrink
// and expand are CUDA-core FFMA loops.
//
// Warp roles: 8 consumer warps (shrink, expand), a producer warp streaming A
// and B row slices with cp.async.bulk (TMA engine, SASS UBLKCP) into a ring
// of 8-row slots in the consumers' order, and an exchange warp.  The
// consumers software-pipeline the items kGDepth deep (shrink i+2 before the
// expand of i), so the exchange of item i overlaps two shrinks.  The weights
// are never written by the previous kernel, so the producer streams them
// before griddepcontrol.wait (programmatic dependent launch); x, y, the
// workspace and the counters are only touched after it.
//
// Determinism: every v entry is (each warp's mma chain over its k-range)
// summed over the 8 warps in order, then over the C slices in order; every y
// element is one fixed-order mma accumulation.  Results depend only on
// (K, C, r), never on page placement, batch order or the group assignment.
//
// Deadlock freedom: a CTA only waits for the CTAs of its own group, which
// process the same list in the same order; the grid never exceeds the number
// of co-resident CTAs (host), so every group is resident as a whole.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "ptx.cuh"
#include "slora_internal.h"

namespace slora {

using namespace ptx;

namespace {

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// diagnostics: event ev of this CTA (CTAs 0-15; events < 256: 0-63 phases, 64-159 consumer slot
// k ready, 160-255 producer slot k issued)
#define GTRACE(ev)                                                                                 \
    do {                                                                                           \
        if (p.trace && blockIdx.x < 16 && (ev) < 256) p.trace[blockIdx.x * 256 + (ev)] = gtimer(); \
    } while (0)
// diagnostics: per-CTA summary [CTA < 512][4]: 0 start, 1 consumers past griddepcontrol.wait,
// 2 first slot ready, 3 consumers done
#define GTRACE_ALL(ev)                                                                          \
    do {                                                                                        \
        if (p.trace && blockIdx.x < 512) p.trace[16 * 256 + blockIdx.x * 4 + (ev)] = gtimer(); \
    } while (0)

constexpr int kIdRing = 8;  // page-id ring entries (items)

struct GSmem {
    uint64_t* full;   // [kGMaxSlots] slot filled (producer expect_tx + TMA bytes)
    uint64_t* empty;  // [kGMaxSlots] slot released (one arrival per consumer warp)
    uint64_t* dbar;   // item descriptors staged
    uint64_t* vfull;  // [2] v of item i ready (exchange warp)
    uint64_t* vempty; // [2] v of item i consumed (consumer warps)
    uint64_t* idfull; // [kIdRing] page ids of item m landed (cp.async, 32 lanes)
    uint64_t* idempty;// [kIdRing] page ids of item m read by both producer warps
    GItem* desc;      // [kGMaxItems]
    int32_t* ids;     // [kIdRing][128] page ids of items m % kIdRing: A rows then B rows
    float* red;       // [2][8 warps][8 tokens][8 rows] per-slot shrink partials
    float* vbuf;      // [2][nt][r] v of items i % 2 (complete)
    unsigned char* ring;
};
__device__ __forceinline__ GSmem carve(unsigned char* s) {
    GSmem L;
    L.full = reinterpret_cast<uint64_t*>(s);
    L.empty = L.full + kGMaxSlots;
    L.dbar = L.empty + kGMaxSlots;
    L.vfull = L.dbar + 1;
    L.vempty = L.vfull + 2;
    L.idfull = L.vempty + 2;
    L.idempty = L.idfull + kIdRing;
    L.desc = reinterpret_cast<GItem*>(s + 512);
    L.ids = reinterpret_cast<int32_t*>(s + 512 + kGMaxItems * 64);
    L.red = reinterpret_cast<float*>(s + 512 + kGMaxItems * 64 + kIdRing * 128 * 4);
    L.vbuf = L.red + 2 * 8 * 64;
    L.ring = s + kGFixedSmem;
    return L;
}

struct RingPos {
    int slot = 0;
    uint32_t lap = 0;
    __device__ __forceinline__ void advance(int ns) {
        if (++slot == ns) {
            slot = 0;
            ++lap;
        }
    }
};

// ------------------------------------------------------------ producers
// Stream, per item m of the group, its A row slices (shrink) and B row slices
// (expand) in the consumers' order A0, A1, A2, B0, A3, B1, ..., B(n-1); each
// 8-row slot is one mbarrier transaction of up to 8 bulk copies issued by
// lanes 0-7.  kGProducers warps walk the same sequence and issue alternate
// slots (a warp's bulk copies are issued one lane at a time, ~60 ns each:
// one warp alone caps a CTA near 20-40 GB/s).  Producer 0 fetches the page
// ids five items ahead into an 8-entry ring with cp.async (completion tracked
// by idfull); both producers release an entry (idempty) after its B rows.
template <typename T>
__device__ __forceinline__ void producer(const GroupParams& p, const GSmem& S, int c, int n, int pw, int lane) {
    constexpr int ES = sizeof(T);
    const T* pool = reinterpret_cast<const T*>(p.pool);
    const int64_t P = p.P;
    auto fetch = [&](int m) {
        if (pw != 0 || m >= n) return;
        const int e = m % kIdRing;
        if (m >= kIdRing) mbar_wait(&S.idempty[e], ((m / kIdRing) - 1) & 1);
        const GItem& it = S.desc[m];
        const int r = it.rank;
        const int proj = p.proj_ids[it.pi];
        const int32_t* src = it.tab + int64_t((p.layer * 4 + proj) * 2) * r;  // A ids, then B ids
        int32_t* dst = S.ids + e * 128;
        for (int j = lane; j < 2 * r; j += 32) cp_async4(dst + j, src + j);
        cp_async_mbar_arrive(&S.idfull[e]);
    };
    RingPos rp;
    int k = 0;  // position in the slot stream
    const int ns = p.ns;
    const uint32_t SS = uint32_t(p.SS);
    const bool copy = !(p.dbg & 32);
    auto emit = [&](int m, int kind) {
        const int e = m % kIdRing;
        mbar_wait(&S.idfull[e], (m / kIdRing) & 1);
        const GItem& it = S.desc[m];
        const int r = it.rank;
        const int32_t* id = S.ids + e * 128 + (kind ? r : 0);
        const int eK = kind ? p.Dc : p.Kc;
        const uint32_t rb = uint32_t(eK) * ES;
        const uint32_t rs = rb + 16;
        const int64_t coff = int64_t(c) * eK;
        for (int j0 = 0; j0 < r; j0 += 8, ++k) {
            if (k % kGProducers == pw) {
                const int nr = min(8, r - j0);
                mbar_wait(&S.empty[rp.slot], (rp.lap & 1) ^ 1);
                const int pg = lane < nr ? id[j0 + lane] : 0;
                if (lane == 0) {
                    if (copy)
                        mbar_arrive_expect_tx(&S.full[rp.slot], uint32_t(nr) * rb);
                    else
                        mbar_arrive(&S.full[rp.slot]);
                }
                __syncwarp();
                if (lane < nr && copy)
                    bulk_g2s(S.ring + rp.slot * SS + uint32_t(lane) * rs, pool + int64_t(pg) * P + coff, rb,
                             &S.full[rp.slot]);
                if (lane == 0 && p.trace && k < 96) GTRACE(160 + k);
            }
            rp.advance(ns);
        }
        if (kind) {  // the item's ids are no longer needed by this warp
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.idempty[e]);
        }
    };
    for (int m = 0; m < 5; ++m) fetch(m);
    if (lane == 0 && pw == 0) GTRACE(2);
    emit(0, 0);
    if (lane == 0 && pw == 0) GTRACE(3);
    if (n > 1) emit(1, 0);
    for (int i = 0; i < n; ++i) {
        if (i + 2 < n) emit(i + 2, 0);
        emit(i, 1);
        fetch(i + 5);  // entry (i+5) % 8 == (i-3) % 8: released by both producers after emit(i-3, B)
    }
    if (lane == 0 && pw == 0) GTRACE(4);
}

// ------------------------------------------------------------ exchange warp
// v of item i = sum over the group's C partials in slice order, into vbuf[i%2]
// once all C CTAs have released item i; the group's last reader of item i
// resets its two counters (self-resetting: no memset between launches).
__device__ __forceinline__ void exchange(const GroupParams& p, const GSmem& S, int i0, int n, int lane) {
    for (int i = 0; i < n; ++i) {
        if (i >= 2) mbar_wait(&S.vempty[i & 1], ((i >> 1) - 1) & 1);
        const GItem& it = S.desc[i];
        const int tot = it.nt * it.rank;
        int* cnt = p.cnt + 2 * (i0 + i);
        float* vb = S.vbuf + (i & 1) * (kGMaxTok * 64);
        if (!(p.dbg & 1)) {
            if (lane == 0)
                while (ld_acquire(cnt) < p.C) __nanosleep(20);
            __syncwarp();
            const float* ws = p.ws + it.ws;
            if ((tot & 3) == 0) {
                for (int e4 = lane; e4 < (tot >> 2); e4 += 32) {
                    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
                    for (int q = 0; q < p.C; ++q) {
                        const float4 v = ld_cg4(ws + int64_t(q) * tot + 4 * e4);
                        s.x += v.x;
                        s.y += v.y;
                        s.z += v.z;
                        s.w += v.w;
                    }
                    reinterpret_cast<float4*>(vb)[e4] = s;
                }
            } else {
                for (int e = lane; e < tot; e += 32) {
                    float s = 0.f;
                    for (int q = 0; q < p.C; ++q) s += ld_cg(ws + int64_t(q) * tot + e);
                    vb[e] = s;
                }
            }
            __syncwarp();
            if (lane == 0 && atomicAdd(cnt + 1, 1) == p.C - 1) {
                cnt[0] = 0;
                cnt[1] = 0;
            }
        }
        if (lane == 0) mbar_arrive(&S.vfull[i & 1]);
    }
}

// ------------------------------------------------------------ consumers
template <typename T> struct Mma8;  // D[16x8] += A[16x8] B[8x8], fp32 accumulate
template <> struct Mma8<__half> {
    __device__ static void run(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
                     "{%0, %1, %2, %3};"
                     : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                     : "r"(a0), "r"(a1), "r"(b0));
    }
    __device__ static uint32_t pack(float lo, float hi) {
        __half2 h = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static float2 unpack(uint32_t u) { return __half22float2(*reinterpret_cast<__half2*>(&u)); }
};
template <> struct Mma8<__nv_bfloat16> {
    __device__ static void run(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
                     "{%0, %1, %2, %3};"
                     : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                     : "r"(a0), "r"(a1), "r"(b0));
    }
    __device__ static uint32_t pack(float lo, float hi) {
        __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static float2 unpack(uint32_t u) { return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u)); }
};
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T, int KSMAX>
struct Consumer {
    static constexpr int ES = sizeof(T);
    static constexpr bool kF32 = sizeof(T) == 4;
    using V = Vec16<T>;
    static constexpr int VE = V::VE;

    const GroupParams& p;
    const GSmem& S;
    const int c, i0, n, tid, warp, lane;
    RingPos rp;

    __device__ Consumer(const GroupParams& p_, const GSmem& S_, int c_, int i0_, int n_)
        : p(p_), S(S_), c(c_), i0(i0_), n(n_), tid(threadIdx.x), warp(threadIdx.x >> 5), lane(threadIdx.x & 31) {}

    __device__ __forceinline__ const T* xrow(const GItem& it, int t) const {
        return reinterpret_cast<const T*>(p.x) + int64_t(it.tok[t]) * p.ldx + int64_t(c) * p.Kc;
    }
    __device__ __forceinline__ T* yrow(const GItem& it, int t) const {
        const int proj = p.proj_ids[it.pi];
        return reinterpret_cast<T*>(p.y[proj]) + int64_t(it.tok[t]) * p.ldy[proj] + int64_t(c) * p.Dc;
    }
    __device__ __forceinline__ void wait_slot() {
        mbar_wait(&S.full[rp.slot], rp.lap & 1);
        if (tid == 0 && p.trace) {
            const int k = int(rp.lap) * p.ns + rp.slot;
            if (k < 96) GTRACE(64 + k);
        }
    }
    __device__ __forceinline__ void release_slot() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[rp.slot]);
        rp.advance(p.ns);
    }

    // x fragments of item m for this warp's k-range [warp*KW, (warp+1)*KW): token g = lane/4
    __device__ __forceinline__ void load_x(int m, uint32_t (&xa)[KSMAX][2]) const {
        if constexpr (!kF32) {
            const int KW = p.Kc >> 3, KS = KW >> 4;
            const int g = lane >> 2, t4 = lane & 3;
            const T* xr = nullptr;
            if (m < n) {
                const GItem& it = S.desc[m];
                if (g < it.nt && !(p.dbg & 2)) xr = xrow(it, g) + warp * KW + 2 * t4;
            }
#pragma unroll
            for (int ks = 0; ks < KSMAX; ++ks) {
                xa[ks][0] = (ks < KS && xr) ? ld_u32(xr + 16 * ks) : 0u;
                xa[ks][1] = (ks < KS && xr) ? ld_u32(xr + 16 * ks + 8) : 0u;
            }
        }
    }
    // y of item m for the expand epilogue: thread (g, t4) owns token 2*t4 + (g & 1) and the column
    // pairs warp*CW + 16j + (g & ~1) + {0, 8} (+0, +1) of each m-block j (4-byte accesses)
    __device__ __forceinline__ T* ypair(const GItem& it) const {
        const int g = lane >> 2, t4 = lane & 3;
        const int tok = 2 * t4 + (g & 1);
        return tok < it.nt ? yrow(it, tok) + warp * (p.Dc >> 3) + (g & ~1) : nullptr;
    }
    __device__ __forceinline__ void load_y(int m, uint32_t (&yv)[KSMAX][2]) const {
        if constexpr (!kF32) {
            const GItem& it = S.desc[m];
            const int MB = p.Dc >> 7;
            const T* yp = (p.dbg & 4) ? nullptr : ypair(it);
#pragma unroll
            for (int j = 0; j < KSMAX; ++j) {
                yv[j][0] = (j < MB && yp) ? ld_u32(yp + 16 * j) : 0u;
                yv[j][1] = (j < MB && yp) ? ld_u32(yp + 16 * j + 8) : 0u;
            }
        }
    }

    // -- shrink of item m: this CTA's partial v over its K-slice -> workspace, then release.
    // xa holds item m's x fragments on entry and item m+1's on return.
    __device__ __forceinline__ void shrink(int m, uint32_t (&xa)[KSMAX][2]) {
        const GItem& it = S.desc[m];
        const int r = it.rank, nt = it.nt;
        const int nsl = (r + 7) >> 3;
        float* part = p.ws + it.ws + int64_t(c) * nt * r;
        const uint32_t rs = uint32_t(p.Kc) * ES + 16;
        if constexpr (kF32) {
            // warp w: row w of each slot, lanes over 16-byte vectors, fixed-order butterfly
            const int nv = p.Kc >> 2;
            for (int s = 0; s < nsl; ++s) {
                wait_slot();
                const int nr = min(8, r - 8 * s);
                float acc[kGMaxTok];
#pragma unroll
                for (int t = 0; t < kGMaxTok; ++t) acc[t] = 0.f;
                if (warp < nr) {
                    const float4* arow =
                        reinterpret_cast<const float4*>(S.ring + rp.slot * uint32_t(p.SS) + uint32_t(warp) * rs);
                    for (int v = lane; v < nv; v += 32) {
                        const float4 a = arow[v];
#pragma unroll
                        for (int t = 0; t < kGMaxTok; ++t)
                            if (t < nt) {
                                const float4 xv = reinterpret_cast<const float4*>(xrow(it, t))[v];
                                acc[t] = fmaf(a.x, xv.x, acc[t]);
                                acc[t] = fmaf(a.y, xv.y, acc[t]);
                                acc[t] = fmaf(a.z, xv.z, acc[t]);
                                acc[t] = fmaf(a.w, xv.w, acc[t]);
                            }
                    }
                }
                release_slot();
                if (warp < nr) {
#pragma unroll
                    for (int t = 0; t < kGMaxTok; ++t) {
                        float a = acc[t];
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                        if (lane == 0 && t < nt) part[t * r + 8 * s + warp] = a;
                    }
                }
            }
        } else {
            const int KW = p.Kc >> 3, KS = KW >> 4;
            const int g = lane >> 2, t4 = lane & 3;
            uint32_t xc[KSMAX][2];  // this item's fragments; xa is refilled with the next item's now
#pragma unroll
            for (int ks = 0; ks < KSMAX; ++ks) {
                xc[ks][0] = xa[ks][0];
                xc[ks][1] = xa[ks][1];
            }
            load_x(m + 1, xa);
            // ldmatrix: lanes 8*mi .. 8*mi+7 address row rr of matrix mi = k offset 8*mi (two k-steps per x4)
            const int mi = lane >> 3, rr = lane & 7;
            const uint32_t rowoff = uint32_t(rr) * rs + uint32_t(warp * KW + mi * 8) * ES;
            const uint32_t ring = smem_u32(S.ring);
            for (int s = 0; s < nsl; ++s) {
                wait_slot();
                if (m == 0 && s == 0 && tid == 0) {
                    GTRACE(10);
                    GTRACE_ALL(2);
                }
                const uint32_t base = ring + uint32_t(rp.slot) * uint32_t(p.SS) + rowoff;
                float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
                if (!(p.dbg & 8)) {
#pragma unroll
                    for (int kp = 0; kp < KSMAX / 2; ++kp)
                        if (2 * kp < KS) {
                            uint32_t b0, b1, b2, b3;
                            ldsm_x4(base + uint32_t(kp) * 32u * ES, b0, b1, b2, b3);
                            Mma<T>::run(d0, xc[2 * kp][0], xc[2 * kp][1], b0, b1);
                            Mma<T>::run(d1, xc[2 * kp + 1][0], xc[2 * kp + 1][1], b2, b3);
                        }
                }
                release_slot();
                if (p.dbg & 8) continue;
                // d[0], d[1]: token g, rows 2*t4, 2*t4+1 of the slot (rows >= r: discarded below)
                float* rb = S.red + (s & 1) * 512 + warp * 64 + g * 8 + 2 * t4;
                rb[0] = d0[0] + d1[0];
                rb[1] = d0[1] + d1[1];
                bar_sync(1, kGConsumers * 32);
                if (tid < 64) {
                    const int tok = tid >> 3, row = tid & 7;
                    if (tok < nt && 8 * s + row < r) {
                        const float* rd = S.red + (s & 1) * 512 + tok * 8 + row;
                        float sum = 0.f;
#pragma unroll
                        for (int w = 0; w < kGConsumers; ++w) sum += rd[w * 64];
                        part[tok * r + 8 * s + row] = sum;
                    }
                }
            }
        }
        bar_sync(1, kGConsumers * 32);  // every partial of the item is written
        if (tid == 0) {
            __threadfence();
            red_release_add(p.cnt + 2 * (i0 + m), 1);
        }
    }

    // -- expand of item m over this CTA's column slice (v of the item in vbuf[m % 2]);
    // yv: the item's y pairs (load_y)
    __device__ __forceinline__ void expand(int m, const uint32_t (&yv)[KSMAX][2]) {
        const GItem& it = S.desc[m];
        const int r = it.rank, nt = it.nt;
        const float* vb = S.vbuf + (m & 1) * (kGMaxTok * 64);
        const uint32_t rs = uint32_t(p.Dc) * ES + 16;
        const int nsl = (r + 7) >> 3;
        const float scale = it.scale;
        if constexpr (kF32) {
            // thread = (16-byte column vector, token group), FFMA over the rank rows
            const int nv = p.Dc / VE;
            const int tpv = max(1, (kGConsumers * 32) / nv);
            const bool active = tid < nv * tpv;
            const int cv = tid % nv, tg = tid / nv;
            constexpr int TT = kGMaxTok;
            float acc[TT][VE];
#pragma unroll
            for (int k = 0; k < TT; ++k)
#pragma unroll
                for (int e = 0; e < VE; ++e) acc[k][e] = 0.f;
            for (int s = 0; s < nsl; ++s) {
                wait_slot();
                const int nr = min(8, r - 8 * s);
                if (active && !(p.dbg & 16)) {
                    const unsigned char* sb = S.ring + rp.slot * uint32_t(p.SS) + cv * 16;
                    for (int jj = 0; jj < nr; ++jj) {
                        float b[VE];
                        V::to_f32(*reinterpret_cast<const uint4*>(sb + jj * rs), b);
#pragma unroll
                        for (int k = 0; k < TT; ++k) {
                            const int t = tg + k * tpv;
                            if (t < nt) {
                                const float vv = vb[t * r + 8 * s + jj];
#pragma unroll
                                for (int e = 0; e < VE; ++e) acc[k][e] = fmaf(vv, b[e], acc[k][e]);
                            }
                        }
                    }
                }
                release_slot();
            }
            if (!active) return;
#pragma unroll
            for (int k = 0; k < TT; ++k) {
                const int t = tg + k * tpv;
                if (t < nt) {
                    T* yp = yrow(it, t) + cv * VE;
                    float yf[VE];
                    V::to_f32(*reinterpret_cast<const uint4*>(yp), yf);
#pragma unroll
                    for (int e = 0; e < VE; ++e) yf[e] = yf[e] + scale * acc[k][e];
                    *reinterpret_cast<uint4*>(yp) = V::from_f32(yf);
                }
            }
        } else {
            // D[col][tok] over this warp's columns [warp*CW, (warp+1)*CW): m-blocks of 16 columns
            using MF = Mma8<T>;
            const int CW = p.Dc >> 3, MB = CW >> 4;
            const int g = lane >> 2, t4 = lane & 3;
            const int mi = lane >> 3, rr = lane & 7;
            float acc[KSMAX][4];
#pragma unroll
            for (int j = 0; j < KSMAX; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
            const uint32_t ring = smem_u32(S.ring);
            // ldmatrix.trans: lanes 8*mi..8*mi+7 address rank row rr, columns +8*mi of a 32-column pair of m-blocks
            const uint32_t laneoff = uint32_t(rr) * rs + uint32_t(warp * CW + mi * 8) * ES;
            const bool math = !(p.dbg & 16);
            for (int s = 0; s < nsl; ++s) {
                wait_slot();
                const int nr = min(8, r - 8 * s);
                if (math) {
                    // v^T operand (k = rank rows 8s+2t4, +1; n = token g) as hi + lo 16-bit pairs
                    const int j = 8 * s + 2 * t4;
                    const float v0 = (g < nt && j < r) ? vb[g * r + j] : 0.f;
                    const float v1 = (g < nt && j + 1 < r) ? vb[g * r + j + 1] : 0.f;
                    const uint32_t bh = MF::pack(v0, v1);
                    const float2 hf = MF::unpack(bh);
                    const uint32_t bl = MF::pack(v0 - hf.x, v1 - hf.y);
                    // rows >= nr of a partial slot hold stale bytes: zero their A-operand halves
                    const uint32_t keep = 2 * t4 + 1 < nr ? 0xffffffffu : (2 * t4 < nr ? 0x0000ffffu : 0u);
                    const uint32_t base = ring + uint32_t(rp.slot) * uint32_t(p.SS) + laneoff;
#pragma unroll
                    for (int q = 0; q < KSMAX / 2; ++q)
                        if (2 * q < MB) {
                            uint32_t a0, a1, a2, a3;
                            ldsm_x4_t(base + uint32_t(q) * 32u * ES, a0, a1, a2, a3);
                            a0 &= keep;
                            a1 &= keep;
                            a2 &= keep;
                            a3 &= keep;
                            MF::run(acc[2 * q], a0, a1, bh);
                            MF::run(acc[2 * q], a0, a1, bl);
                            MF::run(acc[2 * q + 1], a2, a3, bh);
                            MF::run(acc[2 * q + 1], a2, a3, bl);
                        }
                }
                release_slot();
            }
            if (!math) return;
            // acc[j]: columns warp*CW + 16j + g (c0: token 2t4, c1: 2t4+1) and +8 (c2, c3).  One
            // exchange with lane ^ 4 (column g ^ 1) turns them into column pairs of one token:
            // even g keeps token 2t4 (columns g, g+1), odd g token 2t4+1 (columns g-1, g).
            const bool odd = g & 1;
            T* yp = ypair(it);
#pragma unroll
            for (int jm = 0; jm < KSMAX; ++jm)
                if (jm < MB) {
                    const float s0 = __shfl_xor_sync(0xffffffffu, odd ? acc[jm][0] : acc[jm][1], 4);
                    const float s2 = __shfl_xor_sync(0xffffffffu, odd ? acc[jm][2] : acc[jm][3], 4);
                    const float lo0 = odd ? s0 : acc[jm][0], hi0 = odd ? acc[jm][1] : s0;
                    const float lo8 = odd ? s2 : acc[jm][2], hi8 = odd ? acc[jm][3] : s2;
                    if (yp) {
                        const float2 y0 = MF::unpack(yv[jm][0]);
                        const float2 y8 = MF::unpack(yv[jm][1]);
                        *reinterpret_cast<uint32_t*>(yp + 16 * jm) = MF::pack(y0.x + scale * lo0, y0.y + scale * hi0);
                        *reinterpret_cast<uint32_t*>(yp + 16 * jm + 8) =
                            MF::pack(y8.x + scale * lo8, y8.y + scale * hi8);
                    }
                }
        }
    }

    __device__ __forceinline__ void run() {
        uint32_t xa[KSMAX][2];  // x fragments of the next item to shrink
        uint32_t yv[KSMAX][2];  // y pairs of the item being expanded
        load_x(0, xa);
        for (int m = 0; m < min(n, kGDepth); ++m) shrink(m, xa);
        if (tid == 0) GTRACE(16);
        for (int i = 0; i < n; ++i) {
            if (i + kGDepth < n) shrink(i + kGDepth, xa);
            if (tid == 0) GTRACE(17 + 3 * i);
            load_y(i, yv);  // in flight during the wait for v
            mbar_wait(&S.vfull[i & 1], (i >> 1) & 1);
            if (tid == 0) GTRACE(18 + 3 * i);
            expand(i, yv);
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.vempty[i & 1]);
            if (tid == 0) GTRACE(19 + 3 * i);
        }
        if (tid == 0) {
            GTRACE(63);
            GTRACE_ALL(3);
        }
    }
};

template <typename T, int KSMAX>
__global__ void __launch_bounds__(kGThreads, 2) mbgmv_group_kernel(const __grid_constant__ GroupParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const GSmem S = carve(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int C = p.C;
    const int g = blockIdx.x / C, c = blockIdx.x - g * C;
    const int i0 = p.goff[g], n = p.goff[g + 1] - i0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kGMaxSlots; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], kGConsumers);
        }
        mbar_init(S.dbar, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.vfull[b], 1);
            mbar_init(&S.vempty[b], kGConsumers);
        }
        for (int b = 0; b < kIdRing; ++b) {
            mbar_init(&S.idfull[b], 32);
            mbar_init(&S.idempty[b], kGProducers);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_trigger();  // the next launch may start its prologue (weights only)
    if (threadIdx.x == 0) {
        GTRACE(0);
        GTRACE_ALL(0);
    }
    if (n <= 0) return;
    if (warp >= kGConsumers && warp < kGConsumers + kGProducers) {
        const int pw = warp - kGConsumers;
        if (pw == 0 && lane == 0) {
            mbar_arrive_expect_tx(S.dbar, uint32_t(n) * sizeof(GItem));
            bulk_g2s(S.desc, p.items + i0, uint32_t(n) * sizeof(GItem), S.dbar);
        }
        mbar_wait(S.dbar, 0);
        if (pw == 0 && lane == 0) GTRACE(1);
        producer<T>(p, S, c, n, pw, lane);
    } else if (warp == kGConsumers + kGProducers) {
        pdl_wait();  // the workspace and the counters belong to the previous kernel until here
        mbar_wait(S.dbar, 0);
        exchange(p, S, i0, n, lane);
    } else {
        pdl_wait();  // x, y belong to the previous kernel until here
        if (threadIdx.x == 0) {
            GTRACE(8);
            GTRACE_ALL(1);
        }
        mbar_wait(S.dbar, 0);
        if (threadIdx.x == 0) GTRACE(9);
        Consumer<T, KSMAX> cons(p, S, c, i0, n);
        cons.run();
    }
}

template <typename T, int KSMAX>
void* kptr() {
    return reinterpret_cast<void*>(mbgmv_group_kernel<T, KSMAX>);
}
void* group_kernel_for(int dtype, int ksmax) {
    if (dtype == kF32) return kptr<float, 1>();
    if (dtype == kF16) return ksmax > 8 ? kptr<__half, 16>() : kptr<__half, 8>();
    return ksmax > 8 ? kptr<__nv_bfloat16, 16>() : kptr<__nv_bfloat16, 8>();
}
bool pdl_on() {
    static const bool on = [] {
        const char* s = getenv("SLORA_PDL");
        return !(s && atoi(s) == 0);
    }();
    return on;
}
}  // namespace

cudaError_t configure_mbgmv_group() {
    const void* ks[5] = {kptr<float, 1>(), kptr<__half, 8>(), kptr<__half, 16>(), kptr<__nv_bfloat16, 8>(),
                         kptr<__nv_bfloat16, 16>()};
    for (const void* k : ks) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_mbgmv_group(const GroupParams& p, int dtype, int grid, size_t smem, cudaStream_t s) {
    if (grid <= 0) return cudaSuccess;
    const int KS = (p.Kc / 8) / 16;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = smem;
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
    void* k = group_kernel_for(dtype, KS);
    void* args[] = {const_cast<GroupParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, k, args);
}

}  // namespace slora
