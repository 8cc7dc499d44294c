// mbgmv.cu -- the fused single-GPU MBGMV of the S-LoRA hot path on sm_100a:
// heterogeneous batched LoRA, y_i += scale_a * (x_i A_a) B_a, over adapter
// rows gathered from Unified Paging pages (Sec. 5.3, P:279-289;
// Eq. lora_factored; reading R1: page j of A holds column j of A).
//
// Decomposition.  The host (api.cpp plan_group_call) cuts the batch into
// items = (adapter segment, projection, chunk of <= 8 tokens), sorted largest
// first.  A grid of thread-block clusters of C CTAs claims them dynamically:
// the leader CTA of a cluster takes the next item from a per-launch atomic
// counter and broadcasts its index into every CTA of the cluster (distributed
// shared memory), so clusters that start late or run slow simply take fewer
// items.  All C CTAs of a cluster process the same items; CTA c (cluster rank)
//   shrink:   reads the K-slice c (Kc = K/C elements) of each of the item's r
//             stored A rows and forms partial dot products with the same slice
//             of the tokens' x rows (mma.sync m16n8k16: M = tokens, N = 8 A
//             rows, K = 16, fp32 accumulate) -> its partial v (nt x r fp32)
//             in its own shared memory;
//   exchange: the exchange warp of every CTA reads the C partials of the item
//             through distributed shared memory (after each owner's remote
//             release-arrive) and sums them in rank order -> v (complete);
//   expand:   reads the output-column slice c (Dc = D/C) of the item's r B
//             rows and writes y[tok][slice] = y + scale * sum_j v_j B_j
//             (mma.sync m16n8k8: M = 16 output columns (B^T via
//             ldmatrix.trans), N = tokens, K = 8 rank rows; v enters as a
//             16-bit hi + lo pair so the products keep ~fp32 accuracy; fp32
//             accumulate, one rounding into y).
// fp32 inputs never use tensor cores (no TF32, reading R5): their shrink and
// expand are CUDA-core FFMA loops.
//
// Data movement: two producer warps stream, in the consumers' order, 8-row
// slots into a shared-memory ring with cp.async.bulk (TMA engine, SASS
// UBLKCP): per item an X slot (the tokens' x row slices) then its A row
// slices, and later its B row slices then a Y slot (the tokens' y row
// slices).  The weights are never written by the previous kernel, so weight
// slots are issued before griddepcontrol.wait (programmatic dependent launch);
// X and Y slots of the ring's first lap are deferred until after it.  The
// consumers touch global memory only to store y, and the exchange never leaves
// the cluster: no load sits on the consumers' critical path.
//
// Determinism: every v entry is (each warp's mma chain over its k-range)
// summed over the 8 warps in order, then over the C slices in rank order;
// every y element is one fixed-order mma accumulation.  Results depend only
// on (K, C, r), never on page placement, batch order or which cluster claims
// an item.  Clusters never wait for each other (only on the shared counter).
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
// diagnostics: event ev of this CTA (CTAs 0-15; events < 256: 0-63 phases, 64-127 consumer got
// slot k, 128-191 consumer starts waiting for slot k, 192-255 producer issued weight slot k)
#define GTRACE(ev)                                                                                 \
    do {                                                                                           \
        if (p.trace && blockIdx.x < 16 && (ev) < 256) p.trace[blockIdx.x * 256 + (ev)] = gtimer(); \
    } while (0)
// diagnostics: per-CTA summary [CTA < 512][4]: 0 start, 1 consumers past griddepcontrol.wait,
// 2 items processed, 3 consumers done
#define GTRACE_ALL(ev, val)                                                                  \
    do {                                                                                     \
        if (p.trace && blockIdx.x < 512) p.trace[16 * 256 + blockIdx.x * 4 + (ev)] = (val); \
    } while (0)

constexpr int kIdRing = 4;  // page-id ring entries (items)
constexpr int kNP = 3;      // partial-v buffers (item m uses m % 3)
constexpr int kVB = kGMaxTok * 64;  // floats of one v / partial buffer
constexpr int kQD = kGQueue;        // claimed-item ring (item m uses m % kQD)

struct GSmem {
    uint64_t* full;    // [kGMaxSlots] slot filled (producer expect_tx + TMA bytes)
    uint64_t* empty;   // [kGMaxSlots] slot released (one arrival per consumer warp)
    uint64_t* vfull;   // [2] v of item i ready (exchange warp)
    uint64_t* vempty;  // [2] v of item i consumed (consumer warps)
    uint64_t* idfull;  // [kIdRing] page ids of item m landed (cp.async, 32 lanes)
    uint64_t* idempty; // [kIdRing] page ids of item m read by every producer warp
    uint64_t* pready;  // [kNP] partials of item m ready in all C CTAs (C remote arrivals)
    uint64_t* pfree;   // [kNP] this CTA's partial of item m read by all C CTAs (C remote arrivals)
    uint64_t* qfull;   // [kQD] claimed index of item m written by the leader (remote arrive)
    uint64_t* qempty;  // [kQD] (leader CTA) index of item m read by all C CTAs (C remote arrivals)
    uint64_t* dfull;   // [kQD] descriptor of item m staged (bulk copy, or a stop marker)
    uint64_t* dempty;  // [kQD] descriptor of item m no longer needed (consumer warps)
    int32_t* iq;       // [kQD] claimed global item index of item m (-1: no more items)
    int32_t* deferq;   // [kGProducers][16] deferred activation slots: stream position
    int32_t* deferi;   // [kGProducers][16] deferred activation slots: item * 2 + (0 = X, 1 = Y)
    uint32_t zero16;   // shared address of 16 zero bytes (ldmatrix rows of absent tokens)
    GItem* desc;       // [kQD]
    int32_t* ids;      // [kIdRing][128] page ids of items m % kIdRing: A rows then B rows
    float* red;        // [2][8 warps][8 tokens][8 rows] per-slot shrink partials
    float* vbuf;       // [2][nt][r] v of items i % 2 (complete)
    float* part;       // [kNP][nt][r] this CTA's partial v of items m % kNP
    unsigned char* ring;
};
__device__ __forceinline__ GSmem carve(unsigned char* s) {
    GSmem L;
    L.full = reinterpret_cast<uint64_t*>(s);
    L.empty = L.full + kGMaxSlots;
    L.vfull = L.empty + kGMaxSlots;
    L.vempty = L.vfull + 2;
    L.idfull = L.vempty + 2;
    L.idempty = L.idfull + kIdRing;
    L.pready = L.idempty + kIdRing;
    L.pfree = L.pready + kNP;
    L.qfull = L.pfree + kNP;
    L.qempty = L.qfull + kQD;
    L.dfull = L.qempty + kQD;
    L.dempty = L.dfull + kQD;   // barriers end at 8 * (16+16+2+2+4+4+3+3+4*8) = 656 bytes
    L.zero16 = smem_u32(s + 704);  // 64 zero bytes at 704
    L.iq = reinterpret_cast<int32_t*>(s + 768);
    L.deferq = reinterpret_cast<int32_t*>(s + 832);
    L.deferi = L.deferq + kGProducers * 16;  // ends at 832 + 256 = 1088
    L.desc = reinterpret_cast<GItem*>(s + 1152);
    L.ids = reinterpret_cast<int32_t*>(s + 1152 + kQD * 64);
    L.red = reinterpret_cast<float*>(s + 1152 + kQD * 64 + kIdRing * 128 * 4);
    L.vbuf = L.red + 2 * 8 * 64;
    L.part = L.vbuf + 2 * kVB;
    L.ring = s + kGFixedSmem;
    return L;
}
static_assert(kGFixedSmem == 1152 + kQD * 64 + kIdRing * 128 * 4 + 2 * 8 * 64 * 4 + 2 * kVB * 4 + kNP * kVB * 4,
              "shared-memory layout");

// The slot stream, in the consumers' order: S(0), S(1), then for i = 0, 1, ...:
// S(i+2), E(i), where S(m) = [X(m), A(m) rows in slots of 8] and E(i) =
// [B(i) rows in slots of 8, Y(i)].  nslot(r) = ceil(r / 8).
__device__ __forceinline__ int nslot(int r) { return (r + 7) >> 3; }

// Item m of this cluster (its descriptor in desc[m % kQD]) once staged; nullptr
// after the last one.  Every role of every CTA sees the same sequence.
__device__ __forceinline__ const GItem* item_at(const GSmem& S, int m) {
    mbar_wait(&S.dfull[m % kQD], (m / kQD) & 1);
    const GItem* it = &S.desc[m % kQD];
    return it->rank > 0 ? it : nullptr;
}

// ------------------------------------------------------------ producers
// kGProducers warps walk the stream and issue alternate slots (a warp issues
// its bulk copies one lane at a time, ~60 ns each: one warp alone caps a CTA
// near 20-40 GB/s).  Producer 0 also
//   - (leader CTA only) claims the cluster's items from the launch counter and
//     broadcasts each claimed index into every CTA of the cluster;
//   - stages each item's descriptor (bulk copy) and fetches its page ids three
//     items ahead into a 4-entry ring with cp.async (idfull); every producer
//     releases an id entry (idempty) after the item's B rows.
template <typename T>
__device__ __forceinline__ void producer(const GroupParams& p, const GSmem& S, int c, int pw, int lane) {
    constexpr int ES = sizeof(T);
    const T* pool = reinterpret_cast<const T*>(p.pool);
    const int64_t P = p.P;
    const int ns = p.ns;
    const int C = p.C;
    const uint32_t SS = uint32_t(p.SS);
    const bool copy = !(p.dbg & 32);
    const bool leader = c == 0;
    int last = 1 << 30;    // index of the first absent item (known to producer 0 once resolved)
    bool claiming = true;  // leader: claims left to make
    // leader: claim item m (or learn that none is left) and broadcast the index to the cluster
    auto broadcast = [&](int m, int j) {
        const int e = m % kQD;
        if (m >= kQD) mbar_wait_cluster(&S.qempty[e], ((m / kQD) - 1) & 1);
        if (lane < C) {
            st_dsmem(mapa(smem_u32(&S.iq[e]), uint32_t(lane)), j);
            mbar_arrive_remote(mapa(smem_u32(&S.qfull[e]), uint32_t(lane)));
        }
        __syncwarp();
    };
    auto claim_done = [&]() {  // the cluster made its last claim; the last cluster resets the counter
        if (lane == 0 && atomicAdd(p.ctr + 1, 1) == int(gridDim.x) / C - 1) {
            p.ctr[0] = 0;
            p.ctr[1] = 0;
        }
        __syncwarp();
    };
    auto claim = [&](int m) {
        if (pw != 0 || !leader || !claiming) return;
        int j = 0;
        if (lane == 0) j = atomicAdd(p.ctr, 1);
        j = __shfl_sync(0xffffffffu, j, 0);
        if (j >= p.n_items) {
            j = -1;
            claiming = false;
        }
        broadcast(m, j);
#ifdef SLORA_HANG_DEBUG
        if (lane == 0 && gridDim.x / C <= 32) printf("CLAIM block %d m %d j %d ctr %p\n", blockIdx.x, m, j, p.ctr);
#endif
        if (!claiming) claim_done();
    };
    // producer 0: item m's index -> its descriptor, or the stop marker (at and beyond the first
    // absent item, so that every role's lookahead finds one)
    auto resolve = [&](int m) {
        if (pw != 0) return;
        const int e = m % kQD;
        int j = -1;
        if (m <= last) {  // the leader broadcast an index (or -1) for item m
            mbar_wait_cluster(&S.qfull[e], (m / kQD) & 1);
            j = S.iq[e];
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(mapa(smem_u32(&S.qempty[e]), 0u));
#ifdef SLORA_HANG_DEBUG
            if (lane == 0 && gridDim.x / C <= 32) printf("RESOLVE block %d m %d j %d\n", blockIdx.x, m, j);
#endif
        }
        if (m >= kQD) mbar_wait(&S.dempty[e], ((m / kQD) - 1) & 1);
        if (j >= 0) {
            if (lane == 0) {
                mbar_arrive_expect_tx(&S.dfull[e], sizeof(GItem));
                bulk_g2s(&S.desc[e], p.items + j, sizeof(GItem), &S.dfull[e]);
            }
        } else {
            last = min(last, m);
            if (lane == 0) {
                S.desc[e].rank = 0;
                mbar_arrive(&S.dfull[e]);
            }
        }
        __syncwarp();
    };
    auto fetch = [&](int m) {  // page ids of item m (producer 0)
        if (pw != 0 || m >= last) return;
        const GItem* it = item_at(S, m);
        if (!it) return;
        const int e = m % kIdRing;
        if (m >= kIdRing) mbar_wait(&S.idempty[e], ((m / kIdRing) - 1) & 1);
        const int r = it->rank;
        const int proj = p.proj_ids[it->pi];
        const int32_t* src = it->tab + int64_t((p.layer * 4 + proj) * 2) * r;  // A ids, then B ids
        int32_t* dst = S.ids + e * 128;
        for (int j = lane; j < 2 * r; j += 32) cp_async4(dst + j, src + j);
        cp_async_mbar_arrive(&S.idfull[e]);
    };
    int k = 0;             // stream position
    bool waited = false;   // griddepcontrol.wait done (activation slots may be issued)
    int ndef = 0;          // deferred activation slots of the first lap
    int32_t* dq = S.deferq + pw * 16;
    int32_t* di = S.deferi + pw * 16;
    // X (kind 0) or Y (kind 1) slot of item m into stream position kk (its slot is free)
    auto issue_act = [&](int kk, int m, int kind) {
        const GItem& it = S.desc[m % kQD];
        const int slot = kk % ns;
        const int eK = kind ? p.Dc : p.Kc;
        const uint32_t rb = uint32_t(eK) * ES;
        const uint32_t rs = rb + 16;
        if (lane == 0) mbar_arrive_expect_tx(&S.full[slot], uint32_t(it.nt) * rb);
        __syncwarp();
        if (lane < it.nt) {
            const T* src;
            if (kind == 0) {
                src = reinterpret_cast<const T*>(p.x) + int64_t(it.tok[lane]) * p.ldx + int64_t(c) * p.Kc;
            } else {
                const int proj = p.proj_ids[it.pi];
                src = reinterpret_cast<const T*>(p.y[proj]) + int64_t(it.tok[lane]) * p.ldy[proj] +
                      int64_t(c) * p.Dc;
            }
            bulk_g2s(S.ring + slot * SS + uint32_t(lane) * rs, src, rb, &S.full[slot]);
        }
    };
    auto flush = [&]() {  // griddepcontrol.wait, then the deferred activation slots
        pdl_wait();
        waited = true;
        for (int q = 0; q < ndef; ++q) issue_act(dq[q], di[q] >> 1, di[q] & 1);
        ndef = 0;
    };
    auto act = [&](int m, int kind) {  // one activation slot at position k
        if (k % kGProducers == pw) {
            if (waited) {
                mbar_wait(&S.empty[k % ns], ((k / ns) & 1) ^ 1);
                issue_act(k, m, kind);
            } else if (k < ns) {
                if (lane == 0) {
                    dq[ndef] = k;
                    di[ndef] = m * 2 + kind;
                }
                __syncwarp();
                ++ndef;
            } else {
                flush();
                mbar_wait(&S.empty[k % ns], ((k / ns) & 1) ^ 1);
                issue_act(k, m, kind);
            }
        }
        ++k;
    };
    auto rows = [&](int m, int kind) {  // the item's A (kind 0) or B (kind 1) rows, 8 per slot
        const int e = m % kIdRing;
        mbar_wait(&S.idfull[e], (m / kIdRing) & 1);
        const GItem& it = S.desc[m % kQD];
        const int r = it.rank;
        const int32_t* id = S.ids + e * 128 + (kind ? r : 0);
        const int eK = kind ? p.Dc : p.Kc;
        const uint32_t rb = uint32_t(eK) * ES;
        const uint32_t rs = rb + 16;
        const int64_t coff = int64_t(c) * eK;
        for (int j0 = 0; j0 < r; j0 += 8, ++k) {
            if (k % kGProducers != pw) continue;
            if (k >= ns && !waited) flush();  // the ring wraps: the consumers need the deferred slots first
            const int slot = k % ns;
            const int nr = min(8, r - j0);
            mbar_wait(&S.empty[slot], ((k / ns) & 1) ^ 1);
            const int pg = lane < nr ? id[j0 + lane] : 0;
            if (lane == 0) {
                if (copy)
                    mbar_arrive_expect_tx(&S.full[slot], uint32_t(nr) * rb);
                else
                    mbar_arrive(&S.full[slot]);
            }
            __syncwarp();
            if (lane < nr && copy)
                bulk_g2s(S.ring + slot * SS + uint32_t(lane) * rs, pool + int64_t(pg) * P + coff, rb,
                         &S.full[slot]);
            if (lane == 0 && p.trace && k < 64) GTRACE(192 + k);
        }
        if (kind) {  // the item's ids are no longer needed by this warp
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.idempty[e]);
        }
    };
    // prologue: claims and descriptors of items 0..2, their page ids
    for (int m = 0; m < 3; ++m) {
        claim(m);
        resolve(m);
    }
    for (int m = 0; m < 3; ++m) fetch(m);
    if (lane == 0 && pw == 0) GTRACE(2);
    for (int m = 0; m < kGDepth; ++m)
        if (item_at(S, m)) {
            act(m, 0);
            rows(m, 0);
        }
    if (lane == 0 && pw == 0) GTRACE(3);
    for (int i = 0; item_at(S, i); ++i) {
        if (pw == 0) {  // one more item in flight: claim + stage item i+3
            claim(i + 3);
            resolve(i + 3);
        }
        if (item_at(S, i + kGDepth)) {
            act(i + kGDepth, 0);
            rows(i + kGDepth, 0);
        }
        rows(i, 1);
        act(i, 1);
        fetch(i + 3);  // id entry (i+3) % 4 == (i-1) % 4: released by every producer after rows(i-1, B)
    }
    if (!waited) flush();
    if (lane == 0 && pw == 0) GTRACE(4);
}

// ------------------------------------------------------------ exchange warp
// v of item i = sum over the cluster's C partials in rank order (distributed
// shared memory), into vbuf[i % 2]; then every owner learns (remote arrive on
// its pfree) that its partial buffer may be rewritten.
__device__ __forceinline__ void exchange(const GroupParams& p, const GSmem& S, int lane) {
    const int C = p.C;
    for (int i = 0;; ++i) {
        const GItem* itp = item_at(S, i);
        if (!itp) break;
        const int b = i % kNP;
        if (i >= 2) mbar_wait(&S.vempty[i & 1], ((i >> 1) - 1) & 1);
        mbar_wait_cluster(&S.pready[b], (i / kNP) & 1);
        const int tot = itp->nt * itp->rank;
        float* vb = S.vbuf + (i & 1) * kVB;
        const uint32_t local = smem_u32(S.part + b * kVB);
        if (!(p.dbg & 1)) {
            if ((tot & 3) == 0) {
                for (int e4 = lane; e4 < (tot >> 2); e4 += 32) {
                    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int q = 0; q < C; ++q) {
                        const float4 v = ld_dsmem4(mapa(local, uint32_t(q)) + 16u * uint32_t(e4));
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
                    for (int q = 0; q < C; ++q) s += ld_dsmem(mapa(local, uint32_t(q)) + 4u * uint32_t(e));
                    vb[e] = s;
                }
            }
        }
        __syncwarp();
        if (lane < C) mbar_arrive_remote(mapa(smem_u32(&S.pfree[b]), uint32_t(lane)));
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

template <typename T, int KSMAX>
struct Consumer {
    static constexpr int ES = sizeof(T);
    static constexpr bool kF32 = sizeof(T) == 4;
    using V = Vec16<T>;

    const GroupParams& p;
    const GSmem& S;
    const int c, tid, warp, lane;
    int k = 0;  // stream position

    __device__ Consumer(const GroupParams& p_, const GSmem& S_, int c_)
        : p(p_), S(S_), c(c_), tid(threadIdx.x), warp(threadIdx.x >> 5), lane(threadIdx.x & 31) {}

    __device__ __forceinline__ T* yrow(const GItem& it, int t) const {
        const int proj = p.proj_ids[it.pi];
        return reinterpret_cast<T*>(p.y[proj]) + int64_t(it.tok[t]) * p.ldy[proj] + int64_t(c) * p.Dc;
    }
    __device__ __forceinline__ unsigned char* slot_ptr() const { return S.ring + (k % p.ns) * uint32_t(p.SS); }
    __device__ __forceinline__ uint32_t slot_u32() const {
        return smem_u32(S.ring) + uint32_t(k % p.ns) * uint32_t(p.SS);
    }
    __device__ __forceinline__ void wait_slot() {
        if (tid == 0 && p.trace && k < 64) GTRACE(128 + k);
        mbar_wait(&S.full[k % p.ns], (k / p.ns) & 1);
        if (tid == 0 && p.trace && k < 64) GTRACE(64 + k);
    }
    __device__ __forceinline__ void release_slot() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[k % p.ns]);
        ++k;
    }

    // -- shrink of item m: X slot, then the A slots; this CTA's partial v -> part[m % 3],
    // then a release-arrive on the pready of every CTA of the cluster
    __device__ __forceinline__ void shrink(int m, const GItem& it) {
        const int r = it.rank, nt = it.nt;
        const int nsl = nslot(r);
        const int b = m % kNP;
        float* part = S.part + b * kVB;
        // part[b] was last read (by the cluster) for item m - 3
        if (m >= kNP) mbar_wait_cluster(&S.pfree[b], ((m / kNP) - 1) & 1);
        const uint32_t rsx = uint32_t(p.Kc) * ES + 16;
        if constexpr (kF32) {
            // the X slot stays until the A rows are done (fp32 x rows are read from it directly)
            wait_slot();
            const unsigned char* xs = slot_ptr();
            const int kx = k;
            ++k;
            const int nv = p.Kc >> 2;
            for (int s = 0; s < nsl; ++s) {
                wait_slot();
                const int nr = min(8, r - 8 * s);
                float acc[kGMaxTok];
#pragma unroll
                for (int t = 0; t < kGMaxTok; ++t) acc[t] = 0.f;
                if (warp < nr) {
                    const float4* arow = reinterpret_cast<const float4*>(slot_ptr() + uint32_t(warp) * rsx);
                    for (int v = lane; v < nv; v += 32) {
                        const float4 a = arow[v];
#pragma unroll
                        for (int t = 0; t < kGMaxTok; ++t)
                            if (t < nt) {
                                const float4 xv = reinterpret_cast<const float4*>(xs + t * rsx)[v];
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
            __syncwarp();  // release the X slot (position kx)
            if (lane == 0) mbar_arrive(&S.empty[kx % p.ns]);
        } else {
            const int KW = p.Kc >> 3, KS = KW >> 4;
            const int g = lane >> 2, t4 = lane & 3;
            const int mi = lane >> 3, rr = lane & 7;
            // x fragments of this warp's k-range from the X slot: ldmatrix.x4 covers two k-steps
            // (matrix mi = k offset 8*mi; lanes of absent tokens read 16 zero bytes)
            uint32_t xa[KSMAX][2];
            wait_slot();
            {
                const bool real = rr < nt;
                const uint32_t xb = real ? slot_u32() + uint32_t(rr) * rsx + uint32_t(warp * KW + mi * 8) * ES
                                         : S.zero16;
                const uint32_t xadv = real ? 32u * ES : 0u;
#pragma unroll
                for (int kp = 0; kp < KSMAX / 2; ++kp)
                    if (2 * kp < KS)
                        ldsm_x4(xb + uint32_t(kp) * xadv, xa[2 * kp][0], xa[2 * kp][1], xa[2 * kp + 1][0],
                                xa[2 * kp + 1][1]);
            }
            release_slot();
            const uint32_t rowoff = uint32_t(rr) * rsx + uint32_t(warp * KW + mi * 8) * ES;
            for (int s = 0; s < nsl; ++s) {
                wait_slot();
                const uint32_t base = slot_u32() + rowoff;
                float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
                if (!(p.dbg & 8)) {
#pragma unroll
                    for (int kp = 0; kp < KSMAX / 2; ++kp)
                        if (2 * kp < KS) {
                            uint32_t b0, b1, b2, b3;
                            ldsm_x4(base + uint32_t(kp) * 32u * ES, b0, b1, b2, b3);
                            Mma<T>::run(d0, xa[2 * kp][0], xa[2 * kp][1], b0, b1);
                            Mma<T>::run(d1, xa[2 * kp + 1][0], xa[2 * kp + 1][1], b2, b3);
                        }
                }
                release_slot();
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
        bar_sync(1, kGConsumers * 32);  // every partial of the item is in part[b]
        if (tid < p.C) mbar_arrive_remote(mapa(smem_u32(&S.pready[b]), uint32_t(tid)));
    }

    // -- expand of item m over this CTA's column slice: the B slots, then the Y slot
    // (v of the item in vbuf[m % 2])
    __device__ __forceinline__ void expand(int m, const GItem& it) {
        const int r = it.rank, nt = it.nt;
        const float* vb = S.vbuf + (m & 1) * kVB;
        const uint32_t rs = uint32_t(p.Dc) * ES + 16;
        const int nsl = nslot(r);
        const float scale = it.scale;
        if constexpr (kF32) {
            // thread = (16-byte column vector, token group), FFMA over the rank rows
            constexpr int VE = V::VE;
            const int nv = p.Dc / VE;
            const int tpv = max(1, (kGConsumers * 32) / nv);
            const bool active = tid < nv * tpv;
            const int cv = tid % nv, tg = tid / nv;
            constexpr int TT = kGMaxTok;
            float acc[TT][VE];
#pragma unroll
            for (int q = 0; q < TT; ++q)
#pragma unroll
                for (int e = 0; e < VE; ++e) acc[q][e] = 0.f;
            for (int s = 0; s < nsl; ++s) {
                wait_slot();
                const int nr = min(8, r - 8 * s);
                if (active && !(p.dbg & 16)) {
                    const unsigned char* sb = slot_ptr() + cv * 16;
                    for (int jj = 0; jj < nr; ++jj) {
                        float bf[VE];
                        V::to_f32(*reinterpret_cast<const uint4*>(sb + jj * rs), bf);
#pragma unroll
                        for (int q = 0; q < TT; ++q) {
                            const int t = tg + q * tpv;
                            if (t < nt) {
                                const float vv = vb[t * r + 8 * s + jj];
#pragma unroll
                                for (int e = 0; e < VE; ++e) acc[q][e] = fmaf(vv, bf[e], acc[q][e]);
                            }
                        }
                    }
                }
                release_slot();
            }
            wait_slot();  // Y slot
            if (active)
#pragma unroll
                for (int q = 0; q < TT; ++q) {
                    const int t = tg + q * tpv;
                    if (t < nt) {
                        float yf[VE];
                        V::to_f32(*reinterpret_cast<const uint4*>(slot_ptr() + t * rs + cv * 16), yf);
#pragma unroll
                        for (int e = 0; e < VE; ++e) yf[e] = yf[e] + scale * acc[q][e];
                        *reinterpret_cast<uint4*>(yrow(it, t) + cv * VE) = V::from_f32(yf);
                    }
                }
            release_slot();
        } else {
            // D[col][tok] over this warp's columns [warp*CW, (warp+1)*CW): m-blocks of 16 columns
            using MF = Mma8<T>;
            const int CW = p.Dc >> 3, MB = CW >> 4;
            const int g = lane >> 2, t4 = lane & 3;
            const int mi = lane >> 3, rr = lane & 7;
            float acc[KSMAX][4];
#pragma unroll
            for (int j = 0; j < KSMAX; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
            // ldmatrix.trans: lanes 8*mi..8*mi+7 address rank row rr, columns +8*mi of a 32-column pair
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
                    const uint32_t base = slot_u32() + laneoff;
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
            // acc[j]: columns warp*CW + 16j + g (c0: token 2t4, c1: 2t4+1) and +8 (c2, c3).  One
            // exchange with lane ^ 4 (column g ^ 1) turns them into column pairs of one token:
            // even g keeps token 2t4 (columns g, g+1), odd g token 2t4+1 (columns g-1, g).
            wait_slot();  // Y slot: the tokens' y row slices
            if (math) {
                const bool odd = g & 1;
                const int tok = 2 * t4 + (g & 1);
                const int col = warp * CW + (g & ~1);
                const unsigned char* ys = slot_ptr() + uint32_t(tok) * rs + uint32_t(col) * ES;
                T* yp = tok < nt ? yrow(it, tok) + col : nullptr;
#pragma unroll
                for (int jm = 0; jm < KSMAX; ++jm)
                    if (jm < MB) {
                        const float s0 = __shfl_xor_sync(0xffffffffu, odd ? acc[jm][0] : acc[jm][1], 4);
                        const float s2 = __shfl_xor_sync(0xffffffffu, odd ? acc[jm][2] : acc[jm][3], 4);
                        const float lo0 = odd ? s0 : acc[jm][0], hi0 = odd ? acc[jm][1] : s0;
                        const float lo8 = odd ? s2 : acc[jm][2], hi8 = odd ? acc[jm][3] : s2;
                        if (yp) {
                            const float2 y0 = MF::unpack(*reinterpret_cast<const uint32_t*>(ys + 16 * jm * ES));
                            const float2 y8 =
                                MF::unpack(*reinterpret_cast<const uint32_t*>(ys + (16 * jm + 8) * ES));
                            *reinterpret_cast<uint32_t*>(yp + 16 * jm) =
                                MF::pack(y0.x + scale * lo0, y0.y + scale * hi0);
                            *reinterpret_cast<uint32_t*>(yp + 16 * jm + 8) =
                                MF::pack(y8.x + scale * lo8, y8.y + scale * hi8);
                        }
                    }
            }
            release_slot();
        }
    }

    __device__ __forceinline__ void run() {
        for (int m = 0; m < kGDepth; ++m)
            if (const GItem* it = item_at(S, m)) shrink(m, *it);
        if (tid == 0) GTRACE(16);
        int i = 0;
        for (;; ++i) {
            const GItem* it = item_at(S, i);
            if (!it) break;
            if (const GItem* nx = item_at(S, i + kGDepth)) shrink(i + kGDepth, *nx);
            if (tid == 0 && i < 15) GTRACE(17 + 3 * i);
            mbar_wait(&S.vfull[i & 1], (i >> 1) & 1);
            if (tid == 0 && i < 15) GTRACE(18 + 3 * i);
            expand(i, *it);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&S.vempty[i & 1]);
                mbar_arrive(&S.dempty[i % kQD]);
            }
            if (tid == 0 && i < 15) GTRACE(19 + 3 * i);
        }
        if (tid == 0) {
            GTRACE(63);
            GTRACE_ALL(2, i);
            GTRACE_ALL(3, gtimer());
        }
    }
};

template <typename T, int KSMAX>
__global__ void __launch_bounds__(kGThreads, 2) mbgmv_group_kernel(const __grid_constant__ GroupParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const GSmem S = carve(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int C = p.C, c = int(cluster_ctarank());
    if (threadIdx.x == 0) {
        for (int s = 0; s < kGMaxSlots; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], kGConsumers);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.vfull[b], 1);
            mbar_init(&S.vempty[b], kGConsumers);
        }
        for (int b = 0; b < kIdRing; ++b) {
            mbar_init(&S.idfull[b], 32);
            mbar_init(&S.idempty[b], kGProducers);
        }
        for (int b = 0; b < kNP; ++b) {
            mbar_init(&S.pready[b], C);
            mbar_init(&S.pfree[b], C);
        }
        for (int b = 0; b < kQD; ++b) {
            mbar_init(&S.qfull[b], 1);
            mbar_init(&S.qempty[b], C);
            mbar_init(&S.dfull[b], 1);
            mbar_init(&S.dempty[b], kGConsumers);
        }
        fence_mbar_init();
    }
    if (threadIdx.x < 16) reinterpret_cast<uint32_t*>(smem + 704)[threadIdx.x] = 0u;
    cluster_sync();  // every CTA's barriers exist before any remote arrive
    pdl_trigger();   // the next launch may start its prologue (weights only)
    if (threadIdx.x == 0) {
        GTRACE(0);
        GTRACE_ALL(0, gtimer());
    }
    if (warp >= kGConsumers && warp < kGConsumers + kGProducers) {
        producer<T>(p, S, c, warp - kGConsumers, lane);
    } else if (warp == kGConsumers + kGProducers) {
        exchange(p, S, lane);
    } else {
        pdl_wait();  // y stores must follow the previous kernel
        if (threadIdx.x == 0) {
            GTRACE(8);
            GTRACE_ALL(1, gtimer());
        }
        Consumer<T, KSMAX> cons(p, S, c);
        cons.run();
    }
    cluster_sync();  // no CTA leaves while a peer may still read its partials or arrive on its barriers
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
        e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e) return e;
    }
    return cudaSuccess;
}

int mbgmv_group_max_clusters(int dtype, int C, size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(C));
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(C);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, group_kernel_for(dtype, 8), &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

cudaError_t launch_mbgmv_group(const GroupParams& p, int dtype, int grid, size_t smem, cudaStream_t s) {
    if (grid <= 0) return cudaSuccess;
    const int KS = (p.Kc / 8) / 16;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = unsigned(p.C);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
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
