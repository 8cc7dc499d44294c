// kernels.cu -- sm_100a kernels of the S-LoRA hot path.
//
//   lora_unit_kernel<T, MODE>   MBGMV gather-shrink-expand over Unified Paging
//       (Sec. 5.3; Eq. lora_factored).
//       One thread-block cluster of C CTAs per work unit; CTA c owns the c-th
//       1/C slice of the hidden dimension.  Page rows of A and B and the
//       unit's x rows are staged into shared memory by cp.async.bulk
//       (one bulk copy per page slice, completion on an mbarrier), so a single
//       issuing warp puts the whole unit's bytes in flight at once.  Shrink:
//       fp32 dot products over the CTA's K slice with warp-shuffle reductions;
//       the C partial v vectors are combined through distributed shared
//       memory (reduce-scatter + broadcast, fixed order c = 0..C-1); expand:
//       fp32 axpys of the B page slices into y.  The rank-r intermediate never
//       leaves the cluster.  Reduction order depends only on (K, C), never on
//       page placement or batch order.
//   scatter_kernel   adapter load: staging -> pages (A transposed).
//   gather_kernel    test-only page gather.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

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
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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
// 1-D bulk copy global -> own shared memory, completes on `bar` (TMA engine;
// SASS UBLKCP).  bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// ---------------------------------------------------- element conversions
// A 16-byte vector holds VE elements.
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

struct SmemLayout {
    size_t a, b, x, vp, v, bar, total;
};
__host__ __device__ inline SmemLayout smem_layout(const LoraParams& p, int mode, int es) {
    SmemLayout L{};
    const size_t KS = p.K / p.C, DS = p.D / p.C;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
    L.bar = take(16);
    L.a = take(mode == kExpand ? 0 : size_t(p.rcap) * KS * es);
    L.b = take(mode == kShrink ? 0 : size_t(p.rcap) * DS * es);
    L.x = take(mode == kExpand ? 0 : size_t(p.tcap) * KS * es);
    L.vp = take(mode == kExpand ? 0 : size_t(p.vcap) * 4);
    L.v = take(mode == kShrink ? 0 : size_t(p.vcap) * 4);
    L.total = off;
    return L;
}

// ------------------------------------------------------------ the kernel
template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads) lora_unit_kernel(const __grid_constant__ LoraParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    using V = Vec<T>;
    constexpr int VE = V::VE;
    constexpr int ES = sizeof(T);
    const int C = p.C;
    const int unit = blockIdx.x / C;
    const int c = (MODE == kExpand) ? int(blockIdx.x % C) : int(cluster_ctarank());
    const int KS = p.K / C, DS = p.D / C;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const SmemLayout L = smem_layout(p, MODE, ES);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
    T* sA = reinterpret_cast<T*>(smem + L.a);
    T* sB = reinterpret_cast<T*>(smem + L.b);
    T* sX = reinterpret_cast<T*>(smem + L.x);
    float* sVp = reinterpret_cast<float*>(smem + L.vp);
    float* sV = reinterpret_cast<float*>(smem + L.v);

    const DevUnit U = p.units[unit];
    const T* pool = reinterpret_cast<const T*>(p.pool);
    const int64_t P = p.page_elems;

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    // ---------------- issue every page-slice copy of the unit (warp 0) ----
    if (warp == 0) {
        if (lane == 0) {
            uint32_t bytes_ax = 0, bytes_b = 0;
            for (int ii = 0; ii < U.n_items; ++ii) {
                const DevItem it = p.items[U.item_begin + ii];
                const DevSeg sg = p.segs[it.seg];
                const int proj = p.proj_ids[it.pi];
                if (MODE != kExpand) bytes_ax += uint32_t(sg.rank / p.a_div[proj] + it.nt) * KS * ES;
                if (MODE != kShrink) bytes_b += uint32_t(sg.rank) * DS * ES;
            }
            if (MODE != kExpand) mbar_arrive_expect_tx(&bar[0], bytes_ax);
            if (MODE != kShrink) mbar_arrive_expect_tx(&bar[1], bytes_b);
        }
        __syncwarp();
        for (int ii = 0; ii < U.n_items; ++ii) {
            const DevItem it = p.items[U.item_begin + ii];
            const DevSeg sg = p.segs[it.seg];
            const int proj = p.proj_ids[it.pi];
            const int32_t* tab = p.slot_tab[sg.slot] + int64_t((p.layer * 4 + proj) * 2) * sg.rank;
            if (MODE != kExpand) {
                const int rl = sg.rank / p.a_div[proj];
                const int rp = p.a_row_pages[proj];
                const int64_t k0 = int64_t(c) * KS;
                for (int j = lane; j < rl; j += 32) {
                    const int32_t page = tab[j * rp + int(k0 / P)];
                    bulk_g2s(sA + size_t(it.row_off + j) * KS, pool + page * P + (k0 % P), KS * ES, &bar[0]);
                }
                const T* x = reinterpret_cast<const T*>(p.x);
                for (int t = lane; t < it.nt; t += 32) {
                    const int32_t tok = p.tok_idx[sg.tok_off + it.t0 + t];
                    bulk_g2s(sX + size_t(it.tok_slot + t) * KS, x + tok * p.ldx + k0, KS * ES, &bar[0]);
                }
            }
            if (MODE != kShrink) {
                const int32_t* tabB = tab + sg.rank;
                const int64_t d0 = int64_t(c) * DS;
                for (int j = lane; j < sg.rank; j += 32) {
                    const int32_t page = tabB[j];
                    bulk_g2s(sB + size_t(it.row_off + j) * DS, pool + page * P + d0, DS * ES, &bar[1]);
                }
            }
        }
    }

    if (MODE != kExpand) {
        // ---------------- shrink: partial v over this CTA's K slice -------
        mbar_wait(&bar[0], 0);
        const int nvec = KS / VE;
        for (int ii = 0; ii < U.n_items; ++ii) {
            const DevItem it = p.items[U.item_begin + ii];
            const DevSeg sg = p.segs[it.seg];
            const int rl = sg.rank / p.a_div[p.proj_ids[it.pi]];
            for (int j = warp; j < rl; j += kThreads / 32) {
                const T* arow = sA + size_t(it.row_off + j) * KS;
                for (int t = 0; t < it.nt; ++t) {
                    const T* xrow = sX + size_t(it.tok_slot + t) * KS;
                    float acc = 0.f;
                    for (int q = lane; q < nvec; q += 32) {
                        float a[VE], xv[VE];
                        V::to_f32(reinterpret_cast<const uint4*>(arow)[q], a);
                        V::to_f32(reinterpret_cast<const uint4*>(xrow)[q], xv);
#pragma unroll
                        for (int e = 0; e < VE; ++e) acc = fmaf(xv[e], a[e], acc);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    if (lane == 0) sVp[it.v_off / p.a_div[p.proj_ids[it.pi]] + t * rl + j] = acc;
                }
            }
        }
        __syncthreads();
        // ---------------- combine the C partials (DSMEM) -----------------
        // entries of this unit in "local" units (rank / a_div per item)
        int E = 0;
        for (int ii = 0; ii < U.n_items; ++ii) {
            const DevItem it = p.items[U.item_begin + ii];
            E += it.nt * (p.segs[it.seg].rank / p.a_div[p.proj_ids[it.pi]]);
        }
        cluster_sync_all();  // every CTA's sVp is complete and visible
        const int per = (E + C - 1) / C;
        const int e0 = c * per, e1 = min(E, e0 + per);
        for (int e = e0 + tid; e < e1; e += kThreads) {
            const uint32_t a_local = smem_u32(sVp + e);
            float s = 0.f;
            for (int cc = 0; cc < C; ++cc) s += ld_dsmem(mapa_u32(a_local, cc));
            if (MODE == kFused) {
                const uint32_t v_local = smem_u32(sV + e);
                for (int cc = 0; cc < C; ++cc) st_dsmem(mapa_u32(v_local, cc), s);
            } else {
                // locate the item holding entry e, write v in the global layout
                int acc_e = 0;
                for (int ii = 0; ii < U.n_items; ++ii) {
                    const DevItem it = p.items[U.item_begin + ii];
                    const DevSeg sg = p.segs[it.seg];
                    const int div = p.a_div[p.proj_ids[it.pi]];
                    const int n_e = it.nt * (sg.rank / div);
                    if (e < acc_e + n_e) {
                        const int64_t base = int64_t(it.pi) * (p.NR / div) +
                                             (sg.vrow_off + int64_t(it.t0) * sg.rank) / div;
                        p.v_out[base + (e - acc_e)] = s;
                        break;
                    }
                    acc_e += n_e;
                }
            }
        }
        cluster_sync_all();  // all remote reads/writes done (also: safe exit)
    }

    if (MODE == kShrink) return;

    if (MODE == kExpand) {
        // v from global, block layout of slora_lora_expand
        const int vb = p.v_blocks;
        const int64_t stride = int64_t(p.nproj) * (p.NR / vb);
        for (int ii = 0; ii < U.n_items; ++ii) {
            const DevItem it = p.items[U.item_begin + ii];
            const DevSeg sg = p.segs[it.seg];
            const int r = sg.rank, rb = r / vb;
            const int n = it.nt * r;
            const int64_t base = int64_t(it.pi) * (p.NR / vb) + (sg.vrow_off + int64_t(it.t0) * r) / vb;
            for (int e = tid; e < n; e += kThreads) {
                const int t = e / r, j = e % r;
                sV[it.v_off + e] = p.v_in[int64_t(j / rb) * stride + base + int64_t(t) * rb + (j % rb)];
            }
        }
        __syncthreads();
    }

    // ---------------- expand: y += scale * v B over this CTA's D slice ----
    mbar_wait(&bar[1], 0);
    const int ncv = DS / VE;
    int task0 = 0;
    for (int ii = 0; ii < U.n_items; ++ii) {
        const DevItem it = p.items[U.item_begin + ii];
        const DevSeg sg = p.segs[it.seg];
        const int r = sg.rank;
        const int ntask = it.nt * ncv;
        const int proj = p.proj_ids[it.pi];
        T* y = reinterpret_cast<T*>(p.y[proj]);
        // threads continue numbering across items so all stay busy
        int first = (tid - task0) % kThreads;
        if (first < 0) first += kThreads;
        for (int task = first; task < ntask; task += kThreads) {
            const int t = task / ncv, cv = task % ncv;
            float acc[VE];
#pragma unroll
            for (int e = 0; e < VE; ++e) acc[e] = 0.f;
            const float* vrow = sV + it.v_off + t * r;
            for (int j = 0; j < r; ++j) {
                float b[VE];
                V::to_f32(reinterpret_cast<const uint4*>(sB + size_t(it.row_off + j) * DS)[cv], b);
                const float vj = vrow[j];
#pragma unroll
                for (int e = 0; e < VE; ++e) acc[e] = fmaf(vj, b[e], acc[e]);
            }
            const int32_t tok = p.tok_idx[sg.tok_off + it.t0 + t];
            uint4* yp = reinterpret_cast<uint4*>(y + tok * p.ldy[proj] + int64_t(c) * DS) + cv;
            float yv[VE];
            V::to_f32(*yp, yv);
#pragma unroll
            for (int e = 0; e < VE; ++e) yv[e] = yv[e] + sg.scale * acc[e];
            *yp = V::from_f32(yv);
        }
        task0 = (task0 + ntask) % kThreads;
    }
}

size_t lora_smem_bytes(const LoraParams& p, int mode, int esize) { return smem_layout(p, mode, esize).total; }

template <typename T, int MODE>
static cudaError_t launch_t(const LoraParams& p, cudaStream_t s, size_t smem) {
    auto kern = lora_unit_kernel<T, MODE>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(p.n_units) * unsigned(p.C));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (MODE != kExpand) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(p.C);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        na = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kern, p);
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
    if (p.n_units == 0) return cudaSuccess;
    switch (dtype) {
        case kF32: return launch_mode<float>(p, mode, s, smem);
        case kF16: return launch_mode<__half>(p, mode, s, smem);
        default: return launch_mode<__nv_bfloat16>(p, mode, s, smem);
    }
}

template <typename T>
static cudaError_t configure_t() {
    const int max_smem = 227 * 1024;
    cudaError_t e;
    e = cudaFuncSetAttribute(lora_unit_kernel<T, kFused>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
    if (e) return e;
    e = cudaFuncSetAttribute(lora_unit_kernel<T, kShrink>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
    if (e) return e;
    e = cudaFuncSetAttribute(lora_unit_kernel<T, kExpand>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
    if (e) return e;
    e = cudaFuncSetAttribute(lora_unit_kernel<T, kFused>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e) return e;
    return cudaFuncSetAttribute(lora_unit_kernel<T, kShrink>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

cudaError_t configure_lora_kernels(int /*device*/) {
    cudaError_t e = configure_t<float>();
    if (e) return e;
    e = configure_t<__half>();
    if (e) return e;
    return configure_t<__nv_bfloat16>();
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
