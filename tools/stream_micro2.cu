// stream_micro2.cu -- the C2 decode step's data movement alone: 32 layers x
// (q/k/v launch ~560 KB per SM, o launch ~190 KB per SM) of scattered page-row
// slices streamed into a shared-memory ring by NP producer warps (cp.async.bulk,
// 8 lanes per slot), consumed by 8 warps, captured in a CUDA graph with
// programmatic dependent launch (producers stream before griddepcontrol.wait,
// consumers wait first).  Prints the step time and GB/s for each variant.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_micro2 stream_micro2.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                 "l"(src), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ int page_of(uint32_t seed, uint32_t cta, uint32_t row, int npages) {
    uint32_t z = seed * 0x9E3779B9u ^ (cta * 0x85EBCA6Bu) ^ (row * 0xC2B2AE35u);
    z ^= z >> 16; z *= 0x7FEB352Du; z ^= z >> 15; z *= 0x846CA68Bu; z ^= z >> 16;
    return int(z % uint32_t(npages));
}
struct P {
    const unsigned char* pool; int seed; int npages; int nrows; int S; int page_bytes; int ns; int np; int C;
    float* sink; int pdl; int split;
};

__global__ void __launch_bounds__(512, 1) kern(P p) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = (uint64_t*)sm;
    uint64_t* empty = full + 32;
    unsigned char* ring = sm + 1024;
    const int SLOT = 8 * (p.S + 16);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t off = (size_t)(blockIdx.x % p.C) * p.S;
    if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.ns; ++s) { mbar_init(&full[s], p.split ? p.np : 1); mbar_init(&empty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nslots = p.nrows / 8;
    if (warp >= 8 && warp < 8 + p.np && p.split) {
        // every producer warp serves every slot: rows [pw*8/np, (pw+1)*8/np), one lane per row
        const int pw = warp - 8, rpw = 8 / p.np;
        int slot = 0; uint32_t lap = 0;
        for (int s = 0; s < nslots; ++s) {
            mbar_wait(&empty[slot], (lap & 1) ^ 1);
            unsigned char* dst = ring + (size_t)slot * SLOT;
            const int row = pw * rpw + lane;
            const int id = lane < rpw ? page_of(p.seed, blockIdx.x, s * 8 + row, p.npages) : 0;
            if (lane == 0) mbar_expect(&full[slot], rpw * p.S);
            __syncwarp();
            if (lane < rpw) bulk(dst + row * (p.S + 16), p.pool + (size_t)id * p.page_bytes + off, p.S, &full[slot]);
            if (++slot == p.ns) { slot = 0; ++lap; }
        }
    } else if (warp >= 8 && warp < 8 + p.np) {
        const int pw = warp - 8;
        int slot = pw, lap = 0;
        while (slot >= p.ns) { slot -= p.ns; ++lap; }
        for (int s = pw; s < nslots; s += p.np) {
            mbar_wait(&empty[slot], (lap & 1) ^ 1);
            unsigned char* dst = ring + (size_t)slot * SLOT;
            const int id = lane < 8 ? page_of(p.seed, blockIdx.x, s * 8 + lane, p.npages) : 0;
            if (lane == 0) mbar_expect(&full[slot], 8 * p.S);
            __syncwarp();
            if (lane < 8) bulk(dst + lane * (p.S + 16), p.pool + (size_t)id * p.page_bytes + off, p.S, &full[slot]);
            slot += p.np; while (slot >= p.ns) { slot -= p.ns; ++lap; }
        }
    } else if (warp < 8) {
        if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
        int slot = 0; uint32_t lap = 0;
        float acc = 0.f;
        for (int s = 0; s < nslots; ++s) {
            mbar_wait(&full[slot], lap & 1);
            const unsigned char* src = ring + (size_t)slot * SLOT + warp * (p.S + 16);
            for (int k = lane; k < p.S / 16; k += 32) acc += __uint_as_float(((const uint4*)src)[k].x);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == p.ns) { slot = 0; ++lap; }
        }
        if (acc == 1.2345f) p.sink[0] = acc;
    }
}

int main() {
    const size_t pool_bytes = size_t(8) << 30;
    const int page_bytes = 8192;
    const int npages = int(pool_bytes / page_bytes);
    unsigned char* pool; float* sink;
    CK(cudaMalloc(&pool, pool_bytes));
    CK(cudaMemset(pool, 1, pool_bytes));
    CK(cudaMalloc(&sink, 64));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    printf("S ring_kb np cps split  step_us  GB/s  (32 x [560KB, 190KB] per SM, pdl)\n");
    for (int S : {512, 1024, 2048})
      for (int ring_kb : {96, 192})
        for (int np : {1, 2, 4, 8})
          for (int cps : {1, 2})
            for (int split : {0, 1}) {
              const int pdl = 1;
              if (np == 1 && split) continue;
              if (np == 8 && !split) continue;
              if (cps == 2 && ring_kb > 100) continue;
              const int SLOT = 8 * (S + 16);
              const int ns = std::min(32, (ring_kb * 1024) / SLOT);
              if (ns < 2 || ns < np) continue;
              const size_t smem = 1024 + (size_t)ns * SLOT;
              const int grid = sms * cps;
              const int rows_qkv = (560 * 1024 / S) / cps / 8 * 8, rows_o = (190 * 1024 / S) / cps / 8 * 8;
              double bytes = 0;
              cudaGraph_t g; cudaGraphExec_t ge;
              CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
              for (int l = 0; l < 32; ++l)
                for (int c = 0; c < 2; ++c) {
                    P p{pool, 1 + 2 * l + c, npages, c ? rows_o : rows_qkv, S, page_bytes, ns, np, page_bytes / S, sink, pdl, split};
                    bytes += (double)grid * p.nrows * S;
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem; cfg.stream = st;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
                    CK(cudaLaunchKernelEx(&cfg, kern, p));
                }
              CK(cudaStreamEndCapture(st, &g));
              CK(cudaGraphInstantiate(&ge, g, 0));
              for (int it = 0; it < 3; ++it) CK(cudaGraphLaunch(ge, st));
              CK(cudaStreamSynchronize(st));
              const int reps = 10;
              cudaEventRecord(e0, st);
              for (int it = 0; it < reps; ++it) CK(cudaGraphLaunch(ge, st));
              cudaEventRecord(e1, st);
              CK(cudaEventSynchronize(e1));
              float ms; cudaEventElapsedTime(&ms, e0, e1);
              const double us = ms * 1e3 / reps;
              printf("%d %d %d %d %d %.1f %.1f\n", S, ring_kb, np, cps, split, us, bytes / us / 1e3);
              fflush(stdout);
              cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
            }
    return 0;
}
