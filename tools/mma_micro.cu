// mma_micro.cu -- legacy mma.sync (HMMA) throughput on sm_100a: each warp runs
// independent m16n8k16 / m16n8k8 f16 MMAs (4 accumulator chains); 8 warps per
// CTA, grid = 2 x SMs.  Prints MMAs per SM per cycle-equivalent (ns based).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int K>
__global__ void k(float* out, int iters) {
    float d[4][4] = {};
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (K == 16)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            else
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                             : "r"(a0), "r"(a1), "r"(b0));
        }
    }
    float s = 0;
    for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 1.2345f) out[0] = s;
}
int main() {
    float* o; cudaMalloc(&o, 64);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {4, 8, 16}) {
        const int iters = 4096;
        for (int kk : {16, 8}) {
            for (int r = 0; r < 2; ++r) {
                cudaEventRecord(e0);
                if (kk == 16) k<16><<<2 * sms, 32 * warps>>>(o, iters); else k<8><<<2 * sms, 32 * warps>>>(o, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double mmas = 2.0 * sms * warps * iters * 4;
            const double flop = mmas * 2 * 16 * 8 * kk;
            printf("m16n8k%d warps/CTA=%d (2 CTA/SM): %.3f ms  %.2f mma/ns/SM  %.1f TFLOP/s\n", kk, warps, ms,
                   mmas / (ms * 1e6) / sms, flop / (ms * 1e9));
        }
    }
    return 0;
}
