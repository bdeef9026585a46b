// Throughput of scalar FFMA vs packed FFMA2 (fma.rn.f32x2) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_bench ffma2_bench.cu && ./ffma2_bench
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int MODE>
__global__ void k(float *out, int iters, float x) {
    if (MODE == 0) {
        float a[8];
        for (int i = 0; i < 8; ++i) a[i] = x + i + threadIdx.x;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(x), "f"(1.0f));
        float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else {
        u64 a[8];
        u64 xx, one;
        asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
        asm("mov.b64 %0, {%1, %1};" : "=l"(one) : "f"(1.0f));
        for (int i = 0; i < 8; ++i) { float v = x + i + threadIdx.x; asm("mov.b64 %0, {%1, %1};" : "=l"(a[i]) : "f"(v)); }
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], xx, one);
        float s = 0;
        for (int i = 0; i < 8; ++i) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i])); s += lo + hi; }
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    }
}
int main() {
    float *out; cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    const int iters = 20000;
    for (int mode = 0; mode < 2; ++mode) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(out, iters, 0.999f); else k<1><<<148 * 8, 256>>>(out, iters, 0.999f);
            cudaEventRecord(b); cudaEventSynchronize(b);
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        double warp_instr = 148.0 * 8 * 8 /*warps per block*/ * iters * 8;
        double per_smsp_cycle = warp_instr / (148 * 4) / (ms * 1e-3 * 1.965e9);
        printf("mode %d (%s): %.3f ms, %.3f warp-instr/cycle/SMSP, %.1f TFLOP/s\n", mode, mode ? "FFMA2" : "FFMA", ms,
               per_smsp_cycle, warp_instr * 32 * (mode ? 4 : 2) / (ms * 1e-3) / 1e12);
    }
    return 0;
}
