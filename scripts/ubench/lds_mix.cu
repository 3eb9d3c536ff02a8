// Does a SHFL or an L1-hit LDG take shared-memory data-pipe cycles?  (K2 v3's
// code loads: four lanes of a quad fetch the same 8 bytes with LDG.64; moving
// one copy through shuffles only pays if SHFL runs on another path.)
// Not part of the product library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_mix lds_mix.cu
// Each of 16 warps per SM runs `iters` steps of 4 conflict-free LDS.128 (quarter
// warp = one 128-byte row, the R = 32 pattern) + EXTRA other instructions:
//   mode 0: nothing; 1: 2 SHFL (32-bit); 2: one LDG.64 (L1 hit, 4 lanes same
//   address); 3: one LDG.64 with distinct addresses; 4: 4 SHFL.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(int iters, const uint2* __restrict__ g, float* out, long long* cyc) {
    extern __shared__ __align__(16) float sm[];
    for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) sm[i] = (float)(i & 255);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t x = ((threadIdx.x >> 3) + 1) * 2654435761u + blockIdx.x;   // uniform per quarter warp
    float4 a0 = make_float4(0, 0, 0, 0), a1 = a0;
    uint32_t extra = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t rr = ((x >> (8 * k)) & 255u) ^ (uint32_t)k;    // same row per quarter warp
            const float4 v = *reinterpret_cast<const float4*>(reinterpret_cast<const char*>(sm) + rr * 128 + (lane & 7) * 16);
            if (k & 1) { a1.x += v.x; a1.y += v.y; a1.z += v.z; a1.w += v.w; }
            else { a0.x += v.x; a0.y += v.y; a0.z += v.z; a0.w += v.w; }
        }
        if (MODE == 1 || MODE == 4) {
            extra += __shfl_sync(0xffffffffu, extra + it, (lane + 1) & 31);
            extra += __shfl_sync(0xffffffffu, extra, (lane + 5) & 31);
        }
        if (MODE == 4) {
            extra += __shfl_sync(0xffffffffu, extra + it, (lane + 3) & 31);
            extra += __shfl_sync(0xffffffffu, extra, (lane + 7) & 31);
        }
        if (MODE == 2) { const uint2 c = __ldg(g + ((it * 8 + (lane >> 2)) & 4095)); extra += c.x ^ c.y; }
        if (MODE == 3) { const uint2 c = __ldg(g + ((it * 32 + lane) & 4095)); extra += c.x ^ c.y; }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0.x + a0.y + a1.z + a1.w + (float)extra;
}

template <int MODE>
static void run(const char* name, const uint2* g, float* out, long long* cyc) {
    const int iters = 20000;
    cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    kern<MODE><<<148, 512, 128 * 1024>>>(iters, g, out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double lds_wf = 16.0 * iters * 4 * 4;   // warps x iters x LDS.128 x 4 wavefronts
    printf("%-34s cycles %.0f  LDS.128 wavefronts per clock %.3f\n", name, m, lds_wf / m);
}

int main() {
    uint2* g; float* out; long long* cyc;
    cudaMalloc(&g, 4096 * 8); cudaMemset(g, 1, 4096 * 8);
    cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
    run<0>("LDS.128 only", g, out, cyc);
    run<1>("+ 2 SHFL per 4 LDS.128", g, out, cyc);
    run<4>("+ 4 SHFL per 4 LDS.128", g, out, cyc);
    run<2>("+ 1 LDG.64 (quad-shared) per 4", g, out, cyc);
    run<3>("+ 1 LDG.64 (distinct) per 4", g, out, cyc);
    return 0;
}
