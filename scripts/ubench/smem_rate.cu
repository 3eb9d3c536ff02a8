// Shared-memory gather-rate microbenchmark (calibrates K2's smem roofline on
// the box).  Not part of the product library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_rate smem_rate.cu
// Each CTA fills 64 KB..192 KB of shared memory, then every warp performs
// `iters` gathers with one of the access patterns and accumulates with FADD
// (so loads cannot be elided).  Reports bytes/clk/SM and 4-byte lookups/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode 0: LDS.32, lane = bank (row of 128 B per warp, random row)
// mode 1: LDS.128, quarter-warp reads one random 128-B row (R = 32 layout)
// mode 2: LDS.128, quarter-warp = two random 64-B rows in opposite bank halves (R = 16 paired)
// mode 3: LDS.64, half-warp = two random 64-B rows in opposite halves
// mode 4: like 2 but 4 independent chains per lane (more ILP)
template <int MODE>
__global__ void __launch_bounds__(1024, 1) kern(int iters, float* out, long long* cyc) {
    extern __shared__ __align__(16) float sm[];
    const int nwords = 48 * 1024;           // 192 KB
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) sm[i] = (float)(i & 1023);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t seed = hash32(threadIdx.x * 7919u + blockIdx.x);
    float4 acc = make_float4(0, 0, 0, 0);
    float4 acc2 = acc, acc3 = acc, acc4 = acc;
    const char* base = reinterpret_cast<const char*>(sm);
    // precomputed per-lane offsets (16 per lane) so the loop is LDS + FADD only
    uint32_t offs[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t h = hash32(seed ^ (uint32_t)j * 0x9E3779B9u);
        const uint32_t wq = __shfl_sync(0xffffffffu, h, lane & ~7);
        const uint32_t wh = __shfl_sync(0xffffffffu, h, lane & ~15);
        const uint32_t w0 = __shfl_sync(0xffffffffu, h, 0);
        if (MODE == 0) offs[j] = (w0 % 1536) * 128 + lane * 4;
        else if (MODE == 1) offs[j] = (wq % 1536) * 128 + (lane & 7) * 16;
        else if (MODE == 2 || MODE == 4) {
            const uint32_t r = (wq >> ((lane >> 2) & 1) * 11) % 1536;
            offs[j] = ((r & ~1u) | ((lane >> 2) & 1)) * 64 + (lane & 3) * 16;
        } else {
            const uint32_t r = (wh >> ((lane >> 3) & 1) * 11) % 1536;
            offs[j] = ((r & ~1u) | ((lane >> 3) & 1)) * 64 + (lane & 7) * 8;
        }
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t o = offs[j] ^ ((uint32_t)(it & 0x40) << 6);   // vary rows between rounds
            if (MODE == 0) {
                acc.x += *reinterpret_cast<const float*>(base + o);
            } else if (MODE == 1 || MODE == 2 || MODE == 4) {
                const float4 v = *reinterpret_cast<const float4*>(base + o);
                if (MODE == 4 && (j & 1)) { acc2.x += v.x; acc2.y += v.y; acc2.z += v.z; acc2.w += v.w; }
                else { acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
            } else {
                const float2 v = *reinterpret_cast<const float2*>(base + o);
                acc.x += v.x; acc.y += v.y;
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w + acc2.x + acc2.y + acc2.z + acc2.w + acc3.x + acc4.x;
}

template <int MODE>
void run(const char* name, int warps, int iters, int bytes_per_lane) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out; long long* cyc;
    cudaMalloc(&out, (size_t)nsm * 1024 * 4); cudaMalloc(&cyc, nsm * 8);
    cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
    kern<MODE><<<nsm, warps * 32, 192 * 1024>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h[256]; cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < nsm; ++i) mean += h[i]; mean /= nsm;
    const double loads = (double)warps * 32 * iters;
    const double bpc = loads * bytes_per_lane / mean;
    printf("%-34s warps=%2d  %.1f B/clk/SM  (%.1f lookups/clk/SM, %.0f%% of 128 B/clk)\n", name, warps, bpc,
           bpc / 4, bpc / 128 * 100);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {8, 16, 32}) {
        run<0>("LDS.32 conflict-free", w, 20000, 4);
        run<1>("LDS.128 128B row / quarter", w, 20000, 16);
        run<2>("LDS.128 paired 64B rows", w, 20000, 16);
        run<4>("LDS.128 paired, 2 chains", w, 10000, 16);
        run<3>("LDS.64 paired 64B rows", w, 20000, 8);
    }
    return 0;
}
