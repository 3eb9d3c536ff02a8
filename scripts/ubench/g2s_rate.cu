// Global -> shared copy-rate microbenchmark for the B <= 4 kernels' code stream
// (K7: each CTA copies its whole ~69 KB chunk at kernel start; K6: 16 KB
// stages).  Not part of the product library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o g2s_rate g2s_rate.cu
// Each of 148 CTAs copies `bytes` of its own slice of a buffer into shared
// memory with one method and records globaltimer before / after; optionally the
// buffer is made cold by writing a 256 MB scratch buffer first (the bench's L2
// flush).  Methods: 0 one bulk TMA copy per 32 KB piece on one mbarrier; 1 16 x
// 4 KB bulk pieces; 2 cp.async 16 B by every thread; 3 ld.global.v4 by every
// thread + st.shared.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int METHOD>
__global__ void __launch_bounds__(512, 1) kern(const unsigned char* src, uint32_t bytes, long long* t, int* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar;
    long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const unsigned char* s = src + (size_t)blockIdx.x * bytes;
    const uint32_t b0 = smem_u32(&bar);
    if (METHOD <= 1) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b0));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b0), "r"(bytes) : "memory");
            const uint32_t piece = METHOD == 0 ? 32768u : 4096u;
            for (uint32_t o = 0; o < bytes; o += piece)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             :: "r"(smem_u32(sm) + o), "l"(s + o), "r"(min(piece, bytes - o)), "r"(b0) : "memory");
        }
        __syncthreads();
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" :: "r"(b0) : "memory");
    } else if (METHOD == 2) {
        for (uint32_t o = 16u * threadIdx.x; o < bytes; o += 16u * blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(sm) + o), "l"(s + o) : "memory");
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    } else {
        uint4 v[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            const uint32_t o = 16u * (threadIdx.x + i * blockDim.x);
            if (o < bytes) v[i] = *reinterpret_cast<const uint4*>(s + o);
        }
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            const uint32_t o = 16u * (threadIdx.x + i * blockDim.x);
            if (o < bytes) *reinterpret_cast<uint4*>(sm + o) = v[i];
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) { t[2 * blockIdx.x] = t0; t[2 * blockIdx.x + 1] = t1; }
    if (threadIdx.x == 0 && sm[(blockIdx.x * 7) % bytes] == 255 && sm[1] == 254) atomicAdd(sink, 1);
}

template <int M>
static void run(const unsigned char* d, uint32_t bytes, long long* dt, int* sink, unsigned char* flush, bool cold,
                const char* name) {
    auto fn = kern<M>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    std::vector<double> spans, per;
    for (int rep = 0; rep < 12; ++rep) {
        if (cold) cudaMemset(flush, rep & 1, 256u << 20);
        else fn<<<148, 512, bytes, 0>>>(d, bytes, dt, sink);   // warm the slice in L2
        fn<<<148, 512, bytes, 0>>>(d, bytes, dt, sink);
        cudaDeviceSynchronize();
        std::vector<long long> h(296);
        cudaMemcpy(h.data(), dt, 296 * 8, cudaMemcpyDeviceToHost);
        long long mn = h[0], mx = 0;
        double s = 0;
        for (int i = 0; i < 148; ++i) { mn = std::min(mn, h[2 * i]); mx = std::max(mx, h[2 * i + 1]); s += h[2 * i + 1] - h[2 * i]; }
        if (rep >= 2) { spans.push_back((mx - mn) / 1e3); per.push_back(s / 148 / 1e3); }
    }
    std::sort(spans.begin(), spans.end());
    std::sort(per.begin(), per.end());
    printf("%-28s %s bytes/CTA %6u: span %.2f us (all CTAs), mean per-CTA %.2f us -> %.0f GB/s aggregate\n", name,
           cold ? "cold" : "warm", bytes, spans[spans.size() / 2], per[per.size() / 2],
           148.0 * bytes / (spans[spans.size() / 2] * 1e3));
}

int main() {
    unsigned char *d, *flush;
    long long* dt;
    int* sink;
    cudaMalloc(&d, 148u * 200 * 1024);
    cudaMemset(d, 1, 148u * 200 * 1024);
    cudaMalloc(&flush, 256u << 20);
    cudaMalloc(&dt, 296 * 8);
    cudaMalloc(&sink, 4);
    for (uint32_t bytes : {16384u, 69248u, 131072u})
        for (int cold = 0; cold < 2; ++cold) {
            run<0>(d, bytes, dt, sink, flush, cold, "TMA bulk, 32 KB pieces");
            run<1>(d, bytes, dt, sink, flush, cold, "TMA bulk, 4 KB pieces");
            run<2>(d, bytes, dt, sink, flush, cold, "cp.async 16 B x threads");
            if (bytes <= 512u * 16 * 9) run<3>(d, bytes, dt, sink, flush, cold, "ld.v4 + st.shared");
        }
    return 0;
}
