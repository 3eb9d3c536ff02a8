// K1 — sub-id score matrices (Eq. 4):
//   S[u][k][g] = sum_{t < d/m} psi[k][g][t] * phi[u][k*d/m + t]
// phi_k is the k-th contiguous chunk of phi.
//
// Precision (R5): fp32 x fp32 products are exact in fp64, so each
// dot product is accumulated in fp64 and rounded to fp32 once.  This meets the
// 1e-5 relative bound per entry (plain fp32 accumulation does not, near zero)
// and in practice reproduces fl32(exact) bit for bit.  Fixed fp64 order (R5b):
// four partial sums c_j over t = j, j+4, j+8, ... (t < d/m, ascending), then
// S = fl32((c_0 + c_1) + (c_2 + c_3)) -- a quarter of the dependent-add chain
// of a sequential sum; the fused small-batch kernel (k6_query.cu) uses the same
// order, so both produce identical S bits.
//
// Roofline: K1 does 2*B*b*d flops (C4: 0.27 GFLOP fp64) and writes B*m*b*4
// bytes (C4: 16.8 MB) — a few microseconds next to K2's tens of milliseconds,
// so it stays SIMT fp64 (TF32/BF16 tensor cores would break the tolerance; see
// DESIGN.md "K1").
//
// Grid: (m, ceil(B/UB), ceil(b/gchunk)); a block stages psi_k (gchunk x TT tile,
// padded rows) and phi_k for UB users in shared memory and produces the UB x
// gchunk outputs (gchunk = b, halved while the grid is short of two waves).
#include "pq_internal.cuh"

namespace pq {

constexpr int K1_UB = 4;      // users per block
constexpr int K1_TT = 32;     // t-tile (columns of psi_k staged per pass)
constexpr int K1_THREADS = 256;
constexpr int K1_PS = K1_TT + 1;   // padded row (doubles): 2 wavefronts per 64-bit warp load

// psi_k and phi_k tiles are staged in shared memory already converted to fp64
// (each float is converted once per block, not once per use), so the inner
// loop is fp64 fma on shared-memory operands only.
__global__ void __launch_bounds__(K1_THREADS)
k1_subscores(const float* __restrict__ phi, const float* __restrict__ psi, int B, int d,
             int m, int b, float* __restrict__ S, int gchunk) {
    extern __shared__ double k1_sm[];
    double* ps = k1_sm;                             // [gchunk][K1_PS]
    double* fs = k1_sm + (size_t)gchunk * K1_PS;    // [K1_UB][K1_TT]
    const int k = blockIdx.x;
    const int u0 = blockIdx.y * K1_UB;
    const int nu = min(K1_UB, B - u0);
    const int dm = d / m;
    const int g0 = blockIdx.z * gchunk;             // sub-ids [g0, g0 + nb) of split k
    const int nb = min(gchunk, b - g0);
    const int nout = nu * nb;
    constexpr int PER = (K1_UB * 256 + K1_THREADS - 1) / K1_THREADS;   // <= 4
    double acc[PER][4];
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;

    for (int t0 = 0; t0 < dm; t0 += K1_TT) {
        const int tt = min(K1_TT, dm - t0);
        __syncthreads();
        if (tt == K1_TT && (dm & 3) == 0) {
            // full tile, float4-aligned rows: all of a thread's loads are issued
            // before any conversion (the staging is latency-bound otherwise)
            constexpr int Q = K1_TT / 4;                // float4 per row
            const int total = nb * Q;
            for (int x0 = 0; x0 < total; x0 += 8 * K1_THREADS) {
                float4 v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int x = x0 + i * K1_THREADS + threadIdx.x;
                    if (x < total) {
                        const int g = x / Q, c = x - g * Q;
                        v[i] = __ldg(reinterpret_cast<const float4*>(psi + ((int64_t)k * b + g0 + g) * dm + t0) + c);
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int x = x0 + i * K1_THREADS + threadIdx.x;
                    if (x < total) {
                        const int g = x / Q, c = x - g * Q;
                        double* d = ps + g * K1_PS + 4 * c;
                        d[0] = (double)v[i].x; d[1] = (double)v[i].y; d[2] = (double)v[i].z; d[3] = (double)v[i].w;
                    }
                }
            }
        } else {
            for (int x = threadIdx.x; x < nb * tt; x += K1_THREADS) {
                int g = x / tt, t = x - g * tt;
                ps[g * K1_PS + t] = (double)psi[((int64_t)k * b + g0 + g) * dm + t0 + t];
            }
        }
        for (int x = threadIdx.x; x < nu * tt; x += K1_THREADS) {
            int u = x / tt, t = x - u * tt;
            fs[u * K1_TT + t] = (double)phi[(int64_t)(u0 + u) * d + (int64_t)k * dm + t0 + t];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            int o = threadIdx.x + j * K1_THREADS;
            if (o < nout) {
                int u = o / nb, g = o - u * nb;
                const double* pr = ps + g * K1_PS;
                const double* fr = fs + u * K1_TT;
                double a0 = acc[j][0], a1 = acc[j][1], a2 = acc[j][2], a3 = acc[j][3];
                int t = 0;                              // t0 is a multiple of 4: chain = t & 3
                for (; t + 4 <= tt; t += 4) {           // exact products, fp64 sums
                    a0 = fma(pr[t], fr[t], a0);
                    a1 = fma(pr[t + 1], fr[t + 1], a1);
                    a2 = fma(pr[t + 2], fr[t + 2], a2);
                    a3 = fma(pr[t + 3], fr[t + 3], a3);
                }
                if (t < tt) a0 = fma(pr[t], fr[t], a0);
                if (t + 1 < tt) a1 = fma(pr[t + 1], fr[t + 1], a1);
                if (t + 2 < tt) a2 = fma(pr[t + 2], fr[t + 2], a2);
                acc[j][0] = a0; acc[j][1] = a1; acc[j][2] = a2; acc[j][3] = a3;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        int o = threadIdx.x + j * K1_THREADS;
        if (o < nout) {
            int u = o / nb, g = o - u * nb;
            S[((int64_t)(u0 + u) * m + k) * b + g0 + g] =
                (float)((acc[j][0] + acc[j][1]) + (acc[j][2] + acc[j][3]));   // one rounding (RN)
        }
    }
}

void launch_subscores(const float* phi, const float* psi, int B, int d, int m, int b,
                      float* S, cudaStream_t st) {
    if (B <= 0) return;
    // split the sub-ids over blocks while the grid is short of two waves
    int gchunk = b;
    while (gchunk > 32 && (int64_t)m * ceil_div(B, K1_UB) * ceil_div(b, gchunk) < 2 * 148) gchunk = (gchunk + 1) / 2;
    const size_t smem = ((size_t)gchunk * K1_PS + K1_UB * K1_TT) * sizeof(double);
    static std::atomic<uint64_t> attr_set{0};       // per device (bit = ordinal)
    int dev = 0;
    PQ_CUDA(cudaGetDevice(&dev));
    if (dev >= 64 || !(attr_set.load() >> dev & 1)) {   // gchunk <= 256: at most 68.6 KB
        PQ_CUDA(cudaFuncSetAttribute(k1_subscores, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)((256 * K1_PS + K1_UB * K1_TT) * sizeof(double))));
        if (dev < 64) attr_set.fetch_or(1ull << dev);
    }
    dim3 grid(m, (unsigned)ceil_div(B, K1_UB), (unsigned)ceil_div(b, gchunk));
    k1_subscores<<<grid, K1_THREADS, smem, st>>>(phi, psi, B, d, m, b, S, gchunk);
    count_launch();
    check_launch("k1_subscores");
}

}  // namespace pq
