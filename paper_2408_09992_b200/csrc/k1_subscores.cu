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
// gchunk outputs (UB x gchunk <= 2048: up to 8 per thread).  UB = 32 users per
// block for batches (each staged psi tile then serves 32 users instead of 4:
// C2 K1 18 -> see DESIGN.md), fewer for small B; gchunk is halved while the
// grid is short of two waves.
#include <cstdlib>

#include "pq_internal.cuh"
#include "ptx_dev.cuh"

namespace pq {

constexpr int K1_TT = 32;     // t-tile (columns of psi_k staged per pass)
constexpr int K1_MAXOUT = 2048;   // outputs per block (UB x gchunk)
constexpr int K1_THREADS = 256;
constexpr int K1_PS = K1_TT + 1;   // padded row (doubles): 2 wavefronts per 64-bit warp load

// psi_k and phi_k tiles are staged in shared memory already converted to fp64
// (each float is converted once per block, not once per use), so the inner
// loop is fp64 fma on shared-memory operands only.
template <int K1_UB>
__global__ void __launch_bounds__(K1_THREADS)
k1_subscores(const float* __restrict__ phi, const float* __restrict__ psi, int B, int d,
             int m, int b, float* __restrict__ S, int gchunk) {
    extern __shared__ double k1_sm[];
    pdl_wait();                                     // phi / psi may come from the stream predecessor
    pdl_trigger();                                  // the next kernel (tiled tables) may be scheduled
    double* ps = k1_sm;                             // [gchunk][K1_PS]
    double* fs = k1_sm + (size_t)gchunk * K1_PS;    // [K1_UB][K1_TT]
    const int k = blockIdx.x;
    const int u0 = blockIdx.y * K1_UB;
    const int nu = min(K1_UB, B - u0);
    const int dm = d / m;
    const int g0 = blockIdx.z * gchunk;             // sub-ids [g0, g0 + nb) of split k
    const int nb = min(gchunk, b - g0);
    const int nout = nu * nb;
    constexpr int PER = K1_MAXOUT / K1_THREADS;       // outputs per thread (nout <= 2048)
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

template <int UB>
static void launch_k1(const float* phi, const float* psi, int B, int d, int m, int b, float* S,
                      cudaStream_t st) {
    // split the sub-ids over blocks while the grid is short of two waves
    int gchunk = std::min(b, K1_MAXOUT / UB);
    while (gchunk > 32 && (int64_t)m * ceil_div(B, UB) * ceil_div(b, gchunk) < 2 * 148) gchunk = (gchunk + 1) / 2;
    const size_t smem = ((size_t)gchunk * K1_PS + UB * K1_TT) * sizeof(double);
    // gchunk <= 256: at most 256 * 33 * 8 + 32 * 32 * 8 = 75.8 KB (once per device and kernel)
    ensure_max_smem(reinterpret_cast<const void*>(k1_subscores<UB>),
                    (int)((std::min(256, K1_MAXOUT / UB) * K1_PS + UB * K1_TT) * sizeof(double)));
    dim3 grid(m, (unsigned)ceil_div(B, UB), (unsigned)ceil_div(b, gchunk));
    launch_pdl(k1_subscores<UB>, grid, dim3(K1_THREADS), smem, st, phi, psi, B, d, m, b, S, gchunk);
    count_launch();
    check_launch("k1_subscores");
}

void launch_subscores(const float* phi, const float* psi, int B, int d, int m, int b,
                      float* S, cudaStream_t st) {
    if (B <= 0) return;
    // users per block: 32 for batches (a staged psi tile serves 32 users), fewer
    // for small B; PQTOPK_K1_UB forces one (diagnostics A/B)
    static const int forced = [] { const char* e = getenv("PQTOPK_K1_UB"); return e ? atoi(e) : 0; }();
    // (measured, r02: C2 B = 128: 32 -> 14.8 us vs 16.8 at 4-16; C3 / C4: 16 best, 25 / 72 us)
    const int ub = forced ? forced : (B > 128 ? 16 : B >= 32 ? 32 : B >= 16 ? 16 : B >= 8 ? 8 : 4);
    switch (ub) {
        case 32: launch_k1<32>(phi, psi, B, d, m, b, S, st); break;
        case 16: launch_k1<16>(phi, psi, B, d, m, b, S, st); break;
        case 8: launch_k1<8>(phi, psi, B, d, m, b, S, st); break;
        default: launch_k1<4>(phi, psi, B, d, m, b, S, st); break;
    }
}

}  // namespace pq
