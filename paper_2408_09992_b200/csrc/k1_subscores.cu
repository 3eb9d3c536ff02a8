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

// Register-blocked variant (UB >= 16 users per block, d/m % 4 == 0): thread
// (gp, uq) computes the 4 x 2 outputs (users 4 uq .. 4 uq + 3, sub-ids 2 gp,
// 2 gp + 1), each as four fp64 chains over t = j (mod 4) in ascending t --
// exactly K1's order (R5b), so S is bit-identical to the plain kernel's.  The
// tiles are staged transposed ([t][g] and [t][u], fp64), so one t costs one
// 128-bit psi load and two broadcast 128-bit phi loads for 8 fmas (the plain
// kernel: two 64-bit loads per fma; it was shared-memory bound).
constexpr int K1_BTT = 64;    // t-tile of the blocked kernel (one stage for d/m <= 64)

template <int K1_UB>
__global__ void __launch_bounds__(K1_THREADS)
k1_blocked(const float* __restrict__ phi, const float* __restrict__ psi, int B, int d,
           int m, int b, float* __restrict__ S) {
    constexpr int GCH = K1_MAXOUT / K1_UB;          // sub-ids per block (2 per thread column)
    constexpr int NGP = GCH / 2;
    extern __shared__ double k1_sm[];
    pdl_wait();                                     // phi / psi may come from the stream predecessor
    pdl_trigger();
    double* psT = k1_sm;                            // [K1_BTT][GCH]
    double* phT = k1_sm + (size_t)K1_BTT * GCH;     // [K1_BTT][K1_UB]
    const int k = blockIdx.x;
    const int u0 = blockIdx.y * K1_UB;
    const int nu = min(K1_UB, B - u0);
    const int dm = d / m;
    const int g0 = blockIdx.z * GCH;
    const int nb = min(GCH, b - g0);
    const int gp = threadIdx.x % NGP, uq = threadIdx.x / NGP;   // uq < K1_UB / 4
    double acc[4][2][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[u][g][c] = 0.0;
    for (int t0 = 0; t0 < dm; t0 += K1_BTT) {
        const int tt = min(K1_BTT, dm - t0);         // a multiple of 4
        __syncthreads();
        {   // psi_k rows g0 .. g0 + nb, columns t0 .. t0 + tt -> psT[t][g] (zero past nb), and
            // phi_k of the block's users -> phT[t][u]: every load of the stage is issued
            // before the first conversion (the staging is HBM-latency bound otherwise)
            const int q4 = tt / 4;
            constexpr int NPS = K1_BTT / 4 * GCH / K1_THREADS;      // psi float4 per thread (full stage)
            constexpr int NPH = K1_BTT / 4 * K1_UB / K1_THREADS;    // phi float4 per thread
            float4 v[NPS], f[NPH > 0 ? NPH : 1];
#pragma unroll
            for (int i = 0; i < NPS; ++i) {
                const int x = threadIdx.x + i * K1_THREADS, c = x / GCH, g = x - c * GCH;
                v[i] = (c < q4 && g < nb)
                           ? __ldg(reinterpret_cast<const float4*>(psi + ((int64_t)k * b + g0 + g) * dm + t0) + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < NPH; ++i) {
                const int x = threadIdx.x + i * K1_THREADS, u = x / (K1_BTT / 4), c = x - u * (K1_BTT / 4);
                f[i] = (c < q4 && u < nu)
                           ? __ldg(reinterpret_cast<const float4*>(phi + (int64_t)(u0 + u) * d + (int64_t)k * dm + t0) + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < NPS; ++i) {
                const int x = threadIdx.x + i * K1_THREADS, c = x / GCH, g = x - c * GCH;
                if (c < q4) {
                    psT[(4 * c + 0) * GCH + g] = (double)v[i].x;
                    psT[(4 * c + 1) * GCH + g] = (double)v[i].y;
                    psT[(4 * c + 2) * GCH + g] = (double)v[i].z;
                    psT[(4 * c + 3) * GCH + g] = (double)v[i].w;
                }
            }
#pragma unroll
            for (int i = 0; i < NPH; ++i) {
                const int x = threadIdx.x + i * K1_THREADS, u = x / (K1_BTT / 4), c = x - u * (K1_BTT / 4);
                if (c < q4) {
                    phT[(4 * c + 0) * K1_UB + u] = (double)f[i].x;
                    phT[(4 * c + 1) * K1_UB + u] = (double)f[i].y;
                    phT[(4 * c + 2) * K1_UB + u] = (double)f[i].z;
                    phT[(4 * c + 3) * K1_UB + u] = (double)f[i].w;
                }
            }
        }
        __syncthreads();
#pragma unroll 2
        for (int t = 0; t < tt; t += 4) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {               // t0 is a multiple of 4: chain = c
                const double2 p = *reinterpret_cast<const double2*>(psT + (t + c) * GCH + 2 * gp);
                const double2 f01 = *reinterpret_cast<const double2*>(phT + (t + c) * K1_UB + 4 * uq);
                const double2 f23 = *reinterpret_cast<const double2*>(phT + (t + c) * K1_UB + 4 * uq + 2);
                const double f[4] = {f01.x, f01.y, f23.x, f23.y};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc[u][0][c] = fma(p.x, f[u], acc[u][0][c]);
                    acc[u][1][c] = fma(p.y, f[u], acc[u][1][c]);
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int uu = 4 * uq + u, gg = 2 * gp + g;
            if (uu < nu && gg < nb)
                S[((int64_t)(u0 + uu) * m + k) * b + g0 + gg] =
                    (float)((acc[u][g][0] + acc[u][g][1]) + (acc[u][g][2] + acc[u][g][3]));   // one rounding
        }
}

template <int UB>
static void launch_k1_blocked(const float* phi, const float* psi, int B, int d, int m, int b, float* S,
                              cudaStream_t st) {
    constexpr int GCH = K1_MAXOUT / UB;
    const size_t smem = ((size_t)K1_BTT * GCH + (size_t)K1_BTT * UB) * sizeof(double);
    ensure_max_smem(reinterpret_cast<const void*>(k1_blocked<UB>), (int)smem);
    dim3 grid(m, (unsigned)ceil_div(B, UB), (unsigned)ceil_div(b, GCH));
    launch_pdl(k1_blocked<UB>, grid, dim3(K1_THREADS), smem, st, phi, psi, B, d, m, b, S);
    count_launch();
    check_launch("k1_blocked");
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
    static const bool plain = getenv("PQTOPK_K1_PLAIN") != nullptr;   // diagnostics (A/B)
    if (!plain && (d / m) % 4 == 0 && (ub == 32 || ub == 16)) {
        if (ub == 32) launch_k1_blocked<32>(phi, psi, B, d, m, b, S, st);
        else launch_k1_blocked<16>(phi, psi, B, d, m, b, S, st);
        return;
    }
    switch (ub) {
        case 32: launch_k1<32>(phi, psi, B, d, m, b, S, st); break;
        case 16: launch_k1<16>(phi, psi, B, d, m, b, S, st); break;
        case 8: launch_k1<8>(phi, psi, B, d, m, b, S, st); break;
        default: launch_k1<4>(phi, psi, B, d, m, b, S, st); break;
    }
}

}  // namespace pq
