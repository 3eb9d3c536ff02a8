// K4 — the paper's comparison paths.
//  * reconstruction of dense item embeddings (Eq. 2):
//      W[i][k*d/m + t] = psi[k][g_ik][t]
//    pure data movement (N*d*4 bytes written; HBM-bound);
//  * "Transformer Default" scoring r = W phi: a plain fp32 GEMM,
//    done by cuBLAS SGEMM with TF32 disabled (a library GEMM is the right tool
//    for the baseline; the product path is K2);
//  * RecJPQScore (Algorithm 2): split-major accumulation into an
//    N-length score array — one launch per split, in order k = 0..m-1.
#include <cublas_v2.h>
#include <mutex>

#include "pq_internal.cuh"

namespace pq {

// --------------------------------------------------------------------------- reconstruct
__global__ void k4_reconstruct(const uint8_t* __restrict__ codes, const int32_t* __restrict__ perm,
                               const uint8_t* __restrict__ cmap, int64_t rows, int m, int b,
                               int mp, const float* __restrict__ psi, int d,
                               float* __restrict__ W) {
    const int dm = d / m;
    const int64_t total = rows * (int64_t)m;
    for (int64_t x = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); x < total;
         x += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int64_t r = x / m;
        const int k = (int)(x - r * m);
        const int64_t item = perm ? perm[r] : r;
        if (item < 0) continue;                       // padding row
        int g = codes[r * mp + k];
        if (cmap) g = cmap[k * b + g];
        const float* src = psi + ((int64_t)k * b + g) * dm;
        float* dst = W + item * d + (int64_t)k * dm;
        for (int t = threadIdx.x & 31; t < dm; t += 32) dst[t] = src[t];
    }
}

void launch_reconstruct(const pq_index_s* idx, const float* psi, int d, float* W,
                        cudaStream_t st) {
    const int64_t rows = idx->lay.paired ? idx->n_rows : idx->N;
    int64_t warps = rows * idx->m;
    int blocks = (int)std::min<int64_t>(ceil_div(warps, 8), (int64_t)idx->num_sms * 32);
    if (blocks < 1) blocks = 1;
    k4_reconstruct<<<blocks, 256, 0, st>>>(idx->d_codes, idx->lay.paired ? idx->d_perm : nullptr,
                                           idx->lay.paired ? idx->d_cmap : nullptr, rows, idx->m,
                                           idx->b, idx->lay.mp, psi, d, W);
    count_launch();
    check_launch("k4_reconstruct");
}

// --------------------------------------------------------------------------- SGEMM
static std::mutex g_blas_mu;
static cublasHandle_t g_blas[64] = {};

void dense_sgemm(const float* W, int64_t Nc, int d, const float* phi, int B, float* R,
                 cudaStream_t st) {
    int dev = 0;
    PQ_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_blas_mu);
    if (!g_blas[dev]) {
        if (cublasCreate(&g_blas[dev]) != CUBLAS_STATUS_SUCCESS) fail(PQ_ERR_CUDA, "cublasCreate failed");
        // plain fp32 (no TF32 tensor-op math): the baseline computes in fp32
        cublasSetMathMode(g_blas[dev], CUBLAS_DEFAULT_MATH);
    }
    cublasSetStream(g_blas[dev], st);
    const float one = 1.0f, zero = 0.0f;
    // row-major R[B][Nc] = phi[B][d] * W[Nc][d]^T   <=>   col-major R^T = W^T(op) * phi^T
    cublasStatus_t s = cublasSgemm(g_blas[dev], CUBLAS_OP_T, CUBLAS_OP_N, (int)Nc, B, d, &one, W, d,
                                   phi, d, &zero, R, (int)Nc);
    if (s != CUBLAS_STATUS_SUCCESS) fail(PQ_ERR_CUDA, "cublasSgemm failed: status " + std::to_string((int)s));
}

// --------------------------------------------------------------------------- Alg. 2
// R[u][i] += S[u0+u][k][g_ik] for users u < Bc (split k of the sequential loop).
__global__ void k4_recjpq_split(const uint8_t* __restrict__ codes, const int32_t* __restrict__ perm,
                                const uint8_t* __restrict__ cmap, int64_t rows, int mp, int m, int b, int k,
                                const float* __restrict__ S, int u0, int Bc, int64_t N,
                                float* __restrict__ R) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t item = perm ? perm[r] : r;
        if (item < 0) continue;
        int g = codes[r * mp + k];
        if (cmap) g = cmap[k * b + g];
        for (int u = 0; u < Bc; ++u) {
            float* p = R + (int64_t)u * N + item;
            *p = *p + S[((int64_t)(u0 + u) * m + k) * b + g];
        }
    }
}

void launch_recjpq_split(const pq_index_s* idx, const float* S, int B, int u0, int Bc, int k,
                         float* R, cudaStream_t st) {
    (void)B;
    const int64_t rows = idx->lay.paired ? idx->n_rows : idx->N;
    int blocks = (int)std::min<int64_t>(ceil_div(rows, 256), (int64_t)idx->num_sms * 16);
    k4_recjpq_split<<<blocks, 256, 0, st>>>(idx->d_codes, idx->lay.paired ? idx->d_perm : nullptr,
                                            idx->lay.paired ? idx->d_cmap : nullptr,
                                            rows, idx->lay.mp, idx->m, idx->b, k, S, u0, Bc,
                                            idx->N, R);
    count_launch();
    check_launch("k4_recjpq_split");
}

}  // namespace pq
