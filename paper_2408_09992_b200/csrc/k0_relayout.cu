// K0 — code validation + relayout (pq_create; one-time, outside the hot path).
//
// Input : G [N][m] uint8 (Eq. 1), device.
// Output: rows of mp = round_up(m, 4) bytes (zero padding), so the scoring
//         kernel can fetch an item's codes with 4/8/16-byte vector loads.
// Also records the first (lowest linear index i*m+k) code with g >= b.
#include "pq_internal.cuh"

namespace pq {

__global__ void k0_relayout(const uint8_t* __restrict__ src, int64_t N, int m, int b,
                            uint8_t* __restrict__ dst, int mp,
                            unsigned long long* __restrict__ first_bad) {
    const int64_t total = N * (int64_t)mp;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = x / mp;
        int k = (int)(x - i * mp);
        uint8_t v = 0;
        if (k < m) {
            v = src[i * m + k];
            if (v >= b) atomicMin(first_bad, (unsigned long long)(i * m + k));
        }
        dst[x] = v;
    }
}

void launch_relayout(const uint8_t* src, int64_t N, int m, int b, uint8_t* dst, int mp,
                     unsigned long long* first_bad, cudaStream_t st) {
    int64_t total = N * (int64_t)mp;
    int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    if (blocks < 1) blocks = 1;
    k0_relayout<<<blocks, 256, 0, st>>>(src, N, m, b, dst, mp, first_bad);
    count_launch();
    check_launch("k0_relayout");
}

}  // namespace pq
