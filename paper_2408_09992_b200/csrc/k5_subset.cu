// K5 — item subsets (Alg. 1's input V: "V ⊆ I are the items to score")
// and per-user exclusion lists.
//
// Subset V (shared by the batch): the codes of V are gathered into a
// temporary item-order catalogue whose row r maps back to item V[r]; the
// regular fused scoring runs over it (ids through the row -> item map), so the
// result is exactly TopK over V ("subset consistency").  V is sorted
// ascending, so row order is id order and the (score desc, id asc) tie-break
// is unchanged (R3).
//
// Exclusions (e.g. items the user has already seen): the top-(K + E) of the
// full catalogue (E = the longest exclusion list of the batch) contains the
// top-K of I minus any E items, so the kernel below drops the excluded ids
// from each user's top-(K + E) list and keeps the first K: exact, no change
// to the scoring kernels.
#include "pq_internal.cuh"

namespace pq {

// (an entry of V outside [0, N) -- a caller error the asynchronous call does
// not detect -- is read as code 0: memory-safe)
__global__ void k5_gather_codes(const uint8_t* __restrict__ codes, int mp, int64_t N, const int32_t* __restrict__ V,
                                int64_t nV, uint8_t* __restrict__ out) {
    const int64_t total = nV * mp;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = x / mp;
        const int k = (int)(x - r * mp);
        const int32_t v = V[r];
        out[x] = (v >= 0 && v < N) ? codes[(int64_t)v * mp + k] : (uint8_t)0;
    }
}

__global__ void k5_fill_padding(int32_t* __restrict__ ids, float* __restrict__ scores, int64_t n) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        ids[x] = -1;
        scores[x] = -INFINITY;
    }
}

void launch_fill_padding(int32_t* ids, float* scores, int64_t n, cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(n, 256)), 148 * 8);
    k5_fill_padding<<<blocks, 256, 0, st>>>(ids, scores, n);
    count_launch();
    check_launch("k5_fill_padding");
}

__global__ void k5_check_subset(const int32_t* __restrict__ V, int64_t nV, int64_t N,
                                unsigned long long* __restrict__ first_bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nV;
         r += (int64_t)gridDim.x * blockDim.x) {
        const bool bad = V[r] < 0 || V[r] >= N || (r > 0 && V[r] <= V[r - 1]);
        if (bad) atomicMin(first_bad, (unsigned long long)r);
    }
}

void launch_gather_codes(const uint8_t* codes, int mp, int64_t N, const int32_t* V, int64_t nV, uint8_t* out,
                         cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(nV * mp, 256)), 148 * 16);
    k5_gather_codes<<<blocks, 256, 0, st>>>(codes, mp, N, V, nV, out);
    count_launch();
    check_launch("k5_gather_codes");
}

void launch_check_subset(const int32_t* V, int64_t nV, int64_t N, unsigned long long* first_bad,
                         cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(nV, 256)), 148 * 8);
    k5_check_subset<<<blocks, 256, 0, st>>>(V, nV, N, first_bad);
    count_launch();
    check_launch("k5_check_subset");
}

// One warp per user: drop the user's excluded ids (sorted list
// excl[off[u] .. off[u+1])) from its sorted top-K2 list and keep the first K.
__global__ void k5_exclude(const int32_t* __restrict__ ids2, const float* __restrict__ sc2, int B, int K2,
                           const int32_t* __restrict__ excl, const int64_t* __restrict__ off, int K,
                           int32_t* __restrict__ ids, float* __restrict__ scores) {
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (warp >= B) return;
    const int u = warp;
    const int64_t e0 = off[u], e1 = off[u + 1];
    int pos = 0;
    for (int j0 = 0; j0 < K2 && pos < K; j0 += 32) {
        const int j = j0 + lane;
        const int32_t id = j < K2 ? ids2[(int64_t)u * K2 + j] : -1;
        bool keep = j < K2 && id >= 0;
        if (keep) {                                   // binary search in the exclusion list
            int64_t lo = e0, hi = e1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (excl[mid] < id) lo = mid + 1; else hi = mid;
            }
            keep = !(lo < e1 && excl[lo] == id);
        }
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, keep);
        const int p = pos + __popc(bm & ((1u << lane) - 1u));
        if (keep && p < K) {
            ids[(int64_t)u * K + p] = id;
            scores[(int64_t)u * K + p] = sc2[(int64_t)u * K2 + j];
        }
        pos += __popc(bm);
    }
    for (int p = pos + lane; p < K; p += 32) {
        ids[(int64_t)u * K + p] = -1;
        scores[(int64_t)u * K + p] = -INFINITY;
    }
}

void launch_exclude(const int32_t* ids2, const float* sc2, int B, int K2, const int32_t* excl,
                    const int64_t* off, int K, int32_t* ids, float* scores, cudaStream_t st) {
    const int threads = 256;
    const int blocks = (int)ceil_div((int64_t)B * 32, threads);
    k5_exclude<<<blocks, threads, 0, st>>>(ids2, sc2, B, K2, excl, off, K, ids, scores);
    count_launch();
    check_launch("k5_exclude");
}

}  // namespace pq
