// k2_common.cuh — pieces shared by the K2 variants: arguments, the per-lane
// candidate-buffer flush and the end-of-unit CTA merge (see k2_score_select.cu
// for the selection scheme).
#pragma once
#include "select_dev.cuh"

namespace pq {

struct K2Args {
    const uint8_t* codes;      // v1: [N][mp] natural order
    const int32_t* perm;       // row -> local id (-1 = padding row), or null (item order)
    const float* S;            // [B][m][b]
    int64_t N;                 // items
    int m, b, mp;
    int B, K;
    uint32_t id_base;
    int Ug, n_groups, chunks;
    int64_t chunk_items;       // items per chunk
    uint64_t* lanebuf;         // [grid][W][32][cap]
    int cap;
    uint64_t* cand;            // [B][chunks][K]
    uint64_t* mscr;            // [grid][32 * W * K] end-of-unit merge scratch
};

// Shrinks every lane buffer holding more than `trigger` keys to its K best and
// raises the lane's threshold.  All 32 lanes call it.
__device__ __forceinline__ void warp_flush(uint64_t* wbuf, int cap, int& cnt, uint64_t& tau,
                                           float& tau_f, int K, int trigger, uint32_t* hist,
                                           unsigned long long* tau_user) {
    __syncwarp();
    unsigned need = __ballot_sync(FULL, cnt > trigger);
    const int lane = lane_id();
    while (need) {
        const int L = __ffs(need) - 1;
        need &= need - 1;
        const int n = __shfl_sync(FULL, cnt, L);
        uint64_t* buf = wbuf + (int64_t)L * cap;
        const uint64_t kth = warp_kth(buf, n, (uint32_t)K, hist);
        int pos = 0;
        for (int i0 = 0; i0 < n; i0 += 32) {
            int i = i0 + lane;
            uint64_t v = i < n ? buf[i] : 0ull;
            bool keep = (i < n) && (v >= kth);
            unsigned bm = __ballot_sync(FULL, keep);
            __syncwarp();
            if (keep) buf[pos + __popc(bm & lanemask_lt())] = v;
            pos += __popc(bm);
            __syncwarp();
        }
        if (lane == L) {
            cnt = pos;                       // == K (keys are unique)
            if (kth > tau) { tau = kth; tau_f = key_score(kth); }
            atomicMax(tau_user, (unsigned long long)kth);
        }
    }
    __syncwarp();
}

// End of a work unit (whole CTA; every lane has already shrunk its buffer to
// <= K keys, then __syncthreads).  For each user u of the group, only keys >=
// tau_sh[u] can be in the unit's top-K (some lane proved K keys >= it).
//  1. each lane counts its keys >= tau_sh[u] into ucnt[u] (smem atomics);
//  2. if a user's count is <= K they are the answer: lanes append them to
//     cand[user][chunk] directly; otherwise into the CTA's merge scratch;
//  3. one warp per over-full user radix-selects its K-th key in the scratch
//     and compacts the K best into cand; short lists are 0-padded.
// ucnt/ucur (smem, 32 ints each) must be zero on entry.
__device__ __forceinline__ void cta_merge(const K2Args& a, const uint64_t* mybuf, int cnt, bool active,
                                          int my_u, int Ug, int grp, int chunk,
                                          const unsigned long long* tau_sh, int* ucnt, int* ucur,
                                          uint64_t* mscr, int cap_u, uint32_t* whist) {
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint64_t th = active ? tau_sh[my_u] : ~0ull;
    int c = 0;
    if (active)
        for (int e = 0; e < cnt; ++e) c += (mybuf[e] >= th) ? 1 : 0;
    if (c) atomicAdd(&ucnt[my_u], c);
    __syncthreads();
    if (c) {
        const int tot = ucnt[my_u];
        const int gu = grp * Ug + my_u;
        uint64_t* dst = (tot <= a.K) ? a.cand + ((int64_t)gu * a.chunks + chunk) * a.K
                                     : mscr + (int64_t)my_u * cap_u;
        int o = atomicAdd(&ucur[my_u], c);
        for (int e = 0; e < cnt; ++e) {
            const uint64_t v = mybuf[e];
            if (v >= th) dst[o++] = v;
        }
    }
    __syncthreads();
    for (int uu = warp; uu < Ug; uu += W) {
        const int gu = grp * Ug + uu;
        if (gu >= a.B) continue;
        const int t = ucnt[uu];
        uint64_t* out = a.cand + ((int64_t)gu * a.chunks + chunk) * a.K;
        if (t > a.K) {
            const uint64_t* src = mscr + (int64_t)uu * cap_u;
            const uint64_t kth = warp_kth(src, t, (uint32_t)a.K, whist);
            int pos = 0;
            for (int i0 = 0; i0 < t; i0 += 32) {
                const int i = i0 + lane;
                const uint64_t v = i < t ? src[i] : 0ull;
                const bool keep = (i < t) && (v >= kth);
                const unsigned bm = __ballot_sync(FULL, keep);
                if (keep) out[pos + __popc(bm & lanemask_lt())] = v;
                pos += __popc(bm);
            }
        } else {
            for (int j = t + lane; j < a.K; j += 32) out[j] = 0ull;
        }
    }
}

}  // namespace pq
