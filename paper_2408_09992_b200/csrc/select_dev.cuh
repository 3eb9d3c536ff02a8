// select_dev.cuh — device helpers for exact top-K selection on 64-bit keys
// (K2 lane-buffer flushes, K2 CTA merge, K3).  Radix select, 8 bits per pass,
// most significant digit first; keys are unique except the empty key 0.
#pragma once
#include "pq_internal.cuh"

namespace pq {

constexpr unsigned FULL = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Warp-aggregated histogram increment; all 32 lanes must call it.
__device__ __forceinline__ void hist_add(uint32_t* hist, bool ok, uint32_t digit) {
    unsigned d = ok ? digit : 0xFFFFFFFFu;
    unsigned peers = __match_any_sync(FULL, d);
    if (ok && lane_id() == (unsigned)(__ffs(peers) - 1)) atomicAdd(&hist[digit], __popc(peers));
}

// One full warp: given a 256-bin histogram of the keys that match the current
// prefix and krem >= 1 keys still to take (krem <= total), find the digit d*
// holding the krem-th largest key and the count of keys in higher bins.
__device__ __forceinline__ void warp_find_digit(const uint32_t* hist, uint32_t krem,
                                                uint32_t& digit, uint32_t& above_out) {
    const int lane = lane_id();
    const int base = 8 * (31 - lane);          // lane 0 owns the top bins
    uint32_t c[8], local = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { c[j] = hist[base + j]; local += c[j]; }
    uint32_t incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        uint32_t v = __shfl_up_sync(FULL, incl, off);
        if (lane >= off) incl += v;
    }
    uint32_t run = incl - local;               // keys in bins above my range
    int found = -1;
    uint32_t gt = 0;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
        if (found < 0 && run < krem && run + c[j] >= krem) { found = base + j; gt = run; }
        run += c[j];
    }
    unsigned bm = __ballot_sync(FULL, found >= 0);
    int src = bm ? __ffs(bm) - 1 : 0;
    digit = (uint32_t)__shfl_sync(FULL, found, src);
    above_out = __shfl_sync(FULL, gt, src);
}

// Warp-level: the K-th largest of keys buf[0..n) (global or shared), n >= K >= 1.
// hist: 256 words of shared memory private to this warp.  MSD radix select,
// 8 bits per pass; once the selected bin holds exactly the krem keys still to
// take, the K-th key is the smallest key of that bin (one min-reduction pass
// instead of the remaining digit passes).
__device__ __forceinline__ uint64_t warp_kth(const uint64_t* buf, int n, uint32_t K,
                                             uint32_t* hist) {
    uint64_t prefix = 0;
    uint32_t krem = K;
    const int lane = lane_id();
    for (int shift = 56; shift >= 0; shift -= 8) {
        const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
#pragma unroll
        for (int i = lane; i < 256; i += 32) hist[i] = 0;
        __syncwarp();
        constexpr int U = 4;                    // loads in flight per lane
        for (int i0 = 0; i0 < n; i0 += 32 * U) {
            uint64_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * 32 + lane;
                v[u] = i < n ? buf[i] : 0ull;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * 32 + lane;
                const bool ok = (i < n) && ((v[u] & hmask) == prefix);
                hist_add(hist, ok, (uint32_t)(v[u] >> shift) & 255u);
            }
        }
        __syncwarp();
        uint32_t dg, ab;
        warp_find_digit(hist, krem, dg, ab);
        const uint32_t inbin = hist[dg];
        prefix |= (uint64_t)dg << shift;
        krem -= ab;
        __syncwarp();
        if (shift > 0 && inbin == krem) {
            // the K-th key is the minimum of the keys carrying `prefix`
            const uint64_t pmask = ~0ull << shift;
            uint64_t mn = ~0ull;
            for (int i = lane; i < n; i += 32) {
                const uint64_t v = buf[i];
                if ((v & pmask) == prefix && v < mn) mn = v;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const uint64_t t = __shfl_xor_sync(FULL, mn, o);
                mn = t < mn ? t : mn;
            }
            return mn;
        }
    }
    return prefix;
}

// Block-level: the K-th largest of keys buf[0..n) in SHARED memory (n >= K >= 1),
// all threads of the block call it.  MSD radix select (8 bits per pass,
// warp-aggregated histogram increments, early exit as in warp_kth).  hist: 256
// words of shared memory; sc: 4 shared words of scratch.  Returns the key in
// every thread.
__device__ __forceinline__ uint64_t block_kth(const uint64_t* buf, int n, uint32_t K, uint32_t* hist,
                                              unsigned long long* sc) {
    uint64_t prefix = 0;
    uint32_t krem = K;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int shift = 56; shift >= 0; shift -= 8) {
        const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int i0 = 0; i0 < n; i0 += blockDim.x) {
            const int i = i0 + threadIdx.x;
            const uint64_t v = i < n ? buf[i] : 0ull;
            const bool ok = (i < n) && ((v & hmask) == prefix);
            hist_add(hist, ok, (uint32_t)(v >> shift) & 255u);
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t dg, ab;
            warp_find_digit(hist, krem, dg, ab);
            if (lane == 0) { sc[0] = dg; sc[1] = ab; sc[2] = hist[dg]; sc[3] = ~0ull; }
        }
        __syncthreads();
        const uint32_t dg = (uint32_t)sc[0], ab = (uint32_t)sc[1], inbin = (uint32_t)sc[2];
        prefix |= (uint64_t)dg << shift;
        krem -= ab;
        if (shift > 0 && inbin == krem) {        // the K-th is the smallest key of the bin
            const uint64_t pmask = ~0ull << shift;
            uint64_t mn = ~0ull;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const uint64_t v = buf[i];
                if ((v & pmask) == prefix && v < mn) mn = v;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const uint64_t t = __shfl_xor_sync(FULL, mn, o);
                mn = t < mn ? t : mn;
            }
            __syncthreads();                      // everyone has read sc[0..2]
            if (lane == 0) atomicMin(&sc[3], (unsigned long long)mn);
            __syncthreads();
            const uint64_t r = sc[3];
            __syncthreads();
            return r;
        }
        __syncthreads();                          // sc is rewritten by the next pass
    }
    return prefix;
}

// Rank of key buf[self] among buf[0..n) (shared memory, 16-byte aligned): keys
// above it, plus equal keys at a lower index (only repeated keys, which the
// callers' contracts forbid, tie -- the index keeps every output slot
// distinct).  Sixteen keys per step through eight independent 128-bit loads:
// the loop is load-latency bound otherwise.
__device__ __forceinline__ int rank_in_smem(const uint64_t* buf, int n, int self) {
    const uint64_t mine = buf[self];
    int r0 = 0, r1 = 0;
    int j = 0;
    for (; j + 16 <= n; j += 16) {
        ulonglong2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = *reinterpret_cast<const ulonglong2*>(buf + j + 2 * q);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            r0 += (v[q].x > mine || (v[q].x == mine && j + 2 * q < self)) ? 1 : 0;
            r1 += (v[q].y > mine || (v[q].y == mine && j + 2 * q + 1 < self)) ? 1 : 0;
        }
    }
    for (; j < n; ++j) r0 += (buf[j] > mine || (buf[j] == mine && j < self)) ? 1 : 0;
    return r0 + r1;
}

// Block-level bitonic sort (descending) of s[0..n), n a power of two.
__device__ __forceinline__ void block_bitonic_desc(uint64_t* s, int n) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
                int lo = 2 * stride * (i / stride) + (i % stride);
                int hi = lo + stride;
                bool desc = (lo & size) == 0;
                uint64_t a = s[lo], c = s[hi];
                if ((a < c) == desc) { s[lo] = c; s[hi] = a; }
            }
            __syncthreads();
        }
    }
}

__host__ __device__ __forceinline__ int pow2_ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace pq
