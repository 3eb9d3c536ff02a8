// pairing.cu — host-side colour pairing of the catalogue rows for the
// 16-user K2 v3 layout, done once in pq_create (outside the hot path).
//
// 1. Per split k, 2-colour the b sub-ids, balancing the colours by how many
//    items use each sub-id (greedy, largest first, b/2 sub-ids per colour), and
//    renumber them: colour-0 sub-ids get even stored codes, colour-1 odd ones.
//    cmap[k][stored] = original sub-id (the tables are staged through it, so
//    the sums are the paper's sums of the ORIGINAL sub-id scores).
// 2. An item's signature is its colour bit at every split.  Items whose
//    signatures are bitwise complements are paired (A, B); leftovers are paired
//    in arbitrary order (they only lose conflict freedom, not correctness).
// 3. Rows 2p, 2p+1 hold pair p; perm[row] = local item id (-1 = padding).
//    codes16[row][k] = stored code * 64 (byte offset of the 16-user row inside
//    the split's table) for shared-memory splits, and the TMEM column
//    (stored code + 256 * t) for the last `tm` splits.
#include <vector>
#include <cstring>

#include "pq_internal.cuh"

namespace pq {

PairLayout build_pairing(const uint8_t* codes, int64_t N, int m, int b, int tm) {
    PairLayout L;
    L.tm = tm;
    L.cmap.assign((size_t)m * b, 0);
    L.pos.assign((size_t)m * b, 0);
    std::vector<uint8_t> color((size_t)m * 256, 0), stored((size_t)m * 256, 0);
    std::vector<int64_t> hist((size_t)m * 256, 0);
    for (int64_t i = 0; i < N; ++i)
        for (int k = 0; k < m; ++k) hist[(size_t)k * 256 + codes[i * m + k]]++;
    for (int k = 0; k < m; ++k) {
        std::vector<int> order(b);
        for (int g = 0; g < b; ++g) order[g] = g;
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
            return hist[(size_t)k * 256 + x] > hist[(size_t)k * 256 + y];
        });
        const int cap0 = (b + 1) / 2, cap1 = b / 2;
        int n0 = 0, n1 = 0;
        int64_t m0 = 0, m1 = 0;
        for (int g : order) {
            const int64_t w = hist[(size_t)k * 256 + g];
            int c = (n1 >= cap1) ? 0 : (n0 >= cap0) ? 1 : (m0 <= m1 ? 0 : 1);
            color[(size_t)k * 256 + g] = (uint8_t)c;
            const int pos = c == 0 ? 2 * n0++ : 2 * n1++ + 1;
            stored[(size_t)k * 256 + g] = (uint8_t)pos;
            L.cmap[(size_t)k * b + pos] = (uint8_t)g;
            L.pos[(size_t)k * b + g] = (uint8_t)pos;
            (c == 0 ? m0 : m1) += w;
        }
    }
    // Signatures cover the first sm = min(m, 20) splits: with m > 20 (e.g. 64)
    // exact complements of all splits are essentially absent, but pairs that are
    // complementary on 20 of them are plentiful and conflict-free on those splits
    // (about half of the others collide at random either way).
    const int sm = m < 20 ? m : 20;
    const uint32_t mask = (1u << sm) - 1u;
    std::vector<uint32_t> sig((size_t)N);
    for (int64_t i = 0; i < N; ++i) {
        uint32_t s = 0;
        for (int k = 0; k < sm; ++k) s |= (uint32_t)color[(size_t)k * 256 + codes[i * m + k]] << k;
        sig[i] = s;
    }
    // group item ids by signature (ids ascending inside a group)
    std::vector<int64_t> ids((size_t)N);
    std::vector<int64_t> start;
    std::vector<uint32_t> keys;        // distinct signatures, ascending
    if (sm <= 24) {
        const size_t nb = (size_t)1 << sm;
        std::vector<int64_t> cnt(nb + 1, 0);
        for (int64_t i = 0; i < N; ++i) cnt[sig[i] + 1]++;
        for (size_t s = 0; s < nb; ++s) cnt[s + 1] += cnt[s];
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (int64_t i = 0; i < N; ++i) ids[pos[sig[i]]++] = i;
        for (size_t s = 0; s < nb; ++s)
            if (cnt[s + 1] > cnt[s]) { keys.push_back((uint32_t)s); start.push_back(cnt[s]); }
        start.push_back(N);
    } else {
        for (int64_t i = 0; i < N; ++i) ids[i] = i;
        std::stable_sort(ids.begin(), ids.end(), [&](int64_t x, int64_t y) { return sig[x] < sig[y]; });
        for (int64_t i = 0; i < N; ++i)
            if (i == 0 || sig[ids[i]] != sig[ids[i - 1]]) { keys.push_back(sig[ids[i]]); start.push_back(i); }
        start.push_back(N);
    }
    std::vector<int64_t> A, Bv, left;
    A.reserve(N / 2 + 1); Bv.reserve(N / 2 + 1);
    for (size_t q = 0; q < keys.size(); ++q) {
        const uint32_t s = keys[q], c = s ^ mask;
        auto it = std::lower_bound(keys.begin(), keys.end(), c);
        const bool has_c = it != keys.end() && *it == c && c != s;
        if (has_c && c < s) continue;                     // pair handled from the smaller side
        int64_t na = start[q + 1] - start[q], nbb = 0, sb = 0;
        if (has_c) {
            size_t qb = (size_t)(it - keys.begin());
            sb = start[qb];
            nbb = start[qb + 1] - start[qb];
        }
        const int64_t np = std::min(na, nbb);
        for (int64_t t = 0; t < np; ++t) { A.push_back(ids[start[q] + t]); Bv.push_back(ids[sb + t]); }
        for (int64_t t = np; t < na; ++t) left.push_back(ids[start[q] + t]);
        for (int64_t t = np; t < nbb; ++t) left.push_back(ids[sb + t]);
    }
    L.matched_pairs = (int64_t)A.size();
    L.leftover = (int64_t)left.size();
    // Second pass over the leftovers: pair items whose signatures differ from
    // each other's complement in ONE split (those pairs conflict on one split
    // only instead of about m/2).  Greedy, in ascending signature order.
    if (sm <= 20 && !left.empty()) {
        const size_t nb = (size_t)1 << sm;
        std::vector<int64_t> head(nb, -1), nxt(left.size(), -1);
        for (size_t t = left.size(); t-- > 0;) {
            const uint32_t sg = sig[left[t]];
            nxt[t] = head[sg];
            head[sg] = (int64_t)t;
        }
        std::vector<uint8_t> used(left.size(), 0);
        std::vector<int64_t> rest;
        for (size_t t = 0; t < left.size(); ++t) {
            if (used[t]) continue;
            const uint32_t sg = sig[left[t]];
            int64_t mate = -1;
            for (int j = 0; j < sm && mate < 0; ++j) {
                const uint32_t c = (sg ^ mask) ^ (1u << j);
                int64_t& h = head[c];
                while (h >= 0 && used[h]) h = nxt[h];
                if (h >= 0 && (size_t)h != t) { mate = h; }
            }
            used[t] = 1;
            if (mate >= 0) {
                used[mate] = 1;
                A.push_back(left[t]);
                Bv.push_back(left[mate]);
            } else {
                rest.push_back(left[t]);
            }
        }
        left.swap(rest);
    }
    for (size_t t = 0; t + 1 < left.size(); t += 2) { A.push_back(left[t]); Bv.push_back(left[t + 1]); }
    if (left.size() % 2) { A.push_back(left.back()); Bv.push_back(-1); }
    const int64_t np = (int64_t)A.size();
    {   // every item exactly once (cheap one-time self-check)
        std::vector<uint8_t> seen((size_t)N, 0);
        for (int64_t p = 0; p < np; ++p)
            for (int64_t it : {A[p], Bv[p]})
                if (it >= 0) {
                    if (it >= N || seen[it]) fail(PQ_ERR_CUDA, "internal error: pairing is not a permutation");
                    seen[it] = 1;
                }
        for (int64_t i = 0; i < N; ++i)
            if (!seen[i]) fail(PQ_ERR_CUDA, "internal error: pairing dropped an item");
    }
    L.rows = 2 * np;
    L.perm.resize((size_t)L.rows);
    L.codes16.assign((size_t)L.rows * m, 0);
    const int ms = m - tm;
    for (int64_t p = 0; p < np; ++p) {
        for (int hh = 0; hh < 2; ++hh) {
            const int64_t it = hh ? Bv[p] : A[p];
            const int64_t row = 2 * p + hh;
            L.perm[row] = (int32_t)it;
            const int64_t src = it >= 0 ? it : A[p];        // padding row: any valid codes
            for (int k = 0; k < m; ++k) {
                const uint32_t c = stored[(size_t)k * 256 + codes[src * m + k]];
                L.codes16[(size_t)row * m + k] =
                    (uint16_t)(k < ms ? c * 64u : c + (uint32_t)b * (uint32_t)(k - ms));
            }
        }
    }
    return L;
}

}  // namespace pq
