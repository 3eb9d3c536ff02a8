// pq_internal.cuh — internals shared by the libpqtopk translation units.
// (Product path only; the CPU oracle under oracle/ shares nothing with this.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <string>
#include <atomic>
#include <algorithm>
#include <mutex>
#include <vector>

#include "../../include/pqtopk.h"

namespace pq {

// ----------------------------------------------------------------------------
// Error plumbing: every ABI entry point catches and converts to pq_status.
// ----------------------------------------------------------------------------
struct Error {
    pq_status st;
    std::string msg;
};
void set_error(const std::string& msg);
void clear_error();
[[noreturn]] void fail(pq_status st, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
void check_launch(const char* what);        // cudaGetLastError after a launch
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size):
// the plans run on every call and the attribute call is host time on small queries
void ensure_max_smem(const void* fn, int bytes);
extern std::atomic<int64_t> g_launches;     // kernels launched by this library
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define PQ_CUDA(x) ::pq::check_cuda((x), #x)

// Launch with programmatic stream serialization (PDL): only for kernels that
// call pdl_wait() (ptx_dev.cuh) before touching memory a predecessor writes.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, fn, static_cast<KArgs>(args)...), "cudaLaunchKernelEx (PDL)");
}

// ----------------------------------------------------------------------------
// Checked builds (python -m paper_2408_09992_b200.build --checked ->
// libpqtopk_checked.so, -DPQTOPK_CHECKED): device-side bounds / invariant
// checks and bounded spin-waits (PQ_SPIN_LIMIT polls) that report the failing
// site and trap instead of corrupting memory or hanging.  This stands in for
// compute-sanitizer, which this GPU pool does not allow.  Product builds
// compile every check away.
// ----------------------------------------------------------------------------
#ifdef PQTOPK_CHECKED
#define PQ_DCHECK(cond)                                                                      \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("PQ_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,  \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
constexpr long long PQ_SPIN_LIMIT = 1ll << 27;
#define PQ_SPIN_CHECK(counter) PQ_DCHECK(++(counter) < ::pq::PQ_SPIN_LIMIT)
#else
#define PQ_DCHECK(cond) do { } while (0)
#define PQ_SPIN_CHECK(counter) do { } while (0)
#endif

// ----------------------------------------------------------------------------
// Ranking key (reading R3): 64-bit unsigned, larger = ranks earlier.
//   high 32 bits: order-preserving image of the fp32 score bits
//   low  32 bits: 0xFFFFFFFF - global id   (smaller id ranks earlier on ties)
// Key 0 is never produced by a real (score, id) pair and marks "empty".
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t make_key(float s, uint32_t gid) {
    uint32_t u = __float_as_uint(s);
    uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((uint64_t)o << 32) | (uint64_t)(0xFFFFFFFFu - gid);
}
__device__ __forceinline__ float key_score(uint64_t k) {
    uint32_t o = (uint32_t)(k >> 32);
    uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
    return __uint_as_float(u);
}
__device__ __forceinline__ int32_t key_id(uint64_t k) {
    return (int32_t)(0xFFFFFFFFu - (uint32_t)k);
}

// ----------------------------------------------------------------------------
// Index
// ----------------------------------------------------------------------------
struct Layout {
    int32_t mp;            // bytes per item row in d_codes (m rounded up to 4)
    int32_t paired;        // 1: rows are in pair order (see k0), d_perm valid
};

// Colour-paired catalogue rows (pairing.cu), built on the host in pq_create
// for the 16-user K2 v3 layout.
struct PairLayout {
    std::vector<uint16_t> codes16;   // [rows][m]
    std::vector<int32_t> perm;       // [rows]
    std::vector<uint8_t> cmap;       // [m][b] stored -> original
    std::vector<uint8_t> pos;        // [m][b] original -> stored
    int64_t rows = 0, matched_pairs = 0, leftover = 0;
    int tm = 0;
};
PairLayout build_pairing(const uint8_t* codes, int64_t N, int m, int b, int tm);

}  // namespace pq

struct pq_index_s {
    int64_t N = 0;
    int32_t m = 0, b = 0;
    int64_t id_base = 0;
    int device = 0;
    int num_sms = 0;
    size_t smem_optin = 0;
    pq::Layout lay{};
    uint8_t* d_codes = nullptr;    // [N_rows][mp] internal code rows (+ tail pad)
    int32_t* d_perm = nullptr;     // row -> local item id (only if lay.paired)
    uint8_t* d_cmap = nullptr;     // [m][b] stored code -> original code (paired)
    int64_t n_rows = 0;            // rows in d_codes (>= N when paired, padded)
    // K2 v3 ("tiled phases") layout; v3_ok = 0 when not eligible
    int v3_ok = 0;
    int v3_R = 0;                  // users per table row (16: paired layout, 32: item order)
    int64_t v3_tiles = 0;          // tiles of k2_tiled_rows_per_tile(v3_R) rows
    int64_t v3_code_bytes = 0;     // allocated bytes of d_codes3 (incl. V3_CODE_PAD)
    int64_t v3_matched = 0, v3_leftover = 0;
    void* d_codes3 = nullptr;      // [tiles][NP][TR][PS] stored codes, k2_tiled_code_bytes() each (+ pad)
    int32_t* d_perm3 = nullptr;    // [tiles * 4096] row -> local id (-1 = padding)
    uint8_t* d_cmap3 = nullptr;    // [m][b] stored -> original
    // colour-paired ROW-ORDER codes for the small-batch kernels K6 / K7 (built
    // with the R = 16 v3 layout): row r = item d_perm3[r] in stored codes
    // (parity = colour), rows 2p / 2p + 1 complementary; rows < p_rows are all
    // real items (d_codes_p == null: not built)
    uint8_t* d_codes_p = nullptr;
    int64_t p_rows = 0;
    pq_tuning tuning{};
    void* k6_cache = nullptr;      // K6 launch plans by (B, d, K, tuning) (k6_query.cu)
    // optional K2/K3 timing (pq_timing_enable)
    int timing = 0;
    struct EvTriple { cudaEvent_t a, b, c; };
    std::vector<EvTriple>* events = nullptr;
    std::mutex* ev_mu = nullptr;   // guards `events` (calls may come from several threads)
};

namespace pq {

// ---- kernels / launchers implemented in the .cu files ----------------------
// K0 (k0_relayout.cu)
void launch_relayout(const uint8_t* src, int64_t N, int m, int b, uint8_t* dst, int mp,
                     unsigned long long* first_bad, cudaStream_t st);

// K1 (k1_subscores.cu)
void launch_subscores(const float* phi, const float* psi, int B, int d, int m, int b,
                      float* S, cudaStream_t st);

// K2 (k2_score_select.cu)
constexpr int K2_MAX_CUT = 160;   // balanced partition: at most this many CTAs
struct K2Plan {
    int G = 0, Ug = 0, W = 0, J = 0, cap = 0;
    int n_groups = 0, chunks = 0, grid = 0;
    int64_t chunk_items = 0;
    size_t smem = 0;
    size_t lanebuf_bytes = 0;     // grid * W * 32 * cap * 8
    size_t cand_bytes = 0;        // B * chunks * K * 8
    size_t mscr_bytes = 0;        // grid * 32 * W * K * 8 (end-of-unit merge scratch)
    int variant = 1;
    int tm = 0;
    size_t st_bytes = 0;          // v3: tiled S tables [n_groups][m][b][16] fp32 + thresholds, union floors, list counts
    bool qk = false;              // v3: union floors (large K, single-phase tables)
    // v3 balanced partition (single-phase tables): CTA x scores the (group, tile) pairs
    // [cut[x], cut[x + 1]) of the group-major sequence g * n_tiles + t; 0 = legacy units
    int n_cut = 0;
    int32_t cut[K2_MAX_CUT + 1] = {};
};
// K6 (k6_query.cu): the fused single-launch query kernel for B <= 4
struct K6Plan {
    int G = 0, nst = 0, CL = 0, chunks = 0, grid = 0;
    int gridsync = 0;             // 1: cooperative grid mode (S shared through L2), else clusters of CL
    int resident = 0;             // 1: K7 (k7_resident.cu): each CTA's code chunk resident in smem
    int cl = 0;                   // K7 cluster mode: one cluster of cl CTAs per user (no global exchange)
    int paired = 0;               // 1: the colour-paired row-order codes (idx->d_codes_p) with 16 table copies
    int64_t chunk_items = 0;
    size_t smem = 0, cand_bytes = 0;
};
bool k6_query_plan(pq_index_s* idx, int B, int d, int K, K6Plan& p);   // cached per index
void k6_cache_free(pq_index_s* idx);
size_t k6_query_ws_bytes(const K6Plan& p, int B, int E);
// K7 (k7_resident.cu): the chunk-resident single-launch query kernel (B <= 4, small catalogues)
bool k7_resident_plan(const pq_index_s* idx, int B, int d, int K, K6Plan& p);
size_t k7_resident_ws_bytes(const K6Plan& p, int B, int E);
void launch_k7_resident(const pq_index_s* idx, const K6Plan& p, const float* phi, const float* psi, int B,
                        int d, int K, void* ws, float* S_out, int32_t* ids, float* scores, cudaStream_t st);
void launch_k6_query(const pq_index_s* idx, const K6Plan& p, const float* phi, const float* psi, int B,
                     int d, int K, void* ws, float* S_out, int32_t* ids, float* scores, cudaStream_t st);
// v4 helpers (k2_latency.cu): small batches (B <= 4), lane = item
bool k2_latency_supported(const pq_index_s* idx, int B, int K);
void plan_k2_latency(const pq_index_s* idx, int B, int K, K2Plan& p);
void launch_k2_latency(const pq_index_s* idx, const K2Plan& p, const float* S, int B, int K,
                       uint64_t* cand, cudaStream_t st);
// v3 helpers (k2_tiled.cu)
// K2 v3 kernel shape for a catalogue: R users per table row (0 = unsupported),
// m_v "virtual" splits (m - 1 with an exact first-pair table), ps splits per
// phase, pss stored codes per row per phase, bt / bt0 table rows (split 0: bt0)
struct TiledShape { int R = 0, pair = 0, m_v = 0, ps = 0, pss = 0, bt = 0, bt0 = 0; };
TiledShape k2_tiled_shape(int m, int b);
size_t k2_tiled_smem(const TiledShape& t, int W);
// the K2 v3 catalogue layout built on the GPU from d_codes (k0_layout.cu)
void build_v3_layout_gpu(pq_index_s* idx, cudaStream_t st);
bool k2_tiled_supported(int m, int b);
int k2_tiled_users(int m, int b);
int k2_tiled_code_bytes();
int k2_tiled_ps(int m);
int k2_tiled_rows_per_tile(int R);
constexpr int V3_CODE_PAD = 4096;     // bytes after the last tile (prefetch overhang)
void plan_k2_tiled(const pq_index_s* idx, int B, int K, K2Plan& p);
void launch_k2_tiled_prep(const pq_index_s* idx, const K2Plan& p, const float* S, int B, float* St,
                          cudaStream_t st);
void launch_k2_tiled(const pq_index_s* idx, const K2Plan& p, int B, int K,
                     uint64_t* lanebuf, uint64_t* mscr, const float* St, uint64_t* cand, cudaStream_t st);
// v3 writes each unit's list unpadded: entries per (user, chunk) list, [n_groups R][chunks]
const int32_t* k2_tiled_list_counts(const pq_index_s* idx, const K2Plan& p, const float* St);
K2Plan plan_k2(const pq_index_s* idx, int B, int K);
void launch_k2(const pq_index_s* idx, const K2Plan& p, const float* S, int B, int K,
               uint64_t* lanebuf, uint64_t* cand, cudaStream_t st);

// K3 (k3_select.cu): segmented exact top-K
constexpr int K3_SEG = 8192;           // keys per K3 block (smem-resident; 2 blocks per SM; >= 2 PQTOPK_MAX_K so every merge level halves the list)
size_t k3_reduce_scratch_bytes(int64_t L, int B, int K);
// keys [B][L] -> ids/scores [B][K] (sorted), multi-level; scratch from above
// lcnt (optional): keys[u] is lists of K keys of which lcnt[u * L / K + p] are valid (the rest unwritten)
void k3_keys_to_topk(const uint64_t* keys, int64_t L, int B, int K, void* scratch,
                     int32_t* ids, float* scores, cudaStream_t st, const int32_t* lcnt = nullptr);
// pairs [P][B][K] -> ids/scores [B][K]
size_t k3_pairs_scratch_bytes(int P, int B, int K);
void k3_pairs_to_topk(const int32_t* ids_in, const float* sc_in, int64_t pstride, int P, int B,
                      int K, void* scratch, int32_t* ids, float* scores, cudaStream_t st);
// score rows R[B][ld] (cols [0,n)) -> keys appended at out[u][list_off .. ) in
// lists of K; returns the number of lists written per user
int k3_rows_lists(int64_t n);
void k3_rows_to_keys(const float* R, int64_t ld, int64_t n, int B, int K, uint32_t id0,
                     uint64_t* out, int64_t out_lists_per_user, int64_t list_off,
                     cudaStream_t st);

// K5 (k5_subset.cu): item subsets and exclusion lists
void launch_gather_codes(const uint8_t* codes, int mp, int64_t N, const int32_t* V, int64_t nV, uint8_t* out,
                         cudaStream_t st);
void launch_fill_padding(int32_t* ids, float* scores, int64_t n, cudaStream_t st);
void launch_check_subset(const int32_t* V, int64_t nV, int64_t N, unsigned long long* first_bad,
                         cudaStream_t st);
void launch_exclude(const int32_t* ids2, const float* sc2, int B, int K2, const int32_t* excl,
                    const int64_t* off, int K, int32_t* ids, float* scores, cudaStream_t st);

// K4 (k4_dense.cu)
void launch_reconstruct(const pq_index_s* idx, const float* psi, int d, float* W,
                        cudaStream_t st);
void dense_sgemm(const float* W, int64_t Nc, int d, const float* phi, int B, float* R,
                 cudaStream_t st);
void launch_recjpq_split(const pq_index_s* idx, const float* S, int B, int u0, int Bc,
                         int k, float* R, cudaStream_t st);

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace pq
