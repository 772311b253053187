// Internal engine interfaces: device-resident dataset, tree tables, the
// level-synchronous sampler and the graph builder. Host side is C++; every
// heavy loop is an sm_100a kernel in tree.cu / kde.cu / sampler.cu /
// graph.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace fsgg {

// Stream-ordered device allocation (cudaMallocAsync on the handle's pool).
class DevBuf {
public:
  DevBuf() = default;
  DevBuf(size_t bytes, cudaStream_t s) { alloc(bytes, s); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      bytes_ = o.bytes_;
      s_ = o.s_;
      o.p_ = nullptr;
      o.bytes_ = 0;
    }
    return *this;
  }
  void alloc(size_t bytes, cudaStream_t s) {
    release();
    s_ = s;
    bytes_ = bytes;
    if (bytes) FSGG_CUDA(cudaMallocAsync(&p_, bytes, s));
  }
  // Grow-only reallocation (contents not preserved).
  void ensure(size_t bytes, cudaStream_t s) {
    if (bytes > bytes_) alloc(bytes + bytes / 4, s);
  }
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    bytes_ = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  size_t bytes() const { return bytes_; }

private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t s_ = nullptr;
};

// Kernel-family arithmetic parameters (proj/include/fsg/kernel.hpp:28-53).
// The exponent is evaluated in base 2: k = 2^(-scale * dist) where dist is
// ||.||_2^2 (gaussian), ||.||_2 (exponential) or ||.||_1 (laplacian).
struct KernelSpec {
  int family = 0;
  double sigma = 1.0;
  float scale = 0.f;  // log2(e) / sigma^2  or  log2(e) / sigma
};
KernelSpec make_kernel_spec(int family, double sigma);

// Balanced binary partition of [0, n) (split at first + size/2,
// proj/src/sampler.cpp:141, :200), stored heap-ordered: level l occupies
// slots [2^l - 1, 2^(l+1) - 1); slot g's children are 2g+1, 2g+2 in
// global numbering. Nodes below a size-1 node are empty (first == last).
struct TreeTable {
  uint32_t n = 0, d = 0;
  uint32_t depth = 0;  // deepest level index; levels 0..depth
  uint64_t slots = 0;
  bool has_boxes = false;
  DevBuf first, last;  // u32 per slot
  DevBuf lo, hi;       // f32 per slot * d (bounding boxes), d <= kBoxMaxDim
};
constexpr uint32_t kBoxMaxDim = 16;

// Certified pruning (kde.cu): a source sub-chunk is skipped for an entry when
// its bounding-box bound is below 2^-kPruneBits of half the entry's node
// mass. With at most 2^20 sub-chunks per node the skipped mass is below
// 2^-(kPruneBits - 21) of the node mass -- far below the fp32 evaluation
// error -- and the tie guard widens its margin by that bound (sampler.cu).
#ifndef FSGG_PRUNE_BITS
#define FSGG_PRUNE_BITS 48.f
#endif
constexpr float kPruneBits = FSGG_PRUNE_BITS;

struct KdeWorkspace;

struct Dataset {
  int device = 0;
  uint32_t n = 0, d = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  DevBuf pts;  // f32 n*d
  TreeTable tree;
  bool tree_valid = false;
  uint32_t launches = 0;  // kernel launches issued (reset per API call)
  // Grow-only work buffers owned by the handle: repeated builds on one
  // dataset never go back to the allocator (a fresh multi-GB cudaMallocAsync
  // costs hundreds of ms when the pool has to map new memory).
  std::unordered_map<std::string, DevBuf> arena;
  DevBuf& buf(const std::string& name, size_t bytes) {
    DevBuf& b = arena[name];
    b.ensure(bytes ? bytes : 8, stream);
    return b;
  }
  std::unique_ptr<KdeWorkspace> kde_ws;
  // Pinned host words for the per-level counter readbacks: a D2H copy into
  // pageable memory is staged by the driver and costs several microseconds
  // more per level than a DMA straight into page-locked memory.
  struct PinnedWords {
    unsigned long long* p = nullptr;
    ~PinnedWords() {
      if (p) cudaFreeHost(p);
    }
  } pinned;
  unsigned long long* host_words() {
    if (!pinned.p) FSGG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pinned.p), 64 * 8,
                                           cudaHostAllocDefault));
    return pinned.p;
  }
  // tensor-core path (kde_tc.cu): split tf32 hi/lo copies + tensor maps
  bool tc_ready = false;
  bool tie_xn_ready = false;  // fp64 point norms of the batched tie guard (sampler.cu)
  alignas(64) unsigned char tc_blob[1152];
  void release_all();
};

// ---- tree.cu --------------------------------------------------------------
void build_tree(Dataset& ds);

// ---- kde.cu ---------------------------------------------------------------
// One level's entry list: entries grouped by node slot (level-local slot g
// owns entries [goff[g], goff[g+1])).
struct LevelView {
  uint32_t level = 0;
  uint32_t num_slots = 0;  // 2^level
  uint32_t num_entries = 0;
  const uint32_t* eq = nullptr;    // query index per entry
  const float* elm = nullptr;      // log2 of the entry's node mass (nullptr: root)
  int prune = 1;                   // certified pruning of negligible sub-chunks
  float prune_bits = kPruneBits;   // ... below 2^-prune_bits of half the node mass
  const uint32_t* eg = nullptr;    // level-local slot per entry
  const uint32_t* goff = nullptr;  // num_slots + 1
  uint32_t qbase = 0xffffffffu;    // level 0: entries are points qbase.. in order (else ~0)
  // sync-free levels (sampler.cu): the entry count lives on the device and
  // num_entries is only its upper bound; only direct levels accept this
  const uint32_t* dE = nullptr;
};

struct KdeStats {
  uint64_t evals = 0;            // algorithmic (reference-equivalent) evaluations
  uint64_t performed = 0;        // evaluations actually executed
  uint64_t tiled_evals = 0;
  uint64_t tiled_performed = 0;
  double tiled_seconds = 0.0;
  uint32_t tiled_launches = 0;
  uint64_t root_performed = 0;   // symmetric root kernel (kde_sym.cu): pair evaluations
  double root_seconds = 0.0;     // ... and its device time (tile kernel only)
};

struct KdeWorkspace {
  // partials: per entry a row of 2^rd fp64 bucket sums (the node's
  // descendants rd levels down); pyr: the same row's pairwise-sum pyramid,
  // depths 1..rd-1 at offsets 2^m - 2 (a lookup then reads two values).
  DevBuf partials, pyr, blk_off, cub_tmp;
  DevBuf direct_evals;  // u64: evaluations of the direct levels (caller resets/reads)
  uint32_t pyr_depth = 0;  // row depth the pyramid was built for (0: none)
  // symmetric root (kde_sym.cu): block depth Lb of the last root pass (0: the
  // root was not symmetric). Its per-(point, partner block) values stay in
  // the arena ("sym.*") and serve levels whose children are unions of
  // blocks (block_lookup_sums, kde_sym.cu).
  uint32_t sym_Lb = 0;
  uint32_t sym_b0 = 0;       // first query block of that pass
  bool sym_pos = false;      // "sym.pos" holds the partner-position table
  // multi-GPU owner mode: tiles of shard [sym_ready_qb, sym_ready_qe)
  // computed (and remote records received) ahead of the descent
  bool sym_ready = false;
  uint32_t sym_ready_qb = 0, sym_ready_qe = 0, sym_ready_b0 = 0, sym_ready_b1 = 0;
  float sym_ready_scale = 0.f;
  int sym_ready_family = -1;
  float sym_ready_bits = 0.f;
  // pruning threshold of the current call (kPruneBits, or the fast
  // backend's epsilon-derived value: fsgg_config.kde_backend)
  float prune_bits = kPruneBits;
  double sym_ready_seconds = 0.0;     // device time of that tile kernel
  double sym_prepared_seconds = 0.0;  // ... credited to the root level that used it
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  ~KdeWorkspace();
};

inline void Dataset::release_all() {
  kde_ws.reset();
  arena.clear();
  tree.first.release();
  tree.last.release();
  tree.lo.release();
  tree.hi.release();
  pts.release();
}

// Child sums for every entry of the level: g1 = sum over [first, mid),
// g2 = sum over [mid, last), floored at 1e-300 (kde.cpp:68). When groot is
// non-null, also writes the unfloored root sum g1 + g2 (level 0 only).
// Tiled levels keep per-entry partial sums over the node's descendants
// *row_depth levels down in ws.partials (row stride 2^*row_depth), aiming
// for serve_levels >= 1; *row_depth = 0 when no partial rows were kept.
// True when kde_level at `level` runs the low-d direct kernel (or nothing):
// it then accepts a device-resident entry count (LevelView::dE).
bool kde_level_sync_free(const Dataset& ds, const KernelSpec& ks, uint32_t level);
void kde_level(Dataset& ds, const KernelSpec& ks, const LevelView& lv,
               double* g1, double* g2, double* groot, KdeWorkspace& ws,
               KdeStats& stats, uint32_t serve_levels, uint32_t* row_depth);

// ---- kde_tc.cu (tcgen05 / TMEM / TMA, 3xTF32) -------------------------------
constexpr uint32_t kTcMinDim = 64;
bool kde_tc_supported(const Dataset& ds, int family);
// Same work items / partial layout as the tiled kernels with 128 entries per
// block; blk_off must have been computed with 128 entries per block.
// Partials: one per (entry, sub-chunk at depth sdepth below each child),
// row width 2^(sdepth+1).
// Symmetric tensor-core root (each pair once) for a full build's level 0;
// false when it does not apply (kde_tc_tiled then runs the one-sided pass).
bool kde_tc_root_symmetric(Dataset& ds, const KernelSpec& ks, const LevelView& lv, uint32_t rl,
                           double* partials, uint64_t* performed);
void kde_tc_tiled(Dataset& ds, const KernelSpec& ks, const LevelView& lv,
                  const uint32_t* blk_off, uint32_t cdepth, uint32_t sdepth, uint64_t items,
                  double* partials);

// KdeEstimator::eval seam: arbitrary range, arbitrary targets (device).
void kde_range(Dataset& ds, const KernelSpec& ks, uint32_t first,
               uint32_t last, const uint32_t* targets, uint32_t m,
               double* out);

// ---- sampler.cu -----------------------------------------------------------
struct SampleRequest {
  std::vector<uint32_t> queries;  // sorted unique query ids
  std::vector<uint32_t> tickets;  // tickets per query (rounds * multiplicity)
  // Range request (builds and shards): queries [range_begin, range_begin +
  // range_count), range_tickets each; `queries`/`tickets` stay empty and the
  // device lists are generated in place (no host vectors, no upload).
  bool range = false;
  uint32_t range_begin = 0, range_count = 0, range_tickets = 0;
  uint64_t seed = 1;
  int rng_mode = 0;
  int prune = 1;
  // Fast backend (epsilon > 0): certified pruning at
  // prune_bits = 19 + log2((depth + 1) / epsilon) instead of kPruneBits, no
  // tie guard. The skipped mass per level is <= epsilon / (depth + 1) of
  // every node's mass, so each query's sampling distribution is within
  // total variation epsilon of the exact one (K1 fast).
  double fast_epsilon = 0.0;
  bool verify_ties = true;  // reference RNG mode: re-decide near-ties on fp64 sums
  bool dfs_finish = true;   // finish small-node levels depth-first (finish.cu)
  bool walk = true;         // single-ticket entries below kWalkMaxNode walk (walk.cu)
  bool want_root_sums = false;
  // Debug export (fsgg_sample_neighbors_counted_ex): every (node, query)
  // entry's two child sums as the level's KDE kernels produced them, before
  // the tie guard; forces the level-synchronous path (no walks / DFS).
  bool record_sums = false;
};

// One recorded entry: node [first, last) at `level`, children
// [first, first + (last - first) / 2) and [mid, last) (sampler.cpp:141, :200).
struct EntryRecord {
  uint32_t level, query, first, last;
  double left, right;
};

struct SampleResult {
  uint32_t nq = 0;
  uint64_t total_tickets = 0;
  DevBuf uq;       // u32 nq: unique queries
  DevBuf row_off;  // u64 nq+1: leaf row capacity offsets
  DevBuf row_cnt;  // u32 nq: leaves emitted per row
  DevBuf leaf_src, leaf_cnt;  // u32 total_tickets
  DevBuf groot;    // f64 nq: g_full of each query (root sum), if requested
  uint64_t degenerate_draws = 0;
  uint64_t tie_verified = 0;  // entries re-decided on fp64 sums
  std::vector<uint64_t> entries_per_level, tickets_per_level;
  uint64_t peak_entries = 0;
  KdeStats kde;
  std::vector<EntryRecord> records;  // record_sums only
};

void sample_counted(Dataset& ds, const KernelSpec& ks, const SampleRequest& req,
                    SampleResult& out);
// Pruning threshold (log2) of a descent: kPruneBits, or the fast backend's.
float prune_bits_for(const SampleRequest& req, const TreeTable& t);

// Sorted (query, source, count) triples copied to the host.
void sampled_triples_to_host(Dataset& ds, SampleResult& res,
                             std::vector<uint32_t>& triples);

// ---- finish.cu ------------------------------------------------------------
constexpr uint32_t kDfsMaxNode = 0;  // depth-first finish off by default (slower: divergent)
struct DfsArgs {
  uint32_t E = 0, level = 0;
  const uint32_t *eq = nullptr, *et = nullptr, *eg = nullptr;
  uint64_t key_prefix = 0, seed = 0;
  int rng_mode = 0, verify = 1;
  const uint32_t* qrow = nullptr;
  const uint64_t* row_off = nullptr;
  uint32_t *row_cnt = nullptr, *leaf_src = nullptr, *leaf_cnt = nullptr;
  unsigned long long* stats = nullptr;  // [4][64] entries/tickets/evals/degen + ties
};
bool dfs_finish_supported(uint32_t d);
void dfs_finish(Dataset& ds, const KernelSpec& ks, const DfsArgs& args);

// ---- kde_sym.cu -----------------------------------------------------------
// Root level with every pair evaluated once (row + column sums of block
// pairs); writes rows [E][2^rd] for the points [qb, qe). false: unsupported.
// ev0/ev1 (nullable) are recorded around the tile kernel alone.
bool kde_root_symmetric(Dataset& ds, const KernelSpec& ks, uint32_t qb, uint32_t qe,
                        uint32_t rd, double* rows, unsigned long long* d_performed,
                        cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr);
// Depth of the symmetric pass's blocks (0: the pass does not apply).
uint32_t sym_block_depth(const Dataset& ds);
constexpr uint32_t kSymRootServe = 7;  // symmetric root: fp64 rows serve levels 1..6
// Multi-GPU owner mode of the symmetric root (shard bounds on block
// boundaries): compute this shard's tiles, returning the records of values
// owed to other ranks (device, kSymRecordWords 32-bit words each: X, Y,
// first point of X, |X|, kSymStride values). false (no records) when the root is
// not symmetric or the bounds are not block-aligned.
constexpr uint32_t kSymStride = 320;  // values per (block, partner) slot: max block size
constexpr uint32_t kSymRecordWords = 4 + kSymStride;
bool sym_shard_prepare(Dataset& ds, const KernelSpec& ks, uint32_t qb, uint32_t qe,
                       uint32_t* num_records, const uint32_t** records);
// Store records received from other ranks (device) into this shard's values.
void sym_shard_receive(Dataset& ds, const uint32_t* records, uint32_t num_records);
// Block-aligned shard bounds (world + 1 entries) for owner mode, balanced
// by a per-block cost model when the kernel is given (else equal blocks).
void sym_shard_bounds(Dataset& ds, const KernelSpec* ks, uint32_t world, uint32_t* bounds);
// Child sums of level `level` (1 <= level, level + 1 <= ws.sym_Lb) from the
// symmetric root's per-(point, partner block) values: each child of a node
// at this level is a run of whole blocks, so its sum for query q is the sum,
// in ascending partner order, of q's values for the partners in that run.
// Adds the reference-equivalent evaluations to *evals (device counter).
// With dE, E is only an upper bound (the grid) and the count is *dE.
void block_lookup_sums(Dataset& ds, uint32_t E, uint32_t level, const uint32_t* eq,
                       const uint32_t* eg, double* g1, double* g2,
                       unsigned long long* evals, const uint32_t* dE = nullptr);

// ---- walk.cu --------------------------------------------------------------
// Entries holding a single ticket below nodes of kWalkMaxNode points leave
// the level-synchronous lists and finish as one path walk each.
constexpr uint32_t kWalkMaxNode = 128;
struct WalkArgs {
  uint32_t W = 0;  // walks
  const uint32_t* wq = nullptr;  // query
  const uint32_t* wh = nullptr;  // heap index of the start node
  const float* welm = nullptr;   // log2 of the start node's sum
  uint64_t key_prefix = 0, seed = 0;
  int rng_mode = 0, verify = 1;
  const uint32_t* qrow = nullptr;
  const uint64_t* row_off = nullptr;
  uint32_t *row_cnt = nullptr, *leaf_src = nullptr, *leaf_cnt = nullptr;
  unsigned long long* stats = nullptr;  // [5][64]: entries, tickets, evals, degen, ties
  const uint64_t* nlink = nullptr;      // node_link per heap slot (reference RNG)
  // first step from two-deep partial rows: walks whose start node lies one
  // level below rows_level read row wrow (stride 4) instead of evaluating
  const uint32_t* wrow = nullptr;
  const float* wrm = nullptr;           // log2 node mass the rows were pruned against
  const double* rows = nullptr;
  uint32_t rows_level = 0;
};
bool walk_supported(uint32_t d);
void walk_finish(Dataset& ds, const KernelSpec& ks, const WalkArgs& args);

// datasets_dev.cu: device generators (blocking, current device); any of
// p64 / p32 / labels may be null
void make_moons_device(uint32_t n, double noise, uint64_t seed, double* p64, float* p32,
                       uint32_t* labels);
void make_blobs_device(uint32_t n, const double* centers_host, uint32_t k, uint32_t d,
                       double stddev, uint64_t seed, double* p64, float* p32, uint32_t* labels);
void make_image_features_device(uint32_t height, uint32_t width, uint32_t regions, double noise,
                                uint64_t seed, double* p64, float* p32, uint32_t* labels);
void make_gmm_device(uint32_t n, uint32_t d, uint32_t k, double stddev, uint64_t seed,
                     double* p64, float* p32, uint32_t* labels);

// ---- graph.cu -------------------------------------------------------------
struct GraphResult {
  uint32_t n = 0;
  uint64_t m = 0;
  DevBuf u, v, w, row_ptr, degrees;
  double total_weight = 0.0;
  uint64_t underflow = 0;
  DevBuf est;  // fsgg_edge_estimate-compatible records (optional)
  // the finish's transposed order (v ascending, stable: u ascending within
  // a v) with its weights, in arena buffers valid until the next finish on
  // the handle: rows_transposed hands them out instead of sorting again
  const uint32_t* tv_sorted = nullptr;
  const double* tw_sorted = nullptr;
};

// Sorted unique pair keys ((u << 32) | v, u < v) from the leaf rows;
// self samples counted into *self_pairs. Returns count.
uint64_t collapse_pairs(Dataset& ds, SampleResult& res, DevBuf& keys,
                        uint64_t* self_pairs, uint64_t* sampled_pairs);
// Multi-GPU variant: the shard's pair keys ((u << 32) | v, u < v, self
// samples dropped, duplicates kept, unsorted) grouped by the rank owning row
// u under bounds (world + 1 entries, host): counts[r] keys for rank r, in
// rank order. Returns the total. The owner sorts and dedupes what it gets.
uint64_t collapse_pairs_routed(Dataset& ds, SampleResult& res, DevBuf& keys, uint32_t world,
                               const uint32_t* bounds_host, uint64_t* counts,
                               uint64_t* self_pairs, uint64_t* sampled_pairs);

// Row-sharded finish (multi-GPU): the graph's (v, w) stable-sorted by v
// (the degree contributions the owner of v needs), and the degrees of rows
// [rb, re) from the routed lower contributions plus the local rows.
void rows_transposed(Dataset& ds, const GraphResult& g, uint32_t* v_out, double* w_out);
void rows_degrees(Dataset& ds, const GraphResult& g, const uint32_t* lower_v,
                  const double* lower_w, uint64_t nlower, uint32_t rb, uint32_t re,
                  double* deg_out);
// row_ptr[rb .. re) of the rank's rows shifted by the edges of the ranks
// before it: the rank's slice of the gathered graph's global row_ptr.
void rows_row_ptr(Dataset& ds, const GraphResult& g, uint32_t rb, uint32_t re,
                  uint64_t edge_offset, uint64_t* out);

// Host destination of a graph streamed out while it is finished: each
// array's device-to-host copy starts (on its own stream) as soon as the
// array is final, overlapping the rest of the finish. Buffers should be
// pinned; capacity bounds the edge arrays (n * L suffices).
struct HostSink {
  uint32_t* v = nullptr;
  double* w = nullptr;
  uint64_t* row_ptr = nullptr;
  double* degrees = nullptr;
  uint64_t capacity = 0;
};

// Dedupe (keys may repeat across shards), weight, CSR, degrees.
// With chunks (nchunks u-range partitions of unsorted keys, in order, from
// collapse_pairs_routed): each chunk finished and streamed to the sink on
// its own (no estimates), identical output.
void finish_graph(Dataset& ds, const KernelSpec& ks, uint32_t rounds,
                  const double* g_full, const uint64_t* keys, uint64_t nkeys,
                  bool keys_sorted_unique, bool want_estimates,
                  GraphResult& out, const HostSink* sink = nullptr,
                  const uint64_t* chunks = nullptr, uint32_t nchunks = 0);

}  // namespace fsgg
