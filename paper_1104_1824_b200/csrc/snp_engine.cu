// snp_engine.cu — host side of the SNP engine: validation, upload, the level
// pipeline (SURVEY §8(a) a1-a6 / DESIGN.md §2) and the C ABI of include/snp.h.
//
// Every step of the path runs in the kernels of snp_kernels.cu; the host only
// sizes buffers, launches, and reads back per-level counters.  There is no CPU
// fallback: without a CUDA device every compute call fails with SNP_E_CUDA.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/snp.h"
#include "snp_comm.h"
#include "snp_internal.h"

using namespace snp;

namespace {

thread_local std::string g_err;

// SNP_TRACE=1: host-side wall time of allocation / synchronisation sections
// per level, printed to stderr (diagnostics only).
struct HostTrace {
  bool on = getenv("SNP_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0;
  std::string line;
  void start() { if (on) { t0 = std::chrono::steady_clock::now(); line.clear(); } }
  void mark(const char* what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    char buf[64];
    snprintf(buf, sizeof buf, " %s=%.2f", what, std::chrono::duration<double, std::milli>(t - t0).count());
    line += buf;
    t0 = t;
  }
  void flush(const char* tag) { if (on) fprintf(stderr, "[snp-trace] %s%s\n", tag, line.c_str()); }
};
thread_local HostTrace g_trace;

snp_status fail(snp_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      if (e_ == cudaErrorMemoryAllocation) { cudaGetLastError(); return fail(SNP_E_OOM, "%s: %s", #expr, cudaGetErrorString(e_)); } \
      return fail(SNP_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));                      \
    }                                                                                        \
  } while (0)

#define SNP_TRY(expr)            \
  do {                           \
    snp_status s_ = (expr);      \
    if (s_ != SNP_OK) return s_; \
  } while (0)

uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// bytes of a blocked frontier of F configurations (ceil(F/64) blocks of m × 64 counts)
size_t level_bytes(int64_t F, int64_t m, int32_t w) { return (size_t)((F + PB - 1) / PB) * (size_t)m * PB * w; }

// A growable device allocation.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool owned = true;  // false: a piece of a larger allocation (the retained-level pool)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes), owned(o.owned) { o.p = nullptr; o.bytes = 0; o.owned = true; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; owned = o.owned; o.p = nullptr; o.bytes = 0; o.owned = true; }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p && owned) cudaFree(p);
    p = nullptr;
    bytes = 0;
    owned = true;
  }
  snp_status ensure(size_t need, bool slack = true) {
    if (need <= bytes && p) return SNP_OK;
    release();
    size_t want = slack ? need + need / 8 : need;
    if (want < 256) want = 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return fail(SNP_E_OOM, "cudaMalloc(%zu bytes): %s", want, cudaGetErrorString(e));
    }
    bytes = want;
    return SNP_OK;
  }
  template <class U> U* as() const { return reinterpret_cast<U*>(p); }
};

// A non-owning view into an arena allocation.
struct DView {
  void* p = nullptr;
  template <class U> U* as() const { return reinterpret_cast<U*>(p); }
};

// Bump allocator for per-level metadata (kept for the whole exploration):
// a few large cudaMallocs instead of five per level.
struct Arena {
  std::vector<DBuf> chunks;
  size_t chunk = 0, used = 0;
  snp_status alloc(size_t bytes, DView* out) {
    bytes = (bytes + 255) & ~(size_t)255;
    if (chunk < chunks.size() && used + bytes <= chunks[chunk].bytes) {
      out->p = static_cast<uint8_t*>(chunks[chunk].p) + used;
      used += bytes;
      return SNP_OK;
    }
    if (chunk + 1 < chunks.size() && bytes <= chunks[chunk + 1].bytes) {
      ++chunk;
      used = 0;
      return alloc(bytes, out);
    }
    DBuf b;
    SNP_TRY(b.ensure(std::max<size_t>(bytes, (size_t)1 << 30), false));
    chunks.push_back(std::move(b));
    chunk = chunks.size() - 1;
    used = 0;
    return alloc(bytes, out);
  }
  void reset() { chunk = 0; used = 0; }
  size_t capacity() const {
    size_t c = 0;
    for (const DBuf& b : chunks) c += b.bytes;
    return c;
  }
  // one chunk covering `total` bytes beyond what the chunks already hold
  snp_status reserve(size_t total) {
    const size_t have = capacity();
    if (total <= have) return SNP_OK;
    DBuf b;
    SNP_TRY(b.ensure(std::max<size_t>(total - have, (size_t)1 << 30), false));
    chunks.push_back(std::move(b));
    return SNP_OK;
  }
};

// One level of the tree on the device.
struct Level {
  DBuf data;  // blocked counts, ceil(F/64) × m × 64 (may be released when not retained)
  int64_t F = 0;
  DView fp0, fp1, parent, t, halting;
  // keep_all_edges (reading A17): every transition of the expansion that
  // produced this level — the visited ref it reached (EMPTY = not stored),
  // in tag order, and the parents' child offsets (F_parent + 1) to recover
  // (parent, t) of each edge
  DBuf all_ref, all_off;
  int64_t all_T = 0, all_F = 0;
  bool has_data() const { return data.p != nullptr; }
};

}  // namespace

struct snp_system {
  // ---- lifetime: the caller's reference + one per snp_tree taken from it
  int refs = 1;
  // ---- host copy of the system
  int64_t m = 0, n = 0;
  snp_options opt{};
  int32_t bytes = 4;       // storage bytes per count
  int64_t count_max = 0;
  std::vector<int32_t> C0;
  bool binary_emit = true;
  bool small_rules = true;  // every c, p <= 255 (k_sample_cta)
  // ---- device system
  DBuf d_rule_off, d_rules, d_h0, d_h1, d_in_off, d_in_src, d_out_off, d_out_dst, d_R0, d_R1, d_in_pad, d_in_pad16, d_in_pad16x4, d_in_pad_off;
  SysView view{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // ---- exploration state
  uint64_t generation = 0;
  bool begun = false;
  bool horizon_reserved = false;  // reserve_horizon succeeded since the last begin
  std::vector<std::unique_ptr<Level>> levels;
  std::vector<snp_level_counters> counters;
  int64_t n_visited = 0;
  int64_t total_T = 0;
  uint64_t digest = 0;
  bool halting_current_valid = false;
  // hash tables
  DBuf vis, ltab;
  uint64_t vis_cap = 0, ltab_cap = 0, child_cap = 0;
  // scratch
  DBuf psi, off, fpb0, fpb1, ndc, nd, ebits;
  DBuf d_meta, d_tab, d_tab_full, d_ctab, d_ttab, d_elut, d_hsg, d_xyt, d_xyf, d_btile, d_ndl, d_delay, d_cpT;
  DBuf cpar, cfp0, cfp1, verdict, cslot, cref, kept, kpos, kq_off, scan_tmp, ovf, src_index, stored;
  DBuf counters_dev;  // [0] err, [1..] u64 counters
  DBuf edge_scratch;  // snp_level_edges: fp0/fp1 interleave
  DBuf vlist;         // dedup = 0: the transitions to verify
  DBuf vfc;           // dedup = 0: fired (c, p) rows of a verification batch
  DBuf snap_scratch;  // snapshot: packed edge arrays
  DBuf gen;           // generated-number bitmap (out_rule1 > 0)
  std::vector<DBuf> spare;  // released level buffers kept for reuse
  Arena arena;              // per-level metadata
  // retained levels (keep_tree / dedup = 0): their blocked counts carved from
  // one allocation reserved with the horizon, so no cudaMalloc lands inside a
  // level (a 4.3 GB cudaMalloc per level cost ~25 ms at config 3)
  DBuf lpool;
  size_t lpool_used = 0;
  // small frontiers (k_small_bfs): scratch, per-launch level pools (kept until
  // the next snp_begin: the levels they hold are views into them)
  DBuf small_scratch, small_out, small_stored;
  std::vector<DBuf> small_pools;
  std::vector<DBuf> small_spare;  // pools of an earlier exploration, reused (no cudaMalloc per explore)
  size_t small_skip = (size_t)-1;  // levels.size() at which a level had > SMALL_T transitions
  // multi-GPU exploration (snp_dist_*): this rank's share of the frontier and
  // of the visited keys (owner = fmix64(fp1) mod P)
  struct Dist {
    int32_t P = 0;          // 0 = not in distributed mode
    int stage = 0;          // 0 idle, 1 keys ready, 2 packed, 3 owner-deduped, 4 owner-kept, 5 finalized
    bool level0 = false;
    uint64_t T = 0, R = 0;
    int64_t K = 0;
    const uint64_t* recv = nullptr;
    snp_level_counters lc{};
    DBuf raw;               // level-0 rows before the global dedup
    int64_t F0 = 0;
    DBuf fp0, fp1;          // level-0 fingerprints
    DBuf perm, hist, slot, verdict;
    ExpandOut O{};
    int64_t owned = 0;      // keys in this rank's visited shard
    // library-driven levels (snp_dist_init / snp_dist_advance): the transport,
    // exchange buffers and the global view of the exploration
    snp::Comm* comm = nullptr;
    snp::LocalGroup* group = nullptr;
    DBuf sendbuf, recvbuf, vbuf, backbuf, rbuf, mbuf[2];
    double rebalance = 1.1;   // max/mean local frontier above which rows are redistributed (0 = never)
    int64_t F_global = 0, q_off = 0, n_configs = 0, T_total = 0;
    int64_t rebalanced_rows = 0;  // rows this rank sent in the last rebalancing
    int inject_step = -1;         // SNP_DIST_INJECT="rank,step": fail this rank at that protocol step (tests)
  } dist;
  // phase profiling (snp_set_profiling)
  bool profiling = false;
  double prof_ms[SNP_NUM_PHASES] = {0, 0, 0, 0, 0};
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Mark { int phase; cudaEvent_t a, b; };
  std::vector<Mark> marks;
};

struct snp_tree {
  snp_system* sys = nullptr;  // holds a reference (snp_system_free defers until the last tree is freed)
  uint64_t generation = 0;
  int64_t m = 0, n = 0;
  std::vector<int64_t> level_offsets;
  std::vector<int64_t> parent;
  std::vector<uint64_t> t;
  std::vector<uint8_t> halting;
  std::vector<uint64_t> fp;
  std::vector<snp_level_counters> counters;
};

namespace {

// device counter block layout
struct DevCounters {
  int32_t err;
  int32_t pad;
  unsigned long long n_new;
  unsigned long long n_halting;
  unsigned long long n_ovf;
  unsigned long long digest;
  unsigned long long n_verify;
};

snp_status sync(snp_system* s) {
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return SNP_OK;
}

cudaEvent_t pool_event(snp_system* s) {
  if (s->ev_used == s->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    s->ev_pool.push_back(e);
  }
  return s->ev_pool[s->ev_used++];
}

void phase_begin(snp_system* s, int phase) {
  if (!s->profiling) return;
  cudaEvent_t e = pool_event(s);
  cudaEventRecord(e, s->stream);
  s->marks.push_back({phase, e, nullptr});
}

void phase_end(snp_system* s) {
  if (!s->profiling || s->marks.empty()) return;
  cudaEvent_t e = pool_event(s);
  cudaEventRecord(e, s->stream);
  s->marks.back().b = e;
}

// after a stream synchronize: fold the recorded phase intervals into prof_ms
void phase_collect(snp_system* s) {
  for (auto& mk : s->marks) {
    float ms = 0;
    if (mk.b && cudaEventElapsedTime(&ms, mk.a, mk.b) == cudaSuccess) s->prof_ms[mk.phase] += ms;
  }
  s->marks.clear();
  s->ev_used = 0;
}

snp_status read_counters(snp_system* s, DevCounters* h) {
  CUDA_TRY(cudaMemcpyAsync(h, s->counters_dev.p, sizeof(DevCounters), cudaMemcpyDeviceToHost, s->stream));
  return sync(s);
}

snp_status check_err(int32_t err) {
  if (err & ERR_COLLISION) return fail(SNP_E_COLLISION, "two distinct configurations share a 128-bit fingerprint (or a fingerprint equals the empty-slot sentinel)");
  if (err & ERR_TABLE_FULL) return fail(SNP_E_CAPACITY, "hash table full");
  if (err & ERR_CAPACITY) return fail(SNP_E_CAPACITY, "a configuration has more than 2^62 valid spiking vectors");
  if (err & ERR_OVERFLOW) return fail(SNP_E_OVERFLOW, "a spike count leaves the %s storage range", "count_bits");
  return SNP_OK;
}

bool retain_levels(const snp_system* s);

snp_status take_buffer(snp_system* s, size_t bytes, DBuf* out) {
  if (s->lpool.p && retain_levels(s)) {
    const size_t b = (bytes + 255) & ~(size_t)255;
    if (s->lpool_used + b <= s->lpool.bytes) {
      out->release();
      out->p = static_cast<uint8_t*>(s->lpool.p) + s->lpool_used;
      out->bytes = b;
      out->owned = false;
      s->lpool_used += b;
      return SNP_OK;
    }
  }
  // reuse the smallest spare that fits
  int best = -1;
  for (int i = 0; i < (int)s->spare.size(); ++i)
    if (s->spare[i].bytes >= bytes && (best < 0 || s->spare[i].bytes < s->spare[best].bytes)) best = i;
  if (best >= 0) {
    *out = std::move(s->spare[best]);
    s->spare.erase(s->spare.begin() + best);
    return SNP_OK;
  }
  // free spares before a fresh allocation (they are too small)
  s->spare.clear();
  return out->ensure(bytes + bytes / 16, false);
}

void release_level_data(snp_system* s, Level* L) {
  if (L->data.p && !L->data.owned) {  // a view into a pool: nothing to recycle
    L->data.release();
    return;
  }
  if (L->data.p) {
    s->spare.push_back(std::move(L->data));
    while (s->spare.size() > 2) s->spare.erase(s->spare.begin());
  }
}

snp_status ensure_visited(snp_system* s, uint64_t needed_entries) {
  // keep the load <= 1/2; grow 4x at a time so a long run rehashes rarely
  if (2 * needed_entries <= s->vis_cap) return SNP_OK;
  uint64_t want = next_pow2(std::max<uint64_t>(1024, 2 * needed_entries));
  if (s->vis_cap) want = std::max(want, 4 * s->vis_cap);
  DBuf nt;
  SNP_TRY(nt.ensure(want * sizeof(Slot), false));
  CUDA_TRY(cudaMemsetAsync(nt.p, 0xFF, want * sizeof(Slot), s->stream));
  int32_t* err = s->counters_dev.as<int32_t>();
  if (s->vis_cap) launch_rehash(s->vis.as<Slot>(), s->vis_cap, nt.as<Slot>(), want - 1, err, s->stream);
  CUDA_TRY(cudaGetLastError());
  SNP_TRY(sync(s));
  s->vis = std::move(nt);
  s->vis_cap = want;
  return SNP_OK;
}

// Growing the visited table or the level-metadata arena mid-run costs a
// cudaMalloc (tens of ms per GB) plus a rehash inside a level.  Reserve both
// up front for RESERVE_LEVELS levels of Ft configurations, within what the
// device can spare beside the per-level working set (next frontier, emit
// words, child arrays, level table).
snp_status ensure_children(snp_system* s, uint64_t T);
constexpr int64_t RESERVE_LEVELS = 32;
constexpr int64_t RESERVE_CHILDREN = 16;  // T/F reaches 9 at config 3, 6 at config 4
snp_status reserve_horizon(snp_system* s, int64_t Ft) {
  if (Ft <= 0) return SNP_OK;
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  // next level (+10 % thinning slack), emit words, ND lists, child arrays and
  // level table for 16·Ft children, 4 GB of slack
  const size_t working = level_bytes(Ft + Ft / 10, s->m, s->bytes) +
                         (size_t)((Ft + PB - 1) / PB) * ((s->m + 1) & ~1) * 8 + (size_t)Ft * KMAX * 8 +
                         (size_t)Ft * 16 * 60 + next_pow2((uint64_t)Ft * 32) * sizeof(Slot) + ((size_t)4 << 30);
  if (free_b <= working) return SNP_OK;
  // children per level: up to RESERVE_CHILDREN × Ft before the arrays grow.
  // `working` already budgets them (16·Ft·60 B + the level table), so they
  // are reserved first, outside `spare`: left to grow on demand they were
  // reallocated mid-run (cudaFree + cudaMalloc inside a level, 2 to 850 ms
  // measured at config 4's 13th level) once visited + metadata took the spare
  const uint64_t T = (uint64_t)RESERVE_CHILDREN * (uint64_t)Ft;
  if (T > s->child_cap) SNP_TRY(ensure_children(s, T / 2));
  {
    // the level table for 8·Ft transitions (2 slots each): config 4 stays
    // below (T/F <= 6.1); a rarer larger level grows it (a 1 GB reallocation
    // at config 3's tenth level, T/F = 8.8)
    const uint64_t lw = next_pow2(std::max<uint64_t>(1024, 2 * (T / 2)));
    if (lw > s->ltab_cap) {
      SNP_TRY(s->ltab.ensure(lw * sizeof(Slot), false));
      s->ltab_cap = lw;
    }
  }
  size_t spare = free_b - working;
  s->horizon_reserved = true;
  const uint64_t entries = (uint64_t)RESERVE_LEVELS * (uint64_t)Ft;
  const size_t vis_b = next_pow2(2 * entries) * sizeof(Slot);
  if (vis_b <= spare && 2 * entries > s->vis_cap) {
    SNP_TRY(ensure_visited(s, entries));
    spare -= vis_b;
  }
  const size_t meta_b = (size_t)entries * 40;
  if (meta_b <= spare) {
    SNP_TRY(s->arena.reserve(meta_b));
    spare -= meta_b;
  }
  // retained levels: a pool for up to RESERVE_LEVELS more levels of Ft
  // configurations, within what is left (minus 4 GB of slack)
  if (retain_levels(s) && !s->lpool.p) {
    const size_t per = level_bytes(Ft + Ft / 10, s->m, s->bytes) + 256;
    size_t want = per * (size_t)RESERVE_LEVELS;
    const size_t slack = (size_t)4 << 30;
    if (spare > slack && want > spare - slack) want = (spare - slack) / per * per;
    if (spare > slack && want >= per) {
      if (s->lpool.ensure(want, false) == SNP_OK) s->lpool_used = 0;
      else s->lpool.release();
    }
  }
  return SNP_OK;
}

snp_status ensure_ltab(snp_system* s, uint64_t T) {
  uint64_t want = next_pow2(std::max<uint64_t>(1024, 2 * T));
  if (want > s->ltab_cap) {
    SNP_TRY(s->ltab.ensure(want * sizeof(Slot), false));
    s->ltab_cap = want;
  }
  // use only `want` slots this level (smaller clears for small levels)
  CUDA_TRY(cudaMemsetAsync(s->ltab.p, 0xFF, want * sizeof(Slot), s->stream));
  s->ltab_cap = std::max(s->ltab_cap, want);
  return SNP_OK;
}

Tables tables(snp_system* s, uint64_t ltab_slots) {
  return Tables{s->vis.as<Slot>(), s->vis_cap ? s->vis_cap - 1 : 0, s->ltab.as<Slot>(), ltab_slots - 1};
}

snp_status ensure_children(snp_system* s, uint64_t T) {
  // per-level T grows along a run: reallocate rarely, to twice the need
  if (T > s->child_cap) {
    const uint64_t c = std::max<uint64_t>(2 * T, 4096);
    SNP_TRY(s->cpar.ensure(c * 4 + 16, false));
    SNP_TRY(s->cfp0.ensure(c * 8 + 16, false));
    SNP_TRY(s->cfp1.ensure(c * 8 + 16, false));
    SNP_TRY(s->verdict.ensure(c + 16, false));
    SNP_TRY(s->cslot.ensure(c * 8 + 16, false));
    SNP_TRY(s->cref.ensure(c * 8 + 16, false));
    SNP_TRY(s->kept.ensure((c + 1) * 8 + 16, false));
    SNP_TRY(s->kpos.ensure((c + 1) * 8 + 16, false));
    SNP_TRY(s->scan_tmp.ensure(scan_temp_bytes((int64_t)c + 1) + 256, false));
    s->child_cap = c;
  }
  return SNP_OK;
}

ChildArrays child_arrays(snp_system* s) {
  return ChildArrays{s->cpar.as<uint32_t>(), s->cfp0.as<uint64_t>(), s->cfp1.as<uint64_t>(),
                     s->verdict.as<uint8_t>(), s->cslot.as<uint64_t>(), s->cref.as<uint64_t>(),
                     s->kept.as<uint64_t>(), s->kpos.as<uint64_t>()};
}

snp_status alloc_level_meta(snp_system* s, Level* L, int64_t K) {
  size_t k = (size_t)std::max<int64_t>(K, 1);
  SNP_TRY(s->arena.alloc(k * 8, &L->fp0));
  SNP_TRY(s->arena.alloc(k * 8, &L->fp1));
  SNP_TRY(s->arena.alloc(k * 8, &L->parent));
  SNP_TRY(s->arena.alloc(k * 8, &L->t));
  SNP_TRY(s->arena.alloc(k, &L->halting));
  return SNP_OK;
}

bool retain_levels(const snp_system* s) { return s->opt.keep_tree || s->opt.dedup == 0; }

snp_status update_stored_table(snp_system* s) {
  std::vector<StoredLevel> h(s->levels.size());
  for (size_t i = 0; i < s->levels.size(); ++i) h[i] = StoredLevel{s->levels[i]->data.p};
  SNP_TRY(s->stored.ensure(h.size() * sizeof(StoredLevel) + 16));
  CUDA_TRY(cudaMemcpyAsync(s->stored.p, h.data(), h.size() * sizeof(StoredLevel), cudaMemcpyHostToDevice, s->stream));
  return sync(s);  // h is a stack buffer
}

// ---------------------------------------------------------------------------
// validation + upload (snp_load)
// ---------------------------------------------------------------------------
snp_status validate_and_build(snp_system* s, const snp_matrix* M, const snp_rule* rules, int64_t n_rules,
                              const uint64_t* re_bits, std::vector<std::vector<std::pair<int32_t, int32_t>>>* rows,
                              std::vector<std::vector<int32_t>>* out_syn) {
  const int64_t m = s->m, n = n_rules;
  rows->assign(n, {});
  for (int64_t r = 0; r < n; ++r) {
    const snp_rule& R = rules[r];
    if (R.neuron < 0 || R.neuron >= m) return fail(SNP_E_INVALID_SYSTEM, "rule %lld: neuron out of range", (long long)r);
    if (r > 0 && R.neuron < rules[r - 1].neuron) return fail(SNP_E_INVALID_SYSTEM, "rule %lld: rules not grouped by neuron", (long long)r);
    if (R.kind != SNP_RE_EXACT && R.kind != SNP_RE_PERIODIC && R.kind != SNP_RE_UNARY)
      return fail(SNP_E_INVALID_SYSTEM, "rule %lld: bad regex kind", (long long)r);
    if (R.kind == SNP_RE_UNARY && (!re_bits || R.b < 1 || (int64_t)R.a + R.b > 256))
      return fail(SNP_E_INVALID_SYSTEM, "rule %lld: unary regex needs P >= 1, t + P <= 256 and its bit row", (long long)r);
    if (R.consumed < 1) return fail(SNP_E_INVALID_SYSTEM, "rule %lld: c < 1", (long long)r);
    if (R.produced < 0) return fail(SNP_E_INVALID_SYSTEM, "rule %lld: p < 0", (long long)r);
    if (R.a < 0) return fail(SNP_E_INVALID_SYSTEM, "rule %lld: regex exponent < 0", (long long)r);
    if (R.kind == SNP_RE_PERIODIC && R.b < 1) return fail(SNP_E_INVALID_SYSTEM, "rule %lld: period j < 1", (long long)r);
    if (M->dense) {
      for (int64_t j = 0; j < m; ++j) {
        int32_t v = M->dense[r * m + j];
        if (v) (*rows)[r].push_back({(int32_t)j, v});
      }
    } else {
      for (int64_t e = M->row_ptr[r]; e < M->row_ptr[r + 1]; ++e) {
        if (M->col[e] < 0 || M->col[e] >= m) return fail(SNP_E_INVALID_SYSTEM, "M row %lld: column out of range", (long long)r);
        if (M->val[e]) (*rows)[r].push_back({M->col[e], M->val[e]});
      }
    }
  }
  std::vector<int64_t> per(m, 0);
  for (int64_t r = 0; r < n; ++r) per[rules[r].neuron]++;
  for (int64_t j = 0; j < m; ++j)
    if (per[j] > 255) return fail(SNP_E_INVALID_SYSTEM, "neuron %lld: more than 255 rules", (long long)j);
  out_syn->assign(m, {});
  std::vector<char> seen(m, 0);
  for (int64_t r = 0; r < n; ++r) {
    const snp_rule& R = rules[r];
    bool diag = false;
    std::vector<int32_t> targets;
    for (auto& jv : (*rows)[r]) {
      if (jv.first == R.neuron) {
        if (jv.second != -R.consumed) return fail(SNP_E_INVALID_SYSTEM, "M[%lld][%d] != -c", (long long)r, jv.first);
        diag = true;
      } else {
        if (jv.second != R.produced) return fail(SNP_E_INVALID_SYSTEM, "M[%lld][%d] not in {0, p}", (long long)r, jv.first);
        targets.push_back(jv.first);
      }
    }
    if (!diag) return fail(SNP_E_INVALID_SYSTEM, "M[%lld][neuron] != -c", (long long)r);
    std::sort(targets.begin(), targets.end());
    for (size_t i = 1; i < targets.size(); ++i)
      if (targets[i] == targets[i - 1]) return fail(SNP_E_INVALID_SYSTEM, "M row %lld: repeated column", (long long)r);
    if (R.produced > 0) {
      if (!seen[R.neuron]) { seen[R.neuron] = 1; (*out_syn)[R.neuron] = targets; }
      else if ((*out_syn)[R.neuron] != targets)
        return fail(SNP_E_INVALID_SYSTEM, "rule %lld: synapse set differs from neuron's other spiking rules", (long long)r);
    }
  }
  return SNP_OK;
}

template <class U>
snp_status upload(snp_system* s, DBuf& b, const std::vector<U>& v) {
  SNP_TRY(b.ensure(std::max<size_t>(v.size(), 1) * sizeof(U), false));
  if (!v.empty()) CUDA_TRY(cudaMemcpy(b.p, v.data(), v.size() * sizeof(U), cudaMemcpyHostToDevice));
  return SNP_OK;
}

// Row assignment of one half-warp's in-synapse sources for K-c's gather.
// In row r, lane l reads the staged emit word of source lane_row[l][r] (-1:
// padding, the shared zero word).  K-c keeps the 64-bit emit words in shared
// memory, word s in bank pair s mod 16, so the 16 lanes of a half-warp read
// one row in one wavefront when their bank pairs differ.  The order of a
// lane's sources is free (their counts are summed), so the rows are a proper
// edge colouring of the bipartite multigraph lanes × bank pairs (colour =
// row).  König: max-degree colours suffice; with R rows (the group's padded
// row count, >= every in-degree) a bank pair with more than R sources is
// split round-robin into ceil(deg / R) nodes (two of its lanes then share a
// row), so the padding stays that of the plain layout.  Colouring by
// alternating-path swaps.
static void bank_rows(const std::vector<std::vector<int32_t>>& lane_src, int R, std::vector<std::vector<int32_t>>& lane_row) {
  const int NL = (int)lane_src.size();
  int D = R;  // rows available (>= every lane's in-degree)
  for (auto& v : lane_src) D = std::max(D, (int)v.size());
  lane_row.assign(NL, std::vector<int32_t>(D, -1));
  if (D == 0) return;
  int deg[16] = {0};
  for (auto& v : lane_src)
    for (int32_t s : v) deg[s & 15]++;
  int vbase[17] = {0};
  for (int k = 0; k < 16; ++k) vbase[k + 1] = vbase[k] + std::max(1, (deg[k] + D - 1) / D);
  const int NV = vbase[16];
  struct E { int u, v; int32_t s; int c; };
  std::vector<E> es;
  int rr[16] = {0};
  for (int l = 0; l < NL; ++l)
    for (int32_t s : lane_src[l]) {
      const int k = s & 15, nk = vbase[k + 1] - vbase[k];
      es.push_back({l, vbase[k] + (rr[k]++ % nk), s, -1});
    }
  std::vector<int> atL((size_t)NL * D, -1), atV((size_t)NV * D, -1);  // edge id holding colour c at a node
  for (int e = 0; e < (int)es.size(); ++e) {
    const int u = es[e].u, v = es[e].v;
    int a = 0, b = 0;
    while (atL[(size_t)u * D + a] >= 0) ++a;  // free at u (deg u <= D)
    while (atV[(size_t)v * D + b] >= 0) ++b;  // free at v (deg v <= D)
    if (atV[(size_t)v * D + a] >= 0) {
      // swap a/b on the alternating path from v that starts with colour a;
      // bipartite: it never reaches u, so a becomes free at v and stays free at u
      std::vector<int> path;
      int x = v, col = a;
      bool right = true;
      for (;;) {
        const int pe = right ? atV[(size_t)x * D + col] : atL[(size_t)x * D + col];
        if (pe < 0) break;
        path.push_back(pe);
        x = right ? es[pe].u : es[pe].v;
        right = !right;
        col = col == a ? b : a;
      }
      for (int pe : path) {
        atL[(size_t)es[pe].u * D + es[pe].c] = -1;
        atV[(size_t)es[pe].v * D + es[pe].c] = -1;
      }
      for (int pe : path) {
        es[pe].c = es[pe].c == a ? b : a;
        atL[(size_t)es[pe].u * D + es[pe].c] = pe;
        atV[(size_t)es[pe].v * D + es[pe].c] = pe;
      }
    }
    es[e].c = a;
    atL[(size_t)u * D + a] = e;
    atV[(size_t)v * D + a] = e;
  }
  for (auto& e : es) lane_row[e.u][e.c] = e.s;
}

snp_status load_impl(snp_system* s, const snp_matrix* M, const snp_rule* rules, int64_t n_rules, const uint64_t* re_bits,
                     const int32_t* C0) {
  std::vector<std::vector<std::pair<int32_t, int32_t>>> rows;
  std::vector<std::vector<int32_t>> out_syn;
  SNP_TRY(validate_and_build(s, M, rules, n_rules, re_bits, &rows, &out_syn));
  const int64_t m = s->m, n = n_rules;
  s->n = n;
  for (int64_t j = 0; j < m; ++j)
    if (C0[j] < 0 || C0[j] > s->count_max) return fail(SNP_E_OVERFLOW, "C0[%lld] outside the storage range", (long long)j);
  s->C0.assign(C0, C0 + m);
  // rule table
  std::vector<int32_t> rule_off(m + 1, 0);
  std::vector<DevRule> dr(n);
  s->binary_emit = true;
  s->small_rules = true;
  for (int64_t r = 0; r < n; ++r) {
    const snp_rule& R = rules[r];
    rule_off[R.neuron + 1]++;
    DevRule d{};
    d.c = R.consumed;
    d.p = R.produced;
    if (R.kind == SNP_RE_EXACT) {
      d.lo = std::max(R.a, R.consumed);
      d.hi = R.a;
      d.base = R.a;
      d.j = 1;
    } else if (R.kind == SNP_RE_UNARY) {
      d.lo = R.consumed;
      d.hi = 0x7FFFFFFF;
      d.base = R.a;
      d.j = R.b;
      d.unary = 1;
      for (int64_t v = 0; v < (int64_t)R.a + R.b; ++v)
        if ((re_bits[4 * r + v / 64] >> (v % 64)) & 1ULL) d.bits[v / 64] |= 1ULL << (v % 64);
    } else {
      d.lo = std::max(R.a, R.consumed);
      d.hi = 0x7FFFFFFF;
      d.base = R.a;
      d.j = R.b;
    }
    d.jmask = (d.j & (d.j - 1)) == 0 ? d.j - 1 : -1;
    dr[r] = d;
    if (R.produced > 1) s->binary_emit = false;
    if (R.consumed > 255 || R.produced > 255) s->small_rules = false;
  }
  for (int64_t j = 0; j < m; ++j) rule_off[j + 1] += rule_off[j];
  // fingerprint weights R_ℓ[j] = splitmix64(seed_ℓ ^ j) | 1 and h_ℓ[r] = Σ_j M[r][j]·R_ℓ[j]
  std::vector<uint64_t> R0(m), R1(m), h0(n, 0), h1(n, 0);
  for (int64_t j = 0; j < m; ++j) {
    R0[j] = splitmix64(s->opt.fp_seed[0] ^ (uint64_t)j) | 1ULL;
    R1[j] = splitmix64(s->opt.fp_seed[1] ^ (uint64_t)j) | 1ULL;
  }
  for (int64_t r = 0; r < n; ++r)
    for (auto& jv : rows[r]) {
      h0[r] += (uint64_t)(int64_t)jv.second * R0[jv.first];
      h1[r] += (uint64_t)(int64_t)jv.second * R1[jv.first];
    }
  // synapse graph: out-CSR (by source) and in-CSR (by target)
  std::vector<int32_t> out_off(m + 1, 0), out_dst, in_off(m + 1, 0), in_src;
  for (int64_t s_ = 0; s_ < m; ++s_) out_off[s_ + 1] = out_off[s_] + (int32_t)out_syn[s_].size();
  out_dst.reserve(out_off[m]);
  for (int64_t s_ = 0; s_ < m; ++s_) out_dst.insert(out_dst.end(), out_syn[s_].begin(), out_syn[s_].end());
  for (int64_t s_ = 0; s_ < m; ++s_)
    for (int32_t j : out_syn[s_]) in_off[j + 1]++;
  for (int64_t j = 0; j < m; ++j) in_off[j + 1] += in_off[j];
  in_src.assign(in_off[m], 0);
  {
    std::vector<int32_t> fill(in_off.begin(), in_off.end() - 1);
    for (int64_t s_ = 0; s_ < m; ++s_)
      for (int32_t j : out_syn[s_]) in_src[fill[j]++] = (int32_t)s_;
  }
  SNP_TRY(upload(s, s->d_rule_off, rule_off));
  SNP_TRY(upload(s, s->d_rules, dr));
  SNP_TRY(upload(s, s->d_h0, h0));
  SNP_TRY(upload(s, s->d_h1, h1));
  SNP_TRY(upload(s, s->d_in_off, in_off));
  SNP_TRY(upload(s, s->d_in_src, in_src));
  // edge-major padded in-CSR per group of 32 targets (coalesced K-c gathers)
  {
    const int64_t ng = (m + 31) / 32;
    const int32_t pad = (int32_t)((m + 1) & ~1);  // index of the zero emit word
    std::vector<int64_t> pad_off(ng + 1, 0);
    for (int64_t g = 0; g < ng; ++g) {
      int32_t mx = 0;
      for (int64_t j = 32 * g; j < std::min<int64_t>(m, 32 * g + 32); ++j) mx = std::max(mx, in_off[j + 1] - in_off[j]);
      pad_off[g + 1] = pad_off[g] + (mx + 3) / 4 * 4;  // K-c consumes rows in blocks of 8 and 4
    }
    std::vector<int32_t> in_pad((size_t)pad_off[ng] * 32, pad);
    const char* bk = getenv("SNP_INPAD_BANKS");
    const bool banks = !(bk && bk[0] == '0');
    std::vector<std::vector<int32_t>> lane_src(16), lane_row;
    for (int64_t g = 0; g < ng; ++g) {
      if (banks) {
        // each half-warp's rows bank-conflict-free in K-c's staged emit words
        for (int h = 0; h < 2; ++h) {
          for (int l = 0; l < 16; ++l) {
            lane_src[l].clear();
            const int64_t j = 32 * g + 16 * h + l;
            if (j < m) lane_src[l].assign(in_src.begin() + in_off[j], in_src.begin() + in_off[j + 1]);
          }
          const int64_t R = pad_off[g + 1] - pad_off[g];
          bank_rows(lane_src, (int)R, lane_row);
          for (int64_t r = 0; r < R; ++r) {
            // the half-row's padding lanes read one of the EPAD zero words, in
            // a bank pair none of its real sources uses (broadcast, no conflict)
            unsigned used = 0;
            for (int l = 0; l < 16; ++l)
              if (r < (int64_t)lane_row[l].size() && lane_row[l][r] >= 0) used |= 1u << (lane_row[l][r] & 15);
            int z = 0;
            while (z < 15 && ((used >> ((pad + z) & 15)) & 1u)) ++z;
            for (int l = 0; l < 16; ++l) {
              const bool real = r < (int64_t)lane_row[l].size() && lane_row[l][r] >= 0;
              in_pad[(size_t)(pad_off[g] + r) * 32 + 16 * h + l] = real ? lane_row[l][r] : pad + z;
            }
          }
        }
        continue;
      }
      for (int64_t j = 32 * g; j < std::min<int64_t>(m, 32 * g + 32); ++j)
        for (int32_t e = in_off[j]; e < in_off[j + 1]; ++e)
          in_pad[(size_t)(pad_off[g] + (e - in_off[j])) * 32 + (j - 32 * g)] = in_src[e];
    }
    SNP_TRY(upload(s, s->d_in_pad, in_pad));
    if (m + EPAD < 65535) {
      std::vector<uint16_t> in16(in_pad.begin(), in_pad.end());
      SNP_TRY(upload(s, s->d_in_pad16, in16));
      std::vector<uint64_t> in4(in16.size() / 4);  // rows per group are a multiple of 4
      for (size_t q = 0; q < in4.size(); ++q) {
        const size_t rq = q / 32, l = q % 32;
        uint64_t v = 0;
        for (int u = 0; u < 4; ++u) v |= (uint64_t)in16[(4 * rq + u) * 32 + l] << (16 * u);
        in4[q] = v;
      }
      SNP_TRY(upload(s, s->d_in_pad16x4, in4));
    }
    SNP_TRY(upload(s, s->d_in_pad_off, pad_off));
  }
  SNP_TRY(upload(s, s->d_out_off, out_off));
  SNP_TRY(upload(s, s->d_out_dst, out_dst));
  SNP_TRY(upload(s, s->d_R0, R0));
  SNP_TRY(upload(s, s->d_R1, R1));
  // ---- per-neuron outcome-table descriptors: for counts
  // v >= L the applicable set repeats with period P = lcm of the PERIODIC
  // rules' j; counts never exceed count_max.  Neurons with > 15 rules or a
  // table wider than TABW_MAX are evaluated rule by rule (NM_GENERIC).
  std::vector<NeuronMeta> meta(m);
  int64_t tabw = 16;
  for (int64_t j = 0; j < m; ++j) {
    const int32_t r0 = rule_off[j], r1 = rule_off[j + 1];
    int64_t L = 0, P = 1;
    bool ok = (r1 - r0) <= MAX_TABLE_RULES;
    for (int32_t r = r0; r < r1 && ok; ++r) {
      const snp_rule& R = rules[r];
      if (R.kind == SNP_RE_EXACT) {
        L = std::max<int64_t>(L, (int64_t)R.a + 1);
      } else if (R.kind == SNP_RE_UNARY) {  // membership repeats with period P from t on
        L = std::max<int64_t>(L, std::max<int64_t>(R.a, R.consumed));
        const int64_t g = std::__gcd<int64_t>(P, R.b);
        P = P / g * R.b;
        if (P > TABW_MAX) ok = false;
      } else {
        L = std::max<int64_t>(L, std::max<int64_t>(R.a, R.consumed));
        const int64_t g = std::__gcd<int64_t>(P, R.b);
        P = P / g * R.b;
        if (P > TABW_MAX) ok = false;
      }
    }
    if (ok && L > s->count_max + 1) { L = s->count_max + 1; P = 1; }
    if (ok && L + P > TABW_MAX) ok = false;
    NeuronMeta mt{r0, (int32_t)L, (P & (P - 1)) == 0 ? (int32_t)(P - 1) : (int32_t)(-P), ok ? 0 : NM_GENERIC};
    if (!ok) { mt.L = 0; mt.pm = 0; }
    else tabw = std::max<int64_t>(tabw, L + P);
    meta[j] = mt;
  }
  // power of two >= every L + P: a count v < tabw indexes its own entry
  // (every slot holds the outcome at v = slot), larger counts fold
  {
    int64_t w = 16;
    while (w < tabw) w <<= 1;
    tabw = w;
  }
  int32_t max_indeg = 0;
  for (int64_t j = 0; j < m; ++j) max_indeg = std::max(max_indeg, in_off[j + 1] - in_off[j]);
  SNP_TRY(upload(s, s->d_meta, meta));
  SNP_TRY(s->d_tab.ensure((size_t)m * tabw, false));
  SNP_TRY(s->d_ctab.ensure((size_t)m * tabw * s->bytes, false));
  SNP_TRY(s->d_tab_full.ensure((size_t)m * 256, false));  // wide counts: host-side X|Y tables of the TC K-a
  SNP_TRY(s->d_ttab.ensure((size_t)m * (32 + 256), false));  // every width (K-c NARROW for 16/32-bit counts)
  if (s->bytes == 1) SNP_TRY(s->d_elut.ensure((size_t)m * 32, false));
  if (s->bytes == 1) SNP_TRY(s->d_hsg.ensure((size_t)m * 256, false));
  SysView& v = s->view;
  v.tables_ok = 1;
  v.tabw = (int32_t)tabw;
  v.full8 = s->bytes == 1 ? 1 : 0;
  v.max_indeg = max_indeg;
  v.n_in = in_off[m];
  v.meta = s->d_meta.as<NeuronMeta>();
  v.tab = s->d_tab.as<uint8_t>();
  v.tab_full = s->bytes == 1 ? s->d_tab_full.as<uint8_t>() : nullptr;
  v.ctab = s->d_ctab.p;
  v.ttab = s->d_ttab.as<uint8_t>();
  v.elut = s->bytes == 1 ? s->d_elut.as<uint8_t>() : nullptr;
  v.hsg = s->bytes == 1 ? s->d_hsg.as<uint8_t>() : nullptr;
  v.any_generic = 0;
  for (int64_t j = 0; j < m; ++j) v.any_generic |= (meta[j].flags & NM_GENERIC) ? 1 : 0;
  {
    // SNP_KERNELS (tests / tuning): "expand_t" = the 8-configuration-per-lane
    // K-a for uint8 too; "kc_global_e" = K-c reads emit words from global
    // memory even when they fit in shared memory (the large-m path); "kc_tc"
    // = K-c's output permutation on the tensor cores (measured slower)
    const char* k = getenv("SNP_KERNELS");
    v.kernel_flags = 0;
    v.small_cp = s->small_rules ? 1 : 0;  // c, p <= 255: packed (c, p) tables in the verification
    v.aug_rule = -1;  // set by snp_load after the tables are built
    v.aug_neuron = -1;
    if (k && strstr(k, "expand_t")) v.kernel_flags |= KF_EXPAND_T;
    if (k && strstr(k, "kc_global_e")) v.kernel_flags |= KF_KC_GLOBAL_E;
    if (k && strstr(k, "no_tc")) v.kernel_flags |= KF_NO_TC;
    if (k && strstr(k, "kc_tc")) v.kernel_flags |= KF_KC_TC;
    if (k && strstr(k, "kc_wide_exact")) v.kernel_flags |= KF_KC_WIDE_EXACT;  // 16/32-bit K-c in full width
    if (k && strstr(k, "fp_weak")) v.kernel_flags |= KF_FP_WEAK;  // tests: 6-bit child keys (the verification must object)
  }
  v.m = (int32_t)m;
  v.n = n;
  v.binary_emit = s->binary_emit ? 1 : 0;
  v.count_max = s->count_max;
  v.rule_off = s->d_rule_off.as<int32_t>();
  v.rules = s->d_rules.as<DevRule>();
  v.h0 = s->d_h0.as<uint64_t>();
  v.h1 = s->d_h1.as<uint64_t>();
  v.in_off = s->d_in_off.as<int32_t>();
  v.in_src = s->d_in_src.as<int32_t>();
  v.in_pad = s->d_in_pad.as<int32_t>();
  v.in_pad16 = m + EPAD < 65535 ? s->d_in_pad16.as<uint16_t>() : nullptr;
  v.in_pad16x4 = m + EPAD < 65535 ? s->d_in_pad16x4.as<uint64_t>() : nullptr;
  v.in_pad_off = s->d_in_pad_off.as<int64_t>();
  v.out_off = s->d_out_off.as<int32_t>();
  v.out_dst = s->d_out_dst.as<int32_t>();
  v.R0 = s->d_R0.as<uint64_t>();
  v.R1 = s->d_R1.as<uint64_t>();
  SNP_TRY(s->counters_dev.ensure(sizeof(DevCounters), false));
  CUDA_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  s->own_stream = true;
  launch_build_tables(v, s->bytes, s->d_tab.as<uint8_t>(), s->d_ctab.p, s->d_tab_full.as<uint8_t>(),
                      s->d_ttab.as<uint8_t>(),
                      s->bytes == 1 ? s->d_elut.as<uint8_t>() : nullptr,
                      s->bytes == 1 ? s->d_hsg.as<uint8_t>() : nullptr, s->stream);
  CUDA_TRY(cudaGetLastError());
  v.cpT = nullptr;
  if (s->small_rules) {  // count-major first-rule (c, p) for counts < 32 (k_verify_m)
    SNP_TRY(s->d_cpT.ensure((size_t)32 * m * 2, false));
    launch_build_cpT(v, s->d_cpT.as<uint16_t>(), s->stream);
    CUDA_TRY(cudaGetLastError());
    v.cpT = s->d_cpT.as<uint16_t>();
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  // ---- tensor-core K-a (k_expand_tc): X|Y bytes of the first
  // applicable rule per (neuron, count), the B operand chunks (byte planes of
  // −R_ℓ[s] and Rout_ℓ[s] = Σ_{j ∈ out(s)} R_ℓ[j]) and the neurons that can be
  // nondeterministic.  Applies when every rule delta decomposes as
  // h_ℓ[r] = −c_r·R_ℓ[s] + p_r·Rout_ℓ[s] (reading A18) with c <= 15, p <= 1.
  v.tc_ok = 0;
  v.n_nd = 0;
  // the s32 TMEM accumulators of k_expand_tc hold at most m·15·255 (X part)
  // and m·16·255 (Y' part): exact below 2^31 for m <= TC_M_MAX = 2^19
  // 16/32-bit counts (NARROW: low bytes, exact lookups for counts >= 256)
  // when every rule has c <= 15, p <= 1; ND-capable neurons then from the
  // folded table, which covers every count
  bool wide_ok = s->bytes == 1;
  if (s->bytes > 1) {
    wide_ok = true;
    for (int64_t r = 0; r < n; ++r) wide_ok &= rules[r].consumed <= 15 && rules[r].produced <= 1;
  }
  if (wide_ok && !v.any_generic && s->binary_emit && m <= TC_M_MAX) {
    std::vector<uint8_t> tf((size_t)m * 256), tw;
    CUDA_TRY(cudaMemcpy(tf.data(), s->d_tab_full.p, tf.size(), cudaMemcpyDeviceToHost));
    if (s->bytes > 1) {
      tw.resize((size_t)m * tabw);
      CUDA_TRY(cudaMemcpy(tw.data(), s->d_tab.p, tw.size(), cudaMemcpyDeviceToHost));
    }
    bool ok = true;
    std::vector<uint8_t> xyf((size_t)m * 256, 0), xyt((size_t)((m + 63) / 64) * 64 * 32, 0);  // whole chunks
    std::vector<int32_t> ndl;
    for (int64_t j = 0; j < m && ok; ++j) {
      bool nd = false;
      for (int64_t c = 0; c < 256; ++c) {
        const uint8_t e = tf[(size_t)j * 256 + c];
        nd |= (e & TE_ND) != 0;
        const int f = e >> 4;
        if (!f) continue;
        const snp_rule& R = rules[rule_off[j] + f - 1];
        if (R.consumed > 15 || R.produced > 1) { ok = false; break; }
        xyf[(size_t)j * 256 + c] = (uint8_t)(R.consumed | (R.produced << 4));
      }
      if (s->bytes > 1)
        for (int64_t c = 0; c < tabw; ++c) nd |= (tw[(size_t)j * tabw + c] & TE_ND) != 0;
      if (nd) ndl.push_back((int32_t)j);
      std::copy(xyf.begin() + j * 256, xyf.begin() + j * 256 + 32, xyt.begin() + j * 32);
    }
    std::vector<uint64_t> Ro0(m, 0), Ro1(m, 0);
    for (int64_t j = 0; j < m; ++j)
      for (int32_t t : out_syn[j]) { Ro0[j] += R0[t]; Ro1[j] += R1[t]; }
    for (int64_t r = 0; r < n && ok; ++r) {
      const snp_rule& R = rules[r];
      const uint64_t c = (uint64_t)(int64_t)R.consumed, p = (uint64_t)(int64_t)R.produced;
      if (h0[r] != (0 - c) * R0[R.neuron] + p * Ro0[R.neuron] || h1[r] != (0 - c) * R1[R.neuron] + p * Ro1[R.neuron])
        ok = false;
    }
    if ((int64_t)ndl.size() > KMAX) ok = false;
    if (ok) {
      const int64_t nch = (m + 63) / 64;
      std::vector<uint8_t> bt((size_t)nch * 4096, 0);
      for (int64_t j = 0; j < m; ++j) {
        const int64_t ch = j / 64, k = j % 64;
        auto put = [&](int half, int col, uint64_t w) {
          bt[(size_t)ch * 4096 + half * 2048 + (k / 16) * 512 + (col / 8) * 128 + (col % 8) * 16 + k % 16] =
              (uint8_t)w;
        };
        for (int b = 0; b < 8; ++b) {
          put(0, b, (0 - R0[j]) >> (8 * b));
          put(0, 8 + b, (0 - R1[j]) >> (8 * b));
          put(1, b, Ro0[j] >> (8 * b));
          put(1, 8 + b, Ro1[j] >> (8 * b));
        }
        put(0, 16, 1);  // total consumption: 0 <=> halting
      }
      SNP_TRY(upload(s, s->d_xyt, xyt));
      SNP_TRY(upload(s, s->d_xyf, xyf));
      SNP_TRY(upload(s, s->d_btile, bt));
      SNP_TRY(upload(s, s->d_ndl, ndl));
      v.tc_ok = 1;
      v.n_nd = (int32_t)ndl.size();
      v.nd_list = s->d_ndl.as<int32_t>();
      v.xyt = s->d_xyt.as<uint8_t>();
      v.xyf = s->d_xyf.as<uint8_t>();
      v.btile = s->d_btile.as<uint8_t>();
    }
  }
  CUDA_TRY(cudaEventCreate(&s->ev0));
  CUDA_TRY(cudaEventCreate(&s->ev1));
  return SNP_OK;
}

// ---------------------------------------------------------------------------
// exploration
// ---------------------------------------------------------------------------
snp_status reset_state(snp_system* s) {
  s->dist.P = 0;
  s->dist.stage = 0;
  for (double& x : s->prof_ms) x = 0;
  s->marks.clear();
  s->ev_used = 0;
  s->levels.clear();  // pooled level buffers are non-owning: the pool is reused from the start
  s->lpool_used = 0;
  for (auto& pl : s->small_pools)
    if (s->small_spare.size() < 8) s->small_spare.push_back(std::move(pl));
  s->small_pools.clear();
  s->small_skip = (size_t)-1;
  s->arena.reset();
  s->counters.clear();
  s->n_visited = 0;
  s->total_T = 0;
  s->digest = 0;
  s->begun = false;
  s->generation++;
  s->halting_current_valid = false;
  if (s->vis_cap) CUDA_TRY(cudaMemsetAsync(s->vis.p, 0xFF, s->vis_cap * sizeof(Slot), s->stream));
  return SNP_OK;
}

snp_status zero_counters(snp_system* s) {
  CUDA_TRY(cudaMemsetAsync(s->counters_dev.p, 0, sizeof(DevCounters), s->stream));
  return SNP_OK;
}

// entries of the K-c overflow list (2^22; SNP_OVF_CAP overrides it for tests)
uint64_t ovf_capacity() {
  const char* e = getenv("SNP_OVF_CAP");
  const long long v = e ? atoll(e) : 0;
  return v > 0 ? (uint64_t)v : (1ULL << 22);
}
DevCounters* dc(snp_system* s) { return s->counters_dev.as<DevCounters>(); }

// 16/32-bit counts: K-c computes x in bytes (NARROW) and lists every x outside
// [0, 255] for an exact rewrite; a level with more of them than the list holds
// is materialised again in full width (K-c and k_patch overwrite every kept
// child, so nothing of the first pass survives)
snp_status rematerialize_wide(snp_system* s, const LevelView& LV, const ExpandOut& O, const NextArrays& N, int64_t K,
                              uint64_t ovf_cap, int32_t* err, DevCounters* hc) {
  if (hc->n_ovf <= ovf_cap || !materialize_narrow_ok(s->view, s->bytes)) return SNP_OK;
  cudaStream_t st = s->stream;
  SysView wv = s->view;
  wv.kernel_flags |= KF_KC_WIDE_EXACT;
  CUDA_TRY(cudaMemsetAsync(&dc(s)->n_ovf, 0, sizeof(unsigned long long), st));
  phase_begin(s, 3);
  launch_materialize(wv, s->bytes, LV, O, s->kq_off.as<uint64_t>(), N, K, s->ovf.as<uint64_t>(), &dc(s)->n_ovf,
                     ovf_cap, err, st);
  launch_patch(wv, s->bytes, LV, O, N, K, err, st);
  phase_end(s);
  CUDA_TRY(cudaGetLastError());
  return read_counters(s, hc);
}

snp_status begin_impl(snp_system* s, const snp_configs* level0) {
  g_trace.start();
  SNP_TRY(reset_state(s));
  snp_configs c0{};
  if (!level0) {
    c0.data = s->C0.data();
    c0.n_configs = 1;
    c0.elem_bytes = 4;
    c0.layout = SNP_LAYOUT_ROW_MAJOR;
    c0.on_device = 0;
    level0 = &c0;
  }
  const int64_t F0 = level0->n_configs, m = s->m;
  if (F0 < 1 || F0 > 0x7FFFFFFFLL || !level0->data) return fail(SNP_E_ARG, "level0: need 1 <= n_configs < 2^31 and data");
  if (level0->elem_bytes != 1 && level0->elem_bytes != 2 && level0->elem_bytes != 4) return fail(SNP_E_ARG, "level0: elem_bytes");
  if (level0->layout != SNP_LAYOUT_ROW_MAJOR && level0->layout != SNP_LAYOUT_NEURON_MAJOR) return fail(SNP_E_ARG, "level0: layout");
  const int64_t ld = level0->ld ? level0->ld : (level0->layout == SNP_LAYOUT_ROW_MAJOR ? m : F0);
  const size_t in_bytes = (size_t)(level0->layout == SNP_LAYOUT_ROW_MAJOR ? (F0 - 1) * ld + m : (m - 1) * ld + F0) *
                          level0->elem_bytes;
  SNP_TRY(zero_counters(s));
  DBuf raw;
  SNP_TRY(take_buffer(s, level_bytes(F0, m, s->bytes), &raw));
  int32_t* err = &dc(s)->err;
  if (!level0->on_device && level0->layout == SNP_LAYOUT_ROW_MAJOR) {
    // host rows in chunks of R (a multiple of the 64-configuration block, so
    // a chunk's blocks are a contiguous range of the level): two staging
    // buffers, the copy of chunk i + 1 (side stream) overlaps the import of
    // chunk i, and no level-sized staging allocation is needed
    const size_t row_b = (size_t)ld * level0->elem_bytes;
    // chunk bytes: 1 GB (SNP_UPLOAD_CHUNK_BYTES overrides, tests use it to
    // run the multi-chunk path on small inputs); a multiple of 64 rows
    size_t chunk_b = (size_t)1 << 30;
    if (const char* e = getenv("SNP_UPLOAD_CHUNK_BYTES")) chunk_b = std::max<size_t>(1, strtoull(e, nullptr, 10));
    int64_t R = std::max<int64_t>(PB, (int64_t)(chunk_b / row_b) & ~(int64_t)(PB - 1));
    if (R > F0) R = F0;
    DBuf stg[2];
    for (auto& b : stg) SNP_TRY(b.ensure((size_t)((R - 1) * ld + m) * level0->elem_bytes, false));
    // each chunk's copy split over NS side streams (SNP_UPLOAD_STREAMS; 1 by
    // default: 2 streams measured 31 vs 52 GB/s through snp_begin, 3 equal to 1,
    // profiles/r02f/upload_streams.json — one copy engine saturates the link)
    int NS = 1;
    if (const char* e2 = getenv("SNP_UPLOAD_STREAMS")) NS = std::max(1, std::min(4, atoi(e2)));
    cudaStream_t cs[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t copied[2][4] = {}, used[2] = {nullptr, nullptr};
    auto cleanup = [&]() {
      for (int b = 0; b < 2; ++b) {
        for (int k = 0; k < NS; ++k)
          if (copied[b][k]) cudaEventDestroy(copied[b][k]);
        if (used[b]) cudaEventDestroy(used[b]);
      }
      for (int k = 0; k < NS; ++k)
        if (cs[k]) cudaStreamDestroy(cs[k]);
    };
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < NS && e == cudaSuccess; ++k) e = cudaStreamCreateWithFlags(&cs[k], cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
      for (int k = 0; k < NS && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&copied[b][k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&used[b], cudaEventDisableTiming);
    }
    const uint8_t* hsrc = reinterpret_cast<const uint8_t*>(level0->data);
    for (int64_t r0 = 0, i = 0; r0 < F0 && e == cudaSuccess; r0 += R, ++i) {
      const int64_t n = std::min<int64_t>(R, F0 - r0);
      const int b = (int)(i & 1);
      const size_t cb = (size_t)((n - 1) * ld + m) * level0->elem_bytes;
      const size_t piece = (cb / NS + 4095) & ~(size_t)4095;
      for (int k = 0; k < NS && e == cudaSuccess; ++k) {
        const size_t o = (size_t)k * piece;
        if (i >= 2) e = cudaStreamWaitEvent(cs[k], used[b], 0);
        if (e == cudaSuccess && o < cb)
          e = cudaMemcpyAsync(static_cast<uint8_t*>(stg[b].p) + o, hsrc + (size_t)r0 * row_b + o, std::min(piece, cb - o),
                              cudaMemcpyHostToDevice, cs[k]);
        if (e == cudaSuccess) e = cudaEventRecord(copied[b][k], cs[k]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, copied[b][k], 0);
      }
      if (e != cudaSuccess) break;
      launch_import(stg[b].p, level0->elem_bytes, SNP_LAYOUT_ROW_MAJOR, ld, n, (int32_t)m,
                    raw.as<uint8_t>() + (size_t)r0 * m * s->bytes, s->bytes, s->count_max, err, s->stream);
      e = cudaEventRecord(used[b], s->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);  // staging buffers are released below
    cleanup();
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(SNP_E_CUDA, "level0 upload: %s", cudaGetErrorString(e));
    }
  } else {
    // stage other host input on the device in one piece
    DBuf staged;
    const void* src = level0->data;
    if (!level0->on_device) {
      SNP_TRY(staged.ensure(in_bytes, false));
      CUDA_TRY(cudaMemcpyAsync(staged.p, level0->data, in_bytes, cudaMemcpyHostToDevice, s->stream));
      src = staged.p;
    }
    launch_import(src, level0->elem_bytes, level0->layout, ld, F0, (int32_t)m, raw.p, s->bytes, s->count_max, err,
                  s->stream);
    if (!level0->on_device) CUDA_TRY(cudaStreamSynchronize(s->stream));
  }
  CUDA_TRY(cudaGetLastError());
  g_trace.mark("upload");
  // fingerprints of level 0
  DBuf fp0, fp1;
  SNP_TRY(fp0.ensure(F0 * 8, false));
  SNP_TRY(fp1.ensure(F0 * 8, false));
  launch_fingerprint(s->view, s->bytes, raw.p, F0, fp0.as<uint64_t>(), fp1.as<uint64_t>(), s->stream);
  // dedup level 0: first occurrence wins (tags = index)
  SNP_TRY(ensure_children(s, (uint64_t)F0));
  SNP_TRY(ensure_ltab(s, (uint64_t)F0));
  SNP_TRY(ensure_visited(s, 4 * (uint64_t)F0));
  const uint64_t lslots = next_pow2(std::max<uint64_t>(1024, 2 * (uint64_t)F0));
  Tables tb = tables(s, lslots);
  ChildArrays C = child_arrays(s);
  CUDA_TRY(cudaMemcpyAsync(C.cfp0, fp0.p, F0 * 8, cudaMemcpyDeviceToDevice, s->stream));
  CUDA_TRY(cudaMemcpyAsync(C.cfp1, fp1.p, F0 * 8, cudaMemcpyDeviceToDevice, s->stream));
  launch_dedup(C, (uint64_t)F0, 0, tb, 0, err, s->stream);
  launch_winners(C, (uint64_t)F0, 0, tb, &dc(s)->n_new, s->stream);
  launch_keep(C, (uint64_t)F0, 0, tb, 0, 0, s->stream);
  launch_exclusive_scan(s->scan_tmp.p, s->scan_tmp.bytes, C.kept, C.kpos, F0 + 1, s->stream);
  CUDA_TRY(cudaGetLastError());
  DevCounters hc;
  SNP_TRY(read_counters(s, &hc));
  g_trace.mark("fingerprint_dedup");
  SNP_TRY(check_err(hc.err));
  if (s->opt.dedup == 0 && (int64_t)hc.n_new < F0) {
    launch_verify_level0(s->bytes, raw.p, (int32_t)m, C, (uint64_t)F0, tb, err, s->stream);
    CUDA_TRY(cudaGetLastError());
    SNP_TRY(read_counters(s, &hc));
    SNP_TRY(check_err(hc.err));
  }
  const int64_t K = (int64_t)hc.n_new;
  auto L = std::make_unique<Level>();
  SNP_TRY(alloc_level_meta(s, L.get(), K));
  SNP_TRY(ensure_visited(s, (uint64_t)K));
  tb = tables(s, lslots);
  SNP_TRY(s->src_index.ensure(std::max<int64_t>(K, 1) * 8));
  NextArrays N{nullptr, L->parent.as<int64_t>(), L->t.as<uint64_t>(), L->fp0.as<uint64_t>(), L->fp1.as<uint64_t>()};
  launch_level0_compact(C.verdict, C.kept, C.kpos, F0, fp0.as<uint64_t>(), fp1.as<uint64_t>(), N,
                        s->src_index.as<uint64_t>(), tb, 1, err, s->stream);
  if (K == F0) {
    L->data = std::move(raw);
  } else {
    SNP_TRY(take_buffer(s, level_bytes(K, m, s->bytes), &L->data));
    launch_gather_columns(s->bytes, raw.p, s->src_index.as<uint64_t>(), K, (int32_t)m, L->data.p, s->stream);
  }
  N.data = L->data.p;
  launch_zero_tail(s->bytes, L->data.p, K, (int32_t)m, s->stream);
  launch_digest(N, K, 0, 0, 0, &dc(s)->digest, s->stream);
  CUDA_TRY(cudaGetLastError());
  SNP_TRY(read_counters(s, &hc));
  SNP_TRY(check_err(hc.err));
  L->F = K;
  s->digest += hc.digest;
  s->n_visited = K;
  s->levels.push_back(std::move(L));
  s->begun = true;
  s->horizon_reserved = false;
  g_trace.mark("compact_digest");
  const snp_status st = reserve_horizon(s, std::max<int64_t>(K, s->opt.frontier_target));
  g_trace.mark("reserve_horizon");
  g_trace.flush("begin");
  return st;
}

snp_status classify_level(snp_system* s, Level* L) {
  // halting flags of a level that is not expanded (reading A5)
  if (L->F == 0) return SNP_OK;
  SNP_TRY(zero_counters(s));
  ExpandOut O{};
  O.halting = L->halting.as<uint8_t>();
  O.n_halting = &dc(s)->n_halting;
  O.err = &dc(s)->err;
  O.classify_only = 1;
  LevelView LV{L->data.p, L->F, L->fp0.as<uint64_t>(), L->fp1.as<uint64_t>()};
  launch_expand(s->view, s->bytes, LV, O, s->stream);
  CUDA_TRY(cudaGetLastError());
  return sync(s);
}

snp_status advance_impl(snp_system* s, snp_level_counters* out) {
  snp_level_counters lc{};
  Level* cur = s->levels.back().get();
  const int64_t F = cur->F, m = s->m;
  if (F == 0) {
    if (out) *out = lc;
    return SNP_OK;
  }
  if (!cur->has_data()) return fail(SNP_E_STATE, "current level has no data");
  // the parent level of `cur` was kept for snp_level_spiking_vectors until now
  if (!retain_levels(s) && s->levels.size() >= 2) release_level_data(s, s->levels[s->levels.size() - 2].get());
  // the caller may have released its level-0 input since snp_begin
  if (!s->horizon_reserved) SNP_TRY(reserve_horizon(s, std::max<int64_t>(F, s->opt.frontier_target)));
  cudaStream_t st = s->stream;
  g_trace.start();
  CUDA_TRY(cudaEventRecord(s->ev0, st));
  SNP_TRY(zero_counters(s));
  int32_t* err = &dc(s)->err;
  // ---- K-a expand
  SNP_TRY(s->psi.ensure((F + 1) * 8));
  SNP_TRY(s->off.ensure((F + 1) * 8));
  SNP_TRY(s->fpb0.ensure(F * 8));
  SNP_TRY(s->fpb1.ensure(F * 8));
  SNP_TRY(s->ndc.ensure(F * 4));
  SNP_TRY(s->nd.ensure((size_t)F * KMAX * 8));
  g_trace.mark("alloc_a");
  ExpandOut O{};
  O.psi = s->psi.as<uint64_t>();
  O.fpb0 = s->fpb0.as<uint64_t>();
  O.fpb1 = s->fpb1.as<uint64_t>();
  O.ndc = s->ndc.as<int32_t>();
  O.nd = s->nd.as<uint64_t>();
  O.halting = cur->halting.as<uint8_t>();
  O.n_halting = &dc(s)->n_halting;
  O.err = err;
  if (fast_materialize_ok(s->view)) {
    // emit words: one uint64 per (storage block, neuron), rows rounded to even
    SNP_TRY(s->ebits.ensure((size_t)((F + PB - 1) / PB) * (size_t)((m + 1) & ~1) * 8));
    O.ebits = s->ebits.as<uint64_t>();
  }
  CUDA_TRY(cudaMemsetAsync(O.psi + F, 0, 8, st));
  LevelView LV{cur->data.p, F, cur->fp0.as<uint64_t>(), cur->fp1.as<uint64_t>()};
  phase_begin(s, 0);
  launch_expand(s->view, s->bytes, LV, O, st);
  phase_end(s);
  // ---- K-b offsets
  SNP_TRY(s->scan_tmp.ensure(scan_temp_bytes(F + 1) + 256));
  phase_begin(s, 1);
  launch_exclusive_scan(s->scan_tmp.p, s->scan_tmp.bytes, O.psi, s->off.as<uint64_t>(), F + 1, st);
  phase_end(s);
  CUDA_TRY(cudaGetLastError());
  uint64_t T = 0;
  CUDA_TRY(cudaMemcpyAsync(&T, s->off.as<uint64_t>() + F, 8, cudaMemcpyDeviceToHost, st));
  DevCounters hc;
  g_trace.mark("launch_a");
  SNP_TRY(read_counters(s, &hc));
  g_trace.mark("sync_a");
  SNP_TRY(check_err(hc.err));
  lc.parents = F;
  lc.halting = (int64_t)hc.n_halting;
  lc.T = (int64_t)T;
  s->halting_current_valid = true;
  if (s->opt.max_transitions > 0 && (int64_t)T > s->opt.max_transitions)
    return fail(SNP_E_CAPACITY, "level %zu: %llu transitions exceed the budget", s->levels.size() - 1, (unsigned long long)T);
  if (T > 0xFFFFFFFFFFULL) return fail(SNP_E_CAPACITY, "level has more than 2^40 transitions");
  const uint64_t* off = s->off.as<uint64_t>();
  // ---- K-b/K-d children, keys, dedup
  auto next = std::make_unique<Level>();
  int64_t K = 0;
  uint64_t tau = 0;
  if (T > 0) {
    SNP_TRY(ensure_children(s, T));
    SNP_TRY(ensure_ltab(s, T));
    g_trace.mark("alloc_children");
    const uint64_t lslots = next_pow2(std::max<uint64_t>(1024, 2 * T));
    ChildArrays C = child_arrays(s);
    Tables tb = tables(s, lslots);
    const uint64_t tag_base = 0;
    phase_begin(s, 1);
    launch_child_parent(off, F, C.cpar, st);
    if (s->view.delay_m > 0) launch_child_keys_delay(s->view, s->bytes, LV, off, O, T, C, st);
    else launch_child_keys(s->view, off, O, T, C, st);
    if (s->view.aug_rule >= 0) launch_aug_keys(s->view, s->bytes, LV, off, O, T, C, err, st);
    phase_end(s);
    phase_begin(s, 2);
    launch_dedup(C, T, tag_base, tb, 1, err, st);
    launch_winners(C, T, tag_base, tb, &dc(s)->n_new, st);
    phase_end(s);
    CUDA_TRY(cudaGetLastError());
    SNP_TRY(read_counters(s, &hc));
    g_trace.mark("sync_dedup");
    SNP_TRY(check_err(hc.err));
    const int64_t n_new = (int64_t)hc.n_new;
    lc.n_new = n_new;
    const int thin = s->opt.frontier_target > 0 && n_new > s->opt.frontier_target;
    if (thin) {
      unsigned __int128 num = (unsigned __int128)(uint64_t)s->opt.frontier_target << 64;
      tau = (uint64_t)(num / (unsigned __int128)(uint64_t)n_new);
    }
    lc.tau = tau;
    phase_begin(s, 2);
    launch_keep(C, T, tag_base, tb, tau, thin, st);
    launch_exclusive_scan(s->scan_tmp.p, s->scan_tmp.bytes, C.kept, C.kpos, (int64_t)T + 1, st);
    phase_end(s);
    CUDA_TRY(cudaGetLastError());
    uint64_t Kh = 0;
    CUDA_TRY(cudaMemcpyAsync(&Kh, C.kpos + T, 8, cudaMemcpyDeviceToHost, st));
    SNP_TRY(sync(s));
    K = (int64_t)Kh;
    // ---- next level buffers + visited insert
    next->F = K;
    g_trace.mark("sync_keep");
    SNP_TRY(alloc_level_meta(s, next.get(), K));
    g_trace.mark("alloc_meta");
    SNP_TRY(ensure_visited(s, (uint64_t)(s->n_visited + K)));
    g_trace.mark("visited");
    tb = tables(s, lslots);
    NextArrays N{nullptr, next->parent.as<int64_t>(), next->t.as<uint64_t>(), next->fp0.as<uint64_t>(),
                 next->fp1.as<uint64_t>()};
    phase_begin(s, 2);
    launch_compact(C, off, T, N, tb, (uint64_t)s->levels.size() << 40, 1, err, st);
    phase_end(s);
    if (s->opt.keep_all_edges) {  // reading A17: every transition with the configuration it reached
      SNP_TRY(next->all_ref.ensure(T * 8, false));
      SNP_TRY(next->all_off.ensure((size_t)(F + 1) * 8, false));
      launch_all_edges(C, T, tag_base, tb, (uint64_t)s->levels.size() << 40, next->all_ref.as<uint64_t>(), st);
      CUDA_TRY(cudaMemcpyAsync(next->all_off.p, off, (size_t)(F + 1) * 8, cudaMemcpyDeviceToDevice, st));
      next->all_T = (int64_t)T;
      next->all_F = F;
    }
    if (K > 0) {
      SNP_TRY(take_buffer(s, level_bytes(K, m, s->bytes), &next->data));
      g_trace.mark("take_buffer");
      N.data = next->data.p;
      // ---- K-c materialize kept children
      SNP_TRY(s->kq_off.ensure((F + 1) * 8));
      const uint64_t ovf_cap = ovf_capacity();
      SNP_TRY(s->ovf.ensure(ovf_cap * 8));
      phase_begin(s, 3);
      launch_kq_off(off, C.kpos, F, s->kq_off.as<uint64_t>(), st);
      launch_materialize(s->view, s->bytes, LV, O, s->kq_off.as<uint64_t>(), N, K, s->ovf.as<uint64_t>(),
                         &dc(s)->n_ovf, ovf_cap, err, st);
      launch_patch(s->view, s->bytes, LV, O, N, K, err, st);
      phase_end(s);
      CUDA_TRY(cudaGetLastError());
      SNP_TRY(read_counters(s, &hc));
      SNP_TRY(rematerialize_wide(s, LV, O, N, K, ovf_cap, err, &hc));
      if (hc.n_ovf > ovf_cap) return fail(SNP_E_CAPACITY, "too many counts at the storage limit (%llu)", hc.n_ovf);
      lc.overflow_fixes = (int64_t)hc.n_ovf;
      if (hc.n_ovf) {
        phase_begin(s, 3);
        launch_overflow_fix(s->view, s->bytes, LV, O, s->kq_off.as<uint64_t>(), N, s->ovf.as<uint64_t>(), hc.n_ovf,
                            err, st);
        phase_end(s);
        CUDA_TRY(cudaGetLastError());
      }
      if (s->view.aug_rule >= 0) launch_aug_fix(s->view, s->bytes, LV, O, N, K, err, st);
      launch_zero_tail(s->bytes, N.data, K, (int32_t)m, st);
      launch_digest(N, K, (uint64_t)s->levels.size(), 0, 0, &dc(s)->digest, st);
    }
    if (s->opt.dedup == 0) {
      SNP_TRY(update_stored_table(s));
      phase_begin(s, 4);
      SNP_TRY(s->vlist.ensure(std::max<uint64_t>(T, s->child_cap) * 8 + 16));  // sized with the child arrays
      const char* vb = getenv("SNP_VERIFY_BATCH");  // tests: the batched two-pass path
      if (s->view.aug_rule < 0) launch_verify_list(C, T, tag_base, tb, s->vlist.as<uint64_t>(), &dc(s)->n_verify, st);
      if (s->view.aug_rule < 0 && !(vb && vb[0] == '1') &&
          launch_verify_m(s->view, s->bytes, LV, O, off, C, s->vlist.as<uint64_t>(), &dc(s)->n_verify, tag_base, tb,
                          s->stored.as<StoredLevel>(), err, st)) {
        // the key matches listed, then one CTA per match (no host round trip)
      } else if (s->view.aug_rule < 0) {
        // the key matches listed, then verified in batches by the two fully
        // parallel passes (fired (c, p) rows, then one thread per column)
        unsigned long long nv = 0;
        CUDA_TRY(cudaMemcpyAsync(&nv, &dc(s)->n_verify, 8, cudaMemcpyDeviceToHost, st));
        SNP_TRY(sync(s));
        const size_t row = verify2_row_bytes(s->view);
        const uint64_t Bmax = std::max<uint64_t>(1, ((size_t)256 << 20) / row);
        const uint64_t B = std::max<uint64_t>(1, std::min<uint64_t>(nv, Bmax));
        if (nv) SNP_TRY(s->vfc.ensure((size_t)Bmax * row, false));  // one allocation for the run, not per level
        for (uint64_t i0 = 0; i0 < nv; i0 += B)
          launch_verify_batch(s->view, s->bytes, LV, O, off, C, s->vlist.as<uint64_t>(), i0, std::min<uint64_t>(B, nv - i0),
                              tag_base, tb, s->stored.as<StoredLevel>(), s->vfc.p, err, st);
      } else {
        launch_verify(s->view, s->bytes, LV, O, off, C, T, tag_base, tb, s->stored.as<StoredLevel>(),
                      s->vlist.as<uint64_t>(), &dc(s)->n_verify, err, st);
      }
      phase_end(s);
      CUDA_TRY(cudaGetLastError());
    }
  }
  CUDA_TRY(cudaEventRecord(s->ev1, st));
  g_trace.mark("launch_c");
  SNP_TRY(read_counters(s, &hc));
  g_trace.mark("sync_end");
  g_trace.flush("level");
  phase_collect(s);
  SNP_TRY(check_err(hc.err));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  lc.kept = K;
  lc.ms = ms;
  s->digest += hc.digest;
  s->n_visited += K;
  s->total_T += (int64_t)T;
  s->counters.push_back(lc);
  s->levels.push_back(std::move(next));
  s->halting_current_valid = false;
  if (out) *out = lc;
  return SNP_OK;
}

// ---------------------------------------------------------------------------
// small frontiers: up to max_levels levels in one k_small_bfs launch
// (configs 1-2).  *done = levels committed; fewer than asked when a level has
// more than SMALL_T transitions (left for advance_impl), a frontier outgrew
// SMALL_F, or it emptied.  SNP_SMALL=0 turns the path off (tests run both).
// ---------------------------------------------------------------------------
bool small_ok(const snp_system* s) {
  const char* e = getenv("SNP_SMALL");
  const bool off = e && e[0] == '0';
  if (off || s->levels.empty() || s->dist.P != 0 || s->view.aug_rule >= 0 || s->view.delay_m > 0 ||
      s->opt.keep_all_edges || s->levels.size() == s->small_skip)
    return false;
  const Level* cur = s->levels.back().get();
  return cur->F > 0 && cur->F <= SMALL_F && cur->has_data();
}

snp_status advance_small(snp_system* s, int32_t want, int32_t* done) {
  *done = 0;
  Level* cur = s->levels.back().get();
  const int64_t m = s->m, F = cur->F;
  const size_t slot = level_bytes(SMALL_T, m, s->bytes);
  const size_t meta = (size_t)SMALL_T * (8 + 8 + 8 + 8 + 1);
  const size_t per = ((slot + 255) & ~(size_t)255) + ((meta + 255) & ~(size_t)255);
  int32_t L = std::max<int32_t>(1, std::min<int32_t>(want, (int32_t)std::max<size_t>(1, ((size_t)256 << 20) / per)));
  // capacity: every configuration the launch can add enters visited
  SNP_TRY(ensure_visited(s, (uint64_t)s->n_visited + (uint64_t)L * SMALL_F + SMALL_T));
  SNP_TRY(ensure_ltab(s, SMALL_T));
  const uint64_t lslots = next_pow2(std::max<uint64_t>(1024, 2 * (uint64_t)SMALL_T));
  Tables tb = tables(s, lslots);
  // scratch
  const size_t sc_b = (size_t)(SMALL_F + 1) * 8 * 2 + (size_t)SMALL_F * (8 + 8 + 4) + (size_t)SMALL_F * KMAX * 8 +
                      (size_t)SMALL_T * (4 + 8 + 8 + 1 + 8 + 8) + (size_t)(SMALL_T + 1) * 16 + 1024;
  SNP_TRY(s->small_scratch.ensure(sc_b, false));
  uint8_t* sp = s->small_scratch.as<uint8_t>();
  auto take = [&](size_t b) {
    uint8_t* r = sp;
    sp += (b + 15) & ~(size_t)15;
    return r;
  };
  SmallArgs a{};
  a.psi = reinterpret_cast<uint64_t*>(take((SMALL_F + 1) * 8));
  a.off = reinterpret_cast<uint64_t*>(take((SMALL_F + 1) * 8));
  a.fpb0 = reinterpret_cast<uint64_t*>(take(SMALL_F * 8));
  a.fpb1 = reinterpret_cast<uint64_t*>(take(SMALL_F * 8));
  a.ndc = reinterpret_cast<int32_t*>(take(SMALL_F * 4));
  a.nd = reinterpret_cast<uint64_t*>(take((size_t)SMALL_F * KMAX * 8));
  a.cpar = reinterpret_cast<uint32_t*>(take(SMALL_T * 4));
  a.cfp0 = reinterpret_cast<uint64_t*>(take(SMALL_T * 8));
  a.cfp1 = reinterpret_cast<uint64_t*>(take(SMALL_T * 8));
  a.verdict = take(SMALL_T);
  a.cslot = reinterpret_cast<uint64_t*>(take(SMALL_T * 8));
  a.cref = reinterpret_cast<uint64_t*>(take(SMALL_T * 8));
  a.kept = reinterpret_cast<uint64_t*>(take((SMALL_T + 1) * 8));
  a.kpos = reinterpret_cast<uint64_t*>(take((SMALL_T + 1) * 8));
  // pool of the new levels
  DBuf pool;
  for (size_t i = 0; i < s->small_spare.size(); ++i)
    if (s->small_spare[i].bytes >= per * (size_t)L) {
      pool = std::move(s->small_spare[i]);
      s->small_spare.erase(s->small_spare.begin() + (long)i);
      break;
    }
  SNP_TRY(pool.ensure(per * (size_t)L, false));
  uint8_t* pp = pool.as<uint8_t>();
  a.data_pool = pp;
  a.data_stride = (slot + 255) & ~(size_t)255;
  uint8_t* mp = pp + a.data_stride * (size_t)L;
  a.parent_pool = reinterpret_cast<int64_t*>(mp);
  a.t_pool = reinterpret_cast<uint64_t*>(mp + (size_t)L * SMALL_T * 8);
  a.fp0_pool = reinterpret_cast<uint64_t*>(mp + (size_t)L * SMALL_T * 16);
  a.fp1_pool = reinterpret_cast<uint64_t*>(mp + (size_t)L * SMALL_T * 24);
  a.halting_pool = mp + (size_t)L * SMALL_T * 32;
  // dedup = 0: the data of every tree level, the new ones written by the kernel
  std::vector<StoredLevel> st(s->levels.size() + L, StoredLevel{nullptr});
  for (size_t i = 0; i < s->levels.size(); ++i) st[i] = StoredLevel{s->levels[i]->data.p};
  SNP_TRY(s->small_stored.ensure(st.size() * sizeof(StoredLevel) + 16));
  CUDA_TRY(cudaMemcpyAsync(s->small_stored.p, st.data(), st.size() * sizeof(StoredLevel), cudaMemcpyHostToDevice,
                           s->stream));
  SNP_TRY(s->small_out.ensure((size_t)L * sizeof(SmallLevelOut) + 64, false));
  a.data = cur->data.p;
  a.F = F;
  a.fp0 = cur->fp0.as<uint64_t>();
  a.fp1 = cur->fp1.as<uint64_t>();
  a.halting = cur->halting.as<uint8_t>();
  a.level0 = (int32_t)s->levels.size() - 1;
  a.max_levels = L;
  a.tb = tb;
  a.stored = s->small_stored.as<StoredLevel>();
  a.frontier_target = s->opt.frontier_target;
  a.max_transitions = s->opt.max_transitions;
  a.dedup = s->opt.dedup;
  a.out = s->small_out.as<SmallLevelOut>();
  a.levels_done = reinterpret_cast<int32_t*>(s->small_out.as<uint8_t>() + (size_t)L * sizeof(SmallLevelOut));
  CUDA_TRY(cudaMemsetAsync(a.levels_done, 0, 4, s->stream));
  CUDA_TRY(cudaMemsetAsync(a.out, 0, (size_t)L * sizeof(SmallLevelOut), s->stream));
  CUDA_TRY(cudaEventRecord(s->ev0, s->stream));
  launch_small_bfs(s->view, s->bytes, a, s->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(s->ev1, s->stream));
  std::vector<SmallLevelOut> out(L);
  int32_t nd = 0;
  CUDA_TRY(cudaMemcpyAsync(out.data(), a.out, (size_t)L * sizeof(SmallLevelOut), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaMemcpyAsync(&nd, a.levels_done, 4, cudaMemcpyDeviceToHost, s->stream));
  SNP_TRY(sync(s));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  const double ms_lvl = nd > 0 ? ms / nd : 0.0;
  uint8_t* base = pool.as<uint8_t>();
  s->small_pools.push_back(std::move(pool));
  for (int32_t k = 0; k < nd; ++k) {
    Level* prev = s->levels.back().get();
    const SmallLevelOut& o = out[k];
    auto nl = std::make_unique<Level>();
    nl->F = o.kept;
    nl->data.p = base + (size_t)k * a.data_stride;
    nl->data.bytes = slot;
    nl->data.owned = false;
    const size_t mo = a.data_stride * (size_t)L + (size_t)k * SMALL_T * 8;
    nl->parent.p = base + mo;
    nl->t.p = base + mo + (size_t)L * SMALL_T * 8;
    nl->fp0.p = base + mo + (size_t)L * SMALL_T * 16;
    nl->fp1.p = base + mo + (size_t)L * SMALL_T * 24;
    nl->halting.p = base + a.data_stride * (size_t)L + (size_t)L * SMALL_T * 32 + (size_t)k * SMALL_T;
    snp_level_counters lc{};
    lc.parents = prev->F;
    lc.halting = o.n_halting;
    lc.T = o.T;
    lc.n_new = o.n_new;
    lc.kept = o.kept;
    lc.tau = o.tau;
    lc.ms = ms_lvl;
    s->counters.push_back(lc);
    s->digest += o.digest;
    s->n_visited += o.kept;
    s->total_T += o.T;
    s->levels.push_back(std::move(nl));
  }
  // keep_tree = 0: only the newest level and its parent keep their counts
  if (!retain_levels(s))
    for (size_t i = 0; i + 2 < s->levels.size(); ++i)
      if (s->levels[i]->has_data()) release_level_data(s, s->levels[i].get());
  *done = nd;
  if (nd < L && out[nd].stop == 1) s->small_skip = s->levels.size();  // that level goes to advance_impl
  s->halting_current_valid = false;
  if (nd < L && out[nd].err) SNP_TRY(check_err(out[nd].err));
  return SNP_OK;
}

snp_status snapshot(snp_system* s, snp_tree** out) {
  // halting flags of the last level
  Level* last = s->levels.back().get();
  if (!s->halting_current_valid && last->F > 0) {
    if (!last->has_data()) return fail(SNP_E_STATE, "last level has no data");
    SNP_TRY(classify_level(s, last));
    s->halting_current_valid = true;
  }
  auto t = std::make_unique<snp_tree>();
  t->sys = s;
  s->refs++;
  t->generation = s->generation;
  t->m = s->m;
  t->n = s->n;
  t->counters = s->counters;
  int64_t total = 0;
  t->level_offsets.push_back(0);
  for (auto& L : s->levels) {
    total += L->F;
    t->level_offsets.push_back(total);
  }
  t->parent.resize(total);
  t->t.resize(total);
  t->halting.resize(total);
  t->fp.resize(2 * total);
  // every level's arrays packed on the device (one kernel), then one copy per
  // array and one synchronisation (configs 1-2 have hundreds of tiny levels)
  if (total > 0) {
    std::vector<EdgeSrc> src;
    int64_t o = 0, max_F = 0;
    for (auto& L : s->levels) {
      if (L->F)
        src.push_back(EdgeSrc{L->parent.as<int64_t>(), L->t.as<uint64_t>(), L->halting.as<uint8_t>(),
                              L->fp0.as<uint64_t>(), L->fp1.as<uint64_t>(), L->F, o});
      o += L->F;
      max_F = std::max(max_F, L->F);
    }
    const size_t need = src.size() * sizeof(EdgeSrc) + (size_t)total * (8 + 8 + 16 + 1) + 256;
    SNP_TRY(s->snap_scratch.ensure(need));
    uint8_t* b = s->snap_scratch.as<uint8_t>();
    EdgeSrc* d_src = reinterpret_cast<EdgeSrc*>(b);
    int64_t* d_par = reinterpret_cast<int64_t*>(b + ((src.size() * sizeof(EdgeSrc) + 15) & ~(size_t)15));
    uint64_t* d_t = reinterpret_cast<uint64_t*>(d_par + total);
    uint64_t* d_fp = d_t + total;
    uint8_t* d_h = reinterpret_cast<uint8_t*>(d_fp + 2 * total);
    CUDA_TRY(cudaMemcpyAsync(d_src, src.data(), src.size() * sizeof(EdgeSrc), cudaMemcpyHostToDevice, s->stream));
    launch_pack_edges(d_src, (int32_t)src.size(), max_F, d_par, d_t, d_h, d_fp, s->stream);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(t->parent.data(), d_par, (size_t)total * 8, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(t->t.data(), d_t, (size_t)total * 8, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(t->fp.data(), d_fp, (size_t)total * 16, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(t->halting.data(), d_h, (size_t)total, cudaMemcpyDeviceToHost, s->stream));
    SNP_TRY(sync(s));
  }
  *out = t.release();
  return SNP_OK;
}

snp_status tree_check(const snp_tree* t, bool need_data) {
  if (!t) return fail(SNP_E_ARG, "tree is NULL");
  if (need_data) {
    if (!t->sys || t->sys->generation != t->generation) return fail(SNP_E_STATE, "the system has started another exploration since this tree was taken");
    for (size_t i = 0; i + 1 < t->level_offsets.size() && i < t->sys->levels.size(); ++i)
      if (t->sys->levels[i]->F && !t->sys->levels[i]->has_data())
        return fail(SNP_E_STATE, "configurations were not retained (set keep_tree = 1)");
  }
  return SNP_OK;
}

// snp_load_unary / snp_load_delay: validate, widen the state (generated
// numbers: + 1 column; delays: + 2m columns for τ and π), build the device system.
snp_status load_full(const snp_matrix* M, const snp_rule* rules, int64_t n_rules, const uint64_t* re_bits,
                     const int32_t* delays, const int32_t* C0, int64_t m, const snp_options* opt, snp_system** out) {
  if (!M || !C0 || !out || m < 1 || m > 0x7FFFFFFF || n_rules < 0 || (n_rules > 0 && !rules))
    return fail(SNP_E_ARG, "snp_load: bad arguments");
  if (M->n_rules != n_rules || M->n_neurons != m) return fail(SNP_E_ARG, "snp_load: matrix shape != (n_rules, m)");
  if (!M->dense && n_rules > 0 && (!M->row_ptr || !M->col || !M->val)) return fail(SNP_E_ARG, "snp_load: no matrix data");
  snp_options o{};
  o.count_bits = 32;
  o.dedup = 0;
  o.keep_tree = 1;
  o.fp_seed[0] = 0x5EED0;
  o.fp_seed[1] = 0x5EED1;
  if (opt) o = *opt;
  if (o.count_bits != 8 && o.count_bits != 16 && o.count_bits != 32) return fail(SNP_E_ARG, "count_bits must be 8, 16 or 32");
  if (o.dedup != 0 && o.dedup != 1) return fail(SNP_E_ARG, "dedup must be 0 or 1");
  if (o.keep_all_edges != 0 && o.keep_all_edges != 1) return fail(SNP_E_ARG, "keep_all_edges must be 0 or 1");
  if (o.frontier_target < 0 || o.max_transitions < 0) return fail(SNP_E_ARG, "negative frontier_target / max_transitions");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(SNP_E_CUDA, "no CUDA device: the engine has no CPU fallback");
  }
  // generated numbers (include/snp.h): the state gains column m = A, a neuron
  // with no rule and no synapse whose value the engine sets (k_aug_keys,
  // k_aug_fix); M and C0 are widened by one zero column
  const int32_t out_rule = o.out_rule1 - 1;
  if (o.out_rule1 < 0 || out_rule >= n_rules) return fail(SNP_E_ARG, "out_rule1 must be 0 (off) or 1..n_rules");
  // systems with delays (reading A26): + 2m columns τ, π
  if (delays) {
    if (out_rule >= 0) return fail(SNP_E_ARG, "delays and generated numbers cannot be combined");
    if (o.dedup != 1) return fail(SNP_E_ARG, "systems with delays need dedup = 1 (fingerprint keys)");
    for (int64_t r = 0; r < n_rules; ++r)
      if (delays[r] < 0) return fail(SNP_E_ARG, "rule %lld: delay < 0", (long long)r);
  }
  const int64_t extra = out_rule >= 0 ? 1 : (delays ? 2 * m : 0);
  snp_matrix Maug{};
  std::vector<int64_t> arp;
  std::vector<int32_t> acol, aval, aC0;
  if (extra > 0) {
    arp.push_back(0);
    for (int64_t r = 0; r < n_rules; ++r) {
      if (M->dense) {
        for (int64_t j = 0; j < m; ++j)
          if (M->dense[r * m + j]) { acol.push_back((int32_t)j); aval.push_back(M->dense[r * m + j]); }
      } else {
        for (int64_t e = M->row_ptr[r]; e < M->row_ptr[r + 1]; ++e) {
          if (M->col[e] < 0 || M->col[e] >= m) return fail(SNP_E_INVALID_SYSTEM, "M row %lld: column out of range", (long long)r);
          acol.push_back(M->col[e]);
          aval.push_back(M->val[e]);
        }
      }
      arp.push_back((int64_t)acol.size());
    }
    acol.push_back(0);  // keep data() non-null
    aval.push_back(0);
    Maug = snp_matrix{n_rules, m + extra, nullptr, arp.data(), acol.data(), aval.data()};
    aC0.assign(C0, C0 + m);
    aC0.resize(m + extra, 0);
  }
  auto s = std::make_unique<snp_system>();
  s->m = m + extra;
  s->opt = o;
  s->bytes = o.count_bits / 8;
  s->count_max = o.count_bits == 8 ? 255 : o.count_bits == 16 ? 65535 : 0x7FFFFFFF;
  snp_status st = extra > 0 ? load_impl(s.get(), &Maug, rules, n_rules, re_bits, aC0.data())
                            : load_impl(s.get(), M, rules, n_rules, re_bits, C0);
  if (st != SNP_OK) return st;
  s->view.delay_m = 0;
  s->view.delay = nullptr;
  if (delays) {
    SNP_TRY(upload(s.get(), s->d_delay, std::vector<int32_t>(delays, delays + n_rules)));
    s->view.delay_m = (int32_t)m;
    s->view.delay = s->d_delay.as<int32_t>();
    s->view.tc_ok = 0;  // child keys are not linear in the rule choice (reading A26)
  }
  s->view.aug_rule = out_rule;
  s->view.aug_neuron = out_rule >= 0 ? rules[out_rule].neuron : -1;
  s->view.gen_bits = nullptr;
  s->view.gen_cap_bits = 0;
  if (out_rule >= 0) {
    s->view.gen_cap_bits = 1 << 20;
    SNP_TRY(s->gen.ensure((size_t)s->view.gen_cap_bits / 8, false));
    CUDA_TRY(cudaMemset(s->gen.p, 0, (size_t)s->view.gen_cap_bits / 8));
    s->view.gen_bits = s->gen.as<unsigned long long>();
  }
  *out = s.release();
  return SNP_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int snp_abi_version(void) { return SNP_ABI_VERSION; }
const char* snp_last_error(void) { return g_err.c_str(); }

snp_status snp_load(const snp_matrix* M, const snp_rule* rules, int64_t n_rules, const int32_t* C0, int64_t m,
                    const snp_options* opt, snp_system** out) {
  return snp_load_unary(M, rules, n_rules, nullptr, C0, m, opt, out);
}

snp_status snp_load_unary(const snp_matrix* M, const snp_rule* rules, int64_t n_rules, const uint64_t* re_bits,
                          const int32_t* C0, int64_t m, const snp_options* opt, snp_system** out) {
  return load_full(M, rules, n_rules, re_bits, nullptr, C0, m, opt, out);
}

snp_status snp_load_delay(const snp_matrix* M, const snp_rule* rules, int64_t n_rules, const int32_t* delays,
                          const int32_t* C0, int64_t m, const snp_options* opt, snp_system** out) {
  if (!delays && n_rules > 0) return fail(SNP_E_ARG, "snp_load_delay: no delays");
  static const int32_t none = 0;
  return load_full(M, rules, n_rules, nullptr, delays ? delays : &none, C0, m, opt, out);
}

}  // extern "C"

namespace {
void system_destroy(snp_system* s) {
  if (s->stream) cudaStreamSynchronize(s->stream);
  delete s->dist.comm;
  s->dist.comm = nullptr;
  if (s->dist.group) snp::local_group_release(s->dist.group);
  s->levels.clear();
  s->spare.clear();
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  for (auto e : s->ev_pool) cudaEventDestroy(e);
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  delete s;
}
void system_unref(snp_system* s) {
  if (--s->refs == 0) system_destroy(s);
}
}  // namespace

extern "C" {

void snp_system_free(snp_system* s) {
  if (s) system_unref(s);
}

snp_status snp_set_stream(snp_system* s, void* stream) {
  if (!s) return fail(SNP_E_ARG, "NULL system");
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (s->own_stream) cudaStreamDestroy(s->stream);
  if (stream) {
    s->stream = (cudaStream_t)stream;
    s->own_stream = false;
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->own_stream = true;
  }
  return SNP_OK;
}

snp_status snp_begin(snp_system* s, const snp_configs* level0) {
  if (!s) return fail(SNP_E_ARG, "NULL system");
  if (s->view.gen_bits) {
    snp_status z = cudaMemsetAsync(s->view.gen_bits, 0, (size_t)s->view.gen_cap_bits / 8, s->stream) == cudaSuccess
                       ? SNP_OK : fail(SNP_E_CUDA, "clearing the generated-number bitmap failed");
    if (z != SNP_OK) return z;
  }
  snp_status st = begin_impl(s, level0);
  if (st != SNP_OK) s->begun = false;
  return st;
}

snp_status snp_advance(snp_system* s, snp_level_counters* counters) {
  if (!s) return fail(SNP_E_ARG, "NULL system");
  if (!s->begun) return fail(SNP_E_STATE, "snp_advance before snp_begin (or after an error, or in distributed mode)");
  snp_status st = SNP_OK;
  int32_t done = 0;
  if (small_ok(s)) st = advance_small(s, 1, &done);
  if (st == SNP_OK && done == 1) {
    if (counters) *counters = s->counters.back();
  } else if (st == SNP_OK) {
    st = advance_impl(s, counters);
  }
  if (st != SNP_OK) s->begun = false;
  return st;
}

int64_t snp_frontier_size(const snp_system* s) { return (s && !s->levels.empty()) ? s->levels.back()->F : 0; }
int64_t snp_state_width(const snp_system* s) { return s ? s->m : 0; }

snp_status snp_generated_numbers(snp_system* s, uint64_t* words, int64_t n_words, int64_t* max_number) {
  if (!s || n_words < 0) return fail(SNP_E_ARG, "snp_generated_numbers: bad arguments");
  const int64_t nw = s->view.gen_cap_bits / 64;
  std::vector<uint64_t> h((size_t)nw, 0);
  if (nw) {
    CUDA_TRY(cudaMemcpyAsync(h.data(), s->view.gen_bits, (size_t)nw * 8, cudaMemcpyDeviceToHost, s->stream));
    SNP_TRY(sync(s));
  }
  if (words)
    for (int64_t i = 0; i < n_words; ++i) words[i] = i < nw ? h[(size_t)i] : 0;
  if (max_number) {
    *max_number = -1;
    for (int64_t i = nw - 1; i >= 0 && *max_number < 0; --i)
      if (h[(size_t)i]) *max_number = i * 64 + 63 - __builtin_clzll(h[(size_t)i]);
  }
  return SNP_OK;
}
int32_t snp_depth(const snp_system* s) { return s ? (int32_t)s->levels.size() - 1 : -1; }

snp_status snp_summary(const snp_system* s, int64_t* n_configs, int64_t* transitions, uint64_t* digest) {
  if (!s) return fail(SNP_E_ARG, "NULL system");
  if (n_configs) *n_configs = s->n_visited;
  if (transitions) *transitions = s->total_T;
  if (digest) *digest = s->digest;
  return SNP_OK;
}

snp_status snp_set_profiling(snp_system* s, int32_t on) {
  if (!s) return fail(SNP_E_ARG, "NULL system");
  s->profiling = on != 0;
  return SNP_OK;
}

snp_status snp_profile(const snp_system* s, double* ms) {
  if (!s || !ms) return fail(SNP_E_ARG, "snp_profile: bad arguments");
  for (int i = 0; i < SNP_NUM_PHASES; ++i) ms[i] = s->prof_ms[i];
  return SNP_OK;
}

int64_t snp_kernel_launches(void) { return snp::g_kernel_launches.load(); }

snp_status snp_set_device(int32_t device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    return fail(SNP_E_CUDA, "snp_set_device: no CUDA device");
  }
  if (device < 0 || device >= n) return fail(SNP_E_ARG, "snp_set_device: device %d of %d", device, n);
  CUDA_TRY(cudaSetDevice(device));
  return SNP_OK;
}

int32_t snp_kernel_paths(const snp_system* s) {
  if (!s) return 0;
  return (s->view.tc_ok && !(s->view.kernel_flags & (snp::KF_NO_TC | snp::KF_EXPAND_T))) ? SNP_PATH_TC_EXPAND : 0;
}

int64_t snp_level_size(const snp_system* s, int32_t level) {
  if (!s || level < 0 || level >= (int32_t)s->levels.size()) return -1;
  return s->levels[level]->F;
}

snp_status snp_level_edges(snp_system* s, int32_t level, int64_t* parent, uint64_t* t, uint8_t* halting,
                           uint64_t* fp2) {
  if (!s || level < 0 || level >= (int32_t)s->levels.size()) return fail(SNP_E_ARG, "snp_level_edges: bad level");
  Level* L = s->levels[level].get();
  const int64_t F = L->F;
  if (!F) return SNP_OK;
  if (parent) CUDA_TRY(cudaMemcpyAsync(parent, L->parent.p, F * 8, cudaMemcpyDeviceToHost, s->stream));
  if (t) CUDA_TRY(cudaMemcpyAsync(t, L->t.p, F * 8, cudaMemcpyDeviceToHost, s->stream));
  if (halting) {
    // the newest level is classified only once it is expanded (or by
    // snp_explore's snapshot): its flags are not known yet
    if (level == (int32_t)s->levels.size() - 1 && !s->halting_current_valid)
      return fail(SNP_E_STATE, "snp_level_edges: halting flags of level %d are not computed yet (pass halting = NULL)", level);
    CUDA_TRY(cudaMemcpyAsync(halting, L->halting.p, F, cudaMemcpyDeviceToHost, s->stream));
  }
  if (fp2) {  // fp0 / fp1 interleaved on the device (persistent scratch), then one contiguous copy
    SNP_TRY(s->edge_scratch.ensure((size_t)F * 16));
    DBuf& pair = s->edge_scratch;
    CUDA_TRY(cudaMemcpy2DAsync(pair.p, 16, L->fp0.p, 8, 8, F, cudaMemcpyDeviceToDevice, s->stream));
    CUDA_TRY(cudaMemcpy2DAsync(pair.as<uint8_t>() + 8, 16, L->fp1.p, 8, 8, F, cudaMemcpyDeviceToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(fp2, pair.p, (size_t)F * 16, cudaMemcpyDeviceToHost, s->stream));
  }
  return sync(s);
}

snp_status snp_host_alloc(size_t bytes, void** p) {
  if (!p) return fail(SNP_E_ARG, "snp_host_alloc: NULL out pointer");
  *p = nullptr;
  if (!bytes) return SNP_OK;
  if (cudaHostAlloc(p, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(SNP_E_OOM, "snp_host_alloc: cudaHostAlloc failed");
  }
  return SNP_OK;
}

snp_status snp_host_free(void* p) {
  if (p && cudaFreeHost(p) != cudaSuccess) return fail(SNP_E_CUDA, "snp_host_free: cudaFreeHost failed");
  return SNP_OK;
}

snp_status snp_level_columns(snp_system* s, int32_t level, const int64_t* idx, int64_t n, int32_t* out) {
  if (!s || level < 0 || level >= (int32_t)s->levels.size() || (n > 0 && (!idx || !out)))
    return fail(SNP_E_ARG, "snp_level_columns: bad arguments");
  Level* L = s->levels[level].get();
  if (!L->has_data()) return fail(SNP_E_STATE, "level %d counts are not retained", level);
  std::vector<uint64_t> hidx(n);
  for (int64_t i = 0; i < n; ++i) {
    if (idx[i] < 0 || idx[i] >= L->F) return fail(SNP_E_ARG, "snp_level_columns: index out of range");
    hidx[i] = (uint64_t)idx[i];
  }
  if (n == 0) return SNP_OK;
  DBuf didx, cols, rows;
  SNP_TRY(didx.ensure(n * 8, false));
  SNP_TRY(cols.ensure(level_bytes(n, s->m, s->bytes), false));
  SNP_TRY(rows.ensure((size_t)n * s->m * 4, false));
  CUDA_TRY(cudaMemcpyAsync(didx.p, hidx.data(), n * 8, cudaMemcpyHostToDevice, s->stream));
  launch_gather_columns(s->bytes, L->data.p, didx.as<uint64_t>(), n, (int32_t)s->m, cols.p, s->stream);
  launch_export(cols.p, s->bytes, n, (int32_t)s->m, rows.as<int32_t>(), s->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(out, rows.p, (size_t)n * s->m * 4, cudaMemcpyDeviceToHost, s->stream));
  return sync(s);
}

snp_status snp_sample(snp_system* s, int64_t W, int32_t* configs, uint64_t seed, int32_t steps, int32_t input_neuron,
                      const int32_t* train, int32_t train_len, int32_t* halted_step) {
  if (!s || W < 0 || steps < 0 || (W > 0 && (!configs || !halted_step)) || train_len < 0 ||
      (train_len > 0 && !train) || input_neuron >= s->m || input_neuron < -1)
    return fail(SNP_E_ARG, "snp_sample: bad arguments");
  if (s->view.aug_rule >= 0) return fail(SNP_E_STATE, "snp_sample: not available with generated numbers (out_rule1)");
  if (s->view.delay_m > 0) return fail(SNP_E_STATE, "snp_sample: not available for systems with delays");
  const int64_t m = s->m;
  for (int64_t i = 0; i < W * m; ++i)
    if (configs[i] < 0 || configs[i] > s->count_max)
      return fail(SNP_E_ARG, "snp_sample: count %d at walker %lld neuron %lld outside [0, %lld]", configs[i],
                  (long long)(i / m), (long long)(i % m), (long long)s->count_max);
  if (W == 0) return SNP_OK;
  DBuf cur, nxt, fired, halted, dtrain, derr;
  const size_t bytes = (size_t)W * m * 4;
  SNP_TRY(derr.ensure(sizeof(int32_t), false));
  SNP_TRY(cur.ensure(bytes, false));
  SNP_TRY(nxt.ensure(bytes, false));
  SNP_TRY(fired.ensure(2 * bytes, false));
  SNP_TRY(halted.ensure((size_t)W * 4, false));
  SNP_TRY(dtrain.ensure(std::max<size_t>(1, (size_t)train_len) * 4, false));
  CUDA_TRY(cudaMemsetAsync(derr.p, 0, sizeof(int32_t), s->stream));
  CUDA_TRY(cudaMemcpyAsync(cur.p, configs, bytes, cudaMemcpyHostToDevice, s->stream));
  if (train_len > 0)
    CUDA_TRY(cudaMemcpyAsync(dtrain.p, train, (size_t)train_len * 4, cudaMemcpyHostToDevice, s->stream));
  launch_sample(s->view, W, cur.as<int32_t>(), nxt.as<int32_t>(), fired.as<uint64_t>(), seed, steps, input_neuron,
                dtrain.as<int32_t>(), train_len, halted.as<int32_t>(), derr.as<int32_t>(), s->small_rules, s->stream);
  CUDA_TRY(cudaGetLastError());
  int32_t err = 0;
  CUDA_TRY(cudaMemcpyAsync(&err, derr.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (err & ERR_CAPACITY) return fail(SNP_E_CAPACITY, "snp_sample: a walker has more than 2^62 children");
  if (err & ERR_OVERFLOW) return fail(SNP_E_OVERFLOW, "snp_sample: a count left [0, %lld]", (long long)s->count_max);
  CUDA_TRY(cudaMemcpyAsync(configs, cur.p, bytes, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaMemcpyAsync(halted_step, halted.p, (size_t)W * 4, cudaMemcpyDeviceToHost, s->stream));
  return sync(s);
}

snp_status snp_explore(snp_system* s, const snp_configs* level0, int32_t depth, snp_tree** out) {
  if (!s || !out || depth < 0) return fail(SNP_E_ARG, "snp_explore: bad arguments");
  snp_status st = snp_begin(s, level0);
  if (st != SNP_OK) return st;
  for (int32_t d = 0; d < depth;) {
    if (s->levels.back()->F == 0) break;
    int32_t done = 0;
    if (small_ok(s)) {  // several small levels per launch
      st = advance_small(s, depth - d, &done);
      if (st != SNP_OK) {
        s->begun = false;
        return st;
      }
    }
    if (done == 0) {
      st = snp_advance(s, nullptr);
      if (st != SNP_OK) return st;
      done = 1;
    }
    d += done;
    if (s->levels.back()->F == 0) break;
  }
  return snapshot(s, out);
}

snp_status snp_step(snp_system* s, const snp_configs* frontier, snp_tree** out) {
  return snp_explore(s, frontier, 1, out);
}

int32_t snp_tree_num_levels(const snp_tree* t) { return t ? (int32_t)t->level_offsets.size() - 1 : 0; }
int64_t snp_tree_num_configs(const snp_tree* t) { return t ? t->level_offsets.back() : 0; }

snp_status snp_tree_level_offsets(const snp_tree* t, int64_t* out) {
  SNP_TRY(tree_check(t, false));
  std::copy(t->level_offsets.begin(), t->level_offsets.end(), out);
  return SNP_OK;
}

snp_status snp_tree_edges(const snp_tree* t, int64_t* parent, uint64_t* tt, uint8_t* halting, uint64_t* fp2) {
  SNP_TRY(tree_check(t, false));
  if (parent) std::copy(t->parent.begin(), t->parent.end(), parent);
  if (tt) std::copy(t->t.begin(), t->t.end(), tt);
  if (halting) std::copy(t->halting.begin(), t->halting.end(), halting);
  if (fp2) std::copy(t->fp.begin(), t->fp.end(), fp2);
  return SNP_OK;
}

snp_status snp_tree_counters(const snp_tree* t, snp_level_counters* out) {
  SNP_TRY(tree_check(t, false));
  std::copy(t->counters.begin(), t->counters.end(), out);
  return SNP_OK;
}

snp_status snp_tree_configs(const snp_tree* t, int32_t* out) {
  SNP_TRY(tree_check(t, true));
  snp_system* s = t->sys;
  DBuf tmp;
  const int32_t nl = snp_tree_num_levels(t);
  // consecutive levels exported into one staging buffer of up to 1 GB (or one
  // level when larger), one copy and one synchronisation per batch
  const size_t cap = std::max<size_t>((size_t)1 << 30, 0);
  for (int32_t L0 = 0; L0 < nl;) {
    size_t bytes = 0;
    int32_t L1 = L0;
    while (L1 < nl && (L1 == L0 || bytes + (size_t)s->levels[L1]->F * s->m * 4 <= cap))
      bytes += (size_t)s->levels[L1++]->F * s->m * 4;
    if (bytes) {
      SNP_TRY(tmp.ensure(bytes));
      size_t o = 0;
      for (int32_t L = L0; L < L1; ++L) {
        const Level* lv = s->levels[L].get();
        if (!lv->F) continue;
        launch_export(lv->data.p, s->bytes, lv->F, (int32_t)s->m, reinterpret_cast<int32_t*>(tmp.as<uint8_t>() + o),
                      s->stream);
        o += (size_t)lv->F * s->m * 4;
      }
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpyAsync(out + t->level_offsets[L0] * s->m, tmp.p, bytes, cudaMemcpyDeviceToHost, s->stream));
      SNP_TRY(sync(s));
    }
    L0 = L1;
  }
  return SNP_OK;
}

snp_status snp_tree_spiking_vectors(const snp_tree* t, int32_t level, uint8_t* S_out) {
  SNP_TRY(tree_check(t, true));
  snp_system* s = t->sys;
  if (level < 1 || level >= snp_tree_num_levels(t)) return fail(SNP_E_ARG, "level must be in [1, num_levels)");
  if (s->view.delay_m > 0) return fail(SNP_E_STATE, "spiking vectors of systems with delays are not available");
  const Level* par = s->levels[level - 1].get();
  const Level* lv = s->levels[level].get();
  if (!lv->F) return SNP_OK;
  DBuf tmp;
  SNP_TRY(tmp.ensure((size_t)lv->F * s->n));
  launch_spiking_vectors(s->view, s->bytes, par->data.p, lv->parent.as<int64_t>(), lv->t.as<uint64_t>(),
                         lv->F, tmp.as<uint8_t>(), nullptr, s->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(S_out, tmp.p, (size_t)lv->F * s->n, cudaMemcpyDeviceToHost, s->stream));
  return sync(s);
}

void snp_tree_free(snp_tree* t) {
  if (!t) return;
  snp_system* s = t->sys;
  delete t;
  if (s) system_unref(s);
}

snp_status snp_level_spiking_vectors(snp_system* s, int32_t level, const int64_t* idx, int64_t n, uint8_t* S_out) {
  if (!s || level < 1 || level >= (int32_t)s->levels.size() || n < 0 || (n > 0 && (!idx || !S_out)))
    return fail(SNP_E_ARG, "snp_level_spiking_vectors: bad arguments");
  if (s->view.delay_m > 0) return fail(SNP_E_STATE, "spiking vectors of systems with delays are not available");
  const Level* par = s->levels[level - 1].get();
  const Level* lv = s->levels[level].get();
  if (!par->has_data()) return fail(SNP_E_STATE, "level %d counts are not retained (keep_tree = 0: only the newest level's parents)", level - 1);
  if (n == 0) return SNP_OK;
  std::vector<int64_t> hp(n);
  std::vector<uint64_t> ht(n), hi(n);
  for (int64_t i = 0; i < n; ++i) {
    if (idx[i] < 0 || idx[i] >= lv->F) return fail(SNP_E_ARG, "snp_level_spiking_vectors: index out of range");
    hi[i] = (uint64_t)idx[i];
  }
  DBuf didx, dpar, dt, out;
  SNP_TRY(didx.ensure(n * 8, false));
  SNP_TRY(dpar.ensure(n * 8, false));
  SNP_TRY(dt.ensure(n * 8, false));
  SNP_TRY(out.ensure((size_t)n * s->n + 16, false));
  CUDA_TRY(cudaMemcpyAsync(didx.p, hi.data(), n * 8, cudaMemcpyHostToDevice, s->stream));
  // (parent, t) of the requested configurations, gathered on the host side of
  // two small copies (the level's edge arrays stay on the device)
  std::vector<int64_t> allp(lv->F);
  std::vector<uint64_t> allt(lv->F);
  CUDA_TRY(cudaMemcpyAsync(allp.data(), lv->parent.p, lv->F * 8, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaMemcpyAsync(allt.data(), lv->t.p, lv->F * 8, cudaMemcpyDeviceToHost, s->stream));
  SNP_TRY(sync(s));
  for (int64_t i = 0; i < n; ++i) {
    hp[i] = allp[hi[i]];
    ht[i] = allt[hi[i]];
  }
  CUDA_TRY(cudaMemcpyAsync(dpar.p, hp.data(), n * 8, cudaMemcpyHostToDevice, s->stream));
  CUDA_TRY(cudaMemcpyAsync(dt.p, ht.data(), n * 8, cudaMemcpyHostToDevice, s->stream));
  launch_spiking_vectors(s->view, s->bytes, par->data.p, dpar.as<int64_t>(), dt.as<uint64_t>(), n, out.as<uint8_t>(),
                         nullptr, s->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(S_out, out.p, (size_t)n * s->n, cudaMemcpyDeviceToHost, s->stream));
  return sync(s);
}

snp_status snp_spiking_vector(snp_system* s, const int32_t* C, uint64_t t, uint8_t* S_out) {
  if (!s || !C || !S_out) return fail(SNP_E_ARG, "snp_spiking_vector: bad arguments");
  if (s->view.delay_m > 0) return fail(SNP_E_STATE, "spiking vectors of systems with delays are not available");
  const int64_t m = s->m;
  for (int64_t j = 0; j < m; ++j)
    if (C[j] < 0 || C[j] > s->count_max) return fail(SNP_E_ARG, "snp_spiking_vector: count %d at neuron %lld outside [0, %lld]", C[j], (long long)j, (long long)s->count_max);
  DBuf row, blk, dpar, dt, out, derr;
  SNP_TRY(row.ensure((size_t)m * 4, false));
  SNP_TRY(blk.ensure(level_bytes(1, m, s->bytes), false));
  SNP_TRY(dpar.ensure(8, false));
  SNP_TRY(dt.ensure(8, false));
  SNP_TRY(out.ensure((size_t)s->n + 16, false));
  SNP_TRY(derr.ensure(4, false));
  const int64_t zero = 0;
  CUDA_TRY(cudaMemcpyAsync(row.p, C, (size_t)m * 4, cudaMemcpyHostToDevice, s->stream));
  CUDA_TRY(cudaMemcpyAsync(dpar.p, &zero, 8, cudaMemcpyHostToDevice, s->stream));
  CUDA_TRY(cudaMemcpyAsync(dt.p, &t, 8, cudaMemcpyHostToDevice, s->stream));
  CUDA_TRY(cudaMemsetAsync(derr.p, 0, 4, s->stream));
  launch_import(row.p, 4, SNP_LAYOUT_ROW_MAJOR, m, 1, (int32_t)m, blk.p, s->bytes, s->count_max, derr.as<int32_t>(),
                s->stream);
  launch_spiking_vectors(s->view, s->bytes, blk.p, dpar.as<int64_t>(), dt.as<uint64_t>(), 1, out.as<uint8_t>(),
                         derr.as<int32_t>(), s->stream);
  CUDA_TRY(cudaGetLastError());
  int32_t err = 0;
  CUDA_TRY(cudaMemcpyAsync(&err, derr.p, 4, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaMemcpyAsync(S_out, out.p, (size_t)s->n, cudaMemcpyDeviceToHost, s->stream));
  SNP_TRY(sync(s));
  if (err & ERR_CAPACITY) return fail(SNP_E_ARG, "snp_spiking_vector: t = %llu >= Ψ(C)", (unsigned long long)t);
  return SNP_OK;
}

snp_status snp_frontier_copy(snp_system* s, int32_t* configs, int64_t* parent, uint64_t* t, int64_t cap,
                             int64_t* n_out) {
  if (!s || s->levels.empty()) return fail(SNP_E_ARG, "snp_frontier_copy: no exploration");
  const int32_t L = (int32_t)s->levels.size() - 1;
  const int64_t F = s->levels[L]->F;
  if (n_out) *n_out = F;
  if (F > cap) return fail(SNP_E_CAPACITY, "snp_frontier_copy: frontier has %lld configurations > cap %lld", (long long)F, (long long)cap);
  if (parent || t) SNP_TRY(snp_level_edges(s, L, parent, t, nullptr, nullptr));
  if (configs && F) {
    std::vector<int64_t> idx(F);
    for (int64_t i = 0; i < F; ++i) idx[i] = i;
    SNP_TRY(snp_level_columns(s, L, idx.data(), F, configs));
  }
  return SNP_OK;
}

snp_status snp_level_all_edges(snp_system* s, int32_t level, int64_t* parent, uint64_t* t, int64_t* ref, int64_t cap,
                               int64_t* n_edges) {
  if (!s || level < 1 || level >= (int32_t)s->levels.size()) return fail(SNP_E_ARG, "snp_level_all_edges: bad level");
  if (!s->opt.keep_all_edges) return fail(SNP_E_STATE, "snp_level_all_edges needs options.keep_all_edges = 1");
  const Level* lv = s->levels[level].get();
  if (!lv->all_ref.p && lv->all_T) return fail(SNP_E_STATE, "edges of level %d were not recorded", level);
  const int64_t T = lv->all_T;
  if (n_edges) *n_edges = T;
  if (T > cap) return fail(SNP_E_CAPACITY, "snp_level_all_edges: %lld edges > cap %lld", (long long)T, (long long)cap);
  if (!T) return SNP_OK;
  std::vector<uint64_t> raw(T), off(lv->all_F + 1);
  CUDA_TRY(cudaMemcpyAsync(raw.data(), lv->all_ref.p, T * 8, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaMemcpyAsync(off.data(), lv->all_off.p, (lv->all_F + 1) * 8, cudaMemcpyDeviceToHost, s->stream));
  SNP_TRY(sync(s));
  std::vector<int64_t> base(s->levels.size() + 1, 0);
  for (size_t i = 0; i < s->levels.size(); ++i) base[i + 1] = base[i] + s->levels[i]->F;
  for (int64_t p = 0, e = 0; p < lv->all_F; ++p)
    for (uint64_t c = off[p]; c < off[p + 1]; ++c, ++e) {
      if (parent) parent[e] = p;
      if (t) t[e] = c - off[p];
    }
  if (ref)
    for (int64_t e = 0; e < T; ++e) {
      const uint64_t r = raw[e];
      if (r == ~0ULL) { ref[e] = -1; continue; }
      const uint64_t L2 = r >> 40, q = r & ((1ULL << 40) - 1);
      ref[e] = L2 < s->levels.size() ? base[L2] + (int64_t)q : -1;
    }
  return SNP_OK;
}

}  // extern "C"

// ===========================================================================
// multi-GPU exploration.  Each rank holds a contiguous range of
// the global frontier (global order = rank order, then local tag order) and the
// visited keys it owns (owner = fmix64(fp1) mod P).  One level:
//   snp_dist_expand      K-a/K-b on the local frontier: child keys, local T
//   snp_dist_pack        keys bucketed by owner into a caller buffer
//   [caller: all-to-all of keys]
//   snp_dist_owner_dedup visited shard + level table (minimum global tag)
//   [caller: all-reduce of N_new]
//   snp_dist_owner_keep  thinning with the global N_new, visited insert, verdicts
//   [caller: all-to-all of verdicts back]
//   snp_dist_finalize    kept flags of the local children, local K
//   [caller: all-gather of K and F for the global offsets]
//   snp_dist_commit      K-c materialization of the local kept children
// The collectives are the caller's (paper_1104_1824_b200/dist.py, torch
// NCCL); every step of the method runs in the kernels below the ABI.
// ===========================================================================
namespace {

snp_status dist_stage(snp_system* s, int want) {
  if (!s) return fail(SNP_E_ARG, "NULL system");
  if (s->dist.P < 1) return fail(SNP_E_STATE, "not in distributed mode (snp_dist_begin)");
  if (s->dist.stage != want) return fail(SNP_E_STATE, "distributed call out of order (stage %d, expected %d)", s->dist.stage, want);
  return SNP_OK;
}

}  // namespace

extern "C" {

snp_status snp_dist_begin(snp_system* s, const snp_configs* level0, int32_t nranks, int64_t* n_local) {
  if (!s || !level0 || nranks < 1) return fail(SNP_E_ARG, "snp_dist_begin: bad arguments");
  if (s->opt.dedup != 1) return fail(SNP_E_STATE, "distributed exploration needs dedup = 1 (fingerprint keys)");
  if (s->opt.keep_all_edges) return fail(SNP_E_STATE, "keep_all_edges is not available in distributed exploration");
  if (s->view.aug_rule >= 0) return fail(SNP_E_STATE, "distributed exploration does not support generated numbers");
  if (s->view.delay_m > 0) return fail(SNP_E_STATE, "distributed exploration does not support delays");
  const int64_t F0 = level0->n_configs, m = s->m;
  if (F0 < 0 || F0 > 0x7FFFFFFFLL || (F0 > 0 && !level0->data)) return fail(SNP_E_ARG, "level0: bad n_configs / data");
  if (level0->elem_bytes != 1 && level0->elem_bytes != 2 && level0->elem_bytes != 4) return fail(SNP_E_ARG, "level0: elem_bytes");
  SNP_TRY(reset_state(s));
  {  // a fresh level-0 state; the transport and its settings stay
    snp::Comm* comm = s->dist.comm;
    snp::LocalGroup* group = s->dist.group;
    const double rebalance = s->dist.rebalance;
    const int inject = s->dist.inject_step;
    s->dist.comm = nullptr;
    s->dist.group = nullptr;
    s->dist = snp_system::Dist{};
    s->dist.comm = comm;
    s->dist.group = group;
    s->dist.rebalance = rebalance;
    s->dist.inject_step = inject;
  }
  s->dist.P = nranks;
  s->begun = false;
  SNP_TRY(zero_counters(s));
  int32_t* err = &dc(s)->err;
  SNP_TRY(s->dist.raw.ensure(std::max<size_t>(level_bytes(F0, m, s->bytes), 256), false));
  SNP_TRY(s->dist.fp0.ensure(std::max<int64_t>(F0, 1) * 8, false));
  SNP_TRY(s->dist.fp1.ensure(std::max<int64_t>(F0, 1) * 8, false));
  SNP_TRY(ensure_children(s, (uint64_t)std::max<int64_t>(F0, 1)));
  SNP_TRY(ensure_visited(s, 4 * (uint64_t)std::max<int64_t>(F0, 1024)));
  if (F0 > 0) {
    const int64_t ld = level0->ld ? level0->ld : (level0->layout == SNP_LAYOUT_ROW_MAJOR ? m : F0);
    const size_t in_bytes = (size_t)(level0->layout == SNP_LAYOUT_ROW_MAJOR ? (F0 - 1) * ld + m : (m - 1) * ld + F0) *
                            level0->elem_bytes;
    DBuf staged;
    const void* src = level0->data;
    if (!level0->on_device) {
      SNP_TRY(staged.ensure(in_bytes, false));
      CUDA_TRY(cudaMemcpyAsync(staged.p, level0->data, in_bytes, cudaMemcpyHostToDevice, s->stream));
      src = staged.p;
    }
    launch_import(src, level0->elem_bytes, level0->layout, ld, F0, (int32_t)m, s->dist.raw.p, s->bytes, s->count_max,
                  err, s->stream);
    launch_fingerprint(s->view, s->bytes, s->dist.raw.p, F0, s->dist.fp0.as<uint64_t>(), s->dist.fp1.as<uint64_t>(),
                       s->stream);
    ChildArrays C = child_arrays(s);
    CUDA_TRY(cudaMemcpyAsync(C.cfp0, s->dist.fp0.p, F0 * 8, cudaMemcpyDeviceToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(C.cfp1, s->dist.fp1.p, F0 * 8, cudaMemcpyDeviceToDevice, s->stream));
    CUDA_TRY(cudaGetLastError());
  }
  DevCounters hc;
  SNP_TRY(read_counters(s, &hc));
  SNP_TRY(check_err(hc.err));
  s->dist.F0 = F0;
  s->dist.T = (uint64_t)F0;
  s->dist.level0 = true;
  s->dist.stage = 1;
  if (n_local) *n_local = F0;
  return SNP_OK;
}

snp_status snp_dist_expand(snp_system* s, int64_t* T_local) {
  SNP_TRY(dist_stage(s, 0));
  Level* cur = s->levels.back().get();
  const int64_t F = cur->F, m = s->m;
  cudaStream_t st = s->stream;
  snp_level_counters lc{};
  CUDA_TRY(cudaEventRecord(s->ev0, st));
  SNP_TRY(zero_counters(s));
  uint64_t T = 0;
  if (F > 0) {
    if (!cur->has_data()) return fail(SNP_E_STATE, "current level has no data");
    SNP_TRY(s->psi.ensure((F + 1) * 8));
    SNP_TRY(s->off.ensure((F + 1) * 8));
    SNP_TRY(s->fpb0.ensure(F * 8));
    SNP_TRY(s->fpb1.ensure(F * 8));
    SNP_TRY(s->ndc.ensure(F * 4));
    SNP_TRY(s->nd.ensure((size_t)F * KMAX * 8));
    ExpandOut O{};
    O.psi = s->psi.as<uint64_t>();
    O.fpb0 = s->fpb0.as<uint64_t>();
    O.fpb1 = s->fpb1.as<uint64_t>();
    O.ndc = s->ndc.as<int32_t>();
    O.nd = s->nd.as<uint64_t>();
    O.halting = cur->halting.as<uint8_t>();
    O.n_halting = &dc(s)->n_halting;
    O.err = &dc(s)->err;
    if (fast_materialize_ok(s->view)) {
      SNP_TRY(s->ebits.ensure((size_t)((F + PB - 1) / PB) * (size_t)((m + 1) & ~1) * 8));
      O.ebits = s->ebits.as<uint64_t>();
    }
    CUDA_TRY(cudaMemsetAsync(O.psi + F, 0, 8, st));
    LevelView LV{cur->data.p, F, cur->fp0.as<uint64_t>(), cur->fp1.as<uint64_t>()};
    phase_begin(s, 0);
    launch_expand(s->view, s->bytes, LV, O, st);
    phase_end(s);
    SNP_TRY(s->scan_tmp.ensure(scan_temp_bytes(F + 1) + 256));
    phase_begin(s, 1);
    launch_exclusive_scan(s->scan_tmp.p, s->scan_tmp.bytes, O.psi, s->off.as<uint64_t>(), F + 1, st);
    phase_end(s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(&T, s->off.as<uint64_t>() + F, 8, cudaMemcpyDeviceToHost, st));
    DevCounters hc;
    SNP_TRY(read_counters(s, &hc));
    SNP_TRY(check_err(hc.err));
    lc.halting = (int64_t)hc.n_halting;
    if (s->opt.max_transitions > 0 && (int64_t)T > s->opt.max_transitions)
      return fail(SNP_E_CAPACITY, "%llu local transitions exceed the budget", (unsigned long long)T);
    if (T > 0) {
      SNP_TRY(ensure_children(s, T));
      ChildArrays C = child_arrays(s);
      phase_begin(s, 1);
      launch_child_parent(s->off.as<uint64_t>(), F, C.cpar, st);
      launch_child_keys(s->view, s->off.as<uint64_t>(), O, T, C, st);
      phase_end(s);
      CUDA_TRY(cudaGetLastError());
    }
    s->dist.O = O;
  }
  s->halting_current_valid = true;
  lc.parents = F;
  lc.T = (int64_t)T;
  s->dist.lc = lc;
  s->dist.T = T;
  s->dist.level0 = false;
  s->dist.stage = 1;
  if (T_local) *T_local = (int64_t)T;
  return SNP_OK;
}

snp_status snp_dist_pack(snp_system* s, uint64_t tag_base, void* send, int64_t* counts) {
  SNP_TRY(dist_stage(s, 1));
  const uint32_t P = (uint32_t)s->dist.P;
  const uint64_t T = s->dist.T;
  if (!counts || (T > 0 && !send)) return fail(SNP_E_ARG, "snp_dist_pack: bad arguments");
  SNP_TRY(s->dist.perm.ensure(std::max<uint64_t>(T, 1) * 8));
  SNP_TRY(s->dist.hist.ensure(P * 8 + 8));
  auto* hist = s->dist.hist.as<unsigned long long>();
  CUDA_TRY(cudaMemsetAsync(hist, 0, P * 8, s->stream));
  ChildArrays C = child_arrays(s);
  phase_begin(s, 2);
  launch_owner_hist(C.cfp1, T, P, hist, s->stream);
  phase_end(s);
  std::vector<unsigned long long> h(P), cur(P);
  CUDA_TRY(cudaMemcpyAsync(h.data(), hist, P * 8, cudaMemcpyDeviceToHost, s->stream));
  SNP_TRY(sync(s));
  unsigned long long acc = 0;
  for (uint32_t r = 0; r < P; ++r) {
    cur[r] = acc;
    acc += h[r];
    counts[r] = (int64_t)h[r];
  }
  CUDA_TRY(cudaMemcpyAsync(hist, cur.data(), P * 8, cudaMemcpyHostToDevice, s->stream));
  phase_begin(s, 2);
  launch_owner_pack(C.cfp0, C.cfp1, T, P, tag_base, hist, s->dist.perm.as<uint64_t>(), static_cast<uint64_t*>(send),
                    s->stream);
  phase_end(s);
  CUDA_TRY(cudaGetLastError());
  SNP_TRY(sync(s));
  s->dist.stage = 2;
  return SNP_OK;
}

snp_status snp_dist_owner_dedup(snp_system* s, const void* recv, int64_t R, int64_t* n_new_local) {
  SNP_TRY(dist_stage(s, 2));
  if (R < 0 || (R > 0 && !recv)) return fail(SNP_E_ARG, "snp_dist_owner_dedup: bad arguments");
  SNP_TRY(ensure_ltab(s, (uint64_t)std::max<int64_t>(R, 1)));
  const uint64_t lslots = next_pow2(std::max<uint64_t>(1024, 2 * (uint64_t)std::max<int64_t>(R, 1)));
  SNP_TRY(s->dist.slot.ensure(std::max<int64_t>(R, 1) * 8));
  SNP_TRY(s->dist.verdict.ensure(std::max<int64_t>(R, 1)));
  SNP_TRY(zero_counters(s));
  Tables tb = tables(s, lslots);
  const uint64_t* rv = static_cast<const uint64_t*>(recv);
  phase_begin(s, 2);
  launch_owner_dedup(rv, (uint64_t)R, tb, s->dist.verdict.as<uint8_t>(), s->dist.slot.as<uint64_t>(), &dc(s)->err,
                     s->stream);
  launch_owner_winners(rv, (uint64_t)R, tb, s->dist.verdict.as<uint8_t>(), s->dist.slot.as<uint64_t>(),
                       &dc(s)->n_new, s->stream);
  phase_end(s);
  CUDA_TRY(cudaGetLastError());
  DevCounters hc;
  SNP_TRY(read_counters(s, &hc));
  SNP_TRY(check_err(hc.err));
  s->dist.R = (uint64_t)R;
  s->dist.recv = rv;
  s->dist.stage = 3;
  if (n_new_local) *n_new_local = (int64_t)hc.n_new;
  return SNP_OK;
}

snp_status snp_dist_owner_keep(snp_system* s, int64_t n_new_global, void* verdict_out) {
  SNP_TRY(dist_stage(s, 3));
  const uint64_t R = s->dist.R;
  if (R > 0 && !verdict_out) return fail(SNP_E_ARG, "snp_dist_owner_keep: bad arguments");
  uint64_t tau = 0;
  const int thin = !s->dist.level0 && s->opt.frontier_target > 0 && n_new_global > s->opt.frontier_target;
  if (thin) {
    unsigned __int128 num = (unsigned __int128)(uint64_t)s->opt.frontier_target << 64;
    tau = (uint64_t)(num / (unsigned __int128)(uint64_t)n_new_global);
  }
  SNP_TRY(ensure_visited(s, (uint64_t)s->dist.owned + R));
  const uint64_t lslots = next_pow2(std::max<uint64_t>(1024, 2 * std::max<uint64_t>(R, 1)));
  Tables tb = tables(s, lslots);
  SNP_TRY(zero_counters(s));
  phase_begin(s, 2);
  launch_owner_keep(s->dist.recv, R, tb, s->dist.verdict.as<uint8_t>(), s->dist.slot.as<uint64_t>(), tau, thin,
                    static_cast<uint8_t*>(verdict_out), &dc(s)->n_new, &dc(s)->err, s->stream);
  phase_end(s);
  CUDA_TRY(cudaGetLastError());
  DevCounters hc;
  SNP_TRY(read_counters(s, &hc));
  SNP_TRY(check_err(hc.err));
  s->dist.owned += (int64_t)hc.n_new;
  s->dist.lc.n_new = n_new_global;
  s->dist.lc.tau = tau;
  s->dist.stage = 4;
  return SNP_OK;
}

snp_status snp_dist_finalize(snp_system* s, const void* verdict_back, int64_t* K_local) {
  SNP_TRY(dist_stage(s, 4));
  const uint64_t T = s->dist.T;
  if (T > 0 && !verdict_back) return fail(SNP_E_ARG, "snp_dist_finalize: bad arguments");
  ChildArrays C = child_arrays(s);
  phase_begin(s, 2);
  launch_unperm(s->dist.perm.as<uint64_t>(), static_cast<const uint8_t*>(verdict_back), T, C.kept, s->stream);
  launch_exclusive_scan(s->scan_tmp.p, s->scan_tmp.bytes, C.kept, C.kpos, (int64_t)T + 1, s->stream);
  phase_end(s);
  CUDA_TRY(cudaGetLastError());
  uint64_t K = 0;
  CUDA_TRY(cudaMemcpyAsync(&K, C.kpos + T, 8, cudaMemcpyDeviceToHost, s->stream));
  SNP_TRY(sync(s));
  s->dist.K = (int64_t)K;
  s->dist.stage = 5;
  if (K_local) *K_local = (int64_t)K;
  return SNP_OK;
}

snp_status snp_dist_commit(snp_system* s, int64_t parent_offset, int64_t q_offset, snp_level_counters* out) {
  SNP_TRY(dist_stage(s, 5));
  const int64_t K = s->dist.K, m = s->m;
  cudaStream_t st = s->stream;
  SNP_TRY(zero_counters(s));
  int32_t* err = &dc(s)->err;
  ChildArrays C = child_arrays(s);
  Tables tb = tables(s, 1024);
  auto L = std::make_unique<Level>();
  L->F = K;
  SNP_TRY(alloc_level_meta(s, L.get(), K));
  NextArrays N{nullptr, L->parent.as<int64_t>(), L->t.as<uint64_t>(), L->fp0.as<uint64_t>(), L->fp1.as<uint64_t>()};
  if (s->dist.level0) {
    const int64_t F0 = s->dist.F0;
    SNP_TRY(s->src_index.ensure(std::max<int64_t>(K, 1) * 8));
    if (F0 > 0)
      launch_level0_compact(C.verdict, C.kept, C.kpos, F0, s->dist.fp0.as<uint64_t>(), s->dist.fp1.as<uint64_t>(), N,
                            s->src_index.as<uint64_t>(), tb, 0, err, st);
    if (K == F0) {
      L->data = std::move(s->dist.raw);
    } else if (K > 0) {
      SNP_TRY(take_buffer(s, level_bytes(K, m, s->bytes), &L->data));
      launch_gather_columns(s->bytes, s->dist.raw.p, s->src_index.as<uint64_t>(), K, (int32_t)m, L->data.p, st);
    }
    N.data = L->data.p;
    launch_zero_tail(s->bytes, L->data.p, K, (int32_t)m, st);
    launch_digest(N, K, 0, q_offset, 0, &dc(s)->digest, st);
    CUDA_TRY(cudaGetLastError());
    DevCounters hc;
    SNP_TRY(read_counters(s, &hc));
    SNP_TRY(check_err(hc.err));
    s->digest += hc.digest;
    s->n_visited = K;
    s->dist.raw.release();
    s->levels.push_back(std::move(L));
    s->dist.stage = 0;
    s->dist.level0 = false;
    if (out) {
      snp_level_counters lc{};
      lc.parents = s->dist.F0;
      lc.kept = K;
      *out = lc;
    }
    return SNP_OK;
  }
  Level* cur = s->levels.back().get();
  const int64_t F = cur->F;
  const uint64_t T = s->dist.T;
  if (T > 0)
    launch_compact(C, s->off.as<uint64_t>(), T, N, tb, 0, 0, err, st);
  if (K > 0) {
    SNP_TRY(take_buffer(s, level_bytes(K, m, s->bytes), &L->data));
    N.data = L->data.p;
    SNP_TRY(s->kq_off.ensure((F + 1) * 8));
    const uint64_t ovf_cap = ovf_capacity();
    SNP_TRY(s->ovf.ensure(ovf_cap * 8));
    LevelView LV{cur->data.p, F, cur->fp0.as<uint64_t>(), cur->fp1.as<uint64_t>()};
    const ExpandOut& O = s->dist.O;
    phase_begin(s, 3);
    launch_kq_off(s->off.as<uint64_t>(), C.kpos, F, s->kq_off.as<uint64_t>(), st);
    launch_materialize(s->view, s->bytes, LV, O, s->kq_off.as<uint64_t>(), N, K, s->ovf.as<uint64_t>(), &dc(s)->n_ovf,
                       ovf_cap, err, st);
    launch_patch(s->view, s->bytes, LV, O, N, K, err, st);
    phase_end(s);
    CUDA_TRY(cudaGetLastError());
    DevCounters hc;
    SNP_TRY(read_counters(s, &hc));
    SNP_TRY(rematerialize_wide(s, LV, O, N, K, ovf_cap, err, &hc));
    if (hc.n_ovf > ovf_cap) return fail(SNP_E_CAPACITY, "too many counts at the storage limit (%llu)", hc.n_ovf);
    if (hc.n_ovf) {
      launch_overflow_fix(s->view, s->bytes, LV, O, s->kq_off.as<uint64_t>(), N, s->ovf.as<uint64_t>(), hc.n_ovf, err,
                          st);
      CUDA_TRY(cudaGetLastError());
    }
  }
  // parents are indices in the previous level: global = local + parent_offset
  if (K > 0) launch_zero_tail(s->bytes, N.data, K, (int32_t)m, st);
  launch_digest(N, K, (uint64_t)s->levels.size(), q_offset, parent_offset, &dc(s)->digest, st);
  CUDA_TRY(cudaEventRecord(s->ev1, st));
  DevCounters hc;
  SNP_TRY(read_counters(s, &hc));
  phase_collect(s);
  SNP_TRY(check_err(hc.err));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  snp_level_counters lc = s->dist.lc;
  lc.kept = K;
  lc.ms = ms;
  s->digest += hc.digest;
  s->n_visited += K;
  s->total_T += lc.T;
  s->counters.push_back(lc);
  if (!retain_levels(s)) release_level_data(s, cur);
  s->levels.push_back(std::move(L));
  s->halting_current_valid = false;
  s->dist.stage = 0;
  if (out) *out = lc;
  return SNP_OK;
}

}  // extern "C"

// ===========================================================================
// library-driven multi-GPU levels: the steps above with the
// exchanges issued by the library on the system's stream (snp_comm.h).  Each
// step's status is agreed by all ranks at the next collective (it rides in
// the small all-gathers), so a rank that fails (overflow, capacity, an
// injected fault) makes every rank return that same status instead of leaving
// its peers inside a collective.
// ===========================================================================
namespace {

// agreement: every rank contributes (status, values...); returns the status of
// the lowest failing rank (SNP_OK when none failed) and all values in out
snp_status agree(snp_system* s, snp_status mine, const std::vector<int64_t>& vals, std::vector<int64_t>* out) {
  snp::Comm* c = s->dist.comm;
  const int n = 1 + (int)vals.size();
  std::vector<int64_t> in(n), all((size_t)n * c->P);
  in[0] = (int64_t)mine;
  std::copy(vals.begin(), vals.end(), in.begin() + 1);
  std::string msg;
  const std::string my_err = mine != SNP_OK ? g_err : std::string();
  int st = c->allgather_i64(in.data(), n, all.data(), s->stream, &msg);
  if (st != SNP_OK) return fail((snp_status)st, "multi-GPU exchange: %s", msg.c_str());
  if (out) out->assign(all.begin(), all.end());
  for (int r = 0; r < c->P; ++r)
    if (all[(size_t)r * n] != SNP_OK) {
      if (r == c->rank) return fail((snp_status)all[(size_t)r * n], "%s", my_err.c_str());
      return fail((snp_status)all[(size_t)r * n], "rank %d failed (status %lld); every rank stops", r,
                  (long long)all[(size_t)r * n]);
    }
  return SNP_OK;
}

snp_status injected(snp_system* s, int step) {
  if (s->dist.inject_step == step) return fail(SNP_E_CAPACITY, "injected fault (SNP_DIST_INJECT) at step %d", step);
  return SNP_OK;
}

snp_status xfer(snp_system* s, const void* send, const std::vector<int64_t>& sc, void* recv,
                const std::vector<int64_t>& rc, size_t elem) {
  std::string msg;
  int st = s->dist.comm->alltoallv(send, sc.data(), recv, rc.data(), elem, s->stream, &msg);
  if (st != SNP_OK) return fail((snp_status)st, "multi-GPU exchange: %s", msg.c_str());
  return SNP_OK;
}

// one keys round (level 0 when s->dist.level0): pack, key all-to-all, owner
// dedup, N_new, owner keep, verdicts back, finalize, commit; the global
// counters of the level in *g
snp_status keys_round(snp_system* s, snp_status st, int64_t T_local, int64_t halting_local, snp_level_counters* g,
                      snp_level_counters* lo_out = nullptr) {
  snp::Comm* c = s->dist.comm;
  const int P = c->P, me = c->rank;
  std::vector<int64_t> all;
  const int64_t F_local = s->dist.level0 ? 0 : s->levels.back()->F;
  if (st == SNP_OK) st = injected(s, 1);
  SNP_TRY(agree(s, st, {T_local, F_local, halting_local}, &all));
  int64_t tag_base = 0, T_glob = 0, F_glob = 0, H_glob = 0, p_off = 0;
  for (int r = 0; r < P; ++r) {
    if (r < me) { tag_base += all[4 * r + 1]; p_off += all[4 * r + 2]; }
    T_glob += all[4 * r + 1];
    F_glob += all[4 * r + 2];
    H_glob += all[4 * r + 3];
  }
  // keys {fp0, fp1, global tag} grouped by owner
  std::vector<int64_t> sc(P, 0), rc(P, 0);
  st = s->dist.sendbuf.ensure((size_t)std::max<int64_t>(T_local, 1) * 24);
  if (st == SNP_OK) st = snp_dist_pack(s, (uint64_t)tag_base, s->dist.sendbuf.p, sc.data());
  if (st == SNP_OK) st = injected(s, 2);
  SNP_TRY(agree(s, st, sc, &all));
  for (int q = 0; q < P; ++q) rc[q] = all[(size_t)q * (P + 1) + 1 + me];
  int64_t R = 0;
  for (int64_t x : rc) R += x;
  SNP_TRY(s->dist.recvbuf.ensure((size_t)std::max<int64_t>(R, 1) * 24));
  SNP_TRY(xfer(s, s->dist.sendbuf.p, sc, s->dist.recvbuf.p, rc, 24));
  int64_t n_new_local = 0;
  st = snp_dist_owner_dedup(s, s->dist.recvbuf.p, R, &n_new_local);
  if (st == SNP_OK) st = injected(s, 3);
  SNP_TRY(agree(s, st, {n_new_local}, &all));
  int64_t n_new = 0;
  for (int r = 0; r < P; ++r) n_new += all[2 * r + 1];
  st = s->dist.vbuf.ensure((size_t)std::max<int64_t>(R, 1));
  if (st == SNP_OK) st = snp_dist_owner_keep(s, n_new, s->dist.vbuf.p);
  if (st == SNP_OK) st = injected(s, 4);
  SNP_TRY(agree(s, st, {}, nullptr));
  SNP_TRY(s->dist.backbuf.ensure((size_t)std::max<int64_t>(T_local, 1)));
  SNP_TRY(xfer(s, s->dist.vbuf.p, rc, s->dist.backbuf.p, sc, 1));  // verdicts return in send order
  int64_t K = 0;
  st = snp_dist_finalize(s, s->dist.backbuf.p, &K);
  if (st == SNP_OK) st = injected(s, 5);
  SNP_TRY(agree(s, st, {K}, &all));
  int64_t q_off = 0, K_glob = 0;
  std::vector<int64_t> Ks(P);
  for (int r = 0; r < P; ++r) {
    Ks[r] = all[2 * r + 1];
    if (r < me) q_off += Ks[r];
    K_glob += Ks[r];
  }
  snp_level_counters lc{};
  st = snp_dist_commit(s, p_off, q_off, &lc);
  if (st == SNP_OK && !s->levels.empty()) {  // parents as global indices of the previous level
    Level* L = s->levels.back().get();
    if (L->F) launch_add_i64(L->parent.as<int64_t>(), L->F, p_off, s->stream);
    if (cudaGetLastError() != cudaSuccess) st = fail(SNP_E_CUDA, "parent offsets");
  }
  if (st == SNP_OK) st = injected(s, 6);
  std::vector<int64_t> msv;
  SNP_TRY(agree(s, st, {(int64_t)std::llround(lc.ms * 1000.0)}, &msv));
  double ms_max = 0;
  for (int r = 0; r < P; ++r) ms_max = std::max(ms_max, msv[2 * r + 1] / 1000.0);
  s->dist.q_off = q_off;
  s->dist.F_global = K_glob;
  s->dist.n_configs += K_glob;
  if (g) {
    *g = snp_level_counters{};
    g->parents = s->dist.level0 ? 0 : F_glob;
    g->halting = H_glob;
    g->T = s->dist.level0 ? 0 : T_glob;
    g->n_new = n_new;
    g->kept = K_glob;
    g->tau = lc.tau;
    g->ms = ms_max;
    g->overflow_fixes = lc.overflow_fixes;
  }
  if (lo_out) {
    *lo_out = lc;
    lo_out->parents = F_local;
    lo_out->T = T_local;
    lo_out->halting = halting_local;
    lo_out->n_new = n_new_local;
    lo_out->kept = K;
  }
  // rebalancing: the next frontier back to equal contiguous shares
  int64_t kmax = 0;
  for (int64_t k : Ks) kmax = std::max(kmax, k);
  const double mean = (double)K_glob / P;
  if (P > 1 && s->dist.rebalance > 0 && K_glob > 0 && kmax > s->dist.rebalance * mean) {
    // rows [q_off, q_off + K) of the global level move to rank d's target
    // range [K·d/P, K·(d+1)/P); blocked row chunks (padded to 64) plus the
    // per-row metadata travel in four more all-to-alls
    Level* L = s->levels.back().get();
    const int64_t m = s->m;
    std::vector<int64_t> lo(P + 1);
    for (int d = 0; d <= P; ++d) lo[d] = K_glob * d / P;
    std::vector<int64_t> qs(P + 1, 0);
    for (int r = 0; r < P; ++r) qs[r + 1] = qs[r] + Ks[r];
    auto overlap = [&](int src, int dst) {
      const int64_t a = std::max(qs[src], lo[dst]), b = std::min(qs[src + 1], lo[dst + 1]);
      return b > a ? b - a : (int64_t)0;
    };
    std::vector<int64_t> scr(P), rcr(P), scb(P), rcb(P);
    for (int q = 0; q < P; ++q) {
      scr[q] = overlap(me, q);
      rcr[q] = overlap(q, me);
      scb[q] = (int64_t)level_bytes(scr[q], m, s->bytes);
      rcb[q] = (int64_t)level_bytes(rcr[q], m, s->bytes);
    }
    int64_t Snd = 0, Rcv = 0, Kn = 0, Sb = 0, Rb = 0;
    for (int q = 0; q < P; ++q) { Snd += scr[q]; Rcv += rcr[q]; Sb += scb[q]; Rb += rcb[q]; }
    Kn = lo[me + 1] - lo[me];
    // pack this rank's rows as blocked chunks, one per destination
    DBuf pack, recvrows, idx;
    SNP_TRY(pack.ensure((size_t)std::max<int64_t>(Sb, 1), false));
    SNP_TRY(recvrows.ensure((size_t)std::max<int64_t>(Rb, 1), false));
    std::vector<uint64_t> hidx;
    {
      int64_t row = 0, boff = 0;
      for (int q = 0; q < P; ++q) {
        if (scr[q]) {
          hidx.resize(scr[q]);
          for (int64_t i = 0; i < scr[q]; ++i) hidx[i] = (uint64_t)(row + i);
          SNP_TRY(idx.ensure((size_t)scr[q] * 8));
          CUDA_TRY(cudaMemcpyAsync(idx.p, hidx.data(), scr[q] * 8, cudaMemcpyHostToDevice, s->stream));
          launch_gather_columns(s->bytes, L->data.p, idx.as<uint64_t>(), scr[q], (int32_t)m,
                                pack.as<uint8_t>() + boff, s->stream);
          CUDA_TRY(cudaStreamSynchronize(s->stream));  // hidx is reused
        }
        row += scr[q];
        boff += scb[q];
      }
    }
    SNP_TRY(xfer(s, pack.p, scb, recvrows.p, rcb, 1));
    // metadata: parent (global), t, fp0, fp1 — contiguous slices per destination
    auto meta = [&](DView& v, DBuf& out) -> snp_status {
      SNP_TRY(out.ensure((size_t)std::max<int64_t>(Kn, 1) * 8));
      return xfer(s, v.p, scr, out.p, rcr, 8);
    };
    auto nl = std::make_unique<Level>();
    nl->F = Kn;
    SNP_TRY(alloc_level_meta(s, nl.get(), Kn));
    DBuf tmp;
    SNP_TRY(meta(L->parent, tmp));
    CUDA_TRY(cudaMemcpyAsync(nl->parent.p, tmp.p, Kn * 8, cudaMemcpyDeviceToDevice, s->stream));
    SNP_TRY(meta(L->t, tmp));
    CUDA_TRY(cudaMemcpyAsync(nl->t.p, tmp.p, Kn * 8, cudaMemcpyDeviceToDevice, s->stream));
    SNP_TRY(meta(L->fp0, tmp));
    CUDA_TRY(cudaMemcpyAsync(nl->fp0.p, tmp.p, Kn * 8, cudaMemcpyDeviceToDevice, s->stream));
    SNP_TRY(meta(L->fp1, tmp));
    CUDA_TRY(cudaMemcpyAsync(nl->fp1.p, tmp.p, Kn * 8, cudaMemcpyDeviceToDevice, s->stream));
    // received chunks -> one blocked level (chunk q starts at block base_q)
    if (Kn > 0) {
      hidx.resize(Kn);
      int64_t k = 0, base = 0;
      for (int q = 0; q < P; ++q) {
        for (int64_t i = 0; i < rcr[q]; ++i) hidx[k++] = (uint64_t)(base + i);
        base += (rcr[q] + PB - 1) / PB * PB;
      }
      SNP_TRY(idx.ensure((size_t)Kn * 8));
      CUDA_TRY(cudaMemcpyAsync(idx.p, hidx.data(), Kn * 8, cudaMemcpyHostToDevice, s->stream));
      SNP_TRY(take_buffer(s, level_bytes(Kn, m, s->bytes), &nl->data));
      launch_gather_columns(s->bytes, recvrows.p, idx.as<uint64_t>(), Kn, (int32_t)m, nl->data.p, s->stream);
      launch_zero_tail(s->bytes, nl->data.p, Kn, (int32_t)m, s->stream);
      CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    release_level_data(s, L);
    s->levels.back() = std::move(nl);
    s->dist.q_off = lo[me];
    s->dist.rebalanced_rows = Snd - scr[me];
  } else {
    s->dist.rebalanced_rows = 0;
  }
  return SNP_OK;
}

snp_status dist_ready(snp_system* s) {
  if (!s) return fail(SNP_E_ARG, "NULL system");
  if (!s->dist.comm) return fail(SNP_E_STATE, "no multi-GPU transport: call snp_dist_init or snp_dist_init_local first");
  return SNP_OK;
}

void inject_from_env(snp_system* s) {
  s->dist.inject_step = -1;
  if (const char* e = getenv("SNP_DIST_INJECT")) {
    int r = -1, step = -1;
    if (sscanf(e, "%d,%d", &r, &step) == 2 && r == s->dist.comm->rank) s->dist.inject_step = step;
  }
}

}  // namespace

struct snp_local_group { snp::LocalGroup* g; };

extern "C" {

snp_status snp_dist_unique_id(void* id_out) {
  if (!id_out) return fail(SNP_E_ARG, "snp_dist_unique_id: NULL");
  std::string msg;
  int st = snp::nccl_unique_id(id_out, &msg);
  if (st != SNP_OK) return fail((snp_status)st, "%s", msg.c_str());
  return SNP_OK;
}

snp_status snp_dist_init(snp_system* s, const void* id, int32_t rank, int32_t nranks) {
  if (!s || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(SNP_E_ARG, "snp_dist_init: bad arguments");
  delete s->dist.comm;
  s->dist.comm = nullptr;
  std::string msg;
  int st = SNP_OK;
  s->dist.comm = snp::make_nccl_comm(id, rank, nranks, &msg, &st);
  if (!s->dist.comm) return fail((snp_status)st, "%s", msg.c_str());
  inject_from_env(s);
  return SNP_OK;
}

snp_status snp_local_group_create(int32_t nranks, snp_local_group** out) {
  if (!out || nranks < 1) return fail(SNP_E_ARG, "snp_local_group_create: bad arguments");
  *out = new snp_local_group{snp::local_group_create(nranks)};
  return SNP_OK;
}

void snp_local_group_free(snp_local_group* g) {
  if (!g) return;
  snp::local_group_release(g->g);
  delete g;
}

snp_status snp_dist_init_local(snp_system* s, snp_local_group* g, int32_t rank) {
  if (!s || !g || rank < 0 || rank >= snp::local_group_size(g->g)) return fail(SNP_E_ARG, "snp_dist_init_local: bad arguments");
  delete s->dist.comm;
  s->dist.comm = snp::make_local_comm(g->g, rank);
  inject_from_env(s);
  return SNP_OK;
}

snp_status snp_dist_set_rebalance(snp_system* s, double threshold) {
  if (!s || threshold < 0) return fail(SNP_E_ARG, "snp_dist_set_rebalance: bad arguments");
  s->dist.rebalance = threshold;
  return SNP_OK;
}

snp_status snp_dist_start(snp_system* s, const snp_configs* level0_local, int64_t* F_global) {
  SNP_TRY(dist_ready(s));
  int64_t n = 0;
  snp_status st = snp_dist_begin(s, level0_local, s->dist.comm->P, &n);
  s->dist.n_configs = 0;
  s->dist.T_total = 0;
  SNP_TRY(keys_round(s, st, n, 0, nullptr));
  if (F_global) *F_global = s->dist.F_global;
  return SNP_OK;
}

snp_status snp_dist_advance(snp_system* s, snp_level_counters* global, snp_level_counters* local) {
  SNP_TRY(dist_ready(s));
  if (s->dist.P < 1 || s->levels.empty()) return fail(SNP_E_STATE, "snp_dist_advance before snp_dist_start");
  int64_t T = 0;
  snp_status st = snp_dist_expand(s, &T);
  const int64_t h = st == SNP_OK ? s->dist.lc.halting : 0;
  snp_level_counters g{};
  SNP_TRY(keys_round(s, st, T, h, &g, local));
  s->dist.T_total += g.T;
  if (global) *global = g;
  return SNP_OK;
}

snp_status snp_dist_summary(snp_system* s, int64_t* n_configs, int64_t* transitions, uint64_t* digest) {
  SNP_TRY(dist_ready(s));
  std::vector<int64_t> all;
  SNP_TRY(agree(s, SNP_OK, {(int64_t)s->digest}, &all));
  uint64_t d = 0;
  for (int r = 0; r < s->dist.comm->P; ++r) d += (uint64_t)all[2 * r + 1];
  if (n_configs) *n_configs = s->dist.n_configs;
  if (transitions) *transitions = s->dist.T_total;
  if (digest) *digest = d;
  return SNP_OK;
}

snp_status snp_dist_local(const snp_system* s, int64_t* F_local, int64_t* global_offset, int64_t* rebalanced_rows) {
  if (!s || !s->dist.comm) return fail(SNP_E_STATE, "no multi-GPU transport");
  if (F_local) *F_local = s->levels.empty() ? 0 : s->levels.back()->F;
  if (global_offset) *global_offset = s->dist.q_off;
  if (rebalanced_rows) *rebalanced_rows = s->dist.rebalanced_rows;
  return SNP_OK;
}

}  // extern "C"
