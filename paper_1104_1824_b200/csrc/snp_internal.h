// snp_internal.h — launchers shared by the host engine (snp_engine.cu) and the
// kernels (snp_kernels.cu).  Not part of the public ABI (include/snp.h).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include "snp_device.cuh"

namespace snp {

extern std::atomic<int64_t> g_kernel_launches;

// A frontier level on the device (blocked layout, see snp_device.cuh).
struct LevelView {
  const void* data;
  int64_t F;
  const uint64_t* fp0;
  const uint64_t* fp1;
};

struct ExpandOut {
  uint64_t* psi;      // F + 1 (psi[F] = 0 for the exclusive scan)
  uint64_t* fpb0;     // fingerprint of the base child (every neuron fires its first rule)
  uint64_t* fpb1;
  int32_t* ndc;       // number of nondeterministic neurons (d_s >= 2)
  uint64_t* nd;       // F × KMAX entries (s << 32 | count)
  uint8_t* halting;   // F
  uint64_t* ebits;    // binary emits per (block, neuron): bit k = configuration 64·b + k spikes
  unsigned long long* n_halting;
  int32_t* err;
  int classify_only;
};

struct ChildArrays {
  uint32_t* cpar;     // T: parent index of child c
  uint64_t* cfp0;     // T: child fingerprints
  uint64_t* cfp1;
  uint8_t* verdict;   // T: 0 = seen at an earlier level, 1 = inserted into the level table
  uint64_t* cslot;    // T: level-table slot (verdict 1)
  uint64_t* cref;     // T: visited ref (verdict 0)
  uint64_t* kept;     // T + 1: kept flag (0/1), kept[T] = 0
  uint64_t* kpos;     // T + 1: exclusive scan of kept
};

struct NextArrays {
  void* data;         // blocked, ceil(K/64) blocks
  int64_t* parent;    // K
  uint64_t* t;        // K
  uint64_t* fp0;      // K
  uint64_t* fp1;      // K
};

struct StoredLevel {  // device table of retained level buffers (exact verification)
  const void* data;
};

struct Tables {
  Slot* vis;
  uint64_t vmask;
  Slot* ltab;
  uint64_t lmask;
};

// True when the fast kernels apply (outcome tables built, binary emits, the
// per-block emit words of a materialize tile fit in shared memory).
bool fast_expand_ok(const SysView& S);
bool fast_materialize_ok(const SysView& S);
size_t materialize_smem_bytes(const SysView& S, int32_t bytes, bool staged_e);
bool materialize_narrow_ok(const SysView& S, int32_t bytes);
void launch_build_cpT(const SysView& S, uint16_t* cpT, cudaStream_t st);

// ---- launchers (all asynchronous on `st`) ----------------------------------
void launch_build_tables(const SysView& S, int32_t bytes, uint8_t* tab, void* ctab, uint8_t* tab_full,
                         uint8_t* ttab, uint8_t* elut, uint8_t* hsg, cudaStream_t st);
void launch_import(const void* src, int32_t src_bytes, int32_t src_layout, int64_t src_ld, int64_t F, int32_t m,
                   void* dst, int32_t dst_bytes, int64_t count_max, int32_t* err, cudaStream_t st);
void launch_export(const void* src, int32_t bytes, int64_t F, int32_t m, int32_t* dst_rowmajor, cudaStream_t st);
void launch_fingerprint(const SysView& S, int32_t bytes, const void* data, int64_t F, uint64_t* fp0, uint64_t* fp1,
                        cudaStream_t st);
void launch_expand(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, cudaStream_t st);
void launch_child_parent(const uint64_t* off, int64_t F, uint32_t* cpar, cudaStream_t st);
// generated numbers (SysView::aug_rule >= 0): child keys get the augmented
// column's change, terminal children a skip key; kept children get A'
void launch_aug_keys(const SysView& S, int32_t bytes, const LevelView& L, const uint64_t* off, const ExpandOut& O,
                     uint64_t T, const ChildArrays& C, int32_t* err, cudaStream_t st);
void launch_aug_fix(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const NextArrays& N,
                    int64_t K, int32_t* err, cudaStream_t st);
void launch_child_keys(const SysView& S, const uint64_t* off, const ExpandOut& O, uint64_t T, const ChildArrays& C,
                       cudaStream_t st);
void launch_dedup(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, int use_visited, int32_t* err,
                  cudaStream_t st);
void launch_winners(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, unsigned long long* n_new,
                    cudaStream_t st);
void launch_keep(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, uint64_t tau, int thin,
                 cudaStream_t st);
void launch_compact(const ChildArrays& C, const uint64_t* off, uint64_t T, const NextArrays& N, const Tables& tb,
                    uint64_t level_ref, int insert_visited, int32_t* err, cudaStream_t st);
void launch_kq_off(const uint64_t* off, const uint64_t* kpos, int64_t F, uint64_t* kq_off, cudaStream_t st);
void launch_materialize(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O,
                        const uint64_t* kq_off, const NextArrays& N, int64_t K, uint64_t* ovf,
                        unsigned long long* n_ovf, uint64_t ovf_cap, int32_t* err, cudaStream_t st);
void launch_patch(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const NextArrays& N,
                  int64_t K, int32_t* err, cudaStream_t st);
void launch_overflow_fix(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O,
                         const uint64_t* kq_off, const NextArrays& N, const uint64_t* ovf, uint64_t n_ovf,
                         int32_t* err, cudaStream_t st);
void launch_verify(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const uint64_t* off,
                   const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb,
                   const StoredLevel* stored, uint64_t* list, unsigned long long* n_list, int32_t* err,
                   cudaStream_t st);
// dedup = 0 two-pass verification (the list of key matches, then batches)
void launch_verify_list(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, uint64_t* list,
                        unsigned long long* n_list, cudaStream_t st);
size_t verify2_row_bytes(const SysView& S);
bool launch_verify_m(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const uint64_t* off,
                     const ChildArrays& C, const uint64_t* list, const unsigned long long* n_list, uint64_t tag_base,
                     const Tables& tb, const StoredLevel* stored, int32_t* err, cudaStream_t st);
void launch_verify_batch(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const uint64_t* off,
                         const ChildArrays& C, const uint64_t* list, uint64_t i0, uint64_t n, uint64_t tag_base,
                         const Tables& tb, const StoredLevel* stored, void* fc, int32_t* err, cudaStream_t st);
void launch_level0_compact(const uint8_t* verdict, const uint64_t* kept, const uint64_t* kpos, int64_t F0,
                           const uint64_t* fp0, const uint64_t* fp1, const NextArrays& N, uint64_t* src_index,
                           const Tables& tb, int insert_visited, int32_t* err, cudaStream_t st);
void launch_gather_columns(int32_t bytes, const void* src, const uint64_t* src_index, int64_t K, int32_t m, void* dst,
                           cudaStream_t st);
// snapshot: one level's edge arrays and where they go in the packed output
struct EdgeSrc {
  const int64_t* parent;
  const uint64_t* t;
  const uint8_t* halting;
  const uint64_t* fp0;
  const uint64_t* fp1;
  int64_t F, offset;
};
void launch_pack_edges(const EdgeSrc* lv, int32_t nlev, int64_t max_F, int64_t* parent, uint64_t* t,
                       uint8_t* halting, uint64_t* fp2, cudaStream_t st);
// zero the unused configurations of a level's last 64-configuration block
void launch_zero_tail(int32_t bytes, void* data, int64_t F, int32_t m, cudaStream_t st);
// a[i] += add for every a[i] >= 0 (multi-GPU: local -> global parent indices)
void launch_add_i64(int64_t* a, int64_t n, int64_t add, cudaStream_t st);
void launch_verify_level0(int32_t bytes, const void* data, int32_t m, const ChildArrays& C, uint64_t F0,
                          const Tables& tb, int32_t* err, cudaStream_t st);
void launch_rehash(const Slot* old_tab, uint64_t old_cap, Slot* new_tab, uint64_t new_mask, int32_t* err,
                   cudaStream_t st);
void launch_digest(const NextArrays& N, int64_t K, uint64_t level, int64_t q_offset, int64_t parent_offset,
                   unsigned long long* digest, cudaStream_t st);
// multi-GPU dedup ownership
void launch_owner_hist(const uint64_t* fp1, uint64_t T, uint32_t P, unsigned long long* counts, cudaStream_t st);
void launch_owner_pack(const uint64_t* fp0, const uint64_t* fp1, uint64_t T, uint32_t P, uint64_t tag_base,
                       unsigned long long* cursor, uint64_t* perm, uint64_t* send, cudaStream_t st);
void launch_owner_dedup(const uint64_t* recv, uint64_t R, const Tables& tb, uint8_t* verdict, uint64_t* slot,
                        int32_t* err, cudaStream_t st);
void launch_owner_winners(const uint64_t* recv, uint64_t R, const Tables& tb, const uint8_t* verdict,
                          const uint64_t* slot, unsigned long long* n_new, cudaStream_t st);
void launch_owner_keep(const uint64_t* recv, uint64_t R, const Tables& tb, const uint8_t* verdict,
                       const uint64_t* slot, uint64_t tau, int thin, uint8_t* out, unsigned long long* n_kept,
                       int32_t* err, cudaStream_t st);
void launch_unperm(const uint64_t* perm, const uint8_t* back, uint64_t T, uint64_t* kept, cudaStream_t st);
void launch_spiking_vectors(const SysView& S, int32_t bytes, const void* parent_data, const int64_t* parent,
                            const uint64_t* t, int64_t K, uint8_t* S_out, int32_t* err, cudaStream_t st);
// keep_all_edges: the visited ref every transition reached (EMPTY = not stored)
void launch_all_edges(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, uint64_t next_ref,
                      uint64_t* ref, cudaStream_t st);

// systems with delays: child keys of materialised children
void launch_child_keys_delay(const SysView& S, int32_t bytes, const LevelView& L, const uint64_t* off,
                             const ExpandOut& O, uint64_t T, const ChildArrays& C, cudaStream_t st);
// single-path sampling: W walkers, all steps in one launch
void launch_sample(const SysView& S, int64_t W, int32_t* cur, int32_t* nxt, uint64_t* fired, uint64_t seed,
                   int32_t steps, int32_t input_neuron, const int32_t* train, int32_t train_len, int32_t* halted,
                   int32_t* err, bool small_rules, cudaStream_t st);

// Small frontiers (configs 1-2: the paper's Π): whole levels in ONE launch of
// ONE CTA, several levels per launch (k_small_bfs).
constexpr int SMALL_F = 256;    // parents of a level the single CTA expands
constexpr int SMALL_T = 4096;   // transitions of a level it handles
struct SmallLevelOut {
  int64_t T, n_new, kept, n_halting;
  uint64_t tau;
  unsigned long long digest;
  int32_t err;   // ERR_* of this level (the level is not committed)
  int32_t stop;  // 0 committed; 1 more than SMALL_T transitions (nothing committed, level left to the big path)
};
struct SmallArgs {
  const void* data;          // current level (tree level `level0`), blocked counts
  int64_t F;
  const uint64_t* fp0;
  const uint64_t* fp1;
  uint8_t* halting;          // its halting flags (written)
  int32_t level0;
  int32_t max_levels;
  uint8_t* data_pool;        // new level k: data_pool + k · data_stride (blocked, SMALL_T configurations)
  size_t data_stride;
  int64_t* parent_pool;      // new level k: + k · SMALL_T entries
  uint64_t* t_pool;
  uint64_t* fp0_pool;
  uint64_t* fp1_pool;
  uint8_t* halting_pool;
  // scratch
  uint64_t* psi;             // SMALL_F + 1
  uint64_t* off;             // SMALL_F + 1
  uint64_t* fpb0;            // SMALL_F
  uint64_t* fpb1;
  int32_t* ndc;
  uint64_t* nd;              // SMALL_F × KMAX
  uint32_t* cpar;            // SMALL_T
  uint64_t* cfp0;
  uint64_t* cfp1;
  uint8_t* verdict;
  uint64_t* cslot;
  uint64_t* cref;
  uint64_t* kept;            // SMALL_T + 1
  uint64_t* kpos;            // SMALL_T + 1
  Tables tb;                 // visited + a level table of >= 2·SMALL_T slots
  StoredLevel* stored;       // dedup = 0: data of every tree level (new ones written here)
  int64_t frontier_target;
  int64_t max_transitions;   // per-level budget (0 = none)
  int32_t dedup;
  SmallLevelOut* out;        // max_levels
  int32_t* levels_done;
};
void launch_small_bfs(const SysView& S, int32_t bytes, const SmallArgs& a, cudaStream_t st);

// CUB exclusive scan of n uint64 values (temp storage managed by the caller).
size_t scan_temp_bytes(int64_t n);
void launch_exclusive_scan(void* temp, size_t temp_bytes, const uint64_t* in, uint64_t* out, int64_t n,
                           cudaStream_t st);

}  // namespace snp
