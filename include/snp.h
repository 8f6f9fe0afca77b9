/*
 * snp.h — C ABI of the B200-native SNP transition engine (libsnp.so).
 *
 * The engine computes, on the GPU, the batched transition step of Cabarle,
 * Adorna and Martínez-del-Amor's matrix formulation of spiking neural P
 * systems without delays:
 *
 *     C_{k+1} = C_k + S_k · M_Π                     (eq. (2))
 *
 * over a whole breadth-first frontier of configurations: rule applicability
 * (Alg. 2 II-1), enumeration of every valid spiking
 * vector as a mixed-radix product of per-neuron rule choices (eq. (8),
 * PAPER.md:250; Alg. 2 II-2/II-3), the integer transition,
 * and deduplication of the children into the computation tree (Alg. 1,
 * PAPER.md:231-238; stopping criteria PAPER.md:229).  Readings of silent or
 * garbled passages are numbered A1..A22 in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Every call returns snp_status; SNP_OK == 0.  On failure a thread-local
 *     message is available from snp_last_error().  No exception crosses the ABI.
 *   - Caller-owned inputs are deep-copied; the caller may free them on return.
 *   - snp_system / snp_tree / snp_frontier are owned by the library and released
 *     with the matching snp_*_free.  A handle is not thread-safe.
 *   - Integers are little-endian; host arrays are C-contiguous.
 *   - Host-buffer calls are synchronous.  Device-buffer inputs (snp_configs with
 *     on_device = 1) are read on the system's stream (snp_set_stream).
 *   - There is no CPU fallback: without a CUDA device every compute call
 *     returns SNP_E_CUDA.
 */
#ifndef SNP_H_
#define SNP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNP_ABI_VERSION 2

typedef enum {
  SNP_OK = 0,
  SNP_E_ARG = -1,            /* bad argument (NULL, size, enum value)                        */
  SNP_E_INVALID_SYSTEM = -2, /* system violates Def. 1 / Def. 2 (first offending index in msg) */
  SNP_E_OVERFLOW = -3,       /* a stored count leaves the storage range (reading A16)        */
  SNP_E_CAPACITY = -4,       /* Ψ > 2^62, transition budget, or table capacity exceeded      */
  SNP_E_OOM = -5,            /* device allocation failed                                     */
  SNP_E_CUDA = -6,           /* CUDA runtime error (including: no device)                    */
  SNP_E_NCCL = -7,           /* NCCL error (multi-GPU)                                       */
  SNP_E_COLLISION = -8,      /* dedup=0 found two different configurations with equal 128-bit
                                fingerprints (probability < 2^-100; the run is aborted rather
                                than silently merged, reading A18)                            */
  SNP_E_STATE = -9           /* call not valid in the handle's current state                 */
} snp_status;

/* Regular-expression kinds of a rule's E (reading A1):
 *   SNP_RE_EXACT    E = a^a            (form (b-3)): n == a
 *   SNP_RE_PERIODIC E = a^a (a^b)*     (b >= 1):  n >= a && (n - a) % b == 0
 *   SNP_RE_UNARY    any regular E over {a} (the paper's
 *                   future work).  L(E) ⊆ a* is ultimately
 *                   periodic: with threshold t = a >= 0 and period P = b >= 1
 *                   (t + P <= 256), a^n ∈ L(E) iff bit idx of the rule's
 *                   256-bit membership row, idx = n < t + P ? n : t + (n - t) % P.
 *                   The rows are passed to snp_load_unary (reading A24).      */
enum { SNP_RE_EXACT = 0, SNP_RE_PERIODIC = 1, SNP_RE_UNARY = 2 };

/* One rule E/a^c -> a^p of neuron `neuron`.  produced = 0 is a
 * forgetting rule (b-2).  Rules are given in the paper's total order and must be
 * grouped by non-decreasing neuron.  A rule is applicable to
 * a neuron holding n spikes iff a^n ∈ L(E) and n >= consumed.   */
typedef struct {
  int32_t neuron;    /* 0-based neuron index σ(r)               */
  int32_t kind;      /* SNP_RE_EXACT or SNP_RE_PERIODIC         */
  int32_t a;         /* k (EXACT) or i (PERIODIC), >= 0          */
  int32_t b;         /* j >= 1 (PERIODIC), ignored for EXACT     */
  int32_t consumed;  /* c >= 1                                   */
  int32_t produced;  /* p >= 0                                   */
} snp_rule;

/* Spiking transition matrix M_Π (Def. 2): n_rules rows,
 * n_neurons columns; either dense (row-major, eq. (3)) or CSR.
 * Validation: M[r][σ(r)] = -c_r; off-diagonal entries are 0 or p_r; all
 * spiking rules of a neuron share one synapse set; no self-synapse.          */
typedef struct {
  int64_t n_rules;
  int64_t n_neurons;
  const int32_t *dense;    /* n_rules × n_neurons row-major, or NULL           */
  const int64_t *row_ptr;  /* CSR (used when dense == NULL): n_rules + 1 offsets */
  const int32_t *col;
  const int32_t *val;
} snp_matrix;

typedef struct {
  int32_t count_bits;        /* 8, 16 or 32: device storage of spike counts (reading A16)   */
  int32_t dedup;             /* 0 = full-configuration equality, 1 = 128-bit fingerprint    */
  int64_t frontier_target;   /* F for fingerprint thinning (reading A19); 0 = exact BFS      */
  int64_t max_transitions;   /* per-level budget on T; 0 = unlimited                        */
  uint64_t fp_seed[2];       /* fingerprint seeds (reading A18)                             */
  int32_t keep_tree;         /* 1 = retain every level's configurations for snp_tree_configs */
  int32_t out_rule1;         /* 0 = off.  r + 1: generated numbers with
                                rule r of the output neuron (PAPER.md:89 `out`) as its spiking
                                rule — see "Generated numbers" below                          */
  int32_t keep_all_edges;    /* 1 = also record EVERY transition (parent, t) of each level with
                                the configuration it reached (reading A17; the computation tree
                                of Fig. 4, including the edges to configurations
                                already seen): snp_level_all_edges.  Costs 8 B per transition
                                + 8 B per parent of device memory per level.                   */
  int32_t reserved;          /* 0 */
} snp_options;

/* Generated numbers (Π "generates all numbers in N - {1}"; the
 * generated set "is the result of the computation").  The number a computation
 * generates is the count of steps between the first two output spikes; an
 * output spike at step k is rule out_rule1 - 1 firing in S_k.  With out_rule1 >
 * 0 the engine explores the AUGMENTED state (C, A): every configuration has
 * snp_state_width = m + 1 entries, the last one A = 0 before the first output
 * spike, else the number of steps since it.  A transition from (C, A) by S:
 *   - A >= 1 and S fires the output rule: the number A is generated and the
 *     computation ends (the transition counts in T, its child is not stored);
 *   - otherwise the child is (C + S·M, A == 0 ? [output rule fires] : A + 1).
 * Dedup, thinning and halting act on the augmented state; C0 (snp_load) has m
 * entries (A = 0 is appended); level0 rows (snp_begin) have m + 1 columns.
 * Multi-GPU (snp_dist_*) is not available in this mode (SNP_E_STATE).         */

/* A batch of configurations (a frontier).  elem_bytes ∈ {1, 2, 4} (unsigned
 * for 1/2, int32 for 4).  layout ROW_MAJOR: n_configs rows of n_neurons counts
 * (ld = row stride in elements, >= n_neurons; 0 = n_neurons).  NEURON_MAJOR:
 * n_neurons rows of n_configs counts (ld = row stride in elements, >=
 * n_configs; 0 = n_configs).  on_device = 1: data is a CUDA device pointer.   */
enum { SNP_LAYOUT_ROW_MAJOR = 0, SNP_LAYOUT_NEURON_MAJOR = 1 };
typedef struct {
  const void *data;
  int64_t n_configs;
  int64_t ld;
  int32_t elem_bytes;
  int32_t layout;
  int32_t on_device;
  int32_t reserved;
} snp_configs;

/* Per-level counters of one expansion. */
typedef struct {
  int64_t parents;     /* configurations expanded                              */
  int64_t halting;     /* of which halting (no applicable rule, reading A5)    */
  int64_t T;           /* transitions generated = Σ Ψ (every (parent, S) pair)  */
  int64_t n_new;       /* distinct children not seen at an earlier level        */
  int64_t kept;        /* children kept in the next frontier (after thinning)   */
  uint64_t tau;        /* thinning threshold used (0 = no thinning)             */
  double ms;           /* device time of the level (CUDA events)                */
  int64_t overflow_fixes; /* (parent, neuron) base values (every neuron fires its first
                             applicable rule) outside the storage range, for parents with a
                             kept child: their kept children's entries were recomputed
                             exactly (k_overflow_fix); 0 on the paths that compute every
                             entry exactly                                                  */
} snp_level_counters;

typedef struct snp_system snp_system;
typedef struct snp_tree snp_tree;

int         snp_abi_version(void);
const char *snp_last_error(void);

/* Validate and upload a system (host buffers, deep-copied).  C0 (m counts) is
 * the default level 0.  opt may be NULL (defaults: count_bits 32, dedup 0, no
 * thinning, no budget, keep_tree 1).                                          */
snp_status snp_load(const snp_matrix *M, const snp_rule *rules, int64_t n_rules, const int32_t *C0,
                    int64_t m, const snp_options *opt, snp_system **out);
/* snp_load with general unary regexes: re_bits = n_rules × 4 uint64, row r =
 * membership bits of rule r (bit v of word v / 64: a^v ∈ L(E_r), v < t + P);
 * read for SNP_RE_UNARY rules only; may be NULL if there are none.           */
snp_status snp_load_unary(const snp_matrix *M, const snp_rule *rules, int64_t n_rules, const uint64_t *re_bits,
                          const int32_t *C0, int64_t m, const snp_options *opt, snp_system **out);
/* SN P systems WITH delays (the paper treats systems
 * without delays; reading A26 in DESIGN.md §3).  delays: n_rules
 * int32 d >= 0 (host, copied); a rule fired at step t with d >= 1 closes its
 * neuron at steps t .. t+d-1 (it cannot fire; spikes sent to it are lost) and
 * emits its p spikes at step t+d, when the neuron is open again.  The state
 * is the row [C | τ | π] of snp_state_width = 3m entries (spikes, remaining
 * closed steps, pending emission); C0 has m entries (τ = π = 0 appended) and
 * level0 rows (snp_begin) have 3m.  Halting: no open neuron can fire and no
 * neuron is closed.  Requires opt->dedup = 1 (child keys are fingerprints of
 * the materialised children: the child state is not linear in the rule
 * choice) and out_rule1 = 0; snp_sample, snp_dist_* and
 * snp_tree_spiking_vectors return SNP_E_STATE for such a system.
 * Errors as snp_load, plus SNP_E_ARG for a negative delay.                   */
snp_status snp_load_delay(const snp_matrix *M, const snp_rule *rules, int64_t n_rules, const int32_t *delays,
                          const int32_t *C0, int64_t m, const snp_options *opt, snp_system **out);
/* Releases the caller's reference.  Trees taken from the system (snp_tree)
 * keep it alive: the device state is released when the last of the system
 * and its trees is freed, so a tree stays readable after snp_system_free.  */
void       snp_system_free(snp_system *sys);

/* Launch all device work of `sys` on this cudaStream_t (NULL = library stream). */
snp_status snp_set_stream(snp_system *sys, void *cuda_stream);

/* Incremental exploration (what bench.py times one level at a time):
 *   snp_begin    level 0 := distinct configurations of `level0` (first
 *                occurrence kept; NULL = {C0}) (reading A20), visited := level 0.
 *                Host row-major input is uploaded in 1 GB chunks (two device
 *                staging buffers, the copy of the next chunk overlapping the
 *                import of the current one); pinned memory (snp_host_alloc)
 *                copies at full PCIe rate, pageable memory works.  The input
 *                may be released once snp_begin returns.
 *   snp_advance  expand the current frontier by one level (§8(a) a1-a6);
 *                fills *counters (may be NULL).  An empty frontier is a no-op. */
snp_status snp_begin(snp_system *sys, const snp_configs *level0);
snp_status snp_advance(snp_system *sys, snp_level_counters *counters);
int64_t    snp_frontier_size(const snp_system *sys);
/* Entries per configuration: m, or m + 1 with generated numbers (out_rule1 > 0). */
int64_t    snp_state_width(const snp_system *sys);
/* Numbers generated since the last snp_begin (out_rule1 > 0): bit k of
 * words[k / 64] set iff k was generated, for k < 64 · n_words;
 * *max_number = the largest one (-1 if none).  Any pointer may be NULL.      */
snp_status snp_generated_numbers(snp_system *sys, uint64_t *words, int64_t n_words, int64_t *max_number);
int32_t    snp_depth(const snp_system *sys);
/* Summary of the exploration so far: total configurations, total transitions,
 * and an order-sensitive digest of (level, index, parent, t, fingerprint) of
 * every stored configuration.                                  */
snp_status snp_summary(const snp_system *sys, int64_t *n_configs, int64_t *transitions, uint64_t *digest);

/* Direct access to level L (0 <= L <= snp_depth) of the current exploration:
 *   snp_level_size     configurations of level L
 *   snp_level_edges    parent (index in level L-1, -1 at level 0), t, halting
 *                      (valid once level L was expanded or classified), fp (2 per
 *                      configuration); any pointer may be NULL
 *   snp_level_columns  configurations idx[0..n) of level L as n × m int32 rows;
 *                      needs the level's counts on the device (the current level,
 *                      or every level when keep_tree = 1 or dedup = 0).        */
int64_t    snp_level_size(const snp_system *sys, int32_t level);
snp_status snp_level_edges(snp_system *sys, int32_t level, int64_t *parent, uint64_t *t, uint8_t *halting,
                           uint64_t *fp2);
snp_status snp_level_columns(snp_system *sys, int32_t level, const int64_t *idx, int64_t n, int32_t *out);

/* The spiking vectors S ("generate the succeeding C_k's and
 * their corresponding S_k's"; Alg. 2 II-2/II-3, order of
 * reading A7) — n bytes of 0/1 per vector, rule order = the total order of
 * snp_load:
 *   snp_spiking_vector         the t-th valid spiking vector of the host
 *                              configuration C (snp_state_width int32 counts,
 *                              each in the storage range); SNP_E_ARG when
 *                              t >= Ψ(C) (a halting C has no spiking vector).
 *   snp_level_spiking_vectors  the vector that produced configurations
 *                              idx[0..n) of level L >= 1 from their parents;
 *                              needs level L-1's counts on the device: every
 *                              level with keep_tree = 1 or dedup = 0, else
 *                              the newest level (the engine keeps its parent
 *                              level until the next snp_advance).
 * Systems with delays: SNP_E_STATE.  Synchronous.                            */
snp_status snp_spiking_vector(snp_system *sys, const int32_t *C, uint64_t t, uint8_t *S_out /* n */);
snp_status snp_level_spiking_vectors(snp_system *sys, int32_t level, const int64_t *idx, int64_t n,
                                     uint8_t *S_out /* n_idx × n_rules */);

/* The current frontier (the newest level) copied to host buffers, any of them
 * NULL: configs (F × snp_state_width int32, row-major), parent (index in the
 * previous level, -1 at level 0), t (spiking-vector index).  cap = rows the
 * buffers hold; SNP_E_CAPACITY (nothing copied) when F > cap.  *n_out = F.   */
snp_status snp_frontier_copy(snp_system *sys, int32_t *configs, int64_t *parent, uint64_t *t, int64_t cap,
                             int64_t *n_out);

/* Every transition of the expansion that produced level L >= 1 (options
 * keep_all_edges = 1; reading A17): T(L-1) edges in tag order (parents of
 * level L-1 in order, t increasing), edge e = (parent[e], t[e]) reached the
 * configuration ref[e] = its global discovery index (level offsets as in
 * snp_tree: Σ sizes of the earlier levels + index in its level), or -1 when
 * the child was not stored (dropped by thinning, reading A19, or a terminal
 * transition of generated numbers).  The first-discovery edge of a stored
 * child (snp_level_edges) is among them.  *n_edges = T(L-1); the arrays
 * (any may be NULL) must hold cap entries, SNP_E_CAPACITY when T > cap.
 * SNP_E_STATE without keep_all_edges or in distributed mode.                */
snp_status snp_level_all_edges(snp_system *sys, int32_t level, int64_t *parent, uint64_t *t, int64_t *ref,
                               int64_t cap, int64_t *n_edges);

/* Phase timing (CUDA events on the system's stream), accumulated since the
 * last snp_begin while profiling is on.  Phases (SNP_NUM_PHASES):
 *   0 K-a expand (applicability, Ψ, base fingerprint, emits)
 *   1 K-b offsets scan + child keys (mixed-radix decode, fingerprints)
 *   2 K-d dedup (visited probe, level table, winners, thinning, compaction)
 *   3 K-c materialize kept children (gather-add, ND patches)
 *   4 dedup = 0 full-configuration verification                            */
#define SNP_NUM_PHASES 5
snp_status snp_set_profiling(snp_system *sys, int32_t on);
snp_status snp_profile(const snp_system *sys, double *ms /* SNP_NUM_PHASES */);
/* Kernels launched by this process through libsnp.so so far. */
int64_t    snp_kernel_launches(void);
/* Make CUDA device `device` current for the calling thread inside libsnp.so
 * (its CUDA runtime is its own: one process per GPU calls this with its local
 * rank before snp_load, so every allocation, stream and kernel of the systems
 * it loads lives on that GPU).  SNP_E_ARG for a device index out of range,
 * SNP_E_CUDA when no device is present. */
snp_status snp_set_device(int32_t device);
/* Kernel paths the loaded system takes (bit mask, 0 for NULL):
 *   SNP_PATH_TC_EXPAND  K-a on the tensor cores (k_expand_tc: uint8 storage,
 *                       every neuron tabulated, c <= 15, p <= 1, rule deltas
 *                       linear in (c, p) — DESIGN.md §7); otherwise the CUDA-core
 *                       K-a kernels run.  SNP_KERNELS=no_tc at snp_load turns it off. */
#define SNP_PATH_TC_EXPAND 1
int32_t    snp_kernel_paths(const snp_system *sys);

/* Pinned (page-locked) host memory for the host side of the e2e path: the
 * level-0 input of snp_begin and the outputs of snp_level_edges copy at full
 * PCIe rate from/to it (pageable buffers go through the driver's staging).
 *   snp_host_alloc  *p = bytes of pinned host memory (NULL for bytes = 0),
 *                   owned by the caller until snp_host_free; SNP_E_OOM when the
 *                   allocation fails (*p = NULL), SNP_E_ARG for p = NULL.
 *   snp_host_free   releases a pointer from snp_host_alloc (NULL: no-op).    */
snp_status snp_host_alloc(size_t bytes, void **p);
snp_status snp_host_free(void *p);

/* Multi-GPU exploration, step by step (one process per GPU) —
 * the building blocks snp_dist_advance (below) runs with its own exchanges.
 * Rank r holds a contiguous range of the global frontier (global order = rank
 * order, then local tag order) and the visited keys with owner fmix64(fp1)
 * mod P.  A caller driving the steps runs the collectives between them:
 *   snp_dist_begin(level0 rows of this rank)      → keys of the level-0 rows
 *   snp_dist_expand                               → local T (children keys)
 *   snp_dist_pack(tag_base = Σ T of lower ranks, send: device T×3 uint64
 *                 {fp0, fp1, global tag} grouped by owner, counts[P] host)
 *   [all-to-all of keys]
 *   snp_dist_owner_dedup(recv: device R×3)        → N_new of this owner
 *   [all-reduce of N_new]
 *   snp_dist_owner_keep(N_new global, verdict: device R bytes)
 *   [all-to-all of the verdicts back]
 *   snp_dist_finalize(verdict_back: device T bytes, in send order) → local K
 *   [all-gather of K and of the frontier sizes]
 *   snp_dist_commit(parent_offset, q_offset)      → the next local level
 * dedup = 1 only.  Results (configurations, order, digest) equal a 1-GPU run. */
snp_status snp_dist_begin(snp_system *sys, const snp_configs *level0, int32_t nranks, int64_t *n_local);
snp_status snp_dist_expand(snp_system *sys, int64_t *T_local);
snp_status snp_dist_pack(snp_system *sys, uint64_t tag_base, void *send, int64_t *counts);
snp_status snp_dist_owner_dedup(snp_system *sys, const void *recv, int64_t R, int64_t *n_new_local);
snp_status snp_dist_owner_keep(snp_system *sys, int64_t n_new_global, void *verdict_out);
snp_status snp_dist_finalize(snp_system *sys, const void *verdict_back, int64_t *K_local);
snp_status snp_dist_commit(snp_system *sys, int64_t parent_offset, int64_t q_offset, snp_level_counters *out);

/* Library-driven multi-GPU exploration (one process per GPU; DESIGN.md §9;
 * PAPER.md:425 names inter-block communication for very large systems).
 * The library issues every exchange itself, on the system's stream:
 *   snp_dist_unique_id   rank 0: SNP_DIST_ID_BYTES of NCCL unique id, which
 *                        the caller broadcasts once (any host channel)
 *   snp_dist_init        NCCL communicator of rank `rank` of `nranks` (the
 *                        current CUDA device); libnccl.so.2 is opened at run
 *                        time (SNP_E_NCCL when it is missing)
 *   snp_local_group_create / snp_dist_init_local
 *                        the same protocol among nranks snp_system handles of
 *                        ONE process (one host thread each; device-to-device
 *                        copies) — logical ranks on one GPU, used by the tests
 *   snp_dist_start       level 0 := the distinct configurations of the
 *                        concatenation of every rank's level0_local (rank
 *                        order); *F_global = its size
 *   snp_dist_advance     one BFS level over all ranks: local K-a/K-b, key
 *                        all-to-all to owner = fmix64(fp1) mod P, owner-side
 *                        dedup and thinning (τ from the global N_new, A19),
 *                        verdicts back, local K-c; then, when the largest
 *                        local frontier exceeds `rebalance` (default 1.1) ×
 *                        the mean, rows move so that rank r holds the global
 *                        range [F·r/P, F·(r+1)/P).  *global = the level's
 *                        counters summed over ranks (ms = the slowest rank);
 *                        *local = this rank's share (parents, T, kept before
 *                        the redistribution, owner-side n_new, its ms).
 *   snp_dist_summary     (collective) global configurations, transitions and
 *                        the run digest — equal to a 1-GPU run's.
 *   snp_dist_local       this rank's frontier size, its global offset, and
 *                        the rows it sent in the last rebalancing.
 * Every rank must make the same sequence of collective calls.  A failure on
 * any rank (overflow, capacity, a CUDA or NCCL error) is agreed at the next
 * exchange: every rank returns the failing rank's status (the lowest rank's
 * when several fail) rather than waiting for it.  NCCL waits poll
 * ncclCommGetAsyncError and abort after SNP_DIST_TIMEOUT_S seconds (default
 * 600).  Parents reported by snp_level_edges are global indices in this mode.
 * dedup = 1 only; no generated numbers, delays or keep_all_edges.           */
#define SNP_DIST_ID_BYTES 128
typedef struct snp_local_group snp_local_group;
snp_status snp_dist_unique_id(void *id_out /* SNP_DIST_ID_BYTES */);
snp_status snp_dist_init(snp_system *sys, const void *id, int32_t rank, int32_t nranks);
snp_status snp_local_group_create(int32_t nranks, snp_local_group **out);
void       snp_local_group_free(snp_local_group *group);
snp_status snp_dist_init_local(snp_system *sys, snp_local_group *group, int32_t rank);
snp_status snp_dist_set_rebalance(snp_system *sys, double threshold /* 0 = never */);
snp_status snp_dist_start(snp_system *sys, const snp_configs *level0_local, int64_t *F_global);
snp_status snp_dist_advance(snp_system *sys, snp_level_counters *global, snp_level_counters *local /* may be NULL */);
snp_status snp_dist_summary(snp_system *sys, int64_t *n_configs, int64_t *transitions, uint64_t *digest);
snp_status snp_dist_local(const snp_system *sys, int64_t *F_local, int64_t *global_offset, int64_t *rebalanced_rows);

/* Single-path sampling with an input spike train (Def. 1
 * `in`; deep computation trees take long to
 * explore).  Each of W walkers follows ONE computation path for `steps` steps:
 * at step k a walker with Ψ > 0 (eq. (8)) takes the child
 * t = u mod Ψ in the enumeration order of Alg. 2 (reading
 * A7), u = splitmix64(splitmix64(seed ^ (k << 32)) ^ w) (reading A25), i.e.
 * C <- C + S_t·M (eq. (2)); then the input neuron (input_neuron >= 0)
 * receives train[k] spikes from the environment while k < train_len.  A
 * walker with no applicable rule keeps its configuration while input is
 * still to come and stops once it is not: halted_step[w] = k (-1 = still
 * running after `steps` steps; reading A5).
 *   configs      W × m int32 row-major, in/out (host); every count must lie in
 *                [0, storage max] on entry (SNP_E_ARG otherwise)
 *   train        train_len int32 (host), may be NULL when train_len == 0
 *   halted_step  W int32 (host), out
 * Errors: SNP_E_ARG (bad arguments), SNP_E_STATE (system loaded with
 * out_rule1), SNP_E_CAPACITY (some Ψ > 2^62), SNP_E_OVERFLOW (a count left
 * the storage range after a step; capacity is reported first); configs and
 * halted_step are then unspecified.  Synchronous; one kernel launch. */
snp_status snp_sample(snp_system *sys, int64_t W, int32_t *configs, uint64_t seed, int32_t steps,
                      int32_t input_neuron, const int32_t *train, int32_t train_len, int32_t *halted_step);

/* snp_begin + `depth` × snp_advance + halting classification of the last
 * level; the tree is a snapshot owned by the caller.                          */
snp_status snp_explore(snp_system *sys, const snp_configs *level0, int32_t depth, snp_tree **out);
/* One level from an arbitrary frontier: explore with depth 1.                 */
snp_status snp_step(snp_system *sys, const snp_configs *frontier, snp_tree **out);

int32_t    snp_tree_num_levels(const snp_tree *tree);
int64_t    snp_tree_num_configs(const snp_tree *tree);
snp_status snp_tree_level_offsets(const snp_tree *tree, int64_t *out /* num_levels + 1 */);
/* configurations in discovery order, row-major int32 (needs keep_tree).       */
snp_status snp_tree_configs(const snp_tree *tree, int32_t *out /* N × m */);
/* parent = index in the previous level (-1 at level 0), t = spiking-vector index,
 * halting flags, fingerprints (2 per configuration). Any pointer may be NULL. */
snp_status snp_tree_edges(const snp_tree *tree, int64_t *parent, uint64_t *t, uint8_t *halting,
                          uint64_t *fp2);
snp_status snp_tree_counters(const snp_tree *tree, snp_level_counters *out /* num_levels - 1 */);
/* The spiking vector S (n bytes of 0/1) that produced each configuration of
 * level L >= 1 from its parent (needs keep_tree).                             */
snp_status snp_tree_spiking_vectors(const snp_tree *tree, int32_t level, uint8_t *S_out /* count × n */);
void       snp_tree_free(snp_tree *tree);

#ifdef __cplusplus
}
#endif
#endif /* SNP_H_ */
