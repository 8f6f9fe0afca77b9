// snp_device.cuh — device-side data model and helpers of the SNP engine.
//
// Layout in HBM:
//   * a frontier is BLOCKED neuron-major: configurations are grouped in
//     blocks of PB = 64; block b holds the m × 64 counts of its configurations
//     neuron by neuron, so element (configuration p, neuron s) lives at
//         ((p / 64) · m + s) · 64 + p % 64
//     and a block is one contiguous m·64·w-byte stream.  Kernels that walk
//     the neurons of a group of configurations (K-a, K-c) read whole
//     contiguous blocks; every rule descriptor / synapse index is uniform
//     across the lanes that share a neuron.
//   * rules are grouped per neuron (rule_off[s] .. rule_off[s+1]) in the
//     paper's total order.
//   * per-neuron outcome tables: for a count v the first
//     applicable rule, whether it spikes, and whether ≥ 2 rules apply.
//   * the synapse graph is stored twice: in-CSR by target (the gather of the
//     transition) and out-CSR by source (the sparse ND patches).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace snp {

constexpr int64_t TC_M_MAX = 1 << 19;        // k_expand_tc: s32 accumulators exact up to this m
constexpr int EPAD = 16;  // zero emit words after the m real ones: padded in-CSR entries (one per bank pair)
constexpr int KMAX = 64;                    // nondeterministic neurons recorded per parent
constexpr int PB = 64;                      // configurations per storage block
constexpr uint64_t PSI_LIMIT = 1ULL << 62;  // Ψ above this is SNP_E_CAPACITY
constexpr uint64_t EMPTY = ~0ULL;           // empty hash-slot key word
constexpr int TABW_MAX = 512;               // compact outcome-table width limit
constexpr int MAX_TABLE_RULES = 15;         // rules per neuron representable in a table entry

// error bits raised by kernels (ORed into a device word)
enum : int32_t {
  ERR_CAPACITY = 1,
  ERR_OVERFLOW = 2,
  ERR_COLLISION = 4,
  ERR_TABLE_FULL = 8,
};

__host__ __device__ __forceinline__ int64_t eidx(int64_t p, int32_t s, int32_t m) {
  return ((p >> 6) * (int64_t)m + s) * PB + (p & (PB - 1));
}

// Applicability of one rule as an interval + residue test:
//   a^v ∈ L(E) && v >= c   <=>   lo <= v <= hi  &&  (v - base) ≡ 0 (mod j)
//   EXACT(k):      lo = max(k, c), hi = k,       base = k, j = 1
//   PERIODIC(i,j): lo = max(i, c), hi = INT_MAX, base = i, j = j
// or, for a general unary regex (UNARY(t, P)), a
// membership test on the ultimately periodic bit row:
//   lo = c, hi = INT_MAX, base = t, j = P, unary = 1,
//   a^v ∈ L(E)  <=>  bit idx of bits, idx = v < t + P ? v : t + (v - t) mod P
struct DevRule {
  int32_t lo, hi, base, j;
  int32_t jmask;  // j - 1 when j is a power of two, else -1
  int32_t c, p;   // consumed, produced
  int32_t unary;  // 1: membership row below
  uint64_t bits[4];
};

__device__ __forceinline__ bool rule_app(const DevRule& r, int32_t v) {
  if (v < r.lo || v > r.hi) return false;
  if (r.unary) {
    const uint32_t u = (uint32_t)v, t = (uint32_t)r.base, P = (uint32_t)r.j;
    const uint32_t idx = u < t + P ? u : t + (u - t) % P;
    return (r.bits[idx >> 6] >> (idx & 63)) & 1ULL;
  }
  if (r.j == 1) return true;
  int32_t d = v - r.base;
  return r.jmask >= 0 ? ((d & r.jmask) == 0) : (d % r.j == 0);
}

// Per-neuron table descriptor.  For counts v >= L the outcome repeats with
// period P (every PERIODIC rule's j divides P; no EXACT rule applies), so
//   idx(v) = v < L ? v : L + (v - L) mod P.
// pm = P - 1 when P is a power of two, else -P.  flags: bit 0 = no table
// (evaluate the rules), bit 1 = some count makes >= 2 rules applicable.
struct NeuronMeta {
  int32_t rbase;   // first rule of the neuron
  int32_t L;
  int32_t pm;
  int32_t flags;
};
enum : int32_t { NM_GENERIC = 1, NM_ND = 2 };
// outcome-table entry (uint8): bit 0 = the first applicable rule spikes
// (p > 0), bit 1 = >= 2 rules applicable, bits 4-7 = first applicable local
// rule + 1 (0 = none) — pre-shifted so (entry & 0xF0) is the byte offset of
// that rule's 16-B fingerprint delta in a neuron's 256-B slice.
enum : uint32_t { TE_EMIT = 1u, TE_ND = 2u, TE_F = 0xF0u };
// kernel selection flags (SysView::kernel_flags)
enum : int32_t { KF_EXPAND_T = 1, KF_KC_GLOBAL_E = 2, KF_NO_TC = 4, KF_KC_TC = 8, KF_KC_WIDE_EXACT = 16, KF_FP_WEAK = 32 };

__device__ __forceinline__ uint32_t table_index(uint32_t v, const NeuronMeta& mt) {
  // unsigned compare: lanes past F in a partial block may hold any bit
  // pattern (a negative int32 must still land inside the table)
  if (v < (uint32_t)mt.L) return v;
  uint32_t d = v - (uint32_t)mt.L;
  return (uint32_t)mt.L + (mt.pm >= 0 ? (d & (uint32_t)mt.pm) : d % (uint32_t)(-mt.pm));
}

struct SysView {
  int32_t m;
  int32_t binary_emit;   // every p <= 1: emits are one bit per (neuron, config)
  int64_t n;
  int64_t count_max;     // 255 / 65535 / INT32_MAX
  const int32_t* rule_off;   // m + 1
  const DevRule* rules;      // n
  const uint64_t* h0;        // n: h_ℓ[r] = Σ_j M[r][j]·R_ℓ[j] mod 2^64
  const uint64_t* h1;
  const int32_t* in_off;     // m + 1
  const int32_t* in_src;     // sources s with (s, j) ∈ syn, grouped by target j
  // the same in-synapses "edge-major" per group of 32 consecutive targets:
  // group g holds in_pad_off[g+1] - in_pad_off[g] rows of 32 sources (row e,
  // lane l = e-th in-synapse of target 32g + l), padded with the index m_even
  // (a zero word)
  const int32_t* in_pad;
  const uint16_t* in_pad16;    // the same as uint16 when m < 65535 (else null)
  const uint64_t* in_pad16x4;  // the same, 4 rows per lane packed: [row/4][lane] (null with in_pad16)
  const int64_t* in_pad_off;   // m/32 + 1 row offsets (×32 entries)
  const int32_t* out_off;    // m + 1
  const int32_t* out_dst;    // targets j with (s, j) ∈ syn, grouped by source s
  const uint64_t* R0;        // m fingerprint weights (reading A18)
  const uint64_t* R1;
  // outcome tables (valid when tables_ok)
  int32_t tables_ok;         // every neuron is tabulated or flagged generic
  int32_t tabw;              // compact table width (power of two >= every L + P)
  int32_t full8;             // count_bits == 8: tab_full has 256 entries per neuron
  int32_t max_indeg;
  int64_t n_in;              // in-synapses (in_off[m])
  const NeuronMeta* meta;    // m
  const uint8_t* tab;        // m × tabw   (compact)
  const uint8_t* tab_full;   // m × 256    (count_bits == 8)
  const void* ctab;          // m × tabw   consumption of the first rule, storage type
  const uint8_t* ttab;       // (count_bits == 8) v - c_first(v): m × 32 for v < 32, then m × 256 for every v
  const uint8_t* elut;       // m × 32     (count_bits == 8) outcome entries for v < 32
  const uint8_t* hsg;        // m × 256    (count_bits == 8) 16-B fingerprint delta per first-rule slot
  int32_t any_generic;       // some neuron has no table
  int32_t kernel_flags;      // KF_* (SNP_KERNELS environment variable at snp_load; tuning/tests)
  // generated numbers (include/snp.h): the augmented
  // column A is neuron m - 1 (no rule, no synapse); aug_rule = -1 when off
  int32_t aug_rule;          // output neuron's spiking rule
  int32_t aug_neuron;        // its neuron
  unsigned long long* gen_bits;  // generated-number bitmap
  int64_t gen_cap_bits;
  // tensor-core K-a (k_expand_tc), valid when tc_ok: uint8
  // storage, every neuron tabulated, c <= 15, p <= 1 and every rule delta
  // h_ℓ[r] = −c_r·R_ℓ[s] + p_r·Rout_ℓ[s]
  int32_t tc_ok;
  int32_t n_nd;              // neurons with some count making >= 2 rules applicable
  const int32_t* nd_list;    // n_nd, increasing
  const uint8_t* xyt;        // m × 32   first rule c | p << 4 for v < 32 (0 = none)
  const uint16_t* cpT;       // 32 × m   first rule c | p << 8 at count v < 32, count-major (verification; c, p <= 255)
  const uint8_t* xyf;        // m × 256  the same for every uint8 count
  const uint8_t* btile;      // ceil(m/64) × 4096: B chunks (−R bytes | 1, Rout bytes), K-major core matrices
  // SN P systems with delays (reading A26): delay_m > 0
  // real neurons, the state row is [C | τ | π] (m = 3·delay_m columns)
  int32_t delay_m;
  int32_t small_cp;          // every rule has c, p <= 255 (packed fired (c, p) tables)
  const int32_t* delay;      // n: d >= 0 per rule
};
// key of a terminal child (second output spike): skipped by the dedup
constexpr uint64_t KEY_TERMINAL1 = ~0ULL - 1;

// 128-bit hash slot. key (k0,k1) = 128-bit fingerprint; EMPTY/EMPTY = free.
struct alignas(16) Key128 {
  unsigned long long k0, k1;
};
struct alignas(32) Slot {
  unsigned long long k0, k1;
  unsigned long long tag;  // level table: minimum child tag; visited: unused
  unsigned long long ref;  // visited: (level << 40) | column
};

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xFF51AFD7ED558CCDULL;
  k ^= k >> 33;
  k *= 0xC4CEB9FE1A85EC53ULL;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a > PSI_LIMIT / b) return PSI_LIMIT + 1;
  uint64_t r = a * b;
  return r > PSI_LIMIT ? PSI_LIMIT + 1 : r;
}

// 8 consecutive counts of one neuron row inside a block (p0 % 8 == 0)
template <typename T>
__device__ __forceinline__ void load8(const T* data, int64_t p0, int32_t s, int32_t m, int64_t F, uint32_t v[8]);

template <>
__device__ __forceinline__ void load8<uint8_t>(const uint8_t* data, int64_t p0, int32_t s, int32_t m, int64_t F,
                                              uint32_t v[8]) {
  const uint8_t* row = data + eidx(p0, s, m);
  if (p0 + 7 < F) {
    uint2 w = __ldg(reinterpret_cast<const uint2*>(row));
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[k] = (w.x >> (8 * k)) & 0xFF; v[k + 4] = (w.y >> (8 * k)) & 0xFF; }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (p0 + k < F) ? row[k] : 0u;
  }
}
template <>
__device__ __forceinline__ void load8<uint16_t>(const uint16_t* data, int64_t p0, int32_t s, int32_t m, int64_t F,
                                               uint32_t v[8]) {
  const uint16_t* row = data + eidx(p0, s, m);
  if (p0 + 7 < F) {
    uint4 w = __ldg(reinterpret_cast<const uint4*>(row));
    v[0] = w.x & 0xFFFF; v[1] = w.x >> 16; v[2] = w.y & 0xFFFF; v[3] = w.y >> 16;
    v[4] = w.z & 0xFFFF; v[5] = w.z >> 16; v[6] = w.w & 0xFFFF; v[7] = w.w >> 16;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (p0 + k < F) ? row[k] : 0u;
  }
}
template <>
__device__ __forceinline__ void load8<int32_t>(const int32_t* data, int64_t p0, int32_t s, int32_t m, int64_t F,
                                              uint32_t v[8]) {
  const int32_t* row = data + eidx(p0, s, m);
  if (p0 + 7 < F) {
    int4 a = __ldg(reinterpret_cast<const int4*>(row));
    int4 b = __ldg(reinterpret_cast<const int4*>(row) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (p0 + k < F) ? (uint32_t)row[k] : 0u;
  }
}

// ---- TMA bulk copies (cp.async.bulk) and mbarriers --------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// global -> L2 bulk prefetch (bytes % 16 == 0, address 16-aligned); no completion
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace snp
