// snp_device.cuh — device-side data model and helpers of the SNP engine.
//
// Layout in HBM:
//   * a frontier is NEURON-MAJOR: element (s, p) = spike count of neuron s in
//     configuration p, at data[s * pitch + p], stored as uint8/uint16/int32
//     (count_bits, reading A16).  A warp owns a tile of 128 consecutive
//     configurations (4 per lane) and walks the neurons, so every rule
//     descriptor / in-synapse index it reads is warp-uniform (broadcast) and
//     every count load is a coalesced 128-element row segment.
//   * rules are grouped per neuron (rule_off[s] .. rule_off[s+1]) in the
//     paper's total order.
//   * the synapse graph is stored twice: in-CSR by target (the gather of the
//     transition) and out-CSR by source (the sparse ND patches).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace snp {

constexpr int KMAX = 64;                    // nondeterministic neurons recorded per parent
constexpr int TILE = 128;                   // configurations per warp tile (4 per lane)
constexpr uint64_t PSI_LIMIT = 1ULL << 62;  // Ψ above this is SNP_E_CAPACITY
constexpr uint64_t EMPTY = ~0ULL;           // empty hash-slot key word

// error bits raised by kernels (ORed into a device word)
enum : int32_t {
  ERR_CAPACITY = 1,
  ERR_OVERFLOW = 2,
  ERR_COLLISION = 4,
  ERR_TABLE_FULL = 8,
};

// Applicability of one rule as an interval + residue test:
//   a^v ∈ L(E) && v >= c   <=>   lo <= v <= hi  &&  (v - base) ≡ 0 (mod j)
//   EXACT(k):      lo = max(k, c), hi = k,       base = k, j = 1
//   PERIODIC(i,j): lo = max(i, c), hi = INT_MAX, base = i, j = j
struct DevRule {
  int32_t lo, hi, base, j;
  int32_t jmask;  // j - 1 when j is a power of two, else -1
  int32_t c, p;   // consumed, produced
  int32_t pad;
};

__device__ __forceinline__ bool rule_app(const DevRule& r, int32_t v) {
  if (v < r.lo || v > r.hi) return false;
  if (r.j == 1) return true;
  int32_t d = v - r.base;
  return r.jmask >= 0 ? ((d & r.jmask) == 0) : (d % r.j == 0);
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
  const int32_t* out_off;    // m + 1
  const int32_t* out_dst;    // targets j with (s, j) ∈ syn, grouped by source s
  const uint64_t* R0;        // m fingerprint weights (reading A18)
  const uint64_t* R1;
};

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

template <typename T>
__device__ __forceinline__ void load4(const T* row, int64_t p0, int64_t F, int32_t v[4]);

template <>
__device__ __forceinline__ void load4<uint8_t>(const uint8_t* row, int64_t p0, int64_t F, int32_t v[4]) {
  if (p0 + 3 < F) {
    uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(row + p0));
    v[0] = w & 0xFF; v[1] = (w >> 8) & 0xFF; v[2] = (w >> 16) & 0xFF; v[3] = w >> 24;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (p0 + k < F) ? (int32_t)row[p0 + k] : 0;
  }
}
template <>
__device__ __forceinline__ void load4<uint16_t>(const uint16_t* row, int64_t p0, int64_t F, int32_t v[4]) {
  if (p0 + 3 < F) {
    uint2 w = __ldg(reinterpret_cast<const uint2*>(row + p0));
    v[0] = w.x & 0xFFFF; v[1] = w.x >> 16; v[2] = w.y & 0xFFFF; v[3] = w.y >> 16;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (p0 + k < F) ? (int32_t)row[p0 + k] : 0;
  }
}
template <>
__device__ __forceinline__ void load4<int32_t>(const int32_t* row, int64_t p0, int64_t F, int32_t v[4]) {
  if (p0 + 3 < F) {
    int4 w = __ldg(reinterpret_cast<const int4*>(row + p0));
    v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (p0 + k < F) ? row[p0 + k] : 0;
  }
}

}  // namespace snp
