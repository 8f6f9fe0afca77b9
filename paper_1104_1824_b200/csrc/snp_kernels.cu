// snp_kernels.cu — sm_100a kernels of the batched SNP transition step.
//
//   K-a  k_expand        rule applicability per (neuron, configuration)
//                        (Alg. 2 II-1), Ψ (eq. (8),
//                        PAPER.md:250, readings A3/A5), the base-child
//                        fingerprint and the first-choice emits.
//   K-b  CUB scan + k_child_parent + k_child_keys: child offsets, mixed-radix
//                        decode of t (Alg. 2 II-2/II-3, PAPER.md:263-264,
//                        reading A7) and the child fingerprint by linearity.
//   K-d  k_dedup / k_winners / k_keep / k_compact: GPU open-addressing sets
//                        (visited + level table with minimum-tag resolution,
//                        readings A6, A19, A22).
//   K-c  k_materialize + k_patch + k_overflow_fix: C' = C + S·M (eq. (2),
//                        PAPER.md:129) for the kept children only, as a
//                        gather-add over the in-synapses (Def. 2,
//                        PAPER.md:115-119) plus exact sparse ND corrections.
//
// Every kernel is plain CUDA C++ for sm_100a; the path is integer and bound
// by HBM / issue bandwidth, not by tensor cores.
#include <atomic>

#include <cub/cub.cuh>

#include "snp_internal.h"

namespace snp {

std::atomic<int64_t> g_kernel_launches{0};

namespace {

constexpr int BLK = 256;

inline void count_launch(int64_t n = 1) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }

inline unsigned grid_for(uint64_t n, int blk = BLK) {
  uint64_t g = (n + blk - 1) / blk;
  if (g > 0x7FFFFFFFULL) g = 0x7FFFFFFFULL;
  return (unsigned)(g ? g : 1);
}

template <typename T>
__device__ __forceinline__ int32_t ld_count(const void* data, int64_t pitch, int32_t j, int64_t p) {
  return (int32_t) reinterpret_cast<const T*>(data)[(int64_t)j * pitch + p];
}

// Applicable rules of neuron s holding v spikes: count and the x-th one.
__device__ __forceinline__ int count_applicable(const SysView& S, int32_t s, int32_t v) {
  int d = 0;
  for (int r = S.rule_off[s]; r < S.rule_off[s + 1]; ++r) d += rule_app(S.rules[r], v);
  return d;
}
__device__ __forceinline__ int nth_applicable(const SysView& S, int32_t s, int32_t v, int x) {
  for (int r = S.rule_off[s]; r < S.rule_off[s + 1]; ++r) {
    if (rule_app(S.rules[r], v)) {
      if (x == 0) return r;
      --x;
    }
  }
  return -1;
}

// A child described virtually by its parent's nondeterministic neurons and
// the mixed-radix digits of t (least significant digit = last ND neuron).
struct ChildCtx {
  int K;
  int32_t s[KMAX];
  uint8_t x[KMAX];
};

__device__ void decode_child(const SysView& S, const uint64_t* nd_p, int K, uint64_t t, ChildCtx& cx) {
  cx.K = K;
  for (int i = K - 1; i >= 0; --i) {
    uint64_t e = nd_p[i];
    int32_t s = (int32_t)(e >> 32), v = (int32_t)(uint32_t)e;
    uint64_t d = (uint64_t)count_applicable(S, s, v);
    cx.s[i] = s;
    cx.x[i] = (uint8_t)(t % d);
    t /= d;
  }
}

// rule fired by neuron s (count v) in the child: the x-th applicable rule if
// s is nondeterministic in the parent, else its first applicable rule.
__device__ int fired_rule(const SysView& S, int32_t s, int32_t v, const ChildCtx& cx) {
  int lo = 0, hi = cx.K;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cx.s[mid] < s) lo = mid + 1; else hi = mid;
  }
  int x = (lo < cx.K && cx.s[lo] == s) ? cx.x[lo] : 0;
  return nth_applicable(S, s, v, x);
}

// Exact value of the child at neuron j: eq. (2) restricted to column j,
// C'[j] = C[j] - c_{fired(j)} + Σ_{s ∈ in(j)} p_{fired(s)}  (Def. 2).
template <typename T>
__device__ int64_t exact_value(const SysView& S, const void* data, int64_t pitch, int64_t p, int32_t j,
                               const ChildCtx& cx) {
  int32_t vj = ld_count<T>(data, pitch, j, p);
  int rj = fired_rule(S, j, vj, cx);
  int64_t val = (int64_t)vj - (rj >= 0 ? S.rules[rj].c : 0);
  for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) {
    int32_t s = S.in_src[e];
    int rs = fired_rule(S, s, ld_count<T>(data, pitch, s, p), cx);
    if (rs >= 0) val += S.rules[rs].p;
  }
  return val;
}

// ---------------------------------------------------------------------------
// import / export between the ABI's layouts and the device frontier
// ---------------------------------------------------------------------------
template <typename Tin>
__device__ __forceinline__ int64_t ld_in(const void* src, int64_t idx) {
  return (int64_t) reinterpret_cast<const Tin*>(src)[idx];
}

template <typename Tin, typename Tout>
__global__ void k_import(const void* src, int32_t layout, int64_t ld, int64_t F, int32_t m, Tout* dst, int64_t pitch,
                         int64_t count_max, int32_t* err) {
  // 32×32 tiles; row-major input is transposed through shared memory.
  __shared__ int64_t tile[32][33];
  const int64_t p_base = (int64_t)blockIdx.x * 32;
  const int32_t j_base = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 × 8
  bool bad = false;
  if (layout == 0) {  // row-major: element (p, j) at src[p * ld + j]
    for (int r = ty; r < 32; r += 8) {
      int64_t p = p_base + r;
      int32_t j = j_base + tx;
      tile[r][tx] = (p < F && j < m) ? ld_in<Tin>(src, p * ld + j) : 0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      int32_t j = j_base + r;
      int64_t p = p_base + tx;
      if (p < F && j < m) {
        int64_t v = tile[tx][r];
        bad |= (v < 0 || v > count_max);
        dst[(int64_t)j * pitch + p] = (Tout)v;
      }
    }
  } else {  // neuron-major: element (p, j) at src[j * ld + p]
    for (int r = ty; r < 32; r += 8) {
      int32_t j = j_base + r;
      int64_t p = p_base + tx;
      if (p < F && j < m) {
        int64_t v = ld_in<Tin>(src, (int64_t)j * ld + p);
        bad |= (v < 0 || v > count_max);
        dst[(int64_t)j * pitch + p] = (Tout)v;
      }
    }
  }
  if (bad) atomicOr(err, ERR_OVERFLOW);
}

template <typename T>
__global__ void k_export(const T* src, int64_t pitch, int64_t F, int32_t m, int32_t* dst) {
  __shared__ int32_t tile[32][33];
  const int64_t p_base = (int64_t)blockIdx.x * 32;
  const int32_t j_base = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    int32_t j = j_base + r;
    int64_t p = p_base + tx;
    tile[r][tx] = (p < F && j < m) ? (int32_t)src[(int64_t)j * pitch + p] : 0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    int64_t p = p_base + r;
    int32_t j = j_base + tx;
    if (p < F && j < m) dst[p * m + j] = tile[tx][r];
  }
}

// fp_ℓ(C) = Σ_j C[j]·R_ℓ[j] mod 2^64 (reading A18), one column per thread
// slot; warp tiles of 128 configurations as in k_expand.
template <typename T>
__global__ void __launch_bounds__(128) k_fingerprint(SysView S, const T* data, int64_t pitch, int64_t F,
                                                      uint64_t* fp0, uint64_t* fp1) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t p0 = tile * TILE + 4 * lane;
  if (tile * TILE >= F) return;
  uint64_t a[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
  for (int32_t j = 0; j < S.m; ++j) {
    int32_t v[4];
    load4<T>(data + (int64_t)j * pitch, p0, F, v);
    const uint64_t r0 = __ldg(S.R0 + j), r1 = __ldg(S.R1 + j);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[k] += (uint64_t)v[k] * r0;
      b[k] += (uint64_t)v[k] * r1;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (p0 + k < F) { fp0[p0 + k] = a[k]; fp1[p0 + k] = b[k]; }
}

// ---------------------------------------------------------------------------
// K-a: applicability, Ψ, base fingerprint, emits
// ---------------------------------------------------------------------------
template <typename T, bool BIN>
__global__ void __launch_bounds__(128) k_expand(SysView S, LevelView L, ExpandOut O) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t p0 = tile * TILE + 4 * lane;
  if (tile * TILE >= L.F) return;  // warp-uniform
  const T* data = reinterpret_cast<const T*>(L.data);
  uint64_t f0[4], f1[4], psi[4];
  int ndc[4];
  bool any[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool ok = p0 + k < L.F;
    f0[k] = ok ? L.fp0[p0 + k] : 0;
    f1[k] = ok ? L.fp1[p0 + k] : 0;
    psi[k] = 1;
    ndc[k] = 0;
    any[k] = false;
  }
  uint32_t eword = 0;
  for (int32_t s = 0; s < S.m; ++s) {
    int32_t v[4];
    load4<T>(data + (int64_t)s * L.pitch, p0, L.F, v);
    const int r0 = __ldg(S.rule_off + s), r1 = __ldg(S.rule_off + s + 1);
    int first[4] = {-1, -1, -1, -1};
    int d[4] = {0, 0, 0, 0};
    for (int r = r0; r < r1; ++r) {
      const DevRule R = S.rules[r];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (rule_app(R, v[k])) {
          if (d[k] == 0) first[k] = r;
          ++d[k];
        }
      }
    }
    uint32_t nib = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (p0 + k >= L.F) d[k] = 0;
      if (d[k] > 0) {
        any[k] = true;
        f0[k] += __ldg(S.h0 + first[k]);
        f1[k] += __ldg(S.h1 + first[k]);
        if (d[k] >= 2) {
          if (!O.classify_only && ndc[k] < KMAX)
            O.nd[(p0 + k) * KMAX + ndc[k]] = ((uint64_t)(uint32_t)s << 32) | (uint32_t)v[k];
          ++ndc[k];
          psi[k] = sat_mul(psi[k], (uint64_t)d[k]);
        }
        if (BIN && S.rules[first[k]].p > 0) nib |= 1u << k;
      }
    }
    if (!O.classify_only) {
      if (BIN) {
        eword |= nib << (4 * (s & 7));
        if ((s & 7) == 7 || s == S.m - 1) {
          O.ebits[(int64_t)(s >> 3) * O.ebits_ld + tile * 32 + lane] = eword;
          eword = 0;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (p0 + k < L.F) O.evals[(int64_t)s * O.evals_ld + p0 + k] = d[k] > 0 ? S.rules[first[k]].p : 0;
      }
    }
  }
  unsigned nh = 0;
  bool cap = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t p = p0 + k;
    if (p >= L.F) continue;
    const uint64_t ps = any[k] ? psi[k] : 0;  // halting: no children (reading A5)
    cap |= ps > PSI_LIMIT || ndc[k] > KMAX;
    O.halting[p] = any[k] ? 0 : 1;
    nh += any[k] ? 0 : 1;
    if (!O.classify_only) {
      O.psi[p] = ps;
      O.fpb0[p] = f0[k];
      O.fpb1[p] = f1[k];
      O.ndc[p] = ndc[k];
    }
  }
  if (cap && !O.classify_only) atomicOr(O.err, ERR_CAPACITY);
  if (nh) atomicAdd(O.n_halting, (unsigned long long)nh);
}

// ---------------------------------------------------------------------------
// K-b: children of each parent, their fingerprints by linearity
// ---------------------------------------------------------------------------
__global__ void k_child_parent(const uint64_t* off, int64_t F, uint32_t* cpar) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < F; p += (int64_t)gridDim.x * blockDim.x)
    for (uint64_t c = off[p]; c < off[p + 1]; ++c) cpar[c] = (uint32_t)p;
}

// fp(child t) = fp(base) + Σ_{ND s} (h[A_s[x_s]] - h[A_s[0]])  (reading A18),
// x = mixed-radix digits of t, first ND neuron most significant (reading A7).
__global__ void k_child_keys(SysView S, const uint64_t* off, ExpandOut O, uint64_t T, ChildArrays C) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = C.cpar[c];
    uint64_t t = c - off[p];
    uint64_t a = O.fpb0[p], b = O.fpb1[p];
    const int K = O.ndc[p];
    const uint64_t* nd = O.nd + (uint64_t)p * KMAX;
    for (int i = K - 1; i >= 0 && t; --i) {
      const uint64_t e = nd[i];
      const int32_t s = (int32_t)(e >> 32), v = (int32_t)(uint32_t)e;
      const uint64_t d = (uint64_t)count_applicable(S, s, v);
      const int x = (int)(t % d);
      t /= d;
      if (x) {
        const int rf = nth_applicable(S, s, v, 0), rc = nth_applicable(S, s, v, x);
        a += __ldg(S.h0 + rc) - __ldg(S.h0 + rf);
        b += __ldg(S.h1 + rc) - __ldg(S.h1 + rf);
      }
    }
    C.cfp0[c] = a;
    C.cfp1[c] = b;
  }
}

// ---------------------------------------------------------------------------
// K-d: dedup against visited + same-level minimum tag
// ---------------------------------------------------------------------------
__device__ __forceinline__ Key128 ld_key(const Slot* s) { return *reinterpret_cast<const Key128*>(s); }

__global__ void k_dedup(ChildArrays C, uint64_t T, uint64_t tag_base, Tables tb, int use_visited, int32_t* err) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k0 = C.cfp0[c], k1 = C.cfp1[c];
    if (k0 == EMPTY && k1 == EMPTY) {
      atomicOr(err, ERR_COLLISION);
      C.verdict[c] = 0;
      C.cref[c] = EMPTY;
      continue;
    }
    const uint64_t h = fmix64(k0);
    bool old = false;
    if (use_visited) {
      uint64_t i = h & tb.vmask;
      for (uint64_t probes = 0; probes <= tb.vmask; ++probes, i = (i + 1) & tb.vmask) {
        const Key128 key = ld_key(tb.vis + i);
        if (key.k0 == k0 && key.k1 == k1) {
          old = true;
          C.cref[c] = tb.vis[i].ref;
          break;
        }
        if (key.k0 == EMPTY && key.k1 == EMPTY) break;
      }
    }
    if (old) {
      C.verdict[c] = 0;
      continue;
    }
    uint64_t i = h & tb.lmask;
    bool done = false;
    for (uint64_t probes = 0; probes <= tb.lmask; ++probes, i = (i + 1) & tb.lmask) {
      Key128 empty{EMPTY, EMPTY}, mine{k0, k1};
      const Key128 prev = atomicCAS(reinterpret_cast<Key128*>(tb.ltab + i), empty, mine);
      if ((prev.k0 == EMPTY && prev.k1 == EMPTY) || (prev.k0 == k0 && prev.k1 == k1)) {
        atomicMin(&tb.ltab[i].tag, (unsigned long long)(tag_base + c));
        C.cslot[c] = i;
        C.verdict[c] = 1;
        done = true;
        break;
      }
    }
    if (!done) atomicOr(err, ERR_TABLE_FULL);
  }
}

__device__ __forceinline__ bool is_winner(const ChildArrays& C, uint64_t c, uint64_t tag_base, const Tables& tb) {
  return C.verdict[c] == 1 && tb.ltab[C.cslot[c]].tag == tag_base + c;
}

__global__ void k_winners(ChildArrays C, uint64_t T, uint64_t tag_base, Tables tb, unsigned long long* n_new) {
  unsigned long long cnt = 0;
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T; c += (uint64_t)gridDim.x * blockDim.x)
    cnt += is_winner(C, c, tag_base, tb);
  typedef cub::BlockReduce<unsigned long long, BLK> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long tot = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0 && tot) atomicAdd(n_new, tot);
}

// kept = new (winner of its key in this level) and, when thinning, key0 < τ
// where key0 = fmix64(fp0) (reading A19).
__global__ void k_keep(ChildArrays C, uint64_t T, uint64_t tag_base, Tables tb, uint64_t tau, int thin) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c <= T; c += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = 0;
    if (c < T && is_winner(C, c, tag_base, tb)) k = thin ? (fmix64(C.cfp0[c]) < tau) : 1;
    C.kept[c] = k;
  }
}

__device__ void visited_insert(const Tables& tb, uint64_t k0, uint64_t k1, uint64_t ref, int32_t* err) {
  uint64_t i = fmix64(k0) & tb.vmask;
  for (uint64_t probes = 0; probes <= tb.vmask; ++probes, i = (i + 1) & tb.vmask) {
    Key128 empty{EMPTY, EMPTY}, mine{k0, k1};
    const Key128 prev = atomicCAS(reinterpret_cast<Key128*>(tb.vis + i), empty, mine);
    if (prev.k0 == EMPTY && prev.k1 == EMPTY) {
      tb.vis[i].ref = ref;
      return;
    }
    if (prev.k0 == k0 && prev.k1 == k1) {
      atomicOr(err, ERR_COLLISION);  // a kept key cannot already be visited
      return;
    }
  }
  atomicOr(err, ERR_TABLE_FULL);
}

__global__ void k_compact(ChildArrays C, const uint64_t* off, uint64_t T, NextArrays N, Tables tb,
                          uint64_t level_ref, int32_t* err) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T; c += (uint64_t)gridDim.x * blockDim.x) {
    if (!C.kept[c]) continue;
    const uint64_t q = C.kpos[c];
    const uint32_t p = C.cpar[c];
    N.parent[q] = p;
    N.t[q] = c - off[p];
    N.fp0[q] = C.cfp0[c];
    N.fp1[q] = C.cfp1[c];
    visited_insert(tb, C.cfp0[c], C.cfp1[c], level_ref | q, err);
  }
}

__global__ void k_kq_off(const uint64_t* off, const uint64_t* kpos, int64_t F, uint64_t* kq_off) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= F; p += (int64_t)gridDim.x * blockDim.x)
    kq_off[p] = kpos[off[p]];
}

// ---------------------------------------------------------------------------
// K-c: materialize kept children.  Base value per (neuron j, parent):
//   x = C[j] - c_first(j) + Σ_{s ∈ in(j)} p_first(s)
// written to every kept child of the parent; children whose ND digits differ
// from the base are corrected exactly by k_patch.
// ---------------------------------------------------------------------------
template <typename T, bool BIN>
__global__ void __launch_bounds__(128) k_materialize(SysView S, LevelView L, ExpandOut O, const uint64_t* kq_off,
                                                      NextArrays N, uint64_t* ovf, unsigned long long* n_ovf,
                                                      uint64_t ovf_cap) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t p0 = tile * TILE + 4 * lane;
  if (tile * TILE >= L.F) return;
  uint64_t qa[4];
  uint64_t hi = 0;
  if (p0 < L.F) {
#pragma unroll
    for (int k = 0; k < 4; ++k) qa[k] = kq_off[min(p0 + k, L.F)];
    hi = kq_off[min(p0 + 4, L.F)];
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) qa[k] = 0;
  }
  const uint64_t lo = qa[0];
  if (__ballot_sync(0xFFFFFFFFu, hi > lo) == 0) return;
  const T* data = reinterpret_cast<const T*>(L.data);
  T* out = reinterpret_cast<T*>(N.data);
  for (int32_t j = 0; j < S.m; ++j) {
    int32_t v[4];
    load4<T>(data + (int64_t)j * L.pitch, p0, L.F, v);
    const int r0 = __ldg(S.rule_off + j), r1 = __ldg(S.rule_off + j + 1);
    int32_t x[4] = {0, 0, 0, 0};
    bool found[4] = {false, false, false, false};
    for (int r = r0; r < r1; ++r) {
      const DevRule R = S.rules[r];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (!found[k] && rule_app(R, v[k])) { found[k] = true; x[k] = -R.c; }
    }
    for (int e = __ldg(S.in_off + j), e1 = __ldg(S.in_off + j + 1); e < e1; ++e) {
      const int32_t s = __ldg(S.in_src + e);
      if (BIN) {
        const uint32_t w = O.ebits[(int64_t)(s >> 3) * O.ebits_ld + tile * 32 + lane] >> (4 * (s & 7));
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] += (w >> k) & 1;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] += (p0 + k < L.F) ? O.evals[(int64_t)s * O.evals_ld + p0 + k] : 0;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[k] += v[k];
      if ((x[k] > S.count_max || x[k] < 0) && p0 + k < L.F && (k < 3 ? qa[k + 1] : hi) > qa[k]) {
        unsigned long long slot = atomicAdd(n_ovf, 1ULL);
        if (slot < ovf_cap) ovf[slot] = ((uint64_t)(uint32_t)j << 32) | (uint64_t)(p0 + k);
      }
    }
    for (uint64_t q = lo; q < hi; ++q) {
      const int k = (q >= qa[1]) + (q >= qa[2]) + (q >= qa[3]);
      out[(int64_t)j * N.pitch + q] = (T)x[k];
    }
  }
}

// Exact correction of every (neuron, child) touched by a non-first ND choice:
// the ND neuron itself (consumption) and its out-neighbours (emission).
template <typename T>
__global__ void k_patch(SysView S, LevelView L, ExpandOut O, NextArrays N, int64_t K, int32_t* err) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = N.parent[q];
    const uint64_t t = N.t[q];
    if (t == 0) continue;  // all digits 0: the base child
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], t, cx);
    T* out = reinterpret_cast<T*>(N.data);
    for (int i = 0; i < cx.K; ++i) {
      if (!cx.x[i]) continue;
      const int32_t s = cx.s[i];
      for (int e = -1; e < S.out_off[s + 1] - S.out_off[s]; ++e) {
        const int32_t j = e < 0 ? s : S.out_dst[S.out_off[s] + e];
        const int64_t val = exact_value<T>(S, L.data, L.pitch, p, j, cx);
        if (val < 0 || val > S.count_max) atomicOr(err, ERR_OVERFLOW);
        out[(int64_t)j * N.pitch + q] = (T)val;
      }
    }
  }
}

// Base values outside the storage range: recompute exactly for every kept
// child of that parent (a later ND correction may bring it back in range).
template <typename T>
__global__ void k_overflow_fix(SysView S, LevelView L, ExpandOut O, const uint64_t* kq_off, NextArrays N,
                               const uint64_t* ovf, uint64_t n_ovf, int32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_ovf; i += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t j = (int32_t)(ovf[i] >> 32);
    const int64_t p = (int64_t)(uint32_t)ovf[i];
    T* out = reinterpret_cast<T*>(N.data);
    for (uint64_t q = kq_off[p]; q < kq_off[p + 1]; ++q) {
      ChildCtx cx;
      decode_child(S, O.nd + p * KMAX, O.ndc[p], N.t[q], cx);
      const int64_t val = exact_value<T>(S, L.data, L.pitch, p, j, cx);
      if (val < 0 || val > S.count_max) atomicOr(err, ERR_OVERFLOW);
      else out[(int64_t)j * N.pitch + q] = (T)val;
    }
  }
}

// dedup = 0: every fingerprint match is checked by comparing the two full
// configurations (candidate computed exactly from (parent, t)).  A mismatch
// is a 128-bit collision: reported, never merged (reading A18).
template <typename T>
__global__ void k_verify(SysView S, LevelView L, ExpandOut O, const uint64_t* off, ChildArrays C, uint64_t T_,
                         uint64_t tag_base, Tables tb, const StoredLevel* stored, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = warp; c < T_; c += nwarps) {
    const uint8_t vd = C.verdict[c];
    uint64_t other = EMPTY;
    if (vd == 1) {
      const uint64_t wtag = tb.ltab[C.cslot[c]].tag;
      if (wtag == tag_base + c) continue;  // the winner itself
      other = wtag - tag_base;
    } else if (C.cref[c] == EMPTY) {
      continue;
    }
    const uint32_t p = C.cpar[c];
    ChildCtx cx, co;
    decode_child(S, O.nd + (uint64_t)p * KMAX, O.ndc[p], c - off[p], cx);
    uint32_t po = 0;
    if (vd == 1) {
      po = C.cpar[other];
      decode_child(S, O.nd + (uint64_t)po * KMAX, O.ndc[po], other - off[po], co);
    }
    bool diff = false;
    for (int32_t j = lane; j < S.m; j += 32) {
      const int64_t a = exact_value<T>(S, L.data, L.pitch, p, j, cx);
      int64_t b;
      if (vd == 1) {
        b = exact_value<T>(S, L.data, L.pitch, po, j, co);
      } else {
        const uint64_t ref = C.cref[c];
        const StoredLevel sl = stored[ref >> 40];
        b = ld_count<T>(sl.data, sl.pitch, j, (int64_t)(ref & ((1ULL << 40) - 1)));
      }
      diff |= (a != b);
    }
    if (__any_sync(0xFFFFFFFFu, diff) && lane == 0) atomicOr(err, ERR_COLLISION);
  }
}

// level 0 (reading A20): keep the first occurrence of every configuration
__global__ void k_level0_compact(const uint8_t* verdict, const uint64_t* kept, const uint64_t* kpos, int64_t F0,
                                 const uint64_t* fp0, const uint64_t* fp1, NextArrays N, uint64_t* src_index,
                                 Tables tb, int32_t* err) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < F0; c += (int64_t)gridDim.x * blockDim.x) {
    if (!kept[c]) continue;
    const uint64_t q = kpos[c];
    N.parent[q] = -1;
    N.t[q] = 0;
    N.fp0[q] = fp0[c];
    N.fp1[q] = fp1[c];
    src_index[q] = (uint64_t)c;
    visited_insert(tb, fp0[c], fp1[c], q, err);
  }
}

template <typename T>
__global__ void k_gather_columns(const T* src, int64_t src_pitch, const uint64_t* src_index, int64_t K, int32_t m,
                                 T* dst, int64_t dst_pitch) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= K) return;
  const uint64_t c = src_index[q];
  for (int32_t j = blockIdx.y; j < m; j += gridDim.y) dst[(int64_t)j * dst_pitch + q] = src[(int64_t)j * src_pitch + c];
}

template <typename T>
__global__ void k_verify_level0(const T* data, int64_t pitch, int32_t m, ChildArrays C, uint64_t F0, Tables tb,
                                int32_t* err) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = warp; c < F0; c += nwarps) {
    const uint64_t w = tb.ltab[C.cslot[c]].tag;
    if (w == c) continue;
    bool diff = false;
    for (int32_t j = lane; j < m; j += 32) diff |= data[(int64_t)j * pitch + c] != data[(int64_t)j * pitch + w];
    if (__any_sync(0xFFFFFFFFu, diff) && lane == 0) atomicOr(err, ERR_COLLISION);
  }
}

__global__ void k_rehash(const Slot* old_tab, uint64_t old_cap, Slot* new_tab, uint64_t new_mask, int32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < old_cap; i += (uint64_t)gridDim.x * blockDim.x) {
    const Key128 key = ld_key(old_tab + i);
    if (key.k0 == EMPTY && key.k1 == EMPTY) continue;
    Tables tb{new_tab, new_mask, nullptr, 0};
    uint64_t h = fmix64(key.k0) & new_mask;
    bool ok = false;
    for (uint64_t probes = 0; probes <= new_mask; ++probes, h = (h + 1) & new_mask) {
      Key128 empty{EMPTY, EMPTY};
      const Key128 prev = atomicCAS(reinterpret_cast<Key128*>(tb.vis + h), empty, key);
      if (prev.k0 == EMPTY && prev.k1 == EMPTY) {
        new_tab[h].ref = old_tab[i].ref;
        ok = true;
        break;
      }
    }
    if (!ok) atomicOr(err, ERR_TABLE_FULL);
  }
}

// order-sensitive run digest
__global__ void k_digest(NextArrays N, int64_t K, uint64_t level, unsigned long long* digest) {
  unsigned long long acc = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = fmix64((level << 40) ^ (uint64_t)q);
    z = fmix64(z ^ N.fp0[q]);
    z = fmix64(z ^ N.fp1[q]);
    z = fmix64(z ^ (uint64_t)(N.parent[q] + 1));
    z = fmix64(z ^ N.t[q]);
    acc += z;
  }
  typedef cub::BlockReduce<unsigned long long, BLK> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) atomicAdd(digest, tot);
}

// The spiking vector that produced each child (Alg. 2 II-2/II-3 decode).
template <typename T>
__global__ void k_spiking_vectors(SysView S, const T* pdata, int64_t ppitch, const int64_t* parent, const uint64_t* tt,
                                  int64_t K, uint8_t* S_out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = parent[q];
    uint64_t t = tt[q];
    uint8_t* Sq = S_out + q * S.n;
    for (int64_t r = 0; r < S.n; ++r) Sq[r] = 0;
    for (int32_t s = S.m - 1; s >= 0; --s) {  // least significant digit = last neuron
      const int32_t v = (int32_t)pdata[(int64_t)s * ppitch + p];
      const int d = count_applicable(S, s, v);
      if (d == 0) continue;
      const int x = (int)(t % (uint64_t)d);
      t /= (uint64_t)d;
      Sq[nth_applicable(S, s, v, x)] = 1;
    }
  }
}

template <typename F>
void dispatch_bytes(int32_t bytes, F&& f) {
  if (bytes == 1) f(uint8_t{});
  else if (bytes == 2) f(uint16_t{});
  else f(int32_t{});
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================
void launch_import(const void* src, int32_t src_bytes, int32_t src_layout, int64_t src_ld, int64_t F, int32_t m,
                   void* dst, int32_t dst_bytes, int64_t dst_pitch, int64_t count_max, int32_t* err, cudaStream_t st) {
  dim3 grid((unsigned)((F + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  dispatch_bytes(src_bytes, [&](auto tin) {
    using Tin = decltype(tin);
    dispatch_bytes(dst_bytes, [&](auto tout) {
      using Tout = decltype(tout);
      k_import<Tin, Tout><<<grid, block, 0, st>>>(src, src_layout, src_ld, F, m, reinterpret_cast<Tout*>(dst),
                                                  dst_pitch, count_max, err);
      count_launch();
    });
  });
}

void launch_export(const void* src, int32_t bytes, int64_t pitch, int64_t F, int32_t m, int32_t* dst, cudaStream_t st) {
  dim3 grid((unsigned)((F + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_export<T><<<grid, block, 0, st>>>(reinterpret_cast<const T*>(src), pitch, F, m, dst);
    count_launch();
  });
}

static unsigned tiles_grid(int64_t F) { return (unsigned)((F + 4 * TILE - 1) / (4 * TILE)); }

void launch_fingerprint(const SysView& S, int32_t bytes, const void* data, int64_t pitch, int64_t F, uint64_t* fp0,
                        uint64_t* fp1, cudaStream_t st) {
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_fingerprint<T><<<tiles_grid(F), 128, 0, st>>>(S, reinterpret_cast<const T*>(data), pitch, F, fp0, fp1);
    count_launch();
  });
}

void launch_expand(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, cudaStream_t st) {
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    if (S.binary_emit) k_expand<T, true><<<tiles_grid(L.F), 128, 0, st>>>(S, L, O);
    else k_expand<T, false><<<tiles_grid(L.F), 128, 0, st>>>(S, L, O);
    count_launch();
  });
}

void launch_child_parent(const uint64_t* off, int64_t F, uint32_t* cpar, cudaStream_t st) {
  k_child_parent<<<grid_for(F), BLK, 0, st>>>(off, F, cpar);
  count_launch();
}

void launch_child_keys(const SysView& S, const uint64_t* off, const ExpandOut& O, uint64_t T, const ChildArrays& C,
                       cudaStream_t st) {
  k_child_keys<<<grid_for(T), BLK, 0, st>>>(S, off, O, T, C);
  count_launch();
}

void launch_dedup(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, int use_visited, int32_t* err,
                  cudaStream_t st) {
  k_dedup<<<grid_for(T), BLK, 0, st>>>(C, T, tag_base, tb, use_visited, err);
  count_launch();
}

void launch_winners(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, uint64_t, int,
                    unsigned long long* n_new, cudaStream_t st) {
  unsigned g = grid_for(T);
  if (g > 148u * 16u) g = 148u * 16u;
  k_winners<<<g, BLK, 0, st>>>(C, T, tag_base, tb, n_new);
  count_launch();
}

void launch_keep(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, uint64_t tau, int thin,
                 cudaStream_t st) {
  k_keep<<<grid_for(T + 1), BLK, 0, st>>>(C, T, tag_base, tb, tau, thin);
  count_launch();
}

void launch_compact(const ChildArrays& C, const uint64_t* off, uint64_t T, const NextArrays& N, const Tables& tb,
                    uint64_t level_ref, int32_t* err, cudaStream_t st) {
  k_compact<<<grid_for(T), BLK, 0, st>>>(C, off, T, N, tb, level_ref, err);
  count_launch();
}

void launch_kq_off(const uint64_t* off, const uint64_t* kpos, int64_t F, uint64_t* kq_off, cudaStream_t st) {
  k_kq_off<<<grid_for(F + 1), BLK, 0, st>>>(off, kpos, F, kq_off);
  count_launch();
}

void launch_materialize(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O,
                        const uint64_t* kq_off, const NextArrays& N, uint64_t* ovf, unsigned long long* n_ovf,
                        uint64_t ovf_cap, cudaStream_t st) {
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    if (S.binary_emit)
      k_materialize<T, true><<<tiles_grid(L.F), 128, 0, st>>>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap);
    else
      k_materialize<T, false><<<tiles_grid(L.F), 128, 0, st>>>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap);
    count_launch();
  });
}

void launch_patch(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const NextArrays& N,
                  int64_t K, int32_t* err, cudaStream_t st) {
  if (K <= 0) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_patch<T><<<grid_for(K, 128), 128, 0, st>>>(S, L, O, N, K, err);
    count_launch();
  });
}

void launch_overflow_fix(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O,
                         const uint64_t* kq_off, const NextArrays& N, const uint64_t* ovf, uint64_t n_ovf,
                         int32_t* err, cudaStream_t st) {
  if (!n_ovf) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_overflow_fix<T><<<grid_for(n_ovf, 128), 128, 0, st>>>(S, L, O, kq_off, N, ovf, n_ovf, err);
    count_launch();
  });
}

void launch_verify(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const uint64_t* off,
                   const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, const StoredLevel* stored,
                   int32_t* err, cudaStream_t st) {
  if (!T) return;
  unsigned g = grid_for(T * 32, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  dispatch_bytes(bytes, [&](auto tt) {
    using TT = decltype(tt);
    k_verify<TT><<<g, 256, 0, st>>>(S, L, O, off, C, T, tag_base, tb, stored, err);
    count_launch();
  });
}

void launch_level0_compact(const uint8_t* verdict, const uint64_t* kept, const uint64_t* kpos, int64_t F0,
                           const uint64_t* fp0, const uint64_t* fp1, const NextArrays& N, uint64_t* src_index,
                           const Tables& tb, int32_t* err, cudaStream_t st) {
  k_level0_compact<<<grid_for(F0), BLK, 0, st>>>(verdict, kept, kpos, F0, fp0, fp1, N, src_index, tb, err);
  count_launch();
}

void launch_gather_columns(int32_t bytes, const void* src, int64_t src_pitch, const uint64_t* src_index, int64_t K,
                           int32_t m, void* dst, int64_t dst_pitch, cudaStream_t st) {
  if (K <= 0) return;
  dim3 grid(grid_for(K), (unsigned)min(m, 1024));
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_gather_columns<T><<<grid, BLK, 0, st>>>(reinterpret_cast<const T*>(src), src_pitch, src_index, K, m,
                                              reinterpret_cast<T*>(dst), dst_pitch);
    count_launch();
  });
}

void launch_verify_level0(int32_t bytes, const void* data, int64_t pitch, int32_t m, const ChildArrays& C,
                          uint64_t F0, const Tables& tb, int32_t* err, cudaStream_t st) {
  unsigned g = grid_for(F0 * 32, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_verify_level0<T><<<g, 256, 0, st>>>(reinterpret_cast<const T*>(data), pitch, m, C, F0, tb, err);
    count_launch();
  });
}

void launch_rehash(const Slot* old_tab, uint64_t old_cap, Slot* new_tab, uint64_t new_mask, int32_t* err,
                   cudaStream_t st) {
  k_rehash<<<grid_for(old_cap), BLK, 0, st>>>(old_tab, old_cap, new_tab, new_mask, err);
  count_launch();
}

void launch_digest(const NextArrays& N, int64_t K, uint64_t level, unsigned long long* digest, cudaStream_t st) {
  if (K <= 0) return;
  unsigned g = grid_for(K);
  if (g > 148u * 8u) g = 148u * 8u;
  k_digest<<<g, BLK, 0, st>>>(N, K, level, digest);
  count_launch();
}

void launch_spiking_vectors(const SysView& S, int32_t bytes, const void* parent_data, int64_t parent_pitch,
                            const int64_t* parent, const uint64_t* t, int64_t K, uint8_t* S_out, cudaStream_t st) {
  if (K <= 0) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_spiking_vectors<T><<<grid_for(K, 128), 128, 0, st>>>(S, reinterpret_cast<const T*>(parent_data), parent_pitch,
                                                         parent, t, K, S_out);
    count_launch();
  });
}

size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)n);
  return bytes;
}

void launch_exclusive_scan(void* temp, size_t temp_bytes, const uint64_t* in, uint64_t* out, int64_t n,
                           cudaStream_t st) {
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int64_t)n, st);
  count_launch(2);  // init + scan kernels
}

}  // namespace snp
