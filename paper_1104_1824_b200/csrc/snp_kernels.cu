// snp_kernels.cu — sm_100a kernels of the batched SNP transition step.
//
//   K-a  k_expand_t / k_expand_g   rule applicability per (neuron, configuration)
//                        (Alg. 2 II-1), Ψ (eq. (8),
//                        PAPER.md:250, readings A3/A5), the base-child
//                        fingerprint and the first-choice emit bits.
//   K-b  CUB scan + k_child_parent + k_child_keys: child offsets, mixed-radix
//                        decode of t (Alg. 2 II-2/II-3, PAPER.md:263-264,
//                        reading A7) and the child fingerprint by linearity.
//   K-d  k_dedup / k_winners / k_keep / k_compact: GPU open-addressing sets
//                        (visited + level table with minimum-tag resolution,
//                        readings A6, A19, A22).
//   K-c  k_materialize_bs (+ k_patch, k_overflow_fix) or k_materialize_exact:
//                        C' = C + S·M (eq. (2)) for the kept
//                        children only, as a gather-add over the in-synapses
//                        (Def. 2).
//
// Every kernel is plain CUDA C++ / PTX for sm_100a; the path is integer and
// bound by HBM / issue bandwidth, not by tensor cores.
#include <atomic>

#include <cub/cub.cuh>
#include <type_traits>

#include "snp_internal.h"
#include "snp_tc.cuh"

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
__device__ __forceinline__ int32_t ld_count(const void* data, int64_t p, int32_t j, int32_t m) {
  return (int32_t) reinterpret_cast<const T*>(data)[eidx(p, j, m)];
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
__device__ __forceinline__ int first_rule(const SysView& S, int32_t s, int32_t v);

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

// Generated numbers (include/snp.h): the augmented
// column A (neuron m - 1) of the child.  The output spike is the output
// rule firing in the child's spiking vector; A >= 1 and a spike = second
// output spike: *number = A and the child is terminal; else
// A' = (A == 0 ? [spike] : A + 1) and *number = -1.
template <typename T>
__device__ int64_t aug_child(const SysView& S, const void* data, int64_t p, const ChildCtx& cx, int64_t* number) {
  const int64_t a = ld_count<T>(data, p, S.m - 1, S.m);
  const int32_t v = ld_count<T>(data, p, S.aug_neuron, S.m);
  const bool spike = fired_rule(S, S.aug_neuron, v, cx) == S.aug_rule;
  *number = (a >= 1 && spike) ? a : -1;
  return a == 0 ? (spike ? 1 : 0) : a + 1;
}

// Exact value of the child at neuron j: eq. (2) restricted to column j,
// C'[j] = C[j] - c_{fired(j)} + Σ_{s ∈ in(j)} p_{fired(s)}  (Def. 2).
template <typename T>
__device__ int64_t exact_value(const SysView& S, const void* data, int64_t p, int32_t j, const ChildCtx& cx) {
  if (S.aug_rule >= 0 && j == S.m - 1) {
    int64_t number;
    return aug_child<T>(S, data, p, cx, &number);
  }
  int32_t vj = ld_count<T>(data, p, j, S.m);
  int rj = fired_rule(S, j, vj, cx);
  int64_t val = (int64_t)vj - (rj >= 0 ? S.rules[rj].c : 0);
  for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) {
    int32_t s = S.in_src[e];
    int rs = fired_rule(S, s, ld_count<T>(data, p, s, S.m), cx);
    if (rs >= 0) val += S.rules[rs].p;
  }
  return val;
}

// ---------------------------------------------------------------------------
// import / export between the ABI's layouts and the blocked device frontier
// ---------------------------------------------------------------------------
template <typename Tin>
__device__ __forceinline__ int64_t ld_in(const void* src, int64_t idx) {
  return (int64_t) reinterpret_cast<const Tin*>(src)[idx];
}

template <typename Tin, typename Tout>
__global__ void k_import(const void* src, int32_t layout, int64_t ld, int64_t F, int32_t m, Tout* dst,
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
        dst[eidx(p, j, m)] = (Tout)v;
      }
    }
  } else {  // neuron-major: element (p, j) at src[j * ld + p]
    for (int r = ty; r < 32; r += 8) {
      int32_t j = j_base + r;
      int64_t p = p_base + tx;
      if (p < F && j < m) {
        int64_t v = ld_in<Tin>(src, (int64_t)j * ld + p);
        bad |= (v < 0 || v > count_max);
        dst[eidx(p, j, m)] = (Tout)v;
      }
    }
  }
  if (bad) atomicOr(err, ERR_OVERFLOW);
}

template <typename T>
__global__ void k_export(const T* src, int64_t F, int32_t m, int32_t* dst) {
  __shared__ int32_t tile[32][33];
  const int64_t p_base = (int64_t)blockIdx.x * 32;
  const int32_t j_base = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    int32_t j = j_base + r;
    int64_t p = p_base + tx;
    tile[r][tx] = (p < F && j < m) ? (int32_t)src[eidx(p, j, m)] : 0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    int64_t p = p_base + r;
    int32_t j = j_base + tx;
    if (p < F && j < m) dst[p * m + j] = tile[tx][r];
  }
}

// fp_ℓ(C) = Σ_j C[j]·R_ℓ[j] mod 2^64 (reading A18), one configuration per thread.
template <typename T>
__global__ void k_fingerprint(SysView S, const T* data, int64_t F, uint64_t* fp0, uint64_t* fp1) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= F) return;
  uint64_t a = 0, b = 0;
  for (int32_t j = 0; j < S.m; ++j) {
    const uint64_t v = (uint64_t)data[eidx(p, j, S.m)];
    a += v * __ldg(S.R0 + j);
    b += v * __ldg(S.R1 + j);
  }
  fp0[p] = a;
  fp1[p] = b;
}

// ---------------------------------------------------------------------------
// K-a: applicability, Ψ, base fingerprint, emits
// ---------------------------------------------------------------------------
constexpr int XW = 8;       // warps per CTA
constexpr int XPPL = 8;     // configurations per lane
constexpr int XTILE = 256;  // configurations per warp (4 storage blocks)

__device__ __forceinline__ void nd_event(const SysView& S, const ExpandOut& O, int32_t s, uint32_t v, int64_t p,
                                         int& ndc, uint64_t& psi) {
  const int d = count_applicable(S, s, (int32_t)v);
  if (!O.classify_only && ndc < KMAX) O.nd[p * KMAX + ndc] = ((uint64_t)(uint32_t)s << 32) | v;
  ++ndc;
  psi = sat_mul(psi, (uint64_t)d);
}

__device__ __forceinline__ int64_t emit_index(int64_t p, int32_t s, int32_t m) {
  const int64_t mE = (m + 1) & ~1;  // rows per block rounded to even: 16-B aligned block slices
  return ((p >> 6) * mE + s) * 8 + ((p & 63) >> 3);
}

// Evaluate the rules of one neuron for a lane's 8 configurations (no table).
__device__ void expand_generic_neuron(const SysView& S, const ExpandOut& O, int32_t s, const uint32_t v[8],
                                      int64_t p0, int64_t F, uint64_t a[8], uint64_t b[8], uint64_t psi[8],
                                      int ndc[8], uint32_t& anyb, uint32_t& eb) {
  const int r0 = S.rule_off[s], r1 = S.rule_off[s + 1];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int first = -1, d = 0;
    for (int r = r0; r < r1; ++r)
      if (rule_app(S.rules[r], (int32_t)v[k])) {
        if (!d) first = r;
        ++d;
      }
    if (d) {
      a[k] += __ldg(S.h0 + first);
      b[k] += __ldg(S.h1 + first);
      anyb |= 1u << k;
      eb |= (S.rules[first].p > 0 ? 1u : 0u) << k;
      if (d >= 2 && p0 + k < F) {
        if (!O.classify_only && ndc[k] < KMAX) O.nd[(p0 + k) * KMAX + ndc[k]] = ((uint64_t)(uint32_t)s << 32) | v[k];
        ++ndc[k];
        psi[k] = sat_mul(psi[k], (uint64_t)d);
      }
    }
  }
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// bit-sliced full adder: (h, l) = a + b + c per bit position
__device__ __forceinline__ void csa(uint64_t& h, uint64_t& l, uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// 32-byte global load / store (sm_100 LDG.256 / STG.256): one full sector per lane
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, const uint32_t (&r)[8]) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
               "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// t[v] for the four byte counts v < 32 of v4, t = 32 bytes in tt[0..7]:
// bits 0-2 of each count select a byte inside a register pair (one PRMT per
// pair), bits 3 and 4 choose between the pairs (sign-replicate PRMT masks)
__device__ __forceinline__ uint32_t lut32(uint32_t v4, const uint32_t (&tt)[8]) {
  const uint32_t x = v4 & 0x07070707u;
  const uint32_t sel = prmt(x | (x >> 4), 0u, 0x4420u);
  const uint32_t m3 = prmt(v4 << 4, 0u, 0xBA98u);  // 0xFF in bytes whose bit 3 is set
  const uint32_t m4 = prmt(v4 << 3, 0u, 0xBA98u);  // ... bit 4
  const uint32_t a = prmt(tt[0], tt[1], sel), b = prmt(tt[2], tt[3], sel);
  const uint32_t c = prmt(tt[4], tt[5], sel), d = prmt(tt[6], tt[7], sel);
  const uint32_t lo = (a & ~m3) | (b & m3), hi = (c & ~m3) | (d & m3);
  return (lo & ~m4) | (hi & m4);
}

// 4 table entries (one byte each) → 4-bit mask of their TE_EMIT bits
__device__ __forceinline__ uint32_t emit_nibble(uint32_t w4) {
  return ((w4 & 0x01010101u) * 0x01020408u) >> 24;
}

// Table-driven K-a.  A CTA owns 32 storage blocks (2048 configurations; warp w
// owns blocks 4w..4w+3, 8 configurations per lane) and walks the neurons in
// chunks of NC = 16/w.  For every chunk, one thread issues TMA bulk copies of
// the 32 contiguous block slices (NC rows × 64 counts) into a double-buffered
// shared-memory stage one chunk ahead (mbarrier complete_tx), while all
// threads stage the chunk's outcome tables and rule fingerprint deltas.  Per
// (neuron, configuration): one table byte, one 16-B fingerprint delta (slot 0
// of a neuron is zero = "no rule fires"); neurons are consumed in pairs so the
// two deltas enter the 64-bit accumulators through 3-input adds.  Ψ and the
// ND lists are rare and live in global memory.
template <typename T>
struct ExpandGeom {
  static constexpr int NC = 16 / (int)sizeof(T);      // neurons per chunk
  static constexpr int ROWB = PB * (int)sizeof(T);    // bytes of one block row
  static constexpr int BLKB = NC * ROWB;              // bytes of one block slice (1 KB)
  static constexpr int BLKS = BLKB + 64;              // padded slice stride (bank spread)
  static constexpr int CNT_STAGE = 32 * BLKS;         // count bytes per stage
};

template <typename T>
size_t expand_smem_bytes(int W) {
  using G = ExpandGeom<T>;
  return 2 * (size_t)G::CNT_STAGE + 2 * (size_t)G::NC * W + 2 * (size_t)G::NC * 256 + 2 * G::NC * sizeof(NeuronMeta) +
         64;
}

template <typename T>
__device__ __forceinline__ void smem_counts8(const uint8_t* p, uint32_t v[8]) {
  if constexpr (sizeof(T) == 1) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[k] = (w.x >> (8 * k)) & 0xFFu; v[k + 4] = (w.y >> (8 * k)) & 0xFFu; }
  } else if constexpr (sizeof(T) == 2) {
    const uint4 w = *reinterpret_cast<const uint4*>(p);
    const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (x[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
  } else {
    const uint4 a = *reinterpret_cast<const uint4*>(p);
    const uint4 b = *reinterpret_cast<const uint4*>(p + 16);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

template <typename T, bool FULL>
__global__ void __launch_bounds__(256, 2) k_expand_t(SysView S, LevelView L, ExpandOut O) {
  using G = ExpandGeom<T>;
  constexpr int NC = G::NC;
  extern __shared__ __align__(128) uint8_t smem[];
  const int W = FULL ? 256 : S.tabw;
  uint8_t* s_cnt = smem;                                                    // [2][32][BLKS]
  uint8_t* s_tab = s_cnt + 2 * G::CNT_STAGE;                                // [2][NC][W]
  uint8_t* s_hs = s_tab + 2 * NC * W;                                       // [2][NC][256]
  NeuronMeta* s_meta = reinterpret_cast<NeuronMeta*>(s_hs + 2 * NC * 256);  // [2][NC]
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_meta + 2 * NC);             // [2]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t blk0 = (int64_t)blockIdx.x * 32;
  const int64_t nblk_total = (L.F + PB - 1) / PB;
  const int nb = (nblk_total - blk0 < 32) ? (int)(nblk_total - blk0) : 32;
  const int bl = warp * 4 + (lane >> 3);  // this lane's block within the CTA
  const int64_t p0 = (blk0 + bl) * PB + (lane & 7) * 8;
  const int nvalid = p0 >= L.F ? 0 : (L.F - p0 >= 8 ? 8 : (int)(L.F - p0));
  const uint8_t* gtab = FULL ? S.tab_full : S.tab;
  const int m = S.m;
  const int nchunks = (m + NC - 1) / NC;

  uint64_t a[8], b[8];
  uint32_t any0 = 0, any1 = 0, anyb_generic = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const bool ok = k < nvalid;
    a[k] = ok ? L.fp0[p0 + k] : 0;
    b[k] = ok ? L.fp1[p0 + k] : 0;
    if (ok && !O.classify_only) {
      O.psi[p0 + k] = 1;
      O.ndc[p0 + k] = 0;
    }
  }
  uint8_t* ep = nullptr;  // this lane's emit byte of neuron 0; +8 per neuron
  if (O.ebits != nullptr && !O.classify_only && nvalid > 0)
    ep = reinterpret_cast<uint8_t*>(O.ebits) + emit_index(p0, 0, m);

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();

  auto issue = [&](int c) {  // TMA: chunk c's count slices of the CTA's blocks
    if (tid == 0) {
      const int st = c & 1, c0 = c * NC, rows = min(NC, m - c0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(&bar[st], (uint32_t)(nb * rows * G::ROWB));
      const uint8_t* base = reinterpret_cast<const uint8_t*>(L.data);
      for (int bb = 0; bb < nb; ++bb)
        bulk_g2s(s_cnt + st * G::CNT_STAGE + bb * G::BLKS,
                 base + (((blk0 + bb) * (int64_t)m + c0) * PB) * (int64_t)sizeof(T), (uint32_t)(rows * G::ROWB),
                 &bar[st]);
    }
  };
  auto stage_tables = [&](int c) {
    const int st = c & 1, c0 = c * NC, rows = min(NC, m - c0);
    const uint4* src = reinterpret_cast<const uint4*>(gtab + (int64_t)c0 * W);
    uint4* dst = reinterpret_cast<uint4*>(s_tab + st * NC * W);
    for (int i = tid; i < rows * W / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    ulonglong2* hs = reinterpret_cast<ulonglong2*>(s_hs + st * NC * 256);
    for (int i = tid; i < rows * 16; i += blockDim.x) {
      const int sl = i >> 4, f = i & 15;
      const int r0 = __ldg(S.rule_off + c0 + sl), r1 = __ldg(S.rule_off + c0 + sl + 1);
      ulonglong2 h = make_ulonglong2(0ULL, 0ULL);
      if (f >= 1 && f <= r1 - r0 && f <= MAX_TABLE_RULES)
        h = make_ulonglong2(__ldg(S.h0 + r0 + f - 1), __ldg(S.h1 + r0 + f - 1));
      hs[i] = h;
    }
    if (tid < rows) s_meta[st * NC + tid] = S.meta[c0 + tid];
  };

  issue(0);
  stage_tables(0);
  __syncthreads();
  for (int c = 0; c < nchunks; ++c) {
    const int st = c & 1, c0 = c * NC, rows = min(NC, m - c0);
    if (c + 1 < nchunks) {
      issue(c + 1);
      stage_tables(c + 1);
    }
    mbar_wait(&bar[st], (uint32_t)((c >> 1) & 1));
    if (nvalid > 0) {
      const uint8_t* crow = s_cnt + st * G::CNT_STAGE + bl * G::BLKS + (lane & 7) * 8 * (int)sizeof(T);
      const uint8_t* tab = s_tab + st * NC * W;
      const uint8_t* hsb = s_hs + st * NC * 256;
      const NeuronMeta* mts = s_meta + st * NC;
      for (int sl = 0; sl < rows; sl += 2) {
        const bool pair = sl + 1 < rows;
        const NeuronMeta mA = mts[sl];
        const NeuronMeta mB = pair ? mts[sl + 1] : mA;
        if (((mA.flags | mB.flags) & NM_GENERIC) || !pair) {
          // slow path: one neuron at a time (generic neurons, odd tail)
          for (int u = 0; u < (pair ? 2 : 1); ++u) {
            const int su = sl + u;
            const int32_t s = c0 + su;
            const NeuronMeta mt = mts[su];
            uint32_t v[8];
            smem_counts8<T>(crow + su * G::ROWB, v);
            uint32_t eb = 0;
            if (mt.flags & NM_GENERIC) {
              uint64_t psi[8];
              int ndc[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                psi[k] = 1;
                ndc[k] = (!O.classify_only && k < nvalid) ? O.ndc[p0 + k] : 0;
              }
              expand_generic_neuron(S, O, s, v, p0, L.F, a, b, psi, ndc, anyb_generic, eb);
              if (!O.classify_only) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  if (k < nvalid && psi[k] != 1) {
                    O.psi[p0 + k] = sat_mul(O.psi[p0 + k], psi[k]);
                    O.ndc[p0 + k] = ndc[k];
                  }
              }
            } else {
              uint32_t o[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                o[k] = tab[su * W + (FULL ? v[k] : table_index(v[k], mt))];
                const ulonglong2 h = *reinterpret_cast<const ulonglong2*>(hsb + su * 256 + (o[k] & TE_F));
                a[k] += h.x;
                b[k] += h.y;
              }
              const uint32_t w0 = o[0] | (o[1] << 8) | (o[2] << 16) | (o[3] << 24);
              const uint32_t w1 = o[4] | (o[5] << 8) | (o[6] << 16) | (o[7] << 24);
              any0 |= w0;
              any1 |= w1;
              eb = emit_nibble(w0) | (emit_nibble(w1) << 4);
              if (((w0 | w1) & 0x02020202u) && !O.classify_only) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  if ((o[k] & TE_ND) && k < nvalid) {
                    int nk = O.ndc[p0 + k];
                    uint64_t pk = O.psi[p0 + k];
                    nd_event(S, O, s, v[k], p0 + k, nk, pk);
                    O.ndc[p0 + k] = nk;
                    O.psi[p0 + k] = pk;
                  }
              }
            }
            if (ep) ep[(int64_t)s * 8] = (uint8_t)eb;
          }
          continue;
        }
        if constexpr (sizeof(T) == 1 && FULL) {
          // u8 fast path: counts stay packed 4 per word; the first 32 bytes of
          // each neuron's outcome table sit in registers and are looked up 4
          // counts at a time by byte permutes (a count >= 32 reads the table)
          uint32_t ltA[8], ltB[8];
          {
            const uint4* ta = reinterpret_cast<const uint4*>(tab + sl * W);
            const uint4* tb = reinterpret_cast<const uint4*>(tab + (sl + 1) * W);
            const uint4 a0 = ta[0], a1 = ta[1], b0 = tb[0], b1 = tb[1];
            ltA[0] = a0.x; ltA[1] = a0.y; ltA[2] = a0.z; ltA[3] = a0.w;
            ltA[4] = a1.x; ltA[5] = a1.y; ltA[6] = a1.z; ltA[7] = a1.w;
            ltB[0] = b0.x; ltB[1] = b0.y; ltB[2] = b0.z; ltB[3] = b0.w;
            ltB[4] = b1.x; ltB[5] = b1.y; ltB[6] = b1.z; ltB[7] = b1.w;
          }
          const uint2 cA = *reinterpret_cast<const uint2*>(crow + sl * G::ROWB);
          const uint2 cB = *reinterpret_cast<const uint2*>(crow + (sl + 1) * G::ROWB);
          auto look = [&](uint32_t v4, const uint32_t(&lt)[8], const uint8_t* trow) {
            if ((v4 & 0xE0E0E0E0u) == 0) return lut32(v4, lt);
            uint32_t w = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) w |= (uint32_t)trow[(v4 >> (8 * i)) & 0xFFu] << (8 * i);
            return w;
          };
          const uint32_t wA0 = look(cA.x, ltA, tab + sl * W), wA1 = look(cA.y, ltA, tab + sl * W);
          const uint32_t wB0 = look(cB.x, ltB, tab + (sl + 1) * W), wB1 = look(cB.y, ltB, tab + (sl + 1) * W);
          const uint8_t* hA = hsb + sl * 256;
          const uint8_t* hB = hsb + (sl + 1) * 256;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t wa = k < 4 ? wA0 : wA1, wb = k < 4 ? wB0 : wB1;
            const ulonglong2 dA = *reinterpret_cast<const ulonglong2*>(hA + ((wa >> (8 * (k & 3))) & TE_F));
            const ulonglong2 dB = *reinterpret_cast<const ulonglong2*>(hB + ((wb >> (8 * (k & 3))) & TE_F));
            a[k] += dA.x + dB.x;
            b[k] += dA.y + dB.y;
          }
          any0 |= wA0 | wB0;
          any1 |= wA1 | wB1;
          if (ep) {
            ep[(int64_t)(c0 + sl) * 8] = (uint8_t)(emit_nibble(wA0) | (emit_nibble(wA1) << 4));
            ep[(int64_t)(c0 + sl + 1) * 8] = (uint8_t)(emit_nibble(wB0) | (emit_nibble(wB1) << 4));
          }
          if (((wA0 | wA1 | wB0 | wB1) & 0x02020202u) && !O.classify_only) {  // rare: nondeterminism
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              if (k >= nvalid) continue;
              const int sh = 8 * (k & 3);
              const uint32_t wa = k < 4 ? wA0 : wA1, wb = k < 4 ? wB0 : wB1;
              const uint32_t va = ((k < 4 ? cA.x : cA.y) >> sh) & 0xFFu, vb = ((k < 4 ? cB.x : cB.y) >> sh) & 0xFFu;
              if ((wa >> sh) & TE_ND) {
                int nk = O.ndc[p0 + k];
                uint64_t pk = O.psi[p0 + k];
                nd_event(S, O, c0 + sl, va, p0 + k, nk, pk);
                O.ndc[p0 + k] = nk;
                O.psi[p0 + k] = pk;
              }
              if ((wb >> sh) & TE_ND) {
                int nk = O.ndc[p0 + k];
                uint64_t pk = O.psi[p0 + k];
                nd_event(S, O, c0 + sl + 1, vb, p0 + k, nk, pk);
                O.ndc[p0 + k] = nk;
                O.psi[p0 + k] = pk;
              }
            }
          }
          continue;
        }
        // fast path: a pair of tabulated neurons
        uint32_t vA[8], vB[8];
        smem_counts8<T>(crow + sl * G::ROWB, vA);
        smem_counts8<T>(crow + (sl + 1) * G::ROWB, vB);
        uint32_t oA[8], oB[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          oA[k] = tab[sl * W + (FULL ? vA[k] : table_index(vA[k], mA))];
          oB[k] = tab[(sl + 1) * W + (FULL ? vB[k] : table_index(vB[k], mB))];
          const ulonglong2 hA = *reinterpret_cast<const ulonglong2*>(hsb + sl * 256 + (oA[k] & TE_F));
          const ulonglong2 hB = *reinterpret_cast<const ulonglong2*>(hsb + (sl + 1) * 256 + (oB[k] & TE_F));
          a[k] += hA.x + hB.x;
          b[k] += hA.y + hB.y;
        }
        const uint32_t wA0 = oA[0] | (oA[1] << 8) | (oA[2] << 16) | (oA[3] << 24);
        const uint32_t wA1 = oA[4] | (oA[5] << 8) | (oA[6] << 16) | (oA[7] << 24);
        const uint32_t wB0 = oB[0] | (oB[1] << 8) | (oB[2] << 16) | (oB[3] << 24);
        const uint32_t wB1 = oB[4] | (oB[5] << 8) | (oB[6] << 16) | (oB[7] << 24);
        any0 |= wA0 | wB0;
        any1 |= wA1 | wB1;
        if (ep) {
          ep[(int64_t)(c0 + sl) * 8] = (uint8_t)(emit_nibble(wA0) | (emit_nibble(wA1) << 4));
          ep[(int64_t)(c0 + sl + 1) * 8] = (uint8_t)(emit_nibble(wB0) | (emit_nibble(wB1) << 4));
        }
        if (((wA0 | wA1 | wB0 | wB1) & 0x02020202u) && !O.classify_only) {  // rare: nondeterminism
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (k >= nvalid) continue;
            if (oA[k] & TE_ND) {
              int nk = O.ndc[p0 + k];
              uint64_t pk = O.psi[p0 + k];
              nd_event(S, O, c0 + sl, vA[k], p0 + k, nk, pk);
              O.ndc[p0 + k] = nk;
              O.psi[p0 + k] = pk;
            }
            if (oB[k] & TE_ND) {
              int nk = O.ndc[p0 + k];
              uint64_t pk = O.psi[p0 + k];
              nd_event(S, O, c0 + sl + 1, vB[k], p0 + k, nk, pk);
              O.ndc[p0 + k] = nk;
              O.psi[p0 + k] = pk;
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (nvalid == 0) return;
  unsigned nh = 0;
  bool cap = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (k >= nvalid) continue;
    const int64_t p = p0 + k;
    const uint32_t fb = ((k < 4 ? any0 : any1) >> (8 * (k & 3))) & TE_F;
    const bool any = fb != 0 || ((anyb_generic >> k) & 1u);
    O.halting[p] = any ? 0 : 1;
    nh += any ? 0 : 1;
    if (!O.classify_only) {
      if (!any) O.psi[p] = 0;  // halting: no children (reading A5)
      cap |= O.psi[p] > PSI_LIMIT || O.ndc[p] > KMAX;
      O.fpb0[p] = a[k];
      O.fpb1[p] = b[k];
    }
  }
  if (cap) atomicOr(O.err, ERR_CAPACITY);
  if (nh) atomicAdd(O.n_halting, (unsigned long long)nh);
}

// K-a for uint8 counts with every neuron tabulated (the common case): 4
// configurations per lane so that 64 registers suffice and 32 warps share an
// SM.  A CTA owns QB = 16 storage blocks (warp w: blocks 2w, 2w+1; lane l:
// configurations 4(l % 16) .. +3 of its block).  Per chunk of QNC neurons one
// thread issues TMA bulk copies of the 16 count slices, the chunk's
// fingerprint-delta rows (hsg) and outcome-table heads (elut) into a
// double-buffered stage.  Per (neuron, lane): one 32-bit count word, one
// byte-permute table lookup for its 4 counts, one 16-B delta per firing
// configuration; the emit nibbles of lane pairs merge into the E byte by one
// shuffle.
// outcome-table entries of the 4 byte counts of w: byte permutes on the 32-B
// table head staged in shared memory, the full table for a count >= 32
__device__ __forceinline__ uint32_t expand_entries(uint32_t w, const uint8_t* head, const uint8_t* full) {
  if ((w & 0xE0E0E0E0u) == 0) {
    uint32_t t[8];
    const uint4 t0 = reinterpret_cast<const uint4*>(head)[0];
    const uint4 t1 = reinterpret_cast<const uint4*>(head)[1];
    t[0] = t0.x; t[1] = t0.y; t[2] = t0.z; t[3] = t0.w;
    t[4] = t1.x; t[5] = t1.y; t[6] = t1.z; t[7] = t1.w;
    return lut32(w, t);
  }
  uint32_t e = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) e |= (uint32_t)__ldg(full + ((w >> (8 * i)) & 0xFFu)) << (8 * i);
  return e;
}

constexpr int QW = 8;                    // warps per CTA
constexpr int QB = 2 * QW;               // storage blocks per CTA
constexpr int QNC = 16;                  // neurons per chunk
constexpr int QBLKS = QNC * PB + 64;     // padded block slice: the two blocks of a warp on opposite bank halves
constexpr int QSTAGE = QB * QBLKS + QNC * 256 + QNC * 32;

size_t expand_q_smem_bytes() { return 2 * (size_t)QSTAGE + 64; }

__global__ void __launch_bounds__(QW * 32, 3) k_expand_q(SysView S, LevelView L, ExpandOut O) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * QSTAGE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t blk0 = (int64_t)blockIdx.x * QB;
  const int64_t nblk_total = (L.F + PB - 1) / PB;
  const int nb = (nblk_total - blk0 < QB) ? (int)(nblk_total - blk0) : QB;
  const int bl = warp * 2 + (lane >> 4);
  const int64_t p0 = (blk0 + bl) * PB + (lane & 15) * 4;
  const int nvalid = p0 >= L.F ? 0 : (L.F - p0 >= 4 ? 4 : (int)(L.F - p0));
  const int m = S.m;
  const int nchunks = (m + QNC - 1) / QNC;

  uint64_t a[4], b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool ok = k < nvalid;
    a[k] = ok ? L.fp0[p0 + k] : 0;
    b[k] = ok ? L.fp1[p0 + k] : 0;
    if (ok && !O.classify_only) {
      O.psi[p0 + k] = 1;
      O.ndc[p0 + k] = 0;
    }
  }
  // E byte of this lane pair (8 configurations), +8 per neuron; written by the even lane
  uint8_t* ep = nullptr;
  if (O.ebits != nullptr && !O.classify_only && nvalid > 0 && !(lane & 1))
    ep = reinterpret_cast<uint8_t*>(O.ebits) + emit_index(p0, 0, m);
  uint32_t any = 0;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int c) {
    if (tid == 0) {
      const int st = c & 1, c0 = c * QNC, rows = min(QNC, m - c0);
      uint8_t* stg = smem + st * QSTAGE;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(&bar[st], (uint32_t)(nb * rows * PB + rows * 256 + rows * 32));
      const uint8_t* base = reinterpret_cast<const uint8_t*>(L.data);
      for (int bb = 0; bb < nb; ++bb)
        bulk_g2s(stg + bb * QBLKS, base + ((blk0 + bb) * (int64_t)m + c0) * PB, (uint32_t)(rows * PB), &bar[st]);
      bulk_g2s(stg + QB * QBLKS, S.hsg + (int64_t)c0 * 256, (uint32_t)(rows * 256), &bar[st]);
      bulk_g2s(stg + QB * QBLKS + QNC * 256, S.elut + (int64_t)c0 * 32, (uint32_t)(rows * 32), &bar[st]);
    }
  };

  issue(0);
  for (int c = 0; c < nchunks; ++c) {
    const int st = c & 1, c0 = c * QNC, rows = min(QNC, m - c0);
    if (c + 1 < nchunks) issue(c + 1);
    mbar_wait(&bar[st], (uint32_t)((c >> 1) & 1));
    const uint8_t* stg = smem + st * QSTAGE;
    const uint8_t* crow = stg + bl * QBLKS + (lane & 15) * 4;
    const uint8_t* hs = stg + QB * QBLKS;
    const uint8_t* lt = hs + QNC * 256;
    // neurons in pairs: both deltas of a configuration enter its 64-bit
    // accumulators through one 3-input add (slot 0 of a delta row is zero);
    // an odd tail pairs the last neuron with a zero row (sl + 1 == rows)
    for (int sl = 0; sl < rows; sl += 2) {
      const bool pair = sl + 1 < rows;
      const uint32_t wA = *reinterpret_cast<const uint32_t*>(crow + sl * PB);
      const uint32_t wB = pair ? *reinterpret_cast<const uint32_t*>(crow + (sl + 1) * PB) : 0u;
      const uint32_t eA = expand_entries(wA, lt + sl * 32, S.tab_full + (int64_t)(c0 + sl) * 256);
      const uint32_t eB = pair ? expand_entries(wB, lt + (sl + 1) * 32, S.tab_full + (int64_t)(c0 + sl + 1) * 256) : 0u;
      const uint8_t* hA = hs + sl * 256;
      const uint8_t* hB = pair ? hs + (sl + 1) * 256 : hA;  // eB = 0: slot 0 of a loaded row (zero)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const ulonglong2 dA = *reinterpret_cast<const ulonglong2*>(hA + ((eA >> (8 * k)) & TE_F));
        const ulonglong2 dB = *reinterpret_cast<const ulonglong2*>(hB + ((eB >> (8 * k)) & TE_F));
        a[k] += dA.x + dB.x;
        b[k] += dA.y + dB.y;
      }
      any |= eA | eB;
      // emit nibbles of both neurons, merged with the partner lane's in one shuffle
      const uint32_t nib = emit_nibble(eA) | (emit_nibble(eB) << 8);
      const uint32_t hi = __shfl_xor_sync(0xFFFFFFFFu, nib, 1);
      if (ep) {
        ep[(int64_t)(c0 + sl) * 8] = (uint8_t)((nib & 0xFu) | ((hi & 0xFu) << 4));
        if (pair) ep[(int64_t)(c0 + sl + 1) * 8] = (uint8_t)(((nib >> 8) & 0xFu) | (((hi >> 8) & 0xFu) << 4));
      }
      if (((eA | eB) & 0x02020202u) && !O.classify_only) {  // rare: nondeterminism
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k >= nvalid) continue;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const uint32_t e = u ? eB : eA, w = u ? wB : wA;
            if (!((e >> (8 * k)) & TE_ND)) continue;
            int nk = O.ndc[p0 + k];
            uint64_t pk = O.psi[p0 + k];
            nd_event(S, O, c0 + sl + u, (w >> (8 * k)) & 0xFFu, p0 + k, nk, pk);
            O.ndc[p0 + k] = nk;
            O.psi[p0 + k] = pk;
          }
        }
      }
    }
    __syncthreads();
  }
  if (nvalid == 0) return;
  unsigned nh = 0;
  bool cap = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= nvalid) continue;
    const int64_t p = p0 + k;
    const bool fired = ((any >> (8 * k)) & TE_F) != 0;
    O.halting[p] = fired ? 0 : 1;
    nh += fired ? 0 : 1;
    if (!O.classify_only) {
      if (!fired) O.psi[p] = 0;  // halting: no children (reading A5)
      cap |= O.psi[p] > PSI_LIMIT || O.ndc[p] > KMAX;
      O.fpb0[p] = a[k];
      O.fpb1[p] = b[k];
    }
  }
  if (cap) atomicOr(O.err, ERR_CAPACITY);
  if (nh) atomicAdd(O.n_halting, (unsigned long long)nh);
}

// Fingerprint delta rows for k_expand_q: hsg[s][f] (16 B) = (h0, h1) of the
// neuron's f-th rule (f = 1 .. min(#rules, 15)), slot 0 = zero.
__global__ void k_build_hs(SysView S, uint8_t* hsg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)S.m * 16) return;
  const int32_t s = (int32_t)(i >> 4), f = (int32_t)(i & 15);
  const int32_t r0 = S.rule_off[s], r1 = S.rule_off[s + 1];
  ulonglong2 h = make_ulonglong2(0ULL, 0ULL);
  if (f >= 1 && f <= r1 - r0) h = make_ulonglong2(S.h0[r0 + f - 1], S.h1[r0 + f - 1]);
  reinterpret_cast<ulonglong2*>(hsg)[i] = h;
}

// ---------------------------------------------------------------------------
// K-a on the tensor cores (SysView::tc_ok).  The base-child fingerprint is a
// contraction over the neurons (reading A18):
//   fp_ℓ(base(C)) = fp_ℓ(C) + Σ_s X_s·(−R_ℓ[s]) + Σ_s Y_s·Rout_ℓ[s]  (mod 2^64)
// X_s / Y_s = consumption / emission of the first applicable rule of s
// (Def. 2 at 115-119), 0 when none applies.  A CTA owns M = 128
// configurations (two storage blocks) and walks the neurons in chunks of 64:
// thread (h, q, k) loads the 32 counts of neuron c0 + k in half q of block h
// (one 32-B load, one chunk ahead), maps them to X|Y bytes by byte-permute
// lookups in the neuron's 16/32-entry table (the chunk's tables are staged
// in shared memory), writes its half of the block's emit word, and stores X
// and Y into the chunk's A tiles (MN-major, one 16-B store per 16
// configurations); one
// thread issues the chunk's four u8 MMAs (K = 32, N = 32) into a TMEM s32
// accumulator: columns 0-7 / 8-15 are the byte planes of the two
// fingerprint lanes, column 16 the total consumption (0 <=> halting,
// reading A5).  Accumulators stay < 2^31 (m·15·255 + m·255 for m ≤ 2^19).
// Ψ and the ND lists come from k_nd_pass over the few neurons that can be
// nondeterministic.
// ---------------------------------------------------------------------------
constexpr int TCM = 128;                        // configurations per CTA (MMA M)
constexpr int TCK = 64;                         // neurons per chunk
constexpr int TCN = 32;                         // accumulator columns per operand (MMA N)
constexpr int TCT = 256;                        // threads: (block h, half q, neuron k)
constexpr int TC_A_LBO = 1024;                  // A: K-group (8 neurons) stride = 8 MN groups × 128 B
constexpr int TC_B_LBO = 512;                   // B: K-chunk (16 neurons) stride = 4 N groups × 128 B
constexpr int TC_ATILE = TCM * TCK;             // 8 KB
constexpr int TC_BTILE = TCK * TCN;             // 2 KB
constexpr int TC_STAGE = 2 * TC_ATILE;           // X and Y tiles of one chunk
constexpr int TC_STAGES = 2;                     // X|Y tiles: double-buffered
#ifndef SNP_TC_L2PF
#define SNP_TC_L2PF 0  // K-a: L2 bulk prefetch of the counts this many chunks ahead (producer warp); measured slower: 2 / 4 / 8 chunks 19.9 / 20.1 / 20.1 ms vs 19.6 off
#endif
#ifndef SNP_TC_MINB
#define SNP_TC_MINB 4  // K-a: resident CTAs the register budget is sized for (56 registers, 4 CTAs/SM; 1 = 72 registers, 3 CTAs: 24.3 vs 19.2 ms)
#endif
#ifndef SNP_TC_UADDR
#define SNP_TC_UADDR 1  // K-a: mbarrier addresses converted to shared once, outside the chunk loop
#endif
#ifndef SNP_TC_AHEAD
#define SNP_TC_AHEAD 1  // K-a: chunks whose counts are loaded ahead (registers; 2 = two sets in flight)
#endif
#ifndef SNP_TC_WS
#define SNP_TC_WS 1  // producer warp for copies + MMAs (else thread 0 issues them after a CTA barrier)
#endif
constexpr int TC_IN = 3;                         // B tile + tables: a ring of 3 (loaded one chunk ahead)

constexpr int TC_TTAB = TCK * 32;              // the chunk's 32-entry X|Y tables (2 KB)
constexpr int TC_INB = 2 * TC_BTILE + TC_TTAB;  // one input slot: B tiles (X, Y) + tables

size_t expand_tc_smem_bytes() { return (size_t)TC_STAGES * TC_STAGE + (size_t)TC_IN * TC_INB + 64 + 32; }

// t[v] for the four byte counts v < 16 of v4, t = 16 bytes in tt[0..3]
__device__ __forceinline__ uint32_t lut16(uint32_t v4, const uint32_t (&tt)[8]) {
  const uint32_t x = v4 & 0x07070707u;
  const uint32_t sel = prmt(x | (x >> 4), 0u, 0x4420u);
  const uint32_t m3 = prmt(v4 << 4, 0u, 0xBA98u);  // 0xFF in bytes whose bit 3 is set
  const uint32_t a = prmt(tt[0], tt[1], sel), b = prmt(tt[2], tt[3], sel);
  return (a & ~m3) | (b & m3);
}

// WS: a ninth (producer) warp issues the bulk copies and the MMAs; the 256
// compute threads only arrive on a per-stage mbarrier (no CTA barrier per chunk)
// T: count storage; 16/32-bit counts are packed to their low bytes on load
// (NARROW), a warp with a count >= 256 takes the exact per-count rule lookup
template <bool WS, typename T = uint8_t>
__global__ void __launch_bounds__(TCT + 32, SNP_TC_MINB) k_expand_tc(SysView S, LevelView L, ExpandOut O) {
  extern __shared__ __align__(128) uint8_t smem_tc[];
  uint8_t* smem = smem_tc;
  uint8_t* sIn = smem + TC_STAGES * TC_STAGE;                       // [TC_IN][B_X | B_Y | tables]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sIn + TC_IN * TC_INB);  // [2] MMAs done with an X|Y stage
  uint64_t* lbar = bar + TC_STAGES;                                    // [3] an input slot landed
  uint64_t* fbar = lbar + TC_IN;                                       // [2] (WS) X|Y stage written
  uint32_t* tslot = reinterpret_cast<uint32_t*>(fbar + TC_STAGES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t m = S.m;
  const int64_t mE = (m + 1) & ~1;
  const int64_t nblk = (L.F + PB - 1) / PB;
  const int64_t blk0 = (int64_t)blockIdx.x * 2;
  const int k = tid & 63, q = (tid >> 6) & 1, h = tid >> 7;
  const int64_t blk = blk0 + h;
  const bool bvalid = blk < nblk;
  // parents of block blk that exist (the tail block may be partial): mask of this half
  const int64_t nv = bvalid ? (L.F - blk * PB < PB ? L.F - blk * PB : PB) : 0;
  const int64_t nvq = nv - 32 * q;
  const uint32_t vmask = nvq >= 32 ? ~0u : (nvq <= 0 ? 0u : ((1u << nvq) - 1));
  const int nch = (m + TCK - 1) / TCK;
  uint32_t* ew_out = (O.ebits != nullptr && !O.classify_only) ? reinterpret_cast<uint32_t*>(O.ebits) : nullptr;
  const uint8_t* data = reinterpret_cast<const uint8_t*>(L.data);

  if (warp == 0) tc::tmem_alloc(tslot, 64);
  // chunk c's B tiles and X|Y tables (xyt is padded to whole chunks) into
  // input slot c % 3: two bulk copies (TMA engine, no LSU work) on lbar[c % 3]
  auto stage_inputs = [&](int c) {
    const int sl = c % TC_IN;
    mbar_arrive_expect_tx(&lbar[sl], (uint32_t)TC_INB);
    bulk_g2s(sIn + sl * TC_INB, S.btile + (int64_t)c * (2 * TC_BTILE), 2 * TC_BTILE, &lbar[sl]);
    bulk_g2s(sIn + sl * TC_INB + 2 * TC_BTILE, S.xyt + (int64_t)c * TC_TTAB, TC_TTAB, &lbar[sl]);
  };
  if (tid == 0) {
    tc::bar_init(&bar[0], 1);
    tc::bar_init(&bar[1], 1);
    for (int i = 0; i < TC_IN; ++i) tc::bar_init(&lbar[i], 1);
    tc::bar_init(&fbar[0], TCT);
    tc::bar_init(&fbar[1], TCT);
    fence_barrier_init();
    if (!WS) stage_inputs(0);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  [[maybe_unused]] const uint32_t bar_u = tc::smem_u32(bar), lbar_u = tc::smem_u32(lbar), fbar_u = tc::smem_u32(fbar);
  constexpr uint32_t IDESC = tc::idesc_u8(TCM, TCN, true, false);

  // the 32 counts of neuron c·64 + k (block h, half q) of chunk c, loaded
  // one chunk ahead
  uint32_t wbigm = 0;  // NARROW: bit (c & 1) = a count of chunk c's 32 is >= 256
  auto load = [&](int c, uint32_t (&w)[8]) {
    const int32_t s = c * TCK + k;
    bool wbig = false;
    if (c < nch && bvalid && s < m) {
      if constexpr (sizeof(T) == 1) {
        ldg256(data + ((blk * m + s) << 6) + 32 * q, w);
      } else {
        const uint8_t* src = data + (((blk * m + s) << 6) + 32 * q) * (int64_t)sizeof(T);
        uint32_t u[8];
#pragma unroll
        for (int h = 0; h < (int)sizeof(T); ++h) {
          ldg256(src + 32 * h, u);
          if constexpr (sizeof(T) == 2) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              w[4 * h + i] = prmt(u[2 * i], u[2 * i + 1], 0x6420u);
              wbig |= ((u[2 * i] | u[2 * i + 1]) & 0xFF00FF00u) != 0;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              w[2 * h + i] = prmt(prmt(u[4 * i], u[4 * i + 1], 0x0040u), prmt(u[4 * i + 2], u[4 * i + 3], 0x0040u),
                                  0x5410u);
              wbig |= ((u[4 * i] | u[4 * i + 1] | u[4 * i + 2] | u[4 * i + 3]) & 0xFFFFFF00u) != 0;
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = 0;  // count 0 -> entry 0 (nothing fires: padded neurons have zero tables)
    }
    wbigm = (wbigm & ~(1u << (c & 1))) | ((wbig ? 1u : 0u) << (c & 1));
  };
  auto chunk = [&](int c, uint32_t (&w)[8]) {
    const int st = c & 1;
    uint8_t* sX = smem + st * TC_STAGE;
    uint8_t* sY = sX + TC_ATILE;
    const int sl = c % TC_IN;
    uint8_t* sB = sIn + sl * TC_INB;
    const uint8_t* sT = sB + 2 * TC_BTILE;
    const int32_t s = c * TCK + k;
    // entries (c | p << 4) of the 32 counts: 16- or 32-entry byte-permute
    // lookups (warp-uniform choice), the full table for a count >= 32
    uint32_t e[8], tt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#if SNP_TC_UADDR
    tc::bar_wait_u(lbar_u + 8u * sl, (uint32_t)((c / TC_IN) & 1));
#else
    tc::bar_wait(&lbar[sl], (uint32_t)((c / TC_IN) & 1));
#endif
    // the next chunk's inputs go to slot (c + 1) % 3, last read by the MMAs
    // of chunk c - 2 (done: issued two chunks ago) and by the table loads of
    // chunk c - 2 (before every thread's __syncthreads of chunk c - 2)
    if (!WS && tid == 0 && c + 1 < nch) {
      if (c >= 2) tc::bar_wait(&bar[st], (uint32_t)(((c - 2) >> 1) & 1));
      tc::fence_async_smem();
      stage_inputs(c + 1);
    }
    {
      uint32_t hiv = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) hiv |= w[i];
      // the first 16 table entries always; the next 16 only when some count
      // of the warp is >= 16
      const uint4 t0 = reinterpret_cast<const uint4*>(sT + k * 32)[0];
      tt[0] = t0.x; tt[1] = t0.y; tt[2] = t0.z; tt[3] = t0.w;
      const bool small = __all_sync(0xFFFFFFFFu, (hiv & 0xF0F0F0F0u) == 0);
      if (!small) {
        const uint4 t1 = reinterpret_cast<const uint4*>(sT + k * 32)[1];
        tt[4] = t1.x; tt[5] = t1.y; tt[6] = t1.z; tt[7] = t1.w;
      }
      if (sizeof(T) > 1 && __any_sync(0xFFFFFFFFu, (wbigm >> (c & 1)) & 1u)) {
        // NARROW, rare: the entries (c | p << 4) of the first applicable rule
        // from the exact count (tables over the folded domain)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t x = 0;
          if (bvalid && s < m)
            for (int b = 0; b < 4; ++b) {
              const int r = first_rule(S, s, ld_count<T>(L.data, blk * PB + 32 * q + 4 * i + b, s, m));
              if (r >= 0) x |= (uint32_t)(S.rules[r].c | (S.rules[r].p << 4)) << (8 * b);
            }
          e[i] = x;
        }
      } else if (small) {
#pragma unroll
        for (int i = 0; i < 8; ++i) e[i] = lut16(w[i], tt);
      } else if ((hiv & 0xE0E0E0E0u) == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) e[i] = lut32(w[i], tt);
      } else {  // rare
        const uint8_t* xf = S.xyf + (int64_t)s * 256;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if ((w[i] & 0xE0E0E0E0u) == 0) {
            e[i] = lut32(w[i], tt);
          } else {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) x |= (uint32_t)__ldg(xf + ((w[i] >> (8 * b)) & 0xFFu)) << (8 * b);
            e[i] = x;
          }
        }
      }
    }
    load(c + SNP_TC_AHEAD, w);
    uint32_t X[8], Y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      X[i] = e[i] & 0x0F0F0F0Fu;
      Y[i] = e[i] & 0x10101010u;  // 16·p: its accumulator is shifted back in the epilogue
    }
    if (ew_out && bvalid && s < m) {
      // emit bits of configurations 8j..8j+7: bit 0 (4i+b) and bit 4 (4i+4+b)
      // of byte b, gathered into the top byte by one multiply
      uint32_t ew = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t z = (Y[2 * j] >> 4) | Y[2 * j + 1];
        ew = prmt(ew, z * 0x01020408u, (0x3210u & ~(0xFu << (4 * j))) | (7u << (4 * j)));
      }
      ew_out[(blk * mE + s) * 2 + q] = ew & vmask;
    }
    // the MMAs that read this stage two chunks ago must be done
#if SNP_TC_UADDR
    if (c >= 2) tc::bar_wait_u(bar_u + 8u * st, (uint32_t)(((c - 2) >> 1) & 1));
#else
    if (c >= 2) tc::bar_wait(&bar[st], (uint32_t)(((c - 2) >> 1) & 1));
#endif
    {
      const int off = (k >> 3) * TC_A_LBO + (4 * h + 2 * q) * 128 + (k & 7) * 16;
      *reinterpret_cast<uint4*>(sX + off) = make_uint4(X[0], X[1], X[2], X[3]);
      *reinterpret_cast<uint4*>(sX + off + 128) = make_uint4(X[4], X[5], X[6], X[7]);
      *reinterpret_cast<uint4*>(sY + off) = make_uint4(Y[0], Y[1], Y[2], Y[3]);
      *reinterpret_cast<uint4*>(sY + off + 128) = make_uint4(Y[4], Y[5], Y[6], Y[7]);
    }
    // (a per-stage mbarrier that only the MMA-issuing thread waits on, letting
    // the other warps run ahead, measured slower than this barrier)
    tc::fence_async_smem();
    if (WS) {
#if SNP_TC_UADDR
      tc::bar_arrive_u(fbar_u + 8u * st);
#else
      mbar_arrive(&fbar[st]);
#endif
      return;
    }
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
#pragma unroll
      for (int ks = 0; ks < TCK / 32; ++ks) {
        tc::mma_u8(tmem, tc::sdesc(tc::smem_u32(sX + ks * 4 * TC_A_LBO), TC_A_LBO, 128),
                   tc::sdesc(tc::smem_u32(sB + ks * 2 * TC_B_LBO), TC_B_LBO, 128), IDESC, (c > 0 || ks > 0) ? 1u : 0u);
        tc::mma_u8(tmem + TCN, tc::sdesc(tc::smem_u32(sY + ks * 4 * TC_A_LBO), TC_A_LBO, 128),
                   tc::sdesc(tc::smem_u32(sB + TC_BTILE + ks * 2 * TC_B_LBO), TC_B_LBO, 128), IDESC,
                   (c > 0 || ks > 0) ? 1u : 0u);
      }
      tc::commit(&bar[st]);
    }
  };
  if (WS && warp == TCT / 32) {
    // producer: inputs two chunks ahead, the MMAs of each chunk once its
    // X|Y stage is written
    if (lane == 0) {
      stage_inputs(0);
      if (nch > 1) stage_inputs(1);
      for (int c = 0; c < nch; ++c) {
        const int st = c & 1, sl = c % TC_IN;
        uint8_t* sX = smem + st * TC_STAGE;
        uint8_t* sY = sX + TC_ATILE;
        uint8_t* sB = sIn + sl * TC_INB;
#if SNP_TC_L2PF
        // the counts of chunk c + SNP_TC_L2PF (both blocks, 4 KB each) pulled
        // into L2 ahead of the compute warps' loads
        if (c + SNP_TC_L2PF < nch) {
          const int64_t s0 = (int64_t)(c + SNP_TC_L2PF) * TCK;
          const uint32_t nb = (uint32_t)((m - s0 < TCK ? m - s0 : TCK) * PB);
          for (int hh = 0; hh < 2; ++hh)
            if (blk0 + hh < nblk) bulk_prefetch_l2(data + (((blk0 + hh) * m + s0) << 6), nb);
        }
#endif
        tc::bar_wait(&lbar[sl], (uint32_t)((c / TC_IN) & 1));
        tc::bar_wait(&fbar[st], (uint32_t)((c >> 1) & 1));
        tc::fence_after();
#pragma unroll
        for (int ks = 0; ks < TCK / 32; ++ks) {
          tc::mma_u8(tmem, tc::sdesc(tc::smem_u32(sX + ks * 4 * TC_A_LBO), TC_A_LBO, 128),
                     tc::sdesc(tc::smem_u32(sB + ks * 2 * TC_B_LBO), TC_B_LBO, 128), IDESC,
                     (c > 0 || ks > 0) ? 1u : 0u);
          tc::mma_u8(tmem + TCN, tc::sdesc(tc::smem_u32(sY + ks * 4 * TC_A_LBO), TC_A_LBO, 128),
                     tc::sdesc(tc::smem_u32(sB + TC_BTILE + ks * 2 * TC_B_LBO), TC_B_LBO, 128), IDESC,
                     (c > 0 || ks > 0) ? 1u : 0u);
        }
        tc::commit(&bar[st]);
        // slot (c + 2) % 3 was last used by chunk c - 1: its tables were read
        // before fbar(c - 1), its B tiles by the MMAs of chunk c - 1
        if (c + 2 < nch) {
          if (c >= 1) tc::bar_wait(&bar[st ^ 1], (uint32_t)(((c - 1) >> 1) & 1));
          tc::fence_async_smem();
          stage_inputs(c + 2);
        }
      }
    }
  } else {
    uint32_t w[8];
    if (SNP_TC_AHEAD == 1) {
      load(0, w);
      for (int c = 0; c < nch; ++c) chunk(c, w);
    } else {  // two register sets: the counts of chunks c + 1 and c + 2 in flight
      uint32_t w2[8];
      load(0, w);
      load(1, w2);
      for (int c = 0; c < nch; c += 2) {
        chunk(c, w);
        if (c + 1 < nch) chunk(c + 1, w2);
      }
    }
  }
  const int cl = nch - 1;
  tc::bar_wait(&bar[cl & 1], (uint32_t)((cl >> 1) & 1));
  tc::fence_after();
  if (warp < 4) {
    uint32_t rx[32], ry[32];
    tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), rx);
    tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + TCN, ry);
    const int64_t p = blk0 * PB + 32 * warp + lane;
    bool halt = false;
    if (p < L.F) {
      uint64_t a = L.fp0[p], b = L.fp1[p];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a += (uint64_t)(rx[i] + (ry[i] >> 4)) << (8 * i);
        b += (uint64_t)(rx[8 + i] + (ry[8 + i] >> 4)) << (8 * i);
      }
      halt = rx[16] == 0;
      O.halting[p] = halt ? 1 : 0;
      if (!O.classify_only) {
        O.fpb0[p] = a;
        O.fpb1[p] = b;
      }
    }
    const unsigned nh = __popc(__ballot_sync(0xFFFFFFFFu, halt));
    if (lane == 0 && nh) atomicAdd(O.n_halting, (unsigned long long)nh);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

// Ψ (eq. (8), readings A3/A5) and the ND lists for k_expand_tc:
// only neurons in S.nd_list can have d_s >= 2; visited in increasing order so
// the list is in total order (reading A7).
template <typename T>
__global__ void k_nd_pass(SysView S, LevelView L, ExpandOut O) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= L.F) return;
  int ndc = 0;
  uint64_t psi = 1;
  for (int i = 0; i < S.n_nd; ++i) {
    const int32_t s = __ldg(S.nd_list + i);
    const uint32_t v = (uint32_t)ld_count<T>(L.data, p, s, S.m);
    const uint8_t e = sizeof(T) == 1 ? __ldg(S.tab_full + (int64_t)s * 256 + v)
                                     : __ldg(S.tab + (int64_t)s * S.tabw + table_index(v, S.meta[s]));
    if (e & TE_ND) nd_event(S, O, s, v, p, ndc, psi);
  }
  if (O.halting[p]) psi = 0;  // halting: no children (reading A5)
  O.psi[p] = psi;
  O.ndc[p] = ndc;
  if (psi > PSI_LIMIT || ndc > KMAX) atomicOr(O.err, ERR_CAPACITY);
}

// Generic K-a (systems whose neurons cannot all be tabulated): the same walk,
// every rule evaluated from its descriptor.
template <typename T>
__global__ void __launch_bounds__(256) k_expand_g(SysView S, LevelView L, ExpandOut O) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tile = (int64_t)blockIdx.x * XW + warp;
  const int64_t p0 = tile * XTILE + lane * XPPL;
  if (tile * XTILE >= L.F) return;
  const T* data = reinterpret_cast<const T*>(L.data);
  uint64_t a[8], b[8], psi[8];
  int ndc[8];
  uint32_t anyb = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const bool ok = p0 + k < L.F;
    a[k] = ok ? L.fp0[p0 + k] : 0;
    b[k] = ok ? L.fp1[p0 + k] : 0;
    psi[k] = 1;
    ndc[k] = 0;
  }
  uint8_t* Eb = reinterpret_cast<uint8_t*>(O.ebits);
  for (int32_t s = 0; s < S.m; ++s) {
    uint32_t v[8];
    load8<T>(data, p0, s, S.m, L.F, v);
    uint32_t eb = 0;
    expand_generic_neuron(S, O, s, v, p0, L.F, a, b, psi, ndc, anyb, eb);
    if (Eb && !O.classify_only && p0 < L.F) Eb[emit_index(p0, s, S.m)] = (uint8_t)eb;
  }
  unsigned nh = 0;
  bool cap = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t p = p0 + k;
    if (p >= L.F) continue;
    const bool any = (anyb >> k) & 1u;
    const uint64_t ps = any ? psi[k] : 0;
    cap |= ps > PSI_LIMIT || ndc[k] > KMAX;
    O.halting[p] = any ? 0 : 1;
    nh += any ? 0 : 1;
    if (!O.classify_only) {
      O.psi[p] = ps;
      O.fpb0[p] = a[k];
      O.fpb1[p] = b[k];
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
    if (S.kernel_flags & KF_FP_WEAK) {  // tests only: 6-bit keys, so distinct children share keys
      a &= 63;
      b = 0;
    }
    C.cfp0[c] = a;
    C.cfp1[c] = b;
  }
}

// Generated numbers: the child key gets (A' - A)·R_ℓ[m-1] (linearity,
// reading A18); a terminal child records its number and gets the skip key.
template <typename T>
__global__ void k_aug_keys(SysView S, LevelView L, const uint64_t* off, ExpandOut O, uint64_t T_, ChildArrays C,
                           int32_t* err) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T_; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = C.cpar[c];
    ChildCtx cx;
    decode_child(S, O.nd + (uint64_t)p * KMAX, O.ndc[p], c - off[p], cx);
    int64_t number;
    const int64_t a2 = aug_child<T>(S, L.data, p, cx, &number);
    if (number >= 0) {
      if (number < S.gen_cap_bits) atomicOr(S.gen_bits + (number >> 6), 1ULL << (number & 63));
      else atomicOr(err, ERR_CAPACITY);
      C.cfp0[c] = EMPTY;
      C.cfp1[c] = KEY_TERMINAL1;
    } else {
      const uint64_t d = (uint64_t)(a2 - (int64_t)ld_count<T>(L.data, p, S.m - 1, S.m));
      C.cfp0[c] += d * __ldg(S.R0 + S.m - 1);
      C.cfp1[c] += d * __ldg(S.R1 + S.m - 1);
    }
  }
}

// Generated numbers: A' of every kept child (after K-c, which copies A).
template <typename T>
__global__ void k_aug_fix(SysView S, LevelView L, ExpandOut O, NextArrays N, int64_t K, int32_t* err) {
  T* out = reinterpret_cast<T*>(N.data);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = N.parent[q];
    ChildCtx cx;
    decode_child(S, O.nd + (uint64_t)p * KMAX, O.ndc[p], N.t[q], cx);
    int64_t number;
    const int64_t a2 = aug_child<T>(S, L.data, p, cx, &number);
    if (a2 > S.count_max) atomicOr(err, ERR_OVERFLOW);
    out[eidx(q, S.m - 1, S.m)] = (T)a2;
  }
}

// ---------------------------------------------------------------------------
// K-d: dedup against visited + same-level minimum tag
// ---------------------------------------------------------------------------
__device__ __forceinline__ Key128 ld_key(const Slot* s) { return *reinterpret_cast<const Key128*>(s); }

__global__ void k_dedup(ChildArrays C, uint64_t T, uint64_t tag_base, Tables tb, int use_visited, int32_t* err) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k0 = C.cfp0[c], k1 = C.cfp1[c];
    if (k0 == EMPTY && k1 == KEY_TERMINAL1) {  // generated numbers: terminal child (never stored)
      C.verdict[c] = 0;
      C.cref[c] = EMPTY;
      continue;
    }
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

// keep_all_edges (reading A17): the configuration every transition reached,
// as a visited ref (level << 40 | index), or EMPTY when it was not stored
// (thinned, or a terminal transition of generated numbers).  A child seen at
// an earlier level carries the visited ref k_dedup found; a new one points at
// its key's winner (minimum tag) in the next level when that was kept.
__global__ void k_all_edges(ChildArrays C, uint64_t T, uint64_t tag_base, Tables tb, uint64_t next_ref,
                            uint64_t* ref) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T; c += (uint64_t)gridDim.x * blockDim.x) {
    if (C.verdict[c] == 0) {
      ref[c] = C.cref[c];
    } else {
      const uint64_t w = tb.ltab[C.cslot[c]].tag - tag_base;
      ref[c] = C.kept[w] ? (next_ref | C.kpos[w]) : EMPTY;
    }
  }
}

__global__ void k_compact(ChildArrays C, const uint64_t* off, uint64_t T, NextArrays N, Tables tb,
                          uint64_t level_ref, int insert_visited, int32_t* err) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T; c += (uint64_t)gridDim.x * blockDim.x) {
    if (!C.kept[c]) continue;
    const uint64_t q = C.kpos[c];
    const uint32_t p = C.cpar[c];
    N.parent[q] = p;
    N.t[q] = c - off[p];
    N.fp0[q] = C.cfp0[c];
    N.fp1[q] = C.cfp1[c];
    if (insert_visited) visited_insert(tb, C.cfp0[c], C.cfp1[c], level_ref | q, err);
  }
}

// ---------------------------------------------------------------------------
// multi-GPU dedup ownership: owner(key) = fmix64(fp1) mod P
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t key_owner(uint64_t fp1, uint32_t P) { return (uint32_t)(fmix64(fp1) % P); }

// keys per owner: lanes with the same owner aggregated (match_any), one
// shared-memory add per group, one global add per (block, owner) — with P <= 8
// owners a per-key global atomic serialised ~T/P adds on each counter
__global__ void k_owner_hist(const uint64_t* fp1, uint64_t T, uint32_t P, unsigned long long* counts) {
  extern __shared__ unsigned oh_cnt[];  // [P]
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) oh_cnt[i] = 0;
  __syncthreads();
  for (uint64_t c0 = blockIdx.x * (uint64_t)blockDim.x; c0 < T; c0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = c0 + threadIdx.x;
    if (c < T) {
      const uint32_t own = key_owner(fp1[c], P);
      const unsigned grp = __match_any_sync(__activemask(), own);
      if ((threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1)) atomicAdd(&oh_cnt[own], (unsigned)__popc(grp));
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x)
    if (oh_cnt[i]) atomicAdd(&counts[i], (unsigned long long)oh_cnt[i]);
}

// send row pos = {fp0, fp1, global tag}; perm[c] = pos (positions inside an
// owner's bucket are arbitrary: the owner's decisions do not depend on them).
// One key per thread; a block reserves its range of every owner's bucket with
// one global add (ranks inside it from match_any groups and shared memory)
__global__ void k_owner_pack(const uint64_t* fp0, const uint64_t* fp1, uint64_t T, uint32_t P, uint64_t tag_base,
                             unsigned long long* cursor, uint64_t* perm, uint64_t* send) {
  extern __shared__ unsigned long long op_base[];  // [P] bases, then [P] counts
  unsigned* cnt = reinterpret_cast<unsigned*>(op_base + P);
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  uint32_t own = 0;
  unsigned local = 0;
  if (c < T) {
    own = key_owner(fp1[c], P);
    const unsigned grp = __match_any_sync(__activemask(), own);
    const int leader = __ffs(grp) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(&cnt[own], (unsigned)__popc(grp));
    base = __shfl_sync(grp, base, leader);
    local = base + (unsigned)__popc(grp & ((1u << lane) - 1));
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) op_base[i] = cnt[i] ? atomicAdd(&cursor[i], (unsigned long long)cnt[i]) : 0;
  __syncthreads();
  if (c < T) {
    const uint64_t pos = op_base[own] + local;
    perm[c] = pos;
    send[3 * pos] = fp0[c];
    send[3 * pos + 1] = fp1[c];
    send[3 * pos + 2] = tag_base + c;
  }
}

// owner side: received keys against the visited shard, then the level table
// with the minimum global tag (same protocol as k_dedup)
__global__ void k_owner_dedup(const uint64_t* recv, uint64_t R, Tables tb, uint8_t* verdict, uint64_t* slot,
                              int32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < R; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k0 = recv[3 * i], k1 = recv[3 * i + 1], tag = recv[3 * i + 2];
    if (k0 == EMPTY && k1 == EMPTY) {
      atomicOr(err, ERR_COLLISION);
      verdict[i] = 0;
      continue;
    }
    const uint64_t h = fmix64(k0);
    bool old = false;
    uint64_t j = h & tb.vmask;
    for (uint64_t probes = 0; probes <= tb.vmask; ++probes, j = (j + 1) & tb.vmask) {
      const Key128 key = ld_key(tb.vis + j);
      if (key.k0 == k0 && key.k1 == k1) { old = true; break; }
      if (key.k0 == EMPTY && key.k1 == EMPTY) break;
    }
    if (old) { verdict[i] = 0; continue; }
    j = h & tb.lmask;
    bool done = false;
    for (uint64_t probes = 0; probes <= tb.lmask; ++probes, j = (j + 1) & tb.lmask) {
      Key128 empty{EMPTY, EMPTY}, mine{k0, k1};
      const Key128 prev = atomicCAS(reinterpret_cast<Key128*>(tb.ltab + j), empty, mine);
      if ((prev.k0 == EMPTY && prev.k1 == EMPTY) || (prev.k0 == k0 && prev.k1 == k1)) {
        atomicMin(&tb.ltab[j].tag, (unsigned long long)tag);
        slot[i] = j;
        verdict[i] = 1;
        done = true;
        break;
      }
    }
    if (!done) atomicOr(err, ERR_TABLE_FULL);
  }
}

__global__ void k_owner_winners(const uint64_t* recv, uint64_t R, Tables tb, const uint8_t* verdict,
                                const uint64_t* slot, unsigned long long* n_new) {
  unsigned long long cnt = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < R; i += (uint64_t)gridDim.x * blockDim.x)
    cnt += verdict[i] == 1 && tb.ltab[slot[i]].tag == recv[3 * i + 2];
  typedef cub::BlockReduce<unsigned long long, BLK> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long tot = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0 && tot) atomicAdd(n_new, tot);
}

// kept = winner && (no thinning || fmix64(fp0) < τ); kept keys enter the
// owner's visited shard; out[i] = kept byte returned to the producer
__global__ void k_owner_keep(const uint64_t* recv, uint64_t R, Tables tb, const uint8_t* verdict, const uint64_t* slot,
                             uint64_t tau, int thin, uint8_t* out, unsigned long long* n_kept, int32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < R; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k0 = recv[3 * i], k1 = recv[3 * i + 1];
    bool k = verdict[i] == 1 && tb.ltab[slot[i]].tag == recv[3 * i + 2];
    if (k && thin) k = fmix64(k0) < tau;
    out[i] = k ? 1 : 0;
    if (k) visited_insert(tb, k0, k1, 0, err);
    const unsigned b = __ballot_sync(__activemask(), k);  // one add per warp
    if (b && (threadIdx.x & 31) == (unsigned)(__ffs(b) - 1)) atomicAdd(n_kept, (unsigned long long)__popc(b));
  }
}

__global__ void k_unperm(const uint64_t* perm, const uint8_t* back, uint64_t T, uint64_t* kept) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c <= T; c += (uint64_t)gridDim.x * blockDim.x)
    kept[c] = c < T ? (uint64_t)back[perm[c]] : 0;
}

__global__ void k_kq_off(const uint64_t* off, const uint64_t* kpos, int64_t F, uint64_t* kq_off) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= F; p += (int64_t)gridDim.x * blockDim.x)
    kq_off[p] = kpos[off[p]];
}

// ---------------------------------------------------------------------------
// K-c (fast): one CTA per storage block of 64 parents.
//   1. TMA bulk-copies the block's emit words E[s] (bit k = parent k of the
//      block fires a spiking rule at neuron s) into shared memory;
//   2. lane = target neuron j: the in-synapse gather Σ_{s∈in(j)} emit(s, ·) is
//      a bit-sliced counter over the 64 parents (ripple-carry on NPL planes);
//   3. x = C[j] - c_first(j) + count per parent (consumption from the compact
//      outcome table, staged per lane in shared memory), staged per lane and
//      written to every kept child of the parent (row j of the output blocks).
// ND digits ≠ 0 are corrected afterwards by k_patch (exact), out-of-range
// base values by k_overflow_fix.
// ---------------------------------------------------------------------------
#ifndef SNP_KC_WARPS
#define SNP_KC_WARPS 32
#endif
// tuning toggles (tools/gpu_ab.sh), measured at config 4: 32 warps with
// 64 registers beat 24 warps (70.4 ms) and 16 warps (83 ms); loading the row
// before the gather (SNP_KC_PREFETCH=1: 68.6 ms; 64.2 vs 63.7 with the L2 row prefetch on) or one iteration ahead
// (77 ms, spills) loses to loading it where it is used (66.5 ms)
#ifndef SNP_KC_COOP
#define SNP_KC_COOP 1  // warp-cooperative stores of the full 4-child quads (else the per-lane store program).
                       // Measured and rejected in round 2 (config 4, K-c ms): a flat (row, quad) lane list
                       // 68.7 vs 60.6; lane = output quad over all rows 64.3 vs 62.3, with the partial end
                       // quads folded in 87.2; in-degree-sorted lane order (padding 15.9 -> 9.8 gather rows
                       // per lane, but each warp's 32 row loads scattered over 64 KB) +23 ms
#endif
#ifndef SNP_KC_L2PF
#define SNP_KC_L2PF 1  // k > 0: L2 bulk prefetch of the warp's parent rows k - 1 iterations ahead (rolled halves: 0 64.2 ms, 1 64.0, 2 63.7, 3 63.9; unrolled: 1 60.8, 2 61.3)
#endif
#ifndef SNP_KC_BRANCHLESS
#define SNP_KC_BRANCHLESS 0  // cooperative quads: the upper-window permute unconditionally (no per-lane branch); measured 64.1 vs 63.9 ms
#endif
#ifndef SNP_KC_GUNROLL
#define SNP_KC_GUNROLL 2  // the two 32-parent halves unrolled (measured 61.4 vs 63.7 ms rolled)
#endif
#define SNP_PRAGMA_(x) _Pragma(#x)
#define SNP_PRAGMA(x) SNP_PRAGMA_(x)
#ifndef SNP_KC_EDGE
#define SNP_KC_EDGE 1  // boundary bytes of a row end as <= 2 aligned stores (else one byte store per child)
#endif
#ifndef SNP_KC_XS72
#define SNP_KC_XS72 0  // byte staging rows of 72 bytes (8-aligned: x stored as 64-bit words) instead of 68; measured 50.5 vs 50.1 ms
#endif
#ifndef SNP_KC_CARRYU
#define SNP_KC_CARRYU 1  // byte-carry check of x = t + count warp-uniform (a real branch, not predication)
#endif
#ifndef SNP_KC_TAILQ
#define SNP_KC_TAILQ 0  // cooperative quads: the last < 16 quads with several rows per step (measured slower: 54.5 vs 50.7 ms, 64 registers)
#endif
#ifndef SNP_KC_IDX4
#define SNP_KC_IDX4 1  // gather indices: 4 rows' uint16 sources in one 8-byte load per lane
#endif
#ifndef SNP_KC_FULLROWS
#define SNP_KC_FULLROWS 1  // cooperative quads: no per-store row predicate when the warp has all 32 rows
#endif
#ifndef SNP_KC_EDGEPRMT
#define SNP_KC_EDGEPRMT 1  // row-end bytes gathered by the partial quad's byte permute (else byte by byte)
#endif
#ifndef SNP_KC_ABLATE
#define SNP_KC_ABLATE 0  // diagnostics only (wrong results): 1 / 4 skip the per-lane / cooperative stores, 2 the gather
#endif
#ifndef SNP_KC_PREFETCH
#define SNP_KC_PREFETCH 0
#endif
#ifndef SNP_KC_WIDE_COOP
#define SNP_KC_WIDE_COOP 1  // 16/32-bit counts: warp-cooperative row stores (else one lane per row)
#endif
#ifndef SNP_KC_FLATQ
#define SNP_KC_FLATQ 1  // cooperative quads in passes over the CTA's own quad range (else per output block: 61.0 vs 56.4 ms)
#endif
#ifndef SNP_KC_EPF
#define SNP_KC_EPF 0  // k > 0: L2 bulk prefetch of block blk + k's emit words at CTA start (A/B: 148 = one wave ahead)
#endif
constexpr int MW = SNP_KC_WARPS;  // warps per K-c CTA
constexpr int QCAP = 4064;   // outputs per block resolved through the r(q) table (+32 alignment slack)

template <typename T>
__host__ __device__ constexpr int xs_stride() { return sizeof(T) == 1 && SNP_KC_XS72 ? 72 : PB * (int)sizeof(T) + 4; }

// Counts of parents 8k .. 8k+7 as bytes (lo: 8k..8k+3, hi: 8k+4..8k+7) from
// the bit planes: byte k of every plane gathered into one 64-bit word (plane
// b in byte b), then an 8x8 bit-matrix transpose (three delta swaps).
// P = planes used (<= NPL): P = 4 when the warp knows every count < 16.
template <int P, int NPL>
__device__ __forceinline__ void counts8(const uint64_t (&c)[NPL], int k, uint32_t& lo, uint32_t& hi) {
  constexpr int Q = P < NPL ? P : NPL;
  uint32_t p[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) p[b] = b < Q ? (uint32_t)(c[b < Q ? b : 0] >> (32 * (k >> 2))) : 0u;
  const uint32_t s2 = (uint32_t)(k & 3) | ((uint32_t)(4 + (k & 3)) << 4);
  lo = prmt(prmt(p[0], p[1], s2), prmt(p[2], p[3], s2), 0x5410u);
  uint32_t t;
  t = (lo ^ (lo >> 7)) & 0x00AA00AAu; lo ^= t ^ (t << 7);
  t = (lo ^ (lo >> 14)) & 0x0000CCCCu; lo ^= t ^ (t << 14);
  if (Q <= 4) {  // planes 4-7 empty: the last delta swap only moves nibbles out of lo
    t = lo & 0xF0F0F0F0u;
    lo ^= t;
    hi = t >> 4;
    return;
  }
  if (Q == 5) hi = prmt(p[4], 0u, (uint32_t)(k & 3) | 0x4440u);
  else hi = prmt(prmt(p[4], p[5], s2), prmt(p[6], p[7], s2), 0x5410u);
  t = (hi ^ (hi >> 7)) & 0x00AA00AAu; hi ^= t ^ (t << 7);
  t = (hi ^ (hi >> 14)) & 0x0000CCCCu; hi ^= t ^ (t << 14);
  t = (lo ^ (hi << 4)) & 0xF0F0F0F0u; lo ^= t; hi ^= t >> 4;
}

__device__ const uint64_t g_zero_word = 0;  // padded in-synapses when the emit words stay in global memory

// K-c store program (u8): the output range [Q0, Q1) of a CTA split into
// aligned stores, identical for every neuron j of the block, so it is built
// once per CTA into shared memory.  Op (64 bits): bits 0-31 byte offset of
// the store from the row of neuron j in output block Q0 >> 6 (output block
// stride m·64); bits 32-33 kind (0: 1 byte, 1: 4 bytes, 2: 16 bytes, 3: 32
// bytes); bits 48-63 the parent (kind 0) or the quad index (q - Qb) / 4
// (kinds 1-3).  Qb = Q0 rounded down to 32, so the descriptors of a
// 16/32-byte store are one/two aligned 16-B loads.
constexpr int OPCAP = 1100;  // >= 16 ops per output block × (QCAP / 64 + 2)

// K-c store on the tensor cores (TCS, uint8): the output permutation
// out[j][q] = x[j][r(q)] (q = kept child, r(q) its parent in the block) is a
// product with a one-hot matrix, D = X·P, done by tcgen05.mma kind::i8 into
// TMEM instead of byte permutes through shared memory.  A tile = 128 neurons ×
// 64 parents (K-major, no swizzle: addr(m, k) = (k/16)·2048 + (m/8)·128 +
// (m%8)·16 + k%16), written by the 4 warps that computed those rows.  Two
// children per accumulator column: column c of the CTA's child window (Qb =
// Q0 rounded down to 32) holds x(Qb+2c) + 256·x(Qb+2c+1), from two MMAs over
// the same A: P1[k][c] = [r(Qb+2c) = k] + 128·[r(Qb+2c+1) = k] and P2[k][c] =
// 128·[r(Qb+2c+1) = k] (entries <= 129 fit u8).  So 64 columns per tile cover
// 128 children (4 sectors), the 8 tiles of a CTA fill the 512 TMEM columns,
// and one PRMT packs 4 children; each lane then writes whole 32-byte sectors
// of its row (partial ones only at the window's two ends).  CTAs whose window
// exceeds 8 sectors (2 rounds) take a per-lane byte path (rare: ~64 children
// per block once the frontier is thinned).
constexpr int KCT_ATILE = 128 * 64;                // one A tile (bytes)
constexpr int KCT_A_LBO = 2048;                    // A: K-chunk (16 parents) stride
constexpr int KCT_B_LBO = 1024;                    // B: K-chunk stride (64 columns × 16 B)
constexpr int KCT_BHALF = 64 * 64;                 // one B matrix (P1 or P2) of one round
constexpr int KCT_BBYTES = 2 * 2 * KCT_BHALF;      // 2 rounds × (P1, P2)

// ES: the block's emit words are staged in shared memory (m·8 B fit); else
// (large m) the in-synapse gather reads them from global memory (L2/L1).
// MWT: warps per CTA (MW; fewer for wide counts, whose per-lane staging of
// 64 values would not fit shared memory at MW warps — int32 at config 3).
template <typename T, int NPL, bool ES, int MWT = MW, bool TCS = false, bool NARROW = false>
__global__ void __launch_bounds__(MWT * 32) k_materialize_bs(SysView S, LevelView L, ExpandOut O,
                                                             const uint64_t* kq_off, NextArrays N, uint64_t* ovf,
                                                             unsigned long long* n_ovf, uint64_t ovf_cap) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int32_t m = S.m;
  const int64_t mE = (m + 1) & ~1;
  uint64_t* sE = reinterpret_cast<uint64_t*>(smem);                    // mE words + 2 zero words
  uint8_t* sX = smem + (ES ? (mE + EPAD) * 8 : 0);                      // MWT×32×xs_stride (TCS: the A tiles)
  constexpr int XS = NARROW ? xs_stride<uint8_t>() : xs_stride<T>();  // staging row stride (NARROW: bytes)
  uint8_t* sR = sX + (TCS ? (size_t)MWT / 4 * KCT_ATILE + KCT_BBYTES : (size_t)MWT * 32 * XS);  // QCAP + 32
  uint32_t* sD = reinterpret_cast<uint32_t*>(sR + QCAP + 32);           // (QCAP+32)/4 quad descriptors
  uint64_t* sOps = reinterpret_cast<uint64_t*>(sD + (TCS ? 0 : (QCAP + 32) / 4));  // OPCAP store ops
  uint64_t* sQ = sOps + ((TCS || SNP_KC_COOP) ? 0 : OPCAP);             // 65 (+1 pad)
  uint64_t* bar = sQ + 66;
  uint64_t* tbar = bar + 1;                                             // TCS: one mbarrier per A tile
  uint32_t* sMisc = reinterpret_cast<uint32_t*>(tbar + (TCS ? MWT / 4 : 0));  // [0,1] haskids, [2] #ops, [3] TMEM
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t blk = blockIdx.x;
  const int64_t pb0 = blk * PB;
  const int np = (L.F - pb0 < PB) ? (int)(L.F - pb0) : PB;
  const uint64_t Q0 = kq_off[pb0], Q1 = kq_off[pb0 + np];
  if (Q1 == Q0) return;  // no kept child in this block (CTA-uniform)
  const uint32_t ebytes = (uint32_t)(mE * 8);
  if (tid == 0) {
    mbar_init(bar, 1);
    if (TCS)
      for (int t = 0; t < MWT / 4; ++t) mbar_init(&tbar[t], 1);
    fence_barrier_init();
  }
  if (TCS && warp == 0) tc::tmem_alloc(&sMisc[3], 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (ES && tid == 0) {
    mbar_arrive_expect_tx(bar, ebytes);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(O.ebits) + (size_t)blk * ebytes;
    for (uint32_t off = 0; off < ebytes; off += 32768u)
      bulk_g2s(reinterpret_cast<uint8_t*>(sE) + off, src + off, min(32768u, ebytes - off), bar);
#if SNP_KC_EPF
    // the emit words of the block an SM is likely to take next (blocks are
    // handed out in order, one resident CTA per SM) pulled into L2, so that
    // CTA's staging copy does not wait on HBM
    const int64_t nb = blk + SNP_KC_EPF;
    if (nb < (L.F + PB - 1) / PB) {
      const uint8_t* nsrc = reinterpret_cast<const uint8_t*>(O.ebits) + (size_t)nb * ebytes;
      for (uint32_t off = 0; off < ebytes; off += 32768u) bulk_prefetch_l2(nsrc + off, min(32768u, ebytes - off));
    }
#endif
  }
  if (tid <= np) sQ[tid] = kq_off[pb0 + tid];
  if (ES && tid < EPAD) sE[mE + tid] = 0;  // targets of padded in-synapses (one per bank pair)
  const uint64_t* gE = O.ebits + blk * mE;
  __syncthreads();
  const uint64_t nq = Q1 - Q0;
  const bool prog = !TCS && (sizeof(T) == 1 || NARROW) && nq <= QCAP;  // CTA-uniform: the quad stores apply
  const uint64_t Qb = Q0 & ~31ULL;                  // sR[q - Qb]
  const int nsec = (int)((Q1 - Qb + 31) >> 5);      // TCS: 32-child sectors of the window
  const bool tcp = TCS && nsec <= 8;                // CTA-uniform: the tensor-core store applies
  if (nq <= QCAP) {
    if (tid < np)
      for (uint64_t q = sQ[tid]; q < sQ[tid + 1]; ++q) sR[q - Qb] = (uint8_t)tid;
  }
  if (tid < 64) {  // parents with kept children (bit r), for the overflow bookkeeping
    const unsigned b = __ballot_sync(0xFFFFFFFFu, tid < np && sQ[tid + 1] > sQ[tid]);
    if (lane == 0) sMisc[warp] = b;
  }
  __syncthreads();
  // quad descriptors: output quad q..q+3 (q % 4 == 0) whose parents lie in
  // one 8-byte window of the x row = one byte permute of two words (word in
  // bits 16-19, selector in bits 0-15; bit 31 = use the byte path); the
  // store program reads r(q) too, so both run after the r(q) table is built
  if (prog) {
    const uint64_t nquad = (Q1 - Qb + 3) >> 2;
    for (uint64_t i = tid; i < nquad; i += blockDim.x) {
      const uint64_t q = Qb + 4 * i;
      uint32_t d = 0x80000000u;
      // partial quads at the window ends too (positions outside [Q0, Q1)
      // repeat the first valid one): the row-end bytes use the same permute
      const uint64_t qf = q >= Q0 ? q : Q0;
      if (qf < Q1 && qf < q + 4) {
        const uint32_t a = sR[qf - Qb] >> 2;
        uint32_t sel = 0, hb = 0;
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t qk = (q + k >= Q0 && q + k < Q1) ? q + k : qf;
          const uint32_t o = (uint32_t)sR[qk - Qb] - 4 * a;
          ok &= o < 16;
          hb |= (o >> 3) << k;  // byte k from words a+2, a+3
          sel |= (o & 7) << (4 * k);
        }
        if (ok) d = (hb << 24) | (a << 16) | sel;
      }
      sD[i] = d;
    }
  }
  if (TCS && tcp) {
    // the one-hot operands P1 / P2 of both rounds (see KCT_ATILE): item i =
    // (round, matrix, K-chunk, column), one 16-byte core-matrix row each
    for (int i = tid; i < 2 * 2 * 4 * 64; i += blockDim.x) {
      const int n = i & 63, kc = (i >> 6) & 3, h = (i >> 8) & 1, rd = i >> 9;
      const uint64_t q0 = Qb + 2 * (64 * rd + n), q1 = q0 + 1;
      const int r0 = (q0 >= Q0 && q0 < Q1) ? (int)sR[q0 - Qb] : -1;
      const int r1 = (q1 >= Q0 && q1 < Q1) ? (int)sR[q1 - Qb] : -1;
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const int k = 16 * kc + b;
        const uint32_t v = (h == 0 && k == r0 ? 1u : 0u) + (k == r1 ? 128u : 0u);
        w[b >> 2] |= v << (8 * (b & 3));
      }
      *reinterpret_cast<uint4*>(sX + (size_t)MWT / 4 * KCT_ATILE + rd * 2 * KCT_BHALF + h * KCT_BHALF +
                                kc * KCT_B_LBO + (n >> 3) * 128 + (n & 7) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    tc::fence_async_smem();
  }
  if (!SNP_KC_COOP && prog && tid == 64) {  // the store program (one thread; overlaps the emit-word staging)
    int n = 0;
    const uint64_t ob0 = Q0 >> 6;
    for (uint64_t ob = ob0; ob <= (Q1 - 1) >> 6; ++ob) {
      uint64_t q = Q0 > (ob << 6) ? Q0 : (ob << 6);
      const uint64_t qe = Q1 < ((ob + 1) << 6) ? Q1 : ((ob + 1) << 6);
      const uint64_t segoff = ((ob - ob0) * (uint64_t)m) << 6;
      auto op = [&](uint32_t kind, uint64_t qq) {
        const uint64_t idx = kind == 0 ? (uint64_t)sR[qq - Qb] : (qq - Qb) >> 2;
        sOps[n++] = (segoff + (qq & 63)) | ((uint64_t)kind << 32) | (idx << 48);
      };
      for (; q < qe && (q & 3); ++q) op(0, q);
      for (; q + 4 <= qe && (q & 15); q += 4) op(1, q);
      if ((q & 31) && q + 16 <= qe) {
        op(2, q);
        q += 16;
      }
      for (; q + 32 <= qe; q += 32) op(3, q);
      if (q + 16 <= qe) {
        op(2, q);
        q += 16;
      }
      for (; q + 4 <= qe; q += 4) op(1, q);
      for (; q < qe; ++q) op(0, q);
    }
    sMisc[2] = (uint32_t)n;
  }
  __syncthreads();
  const uint64_t haskids = (uint64_t)sMisc[0] | ((uint64_t)sMisc[1] << 32);
  [[maybe_unused]] const int nops = prog ? (int)sMisc[2] : 0;  // the store program (SNP_KC_COOP=0)
  if (ES) mbar_wait(bar, 0);

  const T* data = reinterpret_cast<const T*>(L.data);
  T* out = reinterpret_cast<T*>(N.data);
  // this lane's x row: the staging row (xs_stride), or (TCS) row 32·(warp%4) +
  // lane of the warp's A tile, byte r at (r/16)·KCT_A_LBO + r%16
  uint8_t* xsb = TCS ? sX + (warp >> 2) * KCT_ATILE + (((warp & 3) * 32 + lane) >> 3) * 128 + (lane & 7) * 16
                     : sX + (size_t)(warp * 32 + lane) * XS;
  T* xs = reinterpret_cast<T*>(xsb);
  auto xb = [&](int r) -> uint8_t* { return TCS ? xsb + (r >> 4) * KCT_A_LBO + (r & 15) : xsb + r; };
  const T* ctab = reinterpret_cast<const T*>(S.ctab);
  const int j_iters = (m + MWT * 32 - 1) / (MWT * 32);
  uint32_t tph = 0;  // TCS: parity of this warp's tile mbarrier
  for (int it = 0; it < j_iters; ++it) {
    const int32_t jbase = it * MWT * 32 + warp * 32;
    if (TCS ? it * MWT * 32 + (warp & ~3) * 32 >= m : jbase >= m) break;  // warp- (TCS: tile-) uniform
#if SNP_KC_L2PF
    // the warp's 32 rows of the parent block (2 KB contiguous for u8) pulled
    // into L2 while the gather runs, so the row load after it hits L2
    if (sizeof(T) == 1 && lane == 0) {
      const int32_t jp = jbase + (SNP_KC_L2PF - 1) * MWT * 32;
      if (jp < m) {
        const int32_t nr = (m - jp < 32) ? (m - jp) : 32;
        bulk_prefetch_l2(data + eidx(pb0, jp, m), (uint32_t)(nr * PB * sizeof(T)));
      }
    }
#endif
    const int32_t j = jbase + lane;
    if (j < m) {
    const T* row = data + eidx(pb0, j, m);
#if SNP_KC_PREFETCH
    // the first 32 counts of the row are loaded before the gather so their
    // latency overlaps it; the second half is loaded at the top of half 0
    uint32_t vw[8];
    if (sizeof(T) == 1) ldg256(row, vw);
#endif
    // ---- bit-sliced in-synapse count over the 64 parents of the block
    uint64_t c[NPL];
#pragma unroll
    for (int b = 0; b < NPL; ++b) c[b] = 0;
    {
      // edge-major padded in-CSR: row e of the group holds the e-th source
      // of every lane's target (coalesced), padding points at a zero word;
      // rows come in blocks of 8 (Harley-Seal, 7 full adders), a tail of
      // <= 4 rows in one block of 4 (3 full adders)
      const int64_t g = jbase >> 5;
      const int64_t r0 = __ldg(S.in_pad_off + g), r1 = __ldg(S.in_pad_off + g + 1);
      // rows per group are padded to a multiple of 4 (snp_load), so every
      // index load is in bounds; uint16 indices when m < 65535
      const int ne = (int)(r1 - r0);
      auto word = [&](int32_t s) -> uint64_t { return ES ? sE[s] : __ldg(s < mE ? gE + s : &g_zero_word); };
      auto ripple = [&](int b0, uint64_t carry) {
#pragma unroll
        for (int b = 0; b < NPL; ++b) {
          if (b < b0) continue;
          const uint64_t t = c[b] & carry;
          c[b] ^= carry;
          carry = t;
        }
      };
      // the source of row e (0 <= e < ne) of this lane: u16 rows in 4-row
      // packs (one 8-byte load per 4 rows), else one load per row
      auto srcs4 = [&](const auto* col, int e0, int32_t (&src)[4]) {
        if constexpr (std::is_same<std::remove_cv_t<std::remove_pointer_t<decltype(col)>>, uint64_t>::value) {
          const uint64_t q = __ldg(col + (e0 >> 2) * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u) src[u] = (int32_t)((q >> (16 * u)) & 0xFFFFu);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) src[u] = (int32_t)__ldg(col + (e0 + u) * 32);
        }
      };
      auto gather = [&](const auto* col) {
        int e0 = 0;
        for (; e0 + 8 <= ne; e0 += 8) {
          int32_t src[8];
          {  // batch the loads
            int32_t a4[4], b4[4];
            srcs4(col, e0, a4);
            srcs4(col, e0 + 4, b4);
#pragma unroll
            for (int u = 0; u < 4; ++u) { src[u] = a4[u]; src[4 + u] = b4[u]; }
          }
          uint64_t x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = word(src[u]);
          uint64_t twosA, twosB, foursA, foursB, eightsA;
          csa(twosA, c[0], c[0], x[0], x[1]);
          csa(twosB, c[0], c[0], x[2], x[3]);
          csa(foursA, c[1], c[1], twosA, twosB);
          csa(twosA, c[0], c[0], x[4], x[5]);
          csa(twosB, c[0], c[0], x[6], x[7]);
          csa(foursB, c[1], c[1], twosA, twosB);
          csa(eightsA, c[2], c[2], foursA, foursB);
          ripple(3, eightsA);
        }
        if (e0 < ne) {  // 4 rows left
          int32_t src[4];
          srcs4(col, e0, src);
          uint64_t x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = word(src[u]);
          uint64_t twosA, twosB, foursA;
          csa(twosA, c[0], c[0], x[0], x[1]);
          csa(twosB, c[0], c[0], x[2], x[3]);
          csa(foursA, c[1], c[1], twosA, twosB);
          ripple(2, foursA);
        }
      };
      if (SNP_KC_ABLATE & 2) {
      } else if (SNP_KC_IDX4 && S.in_pad16x4) {
        gather(S.in_pad16x4 + (r0 >> 2) * 32 + lane);
      } else if (S.in_pad16) {
        gather(S.in_pad16 + r0 * 32 + lane);
      } else {
        gather(S.in_pad + r0 * 32 + lane);
      }
    }
    // the descriptor is only needed for untabulated neurons and the rare
    // count >= 32 fallback (loaded there)
    NeuronMeta mt{};
    if (S.any_generic || sizeof(T) != 1) mt = S.meta[j];
    const T* crow_g = ctab + (int64_t)j * S.tabw;
    const bool generic = mt.flags & NM_GENERIC;
    uint64_t ovf_bits = 0;
    if ((sizeof(T) == 1 || NARROW) && !generic) {
      // fast path (u8, and NARROW: wide counts < 256 as bytes): the post-consumption table t(v) = v - c_first(v) for
      // v < 32 lives in 8 registers and is looked up 4 parents at a time by
      // byte permutes; the bit-sliced counts become bytes by an 8x8 bit
      // transpose per 8 parents; x = t + count is one 32-bit add per 4 parents
      uint32_t tt[8];
      ldg256(S.ttab + (int64_t)j * 32, tt);
      // counts >= 16 are rare: when no lane of the warp has one, the upper
      // planes are skipped (warp-uniform branch)
      uint64_t up = 0;
#pragma unroll
      for (int b = 4; b < NPL; ++b) up |= c[b];
      const bool upper = __any_sync(__activemask(), up != 0);
      SNP_PRAGMA(unroll SNP_KC_GUNROLL)  // two halves of 32 parents; rolled (1) keeps the hot loop in the instruction cache
      for (int g = 0; g < 2; ++g) {
#if SNP_KC_PREFETCH
        uint32_t vn[8];
        if (g == 0 && np > 32) ldg256(row + 32, vn);
        else
#pragma unroll
          for (int i = 0; i < 8; ++i) vn[i] = 0;
#else
        uint32_t vw[8];
        bool big = false;  // NARROW: a count of this half is >= 256 (or negative)
        if (32 * g >= np) {
#pragma unroll
          for (int i = 0; i < 8; ++i) vw[i] = 0;
        } else if constexpr (sizeof(T) == 1) {
          ldg256(row + 32 * g, vw);
        } else if constexpr (sizeof(T) == 2) {
          // 32 uint16 counts (2 × 32 B): the low bytes, 4 per word
          uint32_t u[8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            ldg256(row + 32 * g + 16 * h, u);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              vw[4 * h + i] = prmt(u[2 * i], u[2 * i + 1], 0x6420u);
              big |= ((u[2 * i] | u[2 * i + 1]) & 0xFF00FF00u) != 0;
            }
          }
        } else {
          // 32 int32 counts (4 × 32 B): the low bytes, 4 per word
          uint32_t u[8];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            ldg256(row + 32 * g + 8 * h, u);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              vw[2 * h + i] = prmt(prmt(u[4 * i], u[4 * i + 1], 0x0040u), prmt(u[4 * i + 2], u[4 * i + 3], 0x0040u),
                                   0x5410u);
              big |= ((u[4 * i] | u[4 * i + 1] | u[4 * i + 2] | u[4 * i + 3]) & 0xFFFFFF00u) != 0;
            }
          }
        }
        if (NARROW && __any_sync(__activemask(), big)) {
          // rare: exact per parent; x is kept as its low byte and every x
          // outside [0, 255] is rewritten exactly by k_overflow_fix
          for (int k = 0; k < 32; ++k) {
            const int r = 32 * g + k;
            const int64_t v = r < np ? (int64_t)row[r] : 0;
            const int32_t cons = (int32_t)crow_g[table_index((uint32_t)v, mt)];
            int32_t cnt = 0;
#pragma unroll
            for (int b = 0; b < NPL; ++b) cnt |= (int32_t)((c[b] >> r) & 1ULL) << b;
            const int64_t x = v - cons + cnt;
            xsb[r] = (uint8_t)x;
            if (x < 0 || x > 255) ovf_bits |= 1ULL << r;
          }
          continue;
        }
#endif
        // t = v - c_first(v) for the 32 counts: byte permutes unless some
        // count >= 32 (rare: that quad folds through the compact table)
        uint32_t t[8], hiv = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) hiv |= vw[i];
        if (__all_sync(__activemask(), (hiv & 0xF0F0F0F0u) == 0)) {  // every count of the warp < 16
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = lut16(vw[i], tt);
        } else if ((hiv & 0xE0E0E0E0u) == 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = lut32(vw[i], tt);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if ((vw[i] & 0xE0E0E0E0u) == 0) {
              t[i] = lut32(vw[i], tt);
            } else {
              t[i] = 0;
#pragma unroll
              for (int b = 0; b < 4; ++b)  // counts >= 32: the neuron's 256-entry row (L2-resident)
                t[i] |= (uint32_t)__ldg(S.ttab + (int64_t)m * 32 + (int64_t)j * 256 + ((vw[i] >> (8 * b)) & 0xFFu))
                        << (8 * b);
            }
          }
        }
        // x = t + count: plain 32-bit adds; a byte can only carry when some
        // operand byte has its top bit set (rare: redo those quads bytewise)
        uint32_t kq[8], chk = 0, xw[8];
        if (upper) {
#pragma unroll
          for (int h = 0; h < 4; ++h) counts8<NPL, NPL>(c, 4 * g + h, kq[2 * h], kq[2 * h + 1]);
        } else {
#pragma unroll
          for (int h = 0; h < 4; ++h) counts8<4, NPL>(c, 4 * g + h, kq[2 * h], kq[2 * h + 1]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) chk |= t[i] | kq[i];
        // a byte can only carry when an operand byte has its top bit set
        // (rare); CARRYU: the test is warp-uniform so the compiler keeps the
        // careful path as a real branch instead of predicating it into every
        // quad (the careful form is exact for every lane)
        const bool carry = (chk & 0x80808080u) != 0;
        if (SNP_KC_CARRYU ? __any_sync(__activemask(), carry) : carry) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t t4 = t[i], k4 = kq[i];
            const uint32_t s7 = (t4 & 0x7F7F7F7Fu) + (k4 & 0x7F7F7F7Fu);
            const uint32_t co = ((t4 & k4) | ((t4 | k4) & s7)) & 0x80808080u;
            const uint32_t x4 = s7 ^ ((t4 ^ k4) & 0x80808080u);
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if ((co >> (8 * b + 7)) & 1u) ovf_bits |= 1ULL << (32 * g + 4 * i + b);
            if (TCS) xw[i] = x4;
            else reinterpret_cast<uint32_t*>(xsb)[8 * g + i] = x4;
          }
        } else if (!TCS && SNP_KC_XS72) {  // 8-aligned rows: x as 64-bit words
#pragma unroll
          for (int i = 0; i < 8; i += 2)
            reinterpret_cast<uint2*>(xsb)[4 * g + i / 2] = make_uint2(t[i] + kq[i], t[i + 1] + kq[i + 1]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t x4 = t[i] + kq[i];
            if (TCS) xw[i] = x4;
            else reinterpret_cast<uint32_t*>(xsb)[8 * g + i] = x4;
          }
        }
        if (TCS) {  // parents 32g .. 32g+31 = K-chunks 2g, 2g+1 of the A row
          *reinterpret_cast<uint4*>(xsb + (2 * g) * KCT_A_LBO) = make_uint4(xw[0], xw[1], xw[2], xw[3]);
          *reinterpret_cast<uint4*>(xsb + (2 * g + 1) * KCT_A_LBO) = make_uint4(xw[4], xw[5], xw[6], xw[7]);
        }
#if SNP_KC_PREFETCH
#pragma unroll
        for (int i = 0; i < 8; ++i) vw[i] = vn[i];
#endif
      }
    } else if (sizeof(T) == 4 && !generic) {
      // int32 counts: the row in 16-byte loads, 16 parents at a time
      for (int r0 = 0; r0 < PB; r0 += 16) {
        int32_t vv[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int4 q4 = r0 + 4 * k < np ? __ldg(reinterpret_cast<const int4*>(row) + (r0 >> 2) + k) : make_int4(0, 0, 0, 0);
          vv[4 * k] = q4.x;
          vv[4 * k + 1] = q4.y;
          vv[4 * k + 2] = q4.z;
          vv[4 * k + 3] = q4.w;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int r = r0 + k;
          const int32_t v = r < np ? vv[k] : 0;
          const int32_t cons = (int32_t)crow_g[table_index((uint32_t)v, mt)];
          int32_t cnt = 0;
#pragma unroll
          for (int b = 0; b < NPL; ++b) cnt |= (int32_t)((c[b] >> r) & 1ULL) << b;
          const int64_t x = (int64_t)v - cons + cnt;
          if (x > S.count_max) ovf_bits |= 1ULL << r;
          if (TCS) *xb(r) = (uint8_t)x;
          else xs[r] = (T)x;
        }
      }
    } else {
      for (int r = 0; r < PB; ++r) {
        const int32_t v = (r < np) ? (int32_t)row[r] : 0;
        int32_t cons;
        if (generic) {
          const int rf = nth_applicable(S, j, v, 0);
          cons = rf >= 0 ? S.rules[rf].c : 0;
        } else {
          cons = (int32_t)crow_g[table_index((uint32_t)v, mt)];
        }
        int32_t cnt = 0;
#pragma unroll
        for (int b = 0; b < NPL; ++b) cnt |= (int32_t)((c[b] >> r) & 1ULL) << b;
        const int64_t x = (int64_t)v - cons + cnt;
        if (x > S.count_max) ovf_bits |= 1ULL << r;
        if (TCS) *xb(r) = (uint8_t)x;
        else xs[r] = (T)x;
      }
    }
    ovf_bits &= haskids;
    while (ovf_bits) {  // rare: base value beyond the storage range
      const int r = __ffsll((long long)ovf_bits) - 1;
      ovf_bits &= ovf_bits - 1;
      unsigned long long slot = atomicAdd(n_ovf, 1ULL);
      if (slot < ovf_cap) ovf[slot] = ((uint64_t)(uint32_t)j << 32) | (uint64_t)(pb0 + r);
    }
    // ---- write x to every kept child of the block's parents (row j of the output)
#if SNP_KC_COOP
    if (prog) {
      // bytes of [Q0, Q1) whose 4-child quad is not inside the range (<= 3
      // at each end): lane = row, one byte store per position for all rows
      uint8_t* orow = reinterpret_cast<uint8_t*>(out);
      const uint64_t qa = (Q0 + 3) & ~3ULL, qb = Q1 & ~3ULL;  // full quads: [qa, qb)
#if SNP_KC_EDGE
      // each end is <= 3 contiguous bytes of one quad of row j: assembled in
      // a register and written by <= 2 aligned stores (a byte, a halfword)
      // instead of one byte store per child
      auto edge = [&](uint64_t q0, uint64_t q1) {
        if (q0 >= q1) return;
        if constexpr (sizeof(T) > 1) {  // NARROW: <= 3 wide values
          for (uint64_t q = q0; q < q1; ++q) out[eidx((int64_t)q, j, m)] = (T)xsb[sR[q - Qb]];
          return;
        }
        uint32_t v = 0;
        const uint32_t dq = sD[(q0 - Qb) >> 2];  // the partial quad's permute (SNP_KC_EDGEPRMT)
        if (SNP_KC_EDGEPRMT && !(dq & 0x80000000u)) {
          const uint32_t* w = reinterpret_cast<const uint32_t*>(xsb) + ((dq >> 16) & 31);
          const uint32_t sel = dq & 0xFFFFu, hb = dq >> 24;
          v = prmt(w[0], w[1], sel);
          if (hb) {
            const uint32_t mask = (hb * 0x00204081u & 0x01010101u) * 0xFFu;
            v = (v & ~mask) | (prmt(w[2], w[3], sel) & mask);
          }
          v >>= 8 * (uint32_t)(q0 & 3);
        } else {
          for (uint64_t q = q0; q < q1; ++q) v |= (uint32_t)xsb[sR[q - Qb]] << (8 * (q - q0));
        }
        uint8_t* d = orow + eidx((int64_t)q0, j, m);
        int n = (int)(q1 - q0);
        if ((q0 & 1) && n) {
          *d = (uint8_t)v;
          v >>= 8; ++d; --n;
        }
        if (n >= 2) {
          *reinterpret_cast<uint16_t*>(d) = (uint16_t)v;
          v >>= 16; d += 2; n -= 2;
        }
        if (n) *d = (uint8_t)v;
      };
      edge(Q0, Q1 < qa ? Q1 : qa);
      edge(qb > qa ? qb : qa, Q1);
#else
      for (uint64_t q = Q0; q < Q1 && q < qa; ++q) orow[eidx((int64_t)q, j, m)] = xsb[sR[q - Qb]];
      for (uint64_t q = (qb > qa ? qb : qa); q < Q1; ++q) orow[eidx((int64_t)q, j, m)] = xsb[sR[q - Qb]];
#endif
    } else
#else
    if (prog) {
      uint8_t* obase = reinterpret_cast<uint8_t*>(out) + (((int64_t)(Q0 >> 6) * m + j) << 6);
      const uint32_t* xw = reinterpret_cast<const uint32_t*>(xsb);
      auto quad = [&](uint32_t d, uint32_t qi) -> uint32_t {
        if (!(d & 0x80000000u)) {
          const uint32_t* w = xw + ((d >> 16) & 31);
          const uint32_t sel = d & 0xFFFFu, hb = d >> 24;
          const uint32_t lo = prmt(w[0], w[1], sel);
          if (!hb) return lo;
          const uint32_t mask = (hb * 0x00204081u & 0x01010101u) * 0xFFu;  // 0xFF in bytes k with bit k of hb
          return (lo & ~mask) | (prmt(w[2], w[3], sel) & mask);
        }
        const uint32_t rr = *reinterpret_cast<const uint32_t*>(sR + 4 * qi);  // 4 parent indices
        return (uint32_t)xsb[rr & 0xFF] | ((uint32_t)xsb[(rr >> 8) & 0xFF] << 8) |
               ((uint32_t)xsb[(rr >> 16) & 0xFF] << 16) | ((uint32_t)xsb[rr >> 24] << 24);
      };
      for (int i = 0; i < ((SNP_KC_ABLATE & 1) ? 0 : nops); ++i) {
        const uint64_t op = sOps[i];
        uint8_t* dst = obase + (uint32_t)op;
        const uint32_t hi = (uint32_t)(op >> 32), kind = hi & 3u, qi = hi >> 16;
        if (kind == 3u) {
          const uint4 d0 = *reinterpret_cast<const uint4*>(sD + qi);
          const uint4 d1 = *reinterpret_cast<const uint4*>(sD + qi + 4);
          uint32_t w[8];
          w[0] = quad(d0.x, qi);
          w[1] = quad(d0.y, qi + 1);
          w[2] = quad(d0.z, qi + 2);
          w[3] = quad(d0.w, qi + 3);
          w[4] = quad(d1.x, qi + 4);
          w[5] = quad(d1.y, qi + 5);
          w[6] = quad(d1.z, qi + 6);
          w[7] = quad(d1.w, qi + 7);
          stg256(dst, w);
        } else if (kind == 2u) {
          const uint4 d0 = *reinterpret_cast<const uint4*>(sD + qi);
          *reinterpret_cast<uint4*>(dst) =
              make_uint4(quad(d0.x, qi), quad(d0.y, qi + 1), quad(d0.z, qi + 2), quad(d0.w, qi + 3));
        } else if (kind == 1u) {
          *reinterpret_cast<uint32_t*>(dst) = quad(sD[qi], qi);
        } else {
          *dst = xsb[qi];
        }
      }
    } else
#endif
    if (TCS) {
      if (!tcp) {  // window > 8 sectors (rare): one byte store per (row, child)
        if (nq <= QCAP) {
          for (uint64_t q = Q0; q < Q1; ++q) out[eidx((int64_t)q, j, m)] = *xb(sR[q - Qb]);
        } else {
          for (int r = 0; r < np; ++r)
            for (uint64_t q = sQ[r]; q < sQ[r + 1]; ++q) out[eidx((int64_t)q, j, m)] = *xb(r);
        }
      }
    } else if (nq <= QCAP) {
      if (!(SNP_KC_WIDE_COOP && sizeof(T) > 1))  // wide counts: the warp-cooperative rows below
        for (uint64_t q = Q0; q < Q1; ++q) out[eidx((int64_t)q, j, m)] = xs[sR[q - Qb]];
    } else {
      for (int r = 0; r < np; ++r)
        for (uint64_t q = sQ[r]; q < sQ[r + 1]; ++q) out[eidx((int64_t)q, j, m)] = NARROW ? (T)xsb[r] : xs[r];
    }
    }  // j < m
    if constexpr (TCS) {
      if (tcp) {
        // the tile's 128 rows are in its A tile: D = X·P on the tensor cores
        // (KCT_ATILE), then every lane writes whole sectors of its row
        const int t = warp >> 2, wq = warp & 3;
        const uint32_t tmem = sMisc[3] + ((uint32_t)(32 * wq) << 16) + 64u * t;
        uint8_t* sA = sX + t * KCT_ATILE;
        const uint8_t* sB = sX + (size_t)MWT / 4 * KCT_ATILE;
        tc::fence_async_smem();  // this thread's A row → the async proxy
        for (int rd = 0; 4 * rd < nsec; ++rd) {
          tc::fence_before();  // the previous round's TMEM loads are complete (wait_ld)
          tc::named_sync(1 + t, 128);
          if (wq == 0 && lane == 0) {
            tc::fence_after();
            const int ns = nsec - 4 * rd < 4 ? nsec - 4 * rd : 4;
            const uint32_t idesc = tc::idesc_u8(128, 16 * ns, false, false);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int ks = 0; ks < 2; ++ks)
                tc::mma_u8(sMisc[3] + 64u * t, tc::sdesc(tc::smem_u32(sA + ks * 2 * KCT_A_LBO), KCT_A_LBO, 128),
                           tc::sdesc(tc::smem_u32(sB + (2 * rd + h) * KCT_BHALF + ks * 2 * KCT_B_LBO), KCT_B_LBO, 128),
                           idesc, (h | ks) ? 1u : 0u);
            tc::commit(&tbar[t]);
          }
          tc::bar_wait(&tbar[t], tph);
          tph ^= 1;
          tc::fence_after();
          for (int sl = 0; sl < 4 && 4 * rd + sl < nsec; ++sl) {
            uint32_t v[16];
            tc::tmem_ld16_nw(tmem + 16u * sl, v);
            tc::wait_ld();
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = prmt(v[2 * i], v[2 * i + 1], 0x5410u);
            const int32_t jj = jbase + lane;
            if (jbase < m && jj < m) {
              const uint64_t q = Qb + 32 * (uint64_t)(4 * rd + sl);
              uint8_t* dst = reinterpret_cast<uint8_t*>(out) + ((((int64_t)(q >> 6) * m + jj) << 6) | (int64_t)(q & 63));
              const int lo = Q0 > q ? (int)(Q0 - q) : 0;
              const int hi = Q1 < q + 32 ? (int)(Q1 - q) : 32;
              if (lo == 0 && hi == 32) {
                stg256(dst, w);
              } else {
                // partial sector at a window end (warp-uniform bounds): the
                // widest aligned pieces inside [lo, hi)
#pragma unroll
                for (int h16 = 0; h16 < 2; ++h16) {
                  if (lo <= 16 * h16 && 16 * h16 + 16 <= hi) {
                    *reinterpret_cast<uint4*>(dst + 16 * h16) =
                        make_uint4(w[4 * h16], w[4 * h16 + 1], w[4 * h16 + 2], w[4 * h16 + 3]);
                    continue;
                  }
#pragma unroll
                  for (int h8 = 0; h8 < 2; ++h8) {
                    const int b8 = 16 * h16 + 8 * h8;
                    if (lo <= b8 && b8 + 8 <= hi) {
                      *reinterpret_cast<uint2*>(dst + b8) = make_uint2(w[b8 >> 2], w[(b8 >> 2) + 1]);
                      continue;
                    }
#pragma unroll
                    for (int h4 = 0; h4 < 2; ++h4) {
                      const int b4 = b8 + 4 * h4;
                      const uint32_t x = w[b4 >> 2];
                      if (lo <= b4 && b4 + 4 <= hi) {
                        *reinterpret_cast<uint32_t*>(dst + b4) = x;
                      } else if (lo < b4 + 4 && hi > b4) {
                        for (int b = (lo > b4 ? lo : b4); b < (hi < b4 + 4 ? hi : b4 + 4); ++b)
                          dst[b] = (uint8_t)(x >> (8 * (b - b4)));
                      }
                    }
                  }
                }
              }
            }
          }
        }
      }
    }
#if SNP_KC_WIDE_COOP
    if (sizeof(T) > 1 && !prog && nq <= QCAP) {
      // 16/32-bit counts: the warp writes its rows one at a time, lane = child,
      // so each store instruction fills 32 consecutive children of one row
      __syncwarp();
      const int32_t jn = m - jbase;
      for (int r = 0; r < 32 && r < jn; ++r) {
        const uint8_t* xr = sX + (size_t)(warp * 32 + r) * XS;
        for (uint64_t q = Q0 + lane; q < Q1; q += 32)
          out[eidx((int64_t)q, jbase + r, m)] = NARROW ? (T)xr[sR[q - Qb]] : reinterpret_cast<const T*>(xr)[sR[q - Qb]];
      }
      __syncwarp();
    }
#endif
#if SNP_KC_COOP
    if (prog) {
      // full 4-child quads, warp-cooperative: a half-warp covers one 64-child
      // output row (lane = quad; a byte permute of the neuron's x row when
      // the 4 parents lie in a 16-byte window, else 4 byte loads), so each
      // 4-byte store instruction of the warp fills 128 contiguous bytes (4
      // whole sectors) instead of touching 32 rows
      __syncwarp();
      const int hl = lane & 15, j0 = lane >> 4;
      const int32_t jn = m - jbase;  // rows of this warp that exist
      // 4 children's values (bytes of v) as T (NARROW: zero-extended)
      auto put4 = [](uint8_t* d, uint32_t v) {
        if constexpr (sizeof(T) == 1) *reinterpret_cast<uint32_t*>(d) = v;
        else if constexpr (sizeof(T) == 2) *reinterpret_cast<uint2*>(d) = make_uint2(prmt(v, 0u, 0x4140u), prmt(v, 0u, 0x4342u));
        else *reinterpret_cast<uint4*>(d) = make_uint4(prmt(v, 0u, 0x4440u), prmt(v, 0u, 0x4441u), prmt(v, 0u, 0x4442u),
                                                       prmt(v, 0u, 0x4443u));
      };
      const uint8_t* xr0 = sX + (size_t)(warp * 32 + j0) * XS;
      const uint64_t qa = (Q0 + 3) & ~3ULL, qb = Q1 & ~3ULL;
#if SNP_KC_FLATQ
      // passes over the CTA's own full quads [qa, qb), 16 per pass (lane
      // hl takes quad qa + 4·(16·pass + hl), whichever output block it is
      // in): one pass when the CTA has <= 16 full quads
      // (SNP_KC_TAILQ: whole passes only; the last < 16 quads below)
      const uint64_t qpass = (SNP_KC_TAILQ && qa < qb) ? qa + ((qb - qa) & ~(uint64_t)63) : qb;
      for (uint64_t q0 = qa; !(SNP_KC_ABLATE & 4) && q0 < qpass; q0 += 64) {
        const uint64_t q = q0 + 4 * hl;
        if (q < qb) {
          const uint64_t ob = q >> 6;
          const uint32_t d = sD[(q - Qb) >> 2];
          uint8_t* dst0 = reinterpret_cast<uint8_t*>(out + ((((int64_t)ob * m + jbase + j0) << 6) + (q & 63)));
#else
      for (uint64_t ob = qa >> 6; !(SNP_KC_ABLATE & 4) && qa < qb && ob <= (qb - 1) >> 6; ++ob) {
        const uint64_t q = (ob << 6) + 4 * hl;
        if (q >= qa && q < qb) {
          const uint32_t d = sD[(q - Qb) >> 2];
          uint8_t* dst0 = reinterpret_cast<uint8_t*>(out + ((((int64_t)ob * m + jbase + j0) << 6) + 4 * hl));
#endif
          if (!(d & 0x80000000u)) {
            const uint32_t* w0 = reinterpret_cast<const uint32_t*>(xr0) + ((d >> 16) & 31);
            const uint32_t sel = d & 0xFFFFu, hb = d >> 24;
            const uint32_t mask = (hb * 0x00204081u & 0x01010101u) * 0xFFu;  // 0xFF in bytes k with bit k of hb
            // FULL: every row of the warp exists (warp-uniform), no per-store predicate
            auto rows = [&](auto full_c) {
              constexpr bool FULL = decltype(full_c)::value;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(w0) +
                                                                      2 * i * XS);
                uint32_t v = prmt(w[0], w[1], sel);
#if SNP_KC_BRANCHLESS
                v = (v & ~mask) | (prmt(w[2], w[3], sel) & mask);  // mask = 0 when hb = 0 (words past the row are masked out)
#else
                if (hb) v = (v & ~mask) | (prmt(w[2], w[3], sel) & mask);
#endif
                if (FULL || j0 + 2 * i < jn) put4(dst0 + i * 128 * (int)sizeof(T), v);
              }
            };
            if (SNP_KC_FULLROWS && jn >= 32) rows(std::true_type{});
            else rows(std::false_type{});
          } else {
            const uint32_t rr = *reinterpret_cast<const uint32_t*>(sR + (q - Qb));  // 4 parent indices
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
              const uint8_t* xr = xr0 + 2 * i * XS;
              const uint32_t v = (uint32_t)xr[rr & 0xFF] | ((uint32_t)xr[(rr >> 8) & 0xFF] << 8) |
                                 ((uint32_t)xr[(rr >> 16) & 0xFF] << 16) | ((uint32_t)xr[rr >> 24] << 24);
              if (j0 + 2 * i < jn) put4(dst0 + i * 128 * (int)sizeof(T), v);
            }
          }
        }
      }
#if SNP_KC_FLATQ && SNP_KC_TAILQ
      // the last nrem < 16 quads: lpr = nrem rounded up to a power of two
      // lanes per row, 32 / lpr rows per step, so a 2-quad tail takes 2 steps
      // instead of a 16-step pass with 14 idle lanes per half-warp
      if (!(SNP_KC_ABLATE & 4) && qpass < qb) {
        const int nrem = (int)((qb - qpass) >> 2);
        const int lpr = nrem <= 1 ? 1 : nrem <= 2 ? 2 : nrem <= 4 ? 4 : nrem <= 8 ? 8 : 16;
        const int rps = 32 / lpr, qi = lane & (lpr - 1), ro = lane / lpr;
        if (qi < nrem) {
          const uint64_t q = qpass + 4 * (uint64_t)qi;
          const uint64_t ob = q >> 6;
          const uint32_t d = sD[(q - Qb) >> 2];
          const uint32_t rr = *reinterpret_cast<const uint32_t*>(sR + (q - Qb));  // 4 parent indices
          const uint32_t sel = d & 0xFFFFu, hb = d >> 24;
          const uint32_t mask = (hb * 0x00204081u & 0x01010101u) * 0xFFu;
          for (int jr = ro; jr < 32 && jr < jn; jr += rps) {
            const uint8_t* xr = sX + (size_t)(warp * 32 + jr) * XS;
            uint32_t v;
            if (!(d & 0x80000000u)) {
              const uint32_t* w = reinterpret_cast<const uint32_t*>(xr) + ((d >> 16) & 31);
              v = prmt(w[0], w[1], sel);
              if (hb) v = (v & ~mask) | (prmt(w[2], w[3], sel) & mask);
            } else {
              v = (uint32_t)xr[rr & 0xFF] | ((uint32_t)xr[(rr >> 8) & 0xFF] << 8) |
                  ((uint32_t)xr[(rr >> 16) & 0xFF] << 16) | ((uint32_t)xr[rr >> 24] << 24);
            }
            put4(reinterpret_cast<uint8_t*>(out + ((((int64_t)ob * m + jbase + jr) << 6) + (q & 63))), v);
          }
        }
      }
#endif
      __syncwarp();
    }
#endif
  }
  if constexpr (TCS) {
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(sMisc[3], 512);
  }
}
// K-c (generic): every (kept child, neuron) computed exactly.
template <typename T>
__global__ void k_materialize_exact(SysView S, LevelView L, ExpandOut O, NextArrays N, int64_t K, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  T* out = reinterpret_cast<T*>(N.data);
  for (int64_t q = warp; q < K; q += nwarps) {
    const int64_t p = N.parent[q];
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], N.t[q], cx);
    bool bad = false;
    for (int32_t j = lane; j < S.m; j += 32) {
      const int64_t val = exact_value<T>(S, L.data, p, j, cx);
      bad |= (val < 0 || val > S.count_max);
      out[eidx(q, j, S.m)] = (T)val;
    }
    if (bad) atomicOr(err, ERR_OVERFLOW);
  }
}

// Correction of every (neuron, child) touched by a non-first ND choice: the
// ND neuron itself (consumption) and its out-neighbours (emission), by the
// linear delta of eq. (2) on K-c's base values.
template <typename T>
__global__ void k_patch(SysView S, LevelView L, ExpandOut O, NextArrays N, int64_t K, int32_t* err) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = N.parent[q];
    const uint64_t t = N.t[q];
    if (t == 0) continue;  // all digits 0: the base child
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], t, cx);
    T* out = reinterpret_cast<T*>(N.data);
    // eq. (2) is linear in S: child = base child + Σ_{ND s, x_s ≠ 0}
    // (M[chosen_s] − M[first_s]), i.e. −(c_chosen − c_first) at s and
    // +(p_chosen − p_first) at every out-neighbour of s, applied to the base
    // values K-c wrote (a base value outside the storage range is rewritten
    // exactly afterwards by k_overflow_fix)
    for (int i = 0; i < cx.K; ++i) {
      if (!cx.x[i]) continue;
      const int32_t s = cx.s[i];
      const int32_t v = (int32_t)(uint32_t)O.nd[p * KMAX + i];
      const DevRule& rf = S.rules[nth_applicable(S, s, v, 0)];
      const DevRule& rc = S.rules[nth_applicable(S, s, v, cx.x[i])];
      const int64_t dc = (int64_t)rc.c - rf.c, dp = (int64_t)rc.p - rf.p;
      for (int e = -1; e < S.out_off[s + 1] - S.out_off[s]; ++e) {
        const int32_t j = e < 0 ? s : S.out_dst[S.out_off[s] + e];
        const int64_t d = e < 0 ? -dc : dp;
        if (!d) continue;
        T* o = out + eidx(q, j, S.m);
        int64_t val = (int64_t)*o + d;
        if (val < 0 || val > S.count_max) {  // rare: recompute exactly (the base may have wrapped)
          val = exact_value<T>(S, L.data, p, j, cx);
          if (val < 0 || val > S.count_max) atomicOr(err, ERR_OVERFLOW);
        }
        *o = (T)val;
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
      const int64_t val = exact_value<T>(S, L.data, p, j, cx);
      if (val < 0 || val > S.count_max) atomicOr(err, ERR_OVERFLOW);
      else out[eidx((int64_t)q, j, S.m)] = (T)val;
    }
  }
}

// first applicable rule of neuron s at count v (tables when tabulated)
__device__ __forceinline__ int first_rule(const SysView& S, int32_t s, int32_t v) {
  if (S.tables_ok) {
    const NeuronMeta mt = S.meta[s];
    if (!(mt.flags & NM_GENERIC)) {
      const uint32_t e = S.full8 ? S.tab_full[(int64_t)s * 256 + ((uint32_t)v & 0xFFu)]
                                 : S.tab[(int64_t)s * S.tabw + table_index((uint32_t)v, mt)];
      return (e >> 4) ? mt.rbase + (int)(e >> 4) - 1 : -1;
    }
  }
  return nth_applicable(S, s, v, 0);
}

// The fired rule's (c, p) of every neuron of one child into a warp's
// shared-memory slice: first applicable rules, then the ND digits of cx.
template <typename T>
__device__ void fired_cp(const SysView& S, const void* data, int64_t p, const ChildCtx& cx, int2* fc, int lane,
                         int32_t* cnt = nullptr) {
  for (int32_t s = lane; s < S.m; s += 32) {
    const int32_t v = ld_count<T>(data, p, s, S.m);
    if (cnt) cnt[s] = v;
    const int r = first_rule(S, s, v);
    fc[s] = r >= 0 ? make_int2(S.rules[r].c, S.rules[r].p) : make_int2(0, 0);
  }
  __syncwarp();
  for (int i = lane; i < cx.K; i += 32) {
    if (!cx.x[i]) continue;
    const int32_t s = cx.s[i];
    const int r = nth_applicable(S, s, ld_count<T>(data, p, s, S.m), cx.x[i]);
    fc[s] = make_int2(S.rules[r].c, S.rules[r].p);
  }
  __syncwarp();
}

// the same with (c, p) packed as c | p << 8 (every rule has c, p <= 255):
// 2 bytes per neuron instead of 8, so 4x the verification warps fit an SM
template <typename T>
__device__ void fired_cp(const SysView& S, const void* data, int64_t p, const ChildCtx& cx, uint16_t* fc, int lane,
                         int32_t* cnt = nullptr) {
  for (int32_t s = lane; s < S.m; s += 32) {
    const int32_t v = ld_count<T>(data, p, s, S.m);
    if (cnt) cnt[s] = v;
    const int r = first_rule(S, s, v);
    fc[s] = r >= 0 ? (uint16_t)(S.rules[r].c | (S.rules[r].p << 8)) : (uint16_t)0;
  }
  __syncwarp();
  for (int i = lane; i < cx.K; i += 32) {
    if (!cx.x[i]) continue;
    const int32_t s = cx.s[i];
    const int r = nth_applicable(S, s, ld_count<T>(data, p, s, S.m), cx.x[i]);
    fc[s] = (uint16_t)(S.rules[r].c | (S.rules[r].p << 8));
  }
  __syncwarp();
}
__device__ __forceinline__ int32_t fc_c(int2 v) { return v.x; }
__device__ __forceinline__ int32_t fc_p(int2 v) { return v.y; }
__device__ __forceinline__ int32_t fc_c(uint16_t v) { return v & 0xFF; }
__device__ __forceinline__ int32_t fc_p(uint16_t v) { return v >> 8; }

// column j of that child: eq. (2) restricted to column j (Def. 2)
template <typename T, typename FC>
__device__ __forceinline__ int64_t fired_value(const SysView& S, const void* data, int64_t p, int32_t j,
                                               const ChildCtx& cx, const FC* fc) {
  if (S.aug_rule >= 0 && j == S.m - 1) return exact_value<T>(S, data, p, j, cx);
  int64_t val = (int64_t)ld_count<T>(data, p, j, S.m) - fc_c(fc[j]);
  for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) val += fc_p(fc[S.in_src[e]]);
  return val;
}

// K-c (generic) with the fired (c, p) of each child in shared memory
template <typename T>
__global__ void __launch_bounds__(256) k_materialize_exact_s(SysView S, LevelView L, ExpandOut O, NextArrays N,
                                                             int64_t K, int32_t* err) {
  extern __shared__ int2 msm[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  int2* fc = msm + (size_t)wl * S.m;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  T* out = reinterpret_cast<T*>(N.data);
  for (int64_t q = warp; q < K; q += nwarps) {
    const int64_t p = N.parent[q];
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], N.t[q], cx);
    fired_cp<T>(S, L.data, p, cx, fc, lane);
    bool bad = false;
    for (int32_t j = lane; j < S.m; j += 32) {
      const int64_t val = fired_value<T>(S, L.data, p, j, cx, fc);
      bad |= (val < 0 || val > S.count_max);
      out[eidx(q, j, S.m)] = (T)val;
    }
    if (bad) atomicOr(err, ERR_OVERFLOW);
    __syncwarp();
  }
}

constexpr int VERIFY_WARPS = 8;
size_t verify_smem_bytes(int32_t m, size_t entry = 8) { return (size_t)VERIFY_WARPS * 2 * entry * (size_t)m; }

// the children whose key matched another configuration (seen at an earlier
// level, or a same-level duplicate that lost to the minimum tag): appended to
// `list` (order irrelevant: each is only compared), so the verification warps
// touch ~2 % of the transitions instead of scanning them all
__global__ void k_verify_need(ChildArrays C, uint64_t T_, uint64_t tag_base, Tables tb, uint64_t* list,
                              unsigned long long* n_list) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < T_; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t vd = C.verdict[c];
    const bool need = vd == 1 ? tb.ltab[C.cslot[c]].tag != tag_base + c : C.cref[c] != EMPTY;
    if (need) list[atomicAdd(n_list, 1ULL)] = c;
  }
}

// k_verify with the fired (c, p) of both children in shared memory, over
// the list k_verify_need built
template <typename T, typename FC>
__global__ void __launch_bounds__(VERIFY_WARPS * 32) k_verify_s(SysView S, LevelView L, ExpandOut O,
                                                                const uint64_t* off, ChildArrays C,
                                                                const uint64_t* list, const unsigned long long* n_list,
                                                                uint64_t tag_base, Tables tb,
                                                                const StoredLevel* stored, int32_t* err) {
  extern __shared__ __align__(16) uint8_t vsm_raw[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  FC* fa = reinterpret_cast<FC*>(vsm_raw) + (size_t)wl * 2 * S.m;
  FC* fb = fa + S.m;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nl = *n_list;
  for (uint64_t i = warp; i < nl; i += nwarps) {
    const uint64_t c = list[i];
    const uint8_t vd = C.verdict[c];
    uint64_t other = EMPTY;
    if (vd == 1) other = tb.ltab[C.cslot[c]].tag - tag_base;
    const uint32_t p = C.cpar[c];
    ChildCtx cx, co;
    decode_child(S, O.nd + (uint64_t)p * KMAX, O.ndc[p], c - off[p], cx);
    fired_cp<T>(S, L.data, p, cx, fa, lane);
    uint32_t po = 0;
    if (vd == 1) {
      po = C.cpar[other];
      decode_child(S, O.nd + (uint64_t)po * KMAX, O.ndc[po], other - off[po], co);
      fired_cp<T>(S, L.data, po, co, fb, lane);
    }
    bool diff = false;
    for (int32_t j = lane; j < S.m; j += 32) {
      const int64_t a = fired_value<T>(S, L.data, p, j, cx, fa);
      int64_t b;
      if (vd == 1) {
        b = fired_value<T>(S, L.data, po, j, co, fb);
      } else {
        const uint64_t ref = C.cref[c];
        b = ld_count<T>(stored[ref >> 40].data, (int64_t)(ref & ((1ULL << 40) - 1)), j, S.m);
      }
      diff |= (a != b);
    }
    if (__any_sync(0xFFFFFFFFu, diff) && lane == 0) atomicOr(err, ERR_COLLISION);
    __syncwarp();
  }
}

// dedup = 0, two fully parallel passes over a batch of the listed key
// matches: (1) a warp per match writes the fired (c, p) of every neuron of
// the child (and, for a same-level duplicate, of its key's winner) to global
// rows; (2) a thread per (match, column) rebuilds the column of eq. (2) from
// them and compares it with the other row (the winner's, or the stored
// configuration of an earlier level).  A mismatch is a 128-bit collision.
// batch row i: 2m fired (c, p) entries (child, other child), then 2m counts
// of their parents (row-major, so the column pass reads them coalesced
// instead of one sector per count from the block layout)
template <typename FC>
__device__ __forceinline__ FC* vrow_fc(uint8_t* base, uint64_t i, int32_t m) {
  return reinterpret_cast<FC*>(base + i * (2 * (uint64_t)m * (sizeof(FC) + 4)));
}
template <typename FC>
__device__ __forceinline__ int32_t* vrow_cnt(uint8_t* base, uint64_t i, int32_t m) {
  return reinterpret_cast<int32_t*>(base + i * (2 * (uint64_t)m * (sizeof(FC) + 4)) + 2 * (uint64_t)m * sizeof(FC));
}

template <typename T, typename FC>
__global__ void k_verify_fc(SysView S, LevelView L, ExpandOut O, const uint64_t* off, ChildArrays C,
                            const uint64_t* list, uint64_t i0, uint64_t n, uint64_t tag_base, Tables tb, uint8_t* fcg) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = warp; i < n; i += nwarps) {
    const uint64_t c = list[i0 + i];
    FC* fa = vrow_fc<FC>(fcg, i, S.m);
    int32_t* ca = vrow_cnt<FC>(fcg, i, S.m);
    const uint32_t p = C.cpar[c];
    ChildCtx cx;
    decode_child(S, O.nd + (uint64_t)p * KMAX, O.ndc[p], c - off[p], cx);
    fired_cp<T>(S, L.data, p, cx, fa, lane, ca);
    if (C.verdict[c] == 1) {
      const uint64_t o = tb.ltab[C.cslot[c]].tag - tag_base;
      const uint32_t po = C.cpar[o];
      ChildCtx co;
      decode_child(S, O.nd + (uint64_t)po * KMAX, O.ndc[po], o - off[po], co);
      fired_cp<T>(S, L.data, po, co, fa + S.m, lane, ca + S.m);
    }
  }
}

template <typename T, typename FC>
__global__ void k_verify_cols(SysView S, LevelView L, ChildArrays C, const uint64_t* list, uint64_t i0, uint64_t n,
                              uint64_t tag_base, Tables tb, uint8_t* fcg, const StoredLevel* stored, int32_t* err) {
  for (uint64_t i = blockIdx.y; i < n; i += gridDim.y) {
    const uint64_t c = list[i0 + i];
    const uint8_t vd = C.verdict[c];
    const FC* fa = vrow_fc<FC>(fcg, i, S.m);
    const int32_t* ca = vrow_cnt<FC>(fcg, i, S.m);
    const uint64_t ref = vd == 1 ? 0 : C.cref[c];
    bool diff = false;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < S.m; j += gridDim.x * blockDim.x) {
      int64_t a = (int64_t)ca[j] - fc_c(fa[j]);
      for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) a += fc_p(fa[S.in_src[e]]);
      int64_t b;
      if (vd == 1) {
        const FC* fb = fa + S.m;
        b = (int64_t)ca[S.m + j] - fc_c(fb[j]);
        for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) b += fc_p(fb[S.in_src[e]]);
      } else {
        b = ld_count<T>(stored[ref >> 40].data, (int64_t)(ref & ((1ULL << 40) - 1)), j, S.m);
      }
      diff |= a != b;
    }
    if (diff) atomicOr(err, ERR_COLLISION);
  }
}

// dedup = 0, one CTA per listed key match (grid-stride): both children's
// parent counts and fired (c, p) of every neuron into shared memory (the
// counts come from the block layout, one sector each: the floor of this
// pass), the ND digits decoded once, then a warp per 32 columns compares eq.
// (2) for both — as the difference (C_a - c_a) - (C_b - c_b) + Σ_in (p_a - p_b)
// — or against the stored configuration of an earlier level.  The in-synapse
// walk uses K-c's padded, bank-coloured in-CSR rows (one coalesced index load
// per row, padding reads a zero entry).  PK: every rule has c, p <= 255, so a
// neuron's (c_a, p_a, c_b, p_b) is one 32-bit word.  A mismatch is a 128-bit
// collision (reading A18).
#ifndef SNP_VM_THREADS
#define SNP_VM_THREADS 256
#endif
constexpr int VM_THREADS = SNP_VM_THREADS;  // threads per match (CTA); CTAs per SM = min(2048 / VM_THREADS, smem)
size_t verify_m_smem_bytes(int32_t m, bool pk) {
  const size_t mE = (size_t)((m + 1) & ~1) + EPAD;
  return mE * (pk ? 4 : 16) + (size_t)m * 8 + 4 * KMAX * 8 + 64;
}

// VM_THREADS compute threads plus one decoder warp: the decoder reads the
// next match's key, parents and ND digits into the other half of a double
// buffer while the compute warps verify the current one (their phase
// barriers are named barriers over the compute threads only; the loop-end
// barrier joins everyone), so the ≈ 6 dependent loads of a decode overlap
// the count loads and the column pass
template <typename T, bool PK>
__global__ void __launch_bounds__(VM_THREADS + 32) k_verify_m(SysView S, LevelView L, ExpandOut O, const uint64_t* off,
                                                              ChildArrays C, const uint64_t* list,
                                                              const unsigned long long* n_list, uint64_t tag_base,
                                                              Tables tb, const StoredLevel* stored, int32_t* err) {
  using FW = typename std::conditional<PK, uint32_t, int4>::type;
  extern __shared__ __align__(16) uint8_t vm_smem[];
  const int32_t m = S.m;
  const int32_t mE = (m + 1) & ~1;
  FW* fc = reinterpret_cast<FW*>(vm_smem);                            // [mE + EPAD] (c_a, p_a, c_b, p_b); zero pads
  int32_t* cnt = reinterpret_cast<int32_t*>(fc + mE + EPAD);          // [2][m]
  int32_t* nds = cnt + 2 * m;                                          // [2 buf][2 sides][KMAX] neuron
  uint8_t* ndx = reinterpret_cast<uint8_t*>(nds + 4 * KMAX);          // [2 buf][2 sides][KMAX] digit
  __shared__ int sK[2][2];
  __shared__ uint32_t sp[2][2];
  __shared__ uint8_t svd[2];
  __shared__ uint64_t sref[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool decoder = tid >= VM_THREADS;
  // fired (c, p) of the first applicable rule of neuron s at count v: counts
  // < 32 from the count-major table (lanes = consecutive neurons share its
  // rows when their counts agree), else the rule tables
  auto first_cp = [&](int32_t s, int32_t v, int& c, int& p) {
    if (S.cpT && (uint32_t)v < 32u) {
      const uint32_t e = __ldg(S.cpT + (int64_t)v * m + s);
      c = (int)(e & 0xFFu);
      p = (int)(e >> 8);
      return;
    }
    const int r = first_rule(S, s, v);
    c = r >= 0 ? S.rules[r].c : 0;
    p = r >= 0 ? S.rules[r].p : 0;
  };
  auto mk = [](int ca, int pa, int cb, int pb) -> FW {
    if constexpr (PK) return (uint32_t)ca | ((uint32_t)pa << 8) | ((uint32_t)cb << 16) | ((uint32_t)pb << 24);
    else return make_int4(ca, pa, cb, pb);
  };
  auto ca_ = [](FW f) -> int32_t { if constexpr (PK) return (int32_t)(f & 0xFF); else return f.x; };
  auto pa_ = [](FW f) -> int32_t { if constexpr (PK) return (int32_t)((f >> 8) & 0xFF); else return f.y; };
  auto cb_ = [](FW f) -> int32_t { if constexpr (PK) return (int32_t)((f >> 16) & 0xFF); else return f.z; };
  auto pb_ = [](FW f) -> int32_t { if constexpr (PK) return (int32_t)(f >> 24); else return f.w; };
  // decoder lanes 0 / 1: side 0 = the listed child, side 1 = its key's winner
  auto decode = [&](uint64_t i, int b) {
    if (lane > 1) return;
    const uint64_t c = list[i];
    const uint8_t vd = C.verdict[c];
    if (lane == 0) {
      svd[b] = vd;
      sref[b] = vd == 1 ? 0 : C.cref[c];
    }
    if (lane == 1 && vd != 1) return;
    const uint64_t cc = lane == 0 ? c : tb.ltab[C.cslot[c]].tag - tag_base;
    const uint32_t p = C.cpar[cc];
    const uint64_t* nd = O.nd + (uint64_t)p * KMAX;
    const int K = O.ndc[p];
    uint64_t t = cc - off[p];
    for (int k = K - 1; k >= 0; --k) {  // mixed radix, first ND neuron most significant (reading A7)
      const int32_t s = (int32_t)(nd[k] >> 32), v = (int32_t)(uint32_t)nd[k];
      const uint64_t d = (uint64_t)count_applicable(S, s, v);
      nds[(2 * b + lane) * KMAX + k] = s;
      ndx[(2 * b + lane) * KMAX + k] = (uint8_t)(t % d);
      t /= d;
    }
    sK[b][lane] = K;
    sp[b][lane] = p;
  };
  if (tid < mE + EPAD - m) fc[m + tid] = mk(0, 0, 0, 0);  // targets of padded in-synapses
  const uint64_t nl = *n_list;
  if (decoder && blockIdx.x < nl) decode(blockIdx.x, 0);
  __syncthreads();
  int b = 0;
  for (uint64_t i = blockIdx.x; i < nl; i += gridDim.x, b ^= 1) {
    bool diff = false;
    if (decoder) {
      if (i + gridDim.x < nl) decode(i + gridDim.x, b ^ 1);
    } else {
      const uint8_t vd = svd[b];
      const int sides = vd == 1 ? 2 : 1;
      const uint32_t p0 = sp[b][0], p1 = sp[b][1];
      for (int32_t s = tid; s < m; s += VM_THREADS) {
        int ca = 0, pa = 0, cb = 0, pb = 0;
        const int32_t va = ld_count<T>(L.data, p0, s, m);
        const int32_t vb = sides == 2 ? ld_count<T>(L.data, p1, s, m) : 0;
        cnt[s] = va;
        first_cp(s, va, ca, pa);
        if (sides == 2) {
          cnt[m + s] = vb;
          first_cp(s, vb, cb, pb);
        }
        fc[s] = mk(ca, pa, cb, pb);
      }
      tc::named_sync(1, VM_THREADS);
      for (int sd = 0; sd < sides; ++sd) {  // ND digits != 0 (a neuron appears once per side)
        if (tid < sK[b][sd] && ndx[(2 * b + sd) * KMAX + tid]) {
          const int32_t s = nds[(2 * b + sd) * KMAX + tid];
          const int r = nth_applicable(S, s, cnt[sd * m + s], ndx[(2 * b + sd) * KMAX + tid]);
          const FW f = fc[s];
          fc[s] = sd == 0 ? mk(S.rules[r].c, S.rules[r].p, cb_(f), pb_(f)) : mk(ca_(f), pa_(f), S.rules[r].c, S.rules[r].p);
        }
        tc::named_sync(1, VM_THREADS);
      }
      const uint64_t ref = sref[b];
      for (int32_t j0 = warp * 32; j0 < m; j0 += VM_THREADS) {
        const int32_t j = j0 + lane;
        const int64_t g = j0 >> 5;
        const int64_t r0 = __ldg(S.in_pad_off + g), r1 = __ldg(S.in_pad_off + g + 1);
        const FW fj = fc[j < m ? j : m];
        if (vd == 1) {
          int64_t d = j < m ? ((int64_t)cnt[j] - ca_(fj)) - ((int64_t)cnt[m + j] - cb_(fj)) : 0;
          for (int64_t r = r0; r < r1; ++r) {
            const int32_t src = S.in_pad16 ? (int32_t)__ldg(S.in_pad16 + r * 32 + lane) : __ldg(S.in_pad + r * 32 + lane);
            const FW f = fc[src];
            d += pa_(f) - pb_(f);
          }
          diff |= d != 0;
        } else {
          int64_t a = j < m ? (int64_t)cnt[j] - ca_(fj) : 0;
          for (int64_t r = r0; r < r1; ++r) {
            const int32_t src = S.in_pad16 ? (int32_t)__ldg(S.in_pad16 + r * 32 + lane) : __ldg(S.in_pad + r * 32 + lane);
            a += pa_(fc[src]);
          }
          if (j < m) diff |= a != ld_count<T>(stored[ref >> 40].data, (int64_t)(ref & ((1ULL << 40) - 1)), j, m);
        }
      }
    }
    if (__syncthreads_or(diff) && tid == 0) atomicOr(err, ERR_COLLISION);
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
      const int64_t a = exact_value<T>(S, L.data, p, j, cx);
      int64_t b;
      if (vd == 1) {
        b = exact_value<T>(S, L.data, po, j, co);
      } else {
        const uint64_t ref = C.cref[c];
        b = ld_count<T>(stored[ref >> 40].data, (int64_t)(ref & ((1ULL << 40) - 1)), j, S.m);
      }
      diff |= (a != b);
    }
    if (__any_sync(0xFFFFFFFFu, diff) && lane == 0) atomicOr(err, ERR_COLLISION);
  }
}

// level 0 (reading A20): keep the first occurrence of every configuration
__global__ void k_level0_compact(const uint8_t* verdict, const uint64_t* kept, const uint64_t* kpos, int64_t F0,
                                 const uint64_t* fp0, const uint64_t* fp1, NextArrays N, uint64_t* src_index,
                                 Tables tb, int insert_visited, int32_t* err) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < F0; c += (int64_t)gridDim.x * blockDim.x) {
    if (!kept[c]) continue;
    const uint64_t q = kpos[c];
    N.parent[q] = -1;
    N.t[q] = 0;
    N.fp0[q] = fp0[c];
    N.fp1[q] = fp1[c];
    src_index[q] = (uint64_t)c;
    if (insert_visited) visited_insert(tb, fp0[c], fp1[c], q, err);
  }
}

// zero the unused tail of a level's last storage block (configurations F ..
// 64·ceil(F/64) - 1 of every neuron row): K-a and K-c load whole 32-byte row
// halves, so the tail is read (and masked out) — zeroed it is also initialised
template <typename T>
__global__ void k_zero_tail(T* data, int64_t F, int32_t m) {
  const int64_t b = F / PB;
  const int r0 = (int)(F % PB);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)m * (PB - r0);
       i += (int64_t)gridDim.x * blockDim.x)
    data[(b * m + i / (PB - r0)) * PB + r0 + i % (PB - r0)] = 0;
}

// snapshot: every level's edge arrays into one contiguous set (one D2H each)
__global__ void k_pack_edges(const EdgeSrc* lv, int32_t nlev, int64_t* parent, uint64_t* t, uint8_t* halting,
                             uint64_t* fp2) {
  for (int32_t L = blockIdx.y; L < nlev; L += gridDim.y) {
    const EdgeSrc e = lv[L];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e.F; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t o = e.offset + i;
      parent[o] = e.parent[i];
      t[o] = e.t[i];
      halting[o] = e.halting[i];
      fp2[2 * o] = e.fp0[i];
      fp2[2 * o + 1] = e.fp1[i];
    }
  }
}

__global__ void k_add_i64(int64_t* a, int64_t n, int64_t add) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (a[i] >= 0) a[i] += add;
}

template <typename T>
__global__ void k_gather_columns(const T* src, const uint64_t* src_index, int64_t K, int32_t m, T* dst) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= K) return;
  const int64_t c = (int64_t)src_index[q];
  for (int32_t j = blockIdx.y; j < m; j += gridDim.y) dst[eidx(q, j, m)] = src[eidx(c, j, m)];
}

template <typename T>
__global__ void k_verify_level0(const T* data, int32_t m, ChildArrays C, uint64_t F0, Tables tb, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = warp; c < F0; c += nwarps) {
    const uint64_t w = tb.ltab[C.cslot[c]].tag;
    if (w == c) continue;
    bool diff = false;
    for (int32_t j = lane; j < m; j += 32) diff |= data[eidx((int64_t)c, j, m)] != data[eidx((int64_t)w, j, m)];
    if (__any_sync(0xFFFFFFFFu, diff) && lane == 0) atomicOr(err, ERR_COLLISION);
  }
}

__global__ void k_rehash(const Slot* old_tab, uint64_t old_cap, Slot* new_tab, uint64_t new_mask, int32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < old_cap; i += (uint64_t)gridDim.x * blockDim.x) {
    const Key128 key = ld_key(old_tab + i);
    if (key.k0 == EMPTY && key.k1 == EMPTY) continue;
    uint64_t h = fmix64(key.k0) & new_mask;
    bool ok = false;
    for (uint64_t probes = 0; probes <= new_mask; ++probes, h = (h + 1) & new_mask) {
      Key128 empty{EMPTY, EMPTY};
      const Key128 prev = atomicCAS(reinterpret_cast<Key128*>(new_tab + h), empty, key);
      if (prev.k0 == EMPTY && prev.k1 == EMPTY) {
        new_tab[h].ref = old_tab[i].ref;
        ok = true;
        break;
      }
    }
    if (!ok) atomicOr(err, ERR_TABLE_FULL);
  }
}

// ---------------------------------------------------------------------------
// Small frontiers (configs 1-2, the paper's Π with <= 5 configurations per
// level): up to `max_levels` whole BFS levels in ONE launch of ONE CTA.  Each
// level runs the steps of the multi-kernel path in order — K-a (first rule,
// Ψ, ND list, base fingerprint, halting), the offsets, K-b child keys by
// linearity, K-d (visited probe, level table with the minimum tag, N_new,
// thinning τ, kept flags, compaction + visited insert), K-c (each kept child
// exactly, eq. (2) column by column), the dedup = 0 verification and the
// digest — on the same device functions and with the same tags, so the tree
// is the one the big path builds (same parity tests).  A level with more
// than SMALL_T transitions is left untouched for the big path; a level whose
// frontier exceeds SMALL_F ends the launch after it is committed.
// ---------------------------------------------------------------------------
// floor(F·2^64 / N) for F < N (reading A19), by restoring long division
__device__ uint64_t tau_div(uint64_t F, uint64_t N) {
  uint64_t q = 0, r = F;  // remainder < N throughout; dividend F·2^64: 64 zero bits enter
  for (int i = 0; i < 64; ++i) {
    const bool carry = (r >> 63) != 0;
    r <<= 1;
    q <<= 1;
    if (carry || r >= N) {
      r -= N;
      q |= 1;
    }
  }
  return q;
}

// NT threads: 1024, or 128 for tiny frontiers (Π: cheaper barriers per level)
template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_small_bfs(SysView S, SmallArgs a) {
  using SmallScan = cub::BlockScan<uint64_t, NT>;
  __shared__ typename SmallScan::TempStorage scan_tmp;
  __shared__ unsigned long long sh_u64[4];  // [0] n_new, [1] n_halting, [2] digest
  __shared__ int32_t sh_err, sh_stop;
  __shared__ uint64_t sh_T, sh_K, sh_tau, sh_part[NT];
  __shared__ int sh_thin;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int32_t m = S.m;
  const void* data = a.data;
  int64_t F = a.F;
  const uint64_t* fp0 = a.fp0;
  const uint64_t* fp1 = a.fp1;
  uint8_t* halting = a.halting;
  int done = 0;
  for (int lev = 0; lev < a.max_levels; ++lev) {
    if (tid == 0) {
      sh_u64[0] = sh_u64[1] = sh_u64[2] = 0;
      sh_err = 0;
      sh_stop = 0;
    }
    __syncthreads();
    // ---- K-a: applicability, Ψ (eq. (8), A3/A5), ND list, base fingerprint
    for (int64_t p = tid; p < F; p += nt) {
      uint64_t fa = fp0[p], fb = fp1[p], psi = 1;
      int ndc = 0;
      bool any = false;
      for (int32_t s = 0; s < m; ++s) {
        const int32_t v = ld_count<T>(data, p, s, m);
        int first = -1, d = 0;
        for (int r = S.rule_off[s]; r < S.rule_off[s + 1]; ++r)
          if (rule_app(S.rules[r], v)) {
            if (!d) first = r;
            ++d;
          }
        if (!d) continue;
        any = true;
        fa += __ldg(S.h0 + first);
        fb += __ldg(S.h1 + first);
        if (d >= 2) {
          if (ndc < KMAX) a.nd[p * KMAX + ndc] = ((uint64_t)(uint32_t)s << 32) | (uint32_t)v;
          ++ndc;
          psi = sat_mul(psi, (uint64_t)d);
        }
      }
      halting[p] = any ? 0 : 1;
      if (!any) atomicAdd(&sh_u64[1], 1ULL);
      a.psi[p] = any ? psi : 0;
      a.fpb0[p] = fa;
      a.fpb1[p] = fb;
      a.ndc[p] = ndc;
      if ((any && psi > PSI_LIMIT) || ndc > KMAX) atomicOr(&sh_err, ERR_CAPACITY);
    }
    __syncthreads();
    if (tid == 0) {
      uint64_t acc = 0;
      for (int64_t p = 0; p < F; ++p) {
        a.off[p] = acc;
        acc += a.psi[p];
        if (acc > (1ULL << 40)) acc = 1ULL << 40;  // saturate: only the SMALL_T test below reads it
      }
      a.off[F] = acc;
      sh_T = acc;
      if (!sh_err && a.max_transitions > 0 && acc > (uint64_t)a.max_transitions) sh_err = ERR_CAPACITY;  // budget
      if (!sh_err && acc > (uint64_t)SMALL_T) sh_stop = 1;
    }
    __syncthreads();
    SmallLevelOut* o = a.out + lev;
    if (sh_err || sh_stop) {
      if (tid == 0) {
        o->err = sh_err;
        o->stop = sh_stop;
        o->T = (int64_t)sh_T;
        o->n_halting = (int64_t)sh_u64[1];
      }
      break;
    }
    const uint64_t Tn = sh_T;
    // ---- K-b: child -> parent, keys by linearity (reading A18), clear the level table
    for (int64_t p = tid; p < F; p += nt)
      for (uint64_t c = a.off[p]; c < a.off[p + 1]; ++c) a.cpar[c] = (uint32_t)p;
    // the level table sized for this level's transitions (>= 2T slots, a power of two)
    Tables tl = a.tb;
    {
      uint64_t sl = 64;
      while (sl < 2 * Tn) sl <<= 1;
      tl.lmask = sl - 1 < a.tb.lmask ? sl - 1 : a.tb.lmask;
    }
    for (uint64_t i = tid; i <= tl.lmask; i += nt) {
      tl.ltab[i].k0 = EMPTY;
      tl.ltab[i].k1 = EMPTY;
      tl.ltab[i].tag = EMPTY;
      tl.ltab[i].ref = EMPTY;
    }
    __syncthreads();
    for (uint64_t c = tid; c < Tn; c += nt) {
      const uint32_t p = a.cpar[c];
      uint64_t t = c - a.off[p];
      uint64_t fa = a.fpb0[p], fb = a.fpb1[p];
      const uint64_t* nd = a.nd + (uint64_t)p * KMAX;
      for (int i = a.ndc[p] - 1; i >= 0 && t; --i) {
        const int32_t s = (int32_t)(nd[i] >> 32), v = (int32_t)(uint32_t)nd[i];
        const uint64_t d = (uint64_t)count_applicable(S, s, v);
        const int x = (int)(t % d);
        t /= d;
        if (x) {
          const int rf = nth_applicable(S, s, v, 0), rc = nth_applicable(S, s, v, x);
          fa += __ldg(S.h0 + rc) - __ldg(S.h0 + rf);
          fb += __ldg(S.h1 + rc) - __ldg(S.h1 + rf);
        }
      }
      a.cfp0[c] = fa;
      a.cfp1[c] = fb;
    }
    __syncthreads();
    // ---- K-d: visited (earlier levels, A6), level table with the minimum tag (A7)
    for (uint64_t c = tid; c < Tn; c += nt) {
      const uint64_t k0 = a.cfp0[c], k1 = a.cfp1[c];
      if (k0 == EMPTY && k1 == EMPTY) {
        atomicOr(&sh_err, ERR_COLLISION);
        a.verdict[c] = 0;
        a.cref[c] = EMPTY;
        continue;
      }
      const uint64_t h = fmix64(k0);
      bool old = false;
      uint64_t i = h & a.tb.vmask;
      for (uint64_t probes = 0; probes <= a.tb.vmask; ++probes, i = (i + 1) & a.tb.vmask) {
        const Key128 key = *reinterpret_cast<const Key128*>(a.tb.vis + i);
        if (key.k0 == k0 && key.k1 == k1) {
          old = true;
          a.cref[c] = a.tb.vis[i].ref;
          break;
        }
        if (key.k0 == EMPTY && key.k1 == EMPTY) break;
      }
      if (old) {
        a.verdict[c] = 0;
        continue;
      }
      bool ins = false;
      i = h & tl.lmask;
      for (uint64_t probes = 0; probes <= tl.lmask; ++probes, i = (i + 1) & tl.lmask) {
        Key128 empty{EMPTY, EMPTY}, mine{k0, k1};
        const Key128 prev = atomicCAS(reinterpret_cast<Key128*>(tl.ltab + i), empty, mine);
        if ((prev.k0 == EMPTY && prev.k1 == EMPTY) || (prev.k0 == k0 && prev.k1 == k1)) {
          atomicMin(&tl.ltab[i].tag, (unsigned long long)c);
          a.cslot[c] = i;
          a.verdict[c] = 1;
          ins = true;
          break;
        }
      }
      if (!ins) atomicOr(&sh_err, ERR_TABLE_FULL);
    }
    __syncthreads();
    for (uint64_t c = tid; c < Tn; c += nt)
      if (a.verdict[c] == 1 && a.tb.ltab[a.cslot[c]].tag == c) atomicAdd(&sh_u64[0], 1ULL);
    __syncthreads();
    if (tid == 0) {
      const uint64_t n_new = sh_u64[0];
      sh_thin = a.frontier_target > 0 && n_new > (uint64_t)a.frontier_target;
      sh_tau = sh_thin ? tau_div((uint64_t)a.frontier_target, n_new) : 0;  // reading A19
    }
    __syncthreads();
    // kept flags and their exclusive scan (contiguous chunks, block scan of the chunk sums)
    const uint64_t per = (Tn + nt - 1) / nt;
    uint64_t sum = 0;
    for (uint64_t c = tid * per; c < Tn && c < (tid + 1) * per; ++c) {
      uint64_t k = 0;
      if (a.verdict[c] == 1 && a.tb.ltab[a.cslot[c]].tag == c) k = sh_thin ? (fmix64(a.cfp0[c]) < sh_tau) : 1;
      a.kept[c] = k;
      sum += k;
    }
    {
      uint64_t excl, total;
      SmallScan(scan_tmp).ExclusiveSum(sum, excl, total);
      sh_part[tid] = excl;
      if (tid == 0) sh_K = total;
    }
    __syncthreads();
    {
      uint64_t acc = sh_part[tid];
      for (uint64_t c = tid * per; c < Tn && c < (tid + 1) * per; ++c) {
        a.kpos[c] = acc;
        acc += a.kept[c];
      }
    }
    __syncthreads();
    const int64_t K = (int64_t)sh_K;
    const uint64_t level = (uint64_t)(a.level0 + lev + 1);
    uint8_t* ndata = a.data_pool + (size_t)lev * a.data_stride;
    int64_t* npar = a.parent_pool + (size_t)lev * SMALL_T;
    uint64_t* nt_ = a.t_pool + (size_t)lev * SMALL_T;
    uint64_t* nfp0 = a.fp0_pool + (size_t)lev * SMALL_T;
    uint64_t* nfp1 = a.fp1_pool + (size_t)lev * SMALL_T;
    // compaction in tag order + visited insert
    for (uint64_t c = tid; c < Tn; c += nt) {
      if (!a.kept[c]) continue;
      const uint64_t q = a.kpos[c];
      const uint32_t p = a.cpar[c];
      npar[q] = p;
      nt_[q] = c - a.off[p];
      nfp0[q] = a.cfp0[c];
      nfp1[q] = a.cfp1[c];
      visited_insert(a.tb, a.cfp0[c], a.cfp1[c], (level << 40) | q, &sh_err);
    }
    __syncthreads();
    // ---- K-c: every kept child exactly (eq. (2) column by column), tail zeroed
    T* nd_out = reinterpret_cast<T*>(ndata);
    for (int64_t q = tid; q < K; q += nt) {
      const int64_t p = npar[q];
      ChildCtx cx;
      decode_child(S, a.nd + p * KMAX, a.ndc[p], nt_[q], cx);
      bool bad = false;
      for (int32_t j = 0; j < m; ++j) {
        const int64_t val = exact_value<T>(S, data, p, j, cx);
        bad |= (val < 0 || val > S.count_max);
        nd_out[eidx(q, j, m)] = (T)val;
      }
      if (bad) atomicOr(&sh_err, ERR_OVERFLOW);
    }
    if (K % PB)
      for (int64_t i = tid; i < (int64_t)m * (PB - K % PB); i += nt)
        nd_out[((K / PB) * m + i / (PB - K % PB)) * PB + K % PB + i % (PB - K % PB)] = 0;
    if (a.dedup == 0 && tid == 0) a.stored[level].data = ndata;
    __syncthreads();
    // ---- dedup = 0: every key match compared as full configurations (A18)
    if (a.dedup == 0) {
      for (uint64_t c = tid; c < Tn; c += nt) {
        const uint8_t vd = a.verdict[c];
        uint64_t other = EMPTY;
        if (vd == 1) {
          const uint64_t wtag = a.tb.ltab[a.cslot[c]].tag;
          if (wtag == c) continue;
          other = wtag;
        } else if (a.cref[c] == EMPTY) {
          continue;
        }
        const uint32_t p = a.cpar[c];
        ChildCtx cx, co;
        decode_child(S, a.nd + (uint64_t)p * KMAX, a.ndc[p], c - a.off[p], cx);
        uint32_t po = 0;
        if (vd == 1) {
          po = a.cpar[other];
          decode_child(S, a.nd + (uint64_t)po * KMAX, a.ndc[po], other - a.off[po], co);
        }
        bool diff = false;
        for (int32_t j = 0; j < m && !diff; ++j) {
          const int64_t x = exact_value<T>(S, data, p, j, cx);
          int64_t y;
          if (vd == 1) {
            y = exact_value<T>(S, data, po, j, co);
          } else {
            const uint64_t ref = a.cref[c];
            y = ld_count<T>(a.stored[ref >> 40].data, (int64_t)(ref & ((1ULL << 40) - 1)), j, m);
          }
          diff = x != y;
        }
        if (diff) atomicOr(&sh_err, ERR_COLLISION);
      }
    }
    // ---- digest
    for (int64_t q = tid; q < K; q += nt) {
      uint64_t z = fmix64((level << 40) ^ (uint64_t)q);
      z = fmix64(z ^ nfp0[q]);
      z = fmix64(z ^ nfp1[q]);
      z = fmix64(z ^ (uint64_t)(npar[q] + 1));
      z = fmix64(z ^ nt_[q]);
      atomicAdd(&sh_u64[2], (unsigned long long)z);
    }
    __syncthreads();
    if (tid == 0) {
      o->T = (int64_t)Tn;
      o->n_new = (int64_t)sh_u64[0];
      o->kept = K;
      o->n_halting = (int64_t)sh_u64[1];
      o->tau = sh_tau;
      o->digest = sh_u64[2];
      o->err = sh_err;
      o->stop = 0;
    }
    __syncthreads();
    if (sh_err) break;
    ++done;
    // the new level becomes the current one
    data = ndata;
    F = K;
    fp0 = nfp0;
    fp1 = nfp1;
    halting = a.halting_pool + (size_t)lev * SMALL_T;
    if (K == 0 || K > SMALL_F) break;
    __syncthreads();
  }
  if (tid == 0) *a.levels_done = done;
}

// order-sensitive run digest
__global__ void k_digest(NextArrays N, int64_t K, uint64_t level, int64_t q_offset, int64_t parent_offset,
                         unsigned long long* digest) {
  unsigned long long acc = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = fmix64((level << 40) ^ (uint64_t)(q + q_offset));
    z = fmix64(z ^ N.fp0[q]);
    z = fmix64(z ^ N.fp1[q]);
    const int64_t par = N.parent[q];
    z = fmix64(z ^ (uint64_t)(par < 0 ? 0 : par + parent_offset + 1));
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
__global__ void k_spiking_vectors(SysView S, const T* pdata, const int64_t* parent, const uint64_t* tt, int64_t K,
                                  uint8_t* S_out, int32_t* err) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = parent[q];
    uint64_t t = tt[q];
    uint8_t* Sq = S_out + q * S.n;
    for (int64_t r = 0; r < S.n; ++r) Sq[r] = 0;
    bool any = false;
    for (int32_t s = S.m - 1; s >= 0; --s) {  // least significant digit = last neuron
      const int32_t v = (int32_t)pdata[eidx(p, s, S.m)];
      const int d = count_applicable(S, s, v);
      if (d == 0) continue;
      any = true;
      const int x = (int)(t % (uint64_t)d);
      t /= (uint64_t)d;
      Sq[nth_applicable(S, s, v, x)] = 1;
    }
    if ((t || !any) && err) atomicOr(err, ERR_CAPACITY);  // t >= Ψ (Ψ = 0 when halting): no such vector
  }
}

// Outcome tables, one thread per (neuron, table index): the
// applicability of every rule at count v evaluated once per
// system instead of once per (neuron, configuration).
template <typename T>
__global__ void k_build_tables(SysView S, uint8_t* tab, T* ctab, uint8_t* tab_full, uint8_t* ttab, uint8_t* elut) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t w = S.tabw;
  const int64_t n_c = (int64_t)S.m * w;
  const int64_t n_f = (tab_full || ttab) ? (int64_t)S.m * 256 : 0;  // ttab alone for wide counts (K-c NARROW)
  if (i >= n_c + n_f) return;
  const bool full = i >= n_c;
  const int32_t s = (int32_t)(full ? (i - n_c) / 256 : i / w);
  const uint32_t slot = (uint32_t)(full ? (i - n_c) % 256 : i % w);
  const NeuronMeta mt = S.meta[s];
  uint32_t entry = 0;
  int32_t cons = 0;
  const bool valid = !(mt.flags & NM_GENERIC);
  if (valid) {
    // every slot holds the outcome at count v = slot (slots >= L + P repeat the
    // periodic part, so idx(v) of table_index lands on the same outcome)
    const int32_t v = (int32_t)slot;
    int first = -1, d = 0;
    for (int r = S.rule_off[s]; r < S.rule_off[s + 1]; ++r)
      if (rule_app(S.rules[r], v)) {
        if (!d) first = r;
        ++d;
      }
    if (d) {
      entry = ((uint32_t)(first - S.rule_off[s] + 1) << 4) | (S.rules[first].p > 0 ? TE_EMIT : 0u) | (d >= 2 ? TE_ND : 0u);
      cons = S.rules[first].c;
    }
  }
  if (full) {
    if (tab_full) tab_full[i - n_c] = (uint8_t)entry;
    // post-consumption value v - c_first(v) (K-c lookups): counts < 32 in
    // the 32-byte rows (one coalesced 32-B load per lane, then byte
    // permutes in registers), every count in the 256-byte rows
    if (slot < 32) ttab[(int64_t)s * 32 + slot] = (uint8_t)(slot - (uint32_t)cons);
    ttab[(int64_t)S.m * 32 + (int64_t)s * 256 + slot] = (uint8_t)(slot - (uint32_t)cons);
    if (slot < 32 && elut) elut[(int64_t)s * 32 + slot] = (uint8_t)entry;
  } else {
    tab[i] = (uint8_t)entry;
    ctab[i] = (T)cons;
  }
}

template <typename F>
void dispatch_bytes(int32_t bytes, F&& f) {
  if (bytes == 1) f(uint8_t{});
  else if (bytes == 2) f(uint16_t{});
  else f(int32_t{});
}

}  // namespace

// ---------------------------------------------------------------------------
// SN P systems WITH delays (reading A26; SysView::
// delay_m = m > 0).  A state is the row [C | τ | π] of width S.m = 3m
// (spikes, remaining closed steps, pending emission).  Open neurons (τ = 0)
// choose rules as without delays; a closed neuron counts down and emits π
// when it reopens; a firing rule with d >= 1 closes its neuron for d steps
// (τ' = d, π' = p); only neurons open after the step receive.  The child
// state is not linear in the rule choice (a neuron that closes loses its
// incoming spikes), so child keys are computed from the materialised child.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_expand_delay(SysView S, LevelView L, ExpandOut O) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = p < L.F;
  bool halt = false;
  if (valid) {
    const int32_t m = S.delay_m;
    int ndc = 0;
    uint64_t psi = 1;
    bool any = false, closed = false;
    for (int32_t s = 0; s < m; ++s) {
      if (ld_count<T>(L.data, p, m + s, S.m) != 0) {
        closed = true;
        continue;
      }
      const int32_t v = ld_count<T>(L.data, p, s, S.m);
      const int d = count_applicable(S, s, v);
      any |= d > 0;
      if (d >= 2 && !O.classify_only) nd_event(S, O, s, (uint32_t)v, p, ndc, psi);
    }
    halt = !any && !closed;  // reading A26: nothing can fire and no clock runs
    O.halting[p] = halt ? 1 : 0;
    if (!O.classify_only) {
      psi = any ? psi : (closed ? 1 : 0);  // only clocks running: one child
      O.psi[p] = psi;
      O.ndc[p] = ndc;
      if (psi > PSI_LIMIT || ndc > KMAX) atomicOr(O.err, ERR_CAPACITY);
    }
  }
  const unsigned nh = __popc(__ballot_sync(0xFFFFFFFFu, halt));
  if ((threadIdx.x & 31) == 0 && nh) atomicAdd(O.n_halting, (unsigned long long)nh);
}

// column j of the child of parent p described by cx (reading A26)
template <typename T>
__device__ int64_t delay_value(const SysView& S, const void* data, int64_t p, int32_t j, const ChildCtx& cx) {
  const int32_t m = S.delay_m;
  auto tau = [&](int32_t s) { return (int64_t)ld_count<T>(data, p, m + s, S.m); };
  auto fired = [&](int32_t s) { return tau(s) ? -1 : fired_rule(S, s, ld_count<T>(data, p, s, S.m), cx); };
  auto tau_next = [&](int32_t s) -> int64_t {
    const int64_t t0 = tau(s);
    if (t0 >= 1) return t0 - 1;
    const int r = fired(s);
    return r >= 0 ? S.delay[r] : 0;
  };
  auto emit = [&](int32_t s) -> int64_t {
    const int64_t t0 = tau(s);
    if (t0 >= 1) return t0 == 1 ? (int64_t)ld_count<T>(data, p, 2 * m + s, S.m) : 0;
    const int r = fired(s);
    return (r >= 0 && S.delay[r] == 0) ? S.rules[r].p : 0;
  };
  if (j >= 2 * m) {  // π'
    const int32_t s = j - 2 * m;
    const int64_t t0 = tau(s);
    if (t0 >= 1) return t0 == 1 ? 0 : (int64_t)ld_count<T>(data, p, 2 * m + s, S.m);
    const int r = fired(s);
    return (r >= 0 && S.delay[r] >= 1) ? S.rules[r].p : 0;
  }
  if (j >= m) return tau_next(j - m);  // τ'
  const int r = fired(j);
  int64_t val = (int64_t)ld_count<T>(data, p, j, S.m) - (r >= 0 ? S.rules[r].c : 0);
  if (tau_next(j) == 0)  // open after the step: receives
    for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) val += emit(S.in_src[e]);
  return val;
}

// Per-neuron step data of one child (reading A26), computed once per neuron
// into the warp's shared-memory slice: consumption, τ', π', emission.
struct DelayCols {
  int32_t* cons;
  int32_t* taun;
  int32_t* pin;
  int32_t* emit;
};

template <typename T>
__device__ void delay_neurons(const SysView& S, const void* data, int64_t p, const ChildCtx& cx, const DelayCols& D,
                              int lane) {
  const int32_t m = S.delay_m;
  for (int32_t s = lane; s < m; s += 32) {
    const int64_t t0 = ld_count<T>(data, p, m + s, S.m);
    int32_t cons = 0, taun = 0, pin = 0, emit = 0;
    if (t0 >= 1) {  // closed: the clock runs, emits π when it reopens
      taun = (int32_t)(t0 - 1);
      const int32_t pi0 = ld_count<T>(data, p, 2 * m + s, S.m);
      pin = taun ? pi0 : 0;
      emit = taun ? 0 : pi0;
    } else {
      const int r = fired_rule(S, s, ld_count<T>(data, p, s, S.m), cx);
      if (r >= 0) {
        cons = S.rules[r].c;
        if (S.delay[r] == 0) emit = S.rules[r].p;
        else { taun = S.delay[r]; pin = S.rules[r].p; }
      }
    }
    D.cons[s] = cons;
    D.taun[s] = taun;
    D.pin[s] = pin;
    D.emit[s] = emit;
  }
  __syncwarp();
}

template <typename T>
__device__ __forceinline__ int64_t delay_column(const SysView& S, const void* data, int64_t p, int32_t j,
                                                const DelayCols& D) {
  const int32_t m = S.delay_m;
  if (j >= 2 * m) return D.pin[j - 2 * m];
  if (j >= m) return D.taun[j - m];
  int64_t val = (int64_t)ld_count<T>(data, p, j, S.m) - D.cons[j];
  if (D.taun[j] == 0)
    for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) val += D.emit[S.in_src[e]];
  return val;
}

constexpr int DELAY_WARPS = 8;
size_t delay_smem_bytes(int32_t m) { return (size_t)DELAY_WARPS * 16 * (size_t)m; }

// child keys (shared-memory variant, 16·m bytes per warp): the per-neuron
// step data once per child, then the 3m columns and their fingerprint
template <typename T>
__global__ void __launch_bounds__(DELAY_WARPS * 32) k_child_keys_delay_s(SysView S, LevelView L, const uint64_t* off,
                                                                         ExpandOut O, uint64_t T_, ChildArrays C) {
  extern __shared__ int32_t dsm[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int32_t m = S.delay_m;
  const DelayCols D{dsm + (size_t)wl * 4 * m, dsm + (size_t)wl * 4 * m + m, dsm + (size_t)wl * 4 * m + 2 * m,
                    dsm + (size_t)wl * 4 * m + 3 * m};
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = warp; c < T_; c += nwarps) {
    const int64_t p = C.cpar[c];
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], c - off[p], cx);
    delay_neurons<T>(S, L.data, p, cx, D, lane);
    uint64_t f0 = 0, f1 = 0;
    for (int32_t j = lane; j < S.m; j += 32) {
      const uint64_t v = (uint64_t)delay_column<T>(S, L.data, p, j, D);
      f0 += v * S.R0[j];
      f1 += v * S.R1[j];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      f0 += __shfl_xor_sync(0xFFFFFFFFu, f0, o);
      f1 += __shfl_xor_sync(0xFFFFFFFFu, f1, o);
    }
    if (lane == 0) {
      C.cfp0[c] = f0;
      C.cfp1[c] = f1;
    }
    __syncwarp();
  }
}

template <typename T>
__global__ void __launch_bounds__(DELAY_WARPS * 32) k_materialize_delay_s(SysView S, LevelView L, ExpandOut O,
                                                                          NextArrays N, int64_t K, int32_t* err) {
  extern __shared__ int32_t dsm[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int32_t m = S.delay_m;
  const DelayCols D{dsm + (size_t)wl * 4 * m, dsm + (size_t)wl * 4 * m + m, dsm + (size_t)wl * 4 * m + 2 * m,
                    dsm + (size_t)wl * 4 * m + 3 * m};
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  T* out = reinterpret_cast<T*>(N.data);
  for (int64_t q = warp; q < K; q += nwarps) {
    const int64_t p = N.parent[q];
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], N.t[q], cx);
    delay_neurons<T>(S, L.data, p, cx, D, lane);
    bool bad = false;
    for (int32_t j = lane; j < S.m; j += 32) {
      const int64_t val = delay_column<T>(S, L.data, p, j, D);
      bad |= val < 0 || val > S.count_max;
      out[eidx(q, j, S.m)] = (T)val;
    }
    if (bad) atomicOr(err, ERR_OVERFLOW);
    __syncwarp();
  }
}

// child keys: warp per child, fingerprint of the materialised child (A18)
template <typename T>
__global__ void k_child_keys_delay(SysView S, LevelView L, const uint64_t* off, ExpandOut O, uint64_t T_,
                                   ChildArrays C) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = warp; c < T_; c += nwarps) {
    const int64_t p = C.cpar[c];
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], c - off[p], cx);
    uint64_t f0 = 0, f1 = 0;
    for (int32_t j = lane; j < S.m; j += 32) {
      const uint64_t v = (uint64_t)delay_value<T>(S, L.data, p, j, cx);
      f0 += v * S.R0[j];
      f1 += v * S.R1[j];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      f0 += __shfl_xor_sync(0xFFFFFFFFu, f0, o);
      f1 += __shfl_xor_sync(0xFFFFFFFFu, f1, o);
    }
    if (lane == 0) {
      C.cfp0[c] = f0;
      C.cfp1[c] = f1;
    }
  }
}

// K-c: every kept child, exactly (warp per child)
template <typename T>
__global__ void k_materialize_delay(SysView S, LevelView L, ExpandOut O, NextArrays N, int64_t K, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  T* out = reinterpret_cast<T*>(N.data);
  for (int64_t q = warp; q < K; q += nwarps) {
    const int64_t p = N.parent[q];
    ChildCtx cx;
    decode_child(S, O.nd + p * KMAX, O.ndc[p], N.t[q], cx);
    bool bad = false;
    for (int32_t j = lane; j < S.m; j += 32) {
      const int64_t val = delay_value<T>(S, L.data, p, j, cx);
      bad |= val < 0 || val > S.count_max;
      out[eidx(q, j, S.m)] = (T)val;
    }
    if (bad) atomicOr(err, ERR_OVERFLOW);
  }
}

// ---------------------------------------------------------------------------
// Single-path sampling with an input spike train (Def. 1
// `in`; deep trees take long to explore).  One
// warp per walker runs every step (walkers are independent: no grid sync).
// Step k: applicable rules per neuron, Ψ = Π_{d_s>0} d_s
// (eq. (8), reading A3; > 2^62 is SNP_E_CAPACITY), the child
// t = u mod Ψ with u = splitmix64(splitmix64(seed ^ (k << 32)) ^ w)
// (reading A25) decoded in mixed radix, first nondeterministic neuron most
// significant (Alg. 2 II-2/II-3, reading A7), C' = C + S_t·M as the column
// sums of Def. 2, then the input neuron gets train[k] spikes (k < train_len).
// A walker with no applicable rule keeps C while input is still to come and
// stops (halted = k) once it is not (reading A5).  Counts outside
// [0, count_max] after a step are SNP_E_OVERFLOW.
// cur / nxt: W × m int32 walker-major scratch (the final states end in cur);
// fired: W × m uint64, the fired rule's c | p << 32 per neuron.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

constexpr int SAMPLE_WARPS = 4;

__global__ void __launch_bounds__(SAMPLE_WARPS * 32) k_sample(SysView S, int64_t W, int32_t* cur, int32_t* nxt,
                                                             uint64_t* fired, uint64_t seed, int32_t steps,
                                                             int32_t input_neuron, const int32_t* train,
                                                             int32_t train_len, int32_t* halted, int32_t* err) {
  __shared__ int32_t nd_s[SAMPLE_WARPS][KMAX];
  __shared__ uint8_t nd_d[SAMPLE_WARPS][KMAX];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= W) return;
  const int32_t m = S.m;
  int32_t* C = cur + w * m;
  int32_t* N = nxt + w * m;
  uint64_t* Fr = fired + w * m;  // fired rule's c | p << 32 per neuron (0: none)
  const bool tab8 = S.tables_ok && S.full8 && S.tab_full != nullptr;
  int32_t hs = -1;
  bool bad = false;
  for (int32_t k = 0; k < steps && !bad; ++k) {
    // first applicable rule and d_s of every neuron; the nondeterministic ones in order
    uint64_t psi = 1;
    bool any = false;
    int nnd = 0;
    for (int32_t base = 0; base < m; base += 32) {
      const int32_t s = base + lane;
      int d = 0, first = -1;
      if (s < m) {
        const int32_t v = C[s];
        if (tab8 && !(S.meta[s].flags & NM_GENERIC)) {  // uint8 tables: first rule, ND flag
          const uint32_t e = __ldg(S.tab_full + (int64_t)s * 256 + (uint32_t)v);
          if (e >> 4) {
            first = S.rule_off[s] + (int)(e >> 4) - 1;
            d = (e & TE_ND) ? count_applicable(S, s, v) : 1;
          }
        } else {
          for (int r = S.rule_off[s]; r < S.rule_off[s + 1]; ++r)
            if (rule_app(S.rules[r], v)) {
              if (!d) first = r;
              ++d;
            }
        }
        // consumption and emission of the fired rule (the ND choices below
        // overwrite theirs)
        Fr[s] = first >= 0 ? ((uint64_t)(uint32_t)S.rules[first].c | ((uint64_t)(uint32_t)S.rules[first].p << 32)) : 0;
      }
      any |= d > 0;
      if (d > 1) psi = sat_mul(psi, (uint64_t)d);
      const unsigned b = __ballot_sync(0xFFFFFFFFu, d >= 2);
      const int pos = nnd + __popc(b & ((1u << lane) - 1));
      if (d >= 2 && pos < KMAX) {
        nd_s[wl][pos] = s;
        nd_d[wl][pos] = (uint8_t)d;
      }
      nnd += __popc(b);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) psi = sat_mul(psi, __shfl_xor_sync(0xFFFFFFFFu, psi, o));
    any = __any_sync(0xFFFFFFFFu, any);
    if (psi > PSI_LIMIT) {
      if (lane == 0) atomicOr(err, ERR_CAPACITY);
      bad = true;
      break;
    }
    const bool input_left = input_neuron >= 0 && k < train_len;
    if (!any && !input_left) {
      hs = k;
      break;
    }
    if (any) {
      __syncwarp();
      if (lane == 0) {
        uint64_t t = splitmix64_dev(splitmix64_dev(seed ^ ((uint64_t)k << 32)) ^ (uint64_t)w) % psi;
        for (int i = nnd - 1; i >= 0; --i) {
          const int32_t s = nd_s[wl][i];
          const uint64_t d = nd_d[wl][i];
          const int r = nth_applicable(S, s, C[s], (int)(t % d));
          Fr[s] = (uint64_t)(uint32_t)S.rules[r].c | ((uint64_t)(uint32_t)S.rules[r].p << 32);
          t /= d;
        }
      }
      __syncwarp();
      for (int32_t j = lane; j < m; j += 32) {
        int64_t val = (int64_t)C[j] - (int64_t)(uint32_t)Fr[j];
        for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) val += (int64_t)(Fr[S.in_src[e]] >> 32);
        if (j == input_neuron && input_left) val += train[k];
        bad |= val < 0 || val > S.count_max;
        N[j] = (int32_t)val;
      }
      __syncwarp();
      int32_t* t_ = C;
      C = N;
      N = t_;
    } else if (lane == 0) {  // nothing fires: only the input arrives
      const int64_t val = (int64_t)C[input_neuron] + train[k];
      bad |= val < 0 || val > S.count_max;
      C[input_neuron] = (int32_t)val;
    }
    bad = __any_sync(0xFFFFFFFFu, bad);
    if (bad && lane == 0) atomicOr(err, ERR_OVERFLOW);
    __syncwarp();
  }
  if (C != cur + w * m)
    for (int32_t j = lane; j < m; j += 32) cur[w * m + j] = C[j];
  if (lane == 0) halted[w] = hs;
}

// Sampling, one CTA per walker (every rule has c, p <= 255): the fired
// rule's (c, p) of every neuron lives in shared memory as 16 bits, so the
// in-synapse gather of the transition reads shared memory; the few neurons
// with >= 2 applicable rules are collected unordered and sorted by thread 0
// (their order is the mixed-radix order, reading A7).  Same arithmetic and
// the same u as k_sample (reading A25).
constexpr int SAMPLE_CTA = 256;

__global__ void __launch_bounds__(SAMPLE_CTA) k_sample_cta(SysView S, int32_t* cur, int32_t* nxt, uint64_t seed,
                                                          int32_t steps, int32_t input_neuron,
                                                          const int32_t* train, int32_t train_len,
                                                          int32_t* halted, int32_t* err) {
  extern __shared__ uint16_t Fs[];  // m entries: c | p << 8 of the fired rule (0: none)
  __shared__ int32_t nd_s[KMAX + 1];
  __shared__ uint8_t nd_d[KMAX + 1];
  __shared__ int32_t nnd;
  __shared__ int32_t verdict;  // 0 go on, 1 halted, 2 capacity
  const int tid = threadIdx.x;
  const int64_t w = blockIdx.x;
  const int32_t m = S.m;
  int32_t* C = cur + w * m;
  int32_t* N = nxt + w * m;
  const bool tab8 = S.tables_ok && S.full8 && S.tab_full != nullptr;
  int32_t hs = -1;
  for (int32_t k = 0; k < steps; ++k) {
    if (tid == 0) nnd = 0;
    __syncthreads();
    int any = 0;
    for (int32_t s = tid; s < m; s += SAMPLE_CTA) {
      const int32_t v = C[s];
      int d = 0, first = -1;
      if (tab8 && !(S.meta[s].flags & NM_GENERIC)) {
        const uint32_t e = __ldg(S.tab_full + (int64_t)s * 256 + (uint32_t)v);
        if (e >> 4) {
          first = S.rule_off[s] + (int)(e >> 4) - 1;
          d = (e & TE_ND) ? count_applicable(S, s, v) : 1;
        }
      } else {
        for (int r = S.rule_off[s]; r < S.rule_off[s + 1]; ++r)
          if (rule_app(S.rules[r], v)) {
            if (!d) first = r;
            ++d;
          }
      }
      Fs[s] = first >= 0 ? (uint16_t)(S.rules[first].c | (S.rules[first].p << 8)) : (uint16_t)0;
      any |= d > 0;
      if (d >= 2) {
        const int i = atomicAdd(&nnd, 1);
        if (i < KMAX) {
          nd_s[i] = s;
          nd_d[i] = (uint8_t)d;
        }
      }
    }
    any = __syncthreads_or(any);
    const bool input_left = input_neuron >= 0 && k < train_len;
    if (tid == 0) {
      verdict = 0;
      const int n = nnd;
      uint64_t psi = 1;
      if (n > KMAX) psi = PSI_LIMIT + 1;  // every factor is >= 2
      for (int i = 0; i < n && i < KMAX; ++i) psi = sat_mul(psi, nd_d[i]);
      if (psi > PSI_LIMIT) {
        verdict = 2;
      } else if (!any && !input_left) {
        verdict = 1;
      } else if (any && n > 0) {
        for (int i = 1; i < n; ++i) {  // insertion sort: increasing neuron (first = most significant)
          const int32_t ks = nd_s[i];
          const uint8_t kd = nd_d[i];
          int j = i - 1;
          for (; j >= 0 && nd_s[j] > ks; --j) {
            nd_s[j + 1] = nd_s[j];
            nd_d[j + 1] = nd_d[j];
          }
          nd_s[j + 1] = ks;
          nd_d[j + 1] = kd;
        }
        uint64_t t = splitmix64_dev(splitmix64_dev(seed ^ ((uint64_t)k << 32)) ^ (uint64_t)w) % psi;
        for (int i = n - 1; i >= 0; --i) {
          const int32_t s = nd_s[i];
          const uint64_t d = nd_d[i];
          const int r = nth_applicable(S, s, C[s], (int)(t % d));
          Fs[s] = (uint16_t)(S.rules[r].c | (S.rules[r].p << 8));
          t /= d;
        }
      }
    }
    __syncthreads();
    if (verdict == 2) {
      if (tid == 0) atomicOr(err, ERR_CAPACITY);
      break;
    }
    if (verdict == 1) {
      hs = k;
      break;
    }
    int ovf = 0;
    if (any) {
      for (int32_t j = tid; j < m; j += SAMPLE_CTA) {
        int64_t val = (int64_t)C[j] - (Fs[j] & 0xFF);
        for (int e = S.in_off[j]; e < S.in_off[j + 1]; ++e) val += Fs[S.in_src[e]] >> 8;
        if (j == input_neuron && input_left) val += train[k];
        ovf |= val < 0 || val > S.count_max;
        N[j] = (int32_t)val;
      }
    } else if (tid == 0) {  // nothing fires: only the input arrives
      const int64_t val = (int64_t)C[input_neuron] + train[k];
      ovf |= val < 0 || val > S.count_max;
      C[input_neuron] = (int32_t)val;
    }
    ovf = __syncthreads_or(ovf);
    if (ovf) {
      if (tid == 0) atomicOr(err, ERR_OVERFLOW);
      break;
    }
    if (any) {
      int32_t* t_ = C;
      C = N;
      N = t_;
    }
  }
  if (C != cur + w * m)
    for (int32_t j = tid; j < m; j += SAMPLE_CTA) cur[w * m + j] = C[j];
  if (tid == 0) halted[w] = hs;
}

// ===========================================================================
// launchers
// ===========================================================================
bool fast_expand_ok(const SysView& S) { return S.tables_ok != 0; }

void launch_build_tables(const SysView& S, int32_t bytes, uint8_t* tab, void* ctab, uint8_t* tab_full,
                         uint8_t* ttab, uint8_t* elut, uint8_t* hsg, cudaStream_t st) {
  const uint64_t n = (uint64_t)S.m * S.tabw + ((tab_full || ttab) ? (uint64_t)S.m * 256 : 0);
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_build_tables<T><<<grid_for(n), BLK, 0, st>>>(S, tab, reinterpret_cast<T*>(ctab), tab_full, ttab, elut);
  });
  count_launch();
  if (hsg) {
    k_build_hs<<<grid_for((uint64_t)S.m * 16), BLK, 0, st>>>(S, hsg);
    count_launch();
  }
}

constexpr size_t KC_SMEM_MAX = 220 * 1024;

// K-c warps per CTA: MW for 1-2 byte counts, 8 for int32 (staging fits)
int kc_warps(int32_t bytes) { return bytes == 4 ? 8 : MW; }
bool materialize_narrow_ok(const SysView& S, int32_t bytes);

// warps per K-c CTA for the byte-staged paths: 8 when m <= 4096 (one or a
// few neuron passes per block, so several CTAs per SM overlap one block's
// setup — emit-word staging, child tables — with another's passes), else MW
int kc_cta_warps(const SysView& S, int32_t bytes, bool staged_e) {
  if (bytes > 1 && !materialize_narrow_ok(S, bytes)) return kc_warps(bytes);
  if (!staged_e) return MW;
  const char* e = getenv("SNP_KC_CTA_WARPS");
  if (e && atoi(e) > 0) return atoi(e) == 8 ? 8 : MW;
  return S.m <= 4096 ? 8 : MW;
}

// wide counts (16/32-bit) computed as bytes (NARROW): every count and x of a
// level < 256 in the common case; staging rows of bytes, so the CTA keeps
// MW warps; x outside [0, 255] goes through the overflow list (exact rewrite)
bool materialize_narrow_ok(const SysView& S, int32_t bytes) {
  return bytes > 1 && S.ttab != nullptr && !(S.kernel_flags & KF_KC_WIDE_EXACT);
}

size_t materialize_smem_bytes(const SysView& S, int32_t bytes, bool staged_e) {
  const size_t mE = (size_t)((S.m + 1) & ~1);
  const size_t xsb = bytes == 1 || materialize_narrow_ok(S, bytes) ? (size_t)xs_stride<uint8_t>() : (size_t)(PB * bytes + 4);
  const size_t xs = (size_t)kc_cta_warps(S, bytes, staged_e) * 32 * xsb;
  return (staged_e ? (mE + EPAD) * 8 : 0) + xs + 2 * (QCAP + 32) + (SNP_KC_COOP ? 0 : 8 * OPCAP) + 67 * 8 + 16 + 16;
}

// the tensor-core store variant (uint8): A tiles + one-hot operands instead of
// the staging rows, descriptors and store program; one mbarrier per tile
size_t materialize_tc_smem_bytes(const SysView& S, bool staged_e) {
  const size_t mE = (size_t)((S.m + 1) & ~1);
  return (staged_e ? (mE + EPAD) * 8 : 0) + (size_t)MW / 4 * KCT_ATILE + KCT_BBYTES + (QCAP + 32) + 66 * 8 + 8 +
         8 * (MW / 4) + 16 + 16;
}

// opt-in (SNP_KERNELS=kc_tc): measured slower at config 4 (K-c 73.2 vs 55.3 ms
// per level, profiles/r02/ab_kc_tc.json): correct, and it moves the shared
// wavefronts off the LSU (1.83e9 -> 0.70e9 at F = 2^20), but each lane's
// sector stores touch 32 rows (16 lines per instruction) and the window ends
// need up to 9 masked pieces, and the per-tile barrier + MMA round trip every
// 1024 neurons leaves warps waiting (long-scoreboard 40 % of the samples)
bool materialize_tc_ok(const SysView& S, int32_t bytes, bool staged_e) {
  return bytes == 1 && (S.kernel_flags & KF_KC_TC) && materialize_tc_smem_bytes(S, staged_e) <= KC_SMEM_MAX;
}

// emit words staged in shared memory when they fit (else read from L2)
bool materialize_stage_e(const SysView& S, int32_t bytes) {
  return !(S.kernel_flags & KF_KC_GLOBAL_E) && materialize_smem_bytes(S, bytes, true) <= KC_SMEM_MAX;
}

bool fast_materialize_ok(const SysView& S) {
  const int32_t w = S.count_max <= 255 ? 1 : S.count_max <= 65535 ? 2 : 4;
  return S.delay_m == 0 && S.tables_ok && S.binary_emit && S.max_indeg < 256 && materialize_smem_bytes(S, w, false) <= KC_SMEM_MAX;
}

void launch_import(const void* src, int32_t src_bytes, int32_t src_layout, int64_t src_ld, int64_t F, int32_t m,
                   void* dst, int32_t dst_bytes, int64_t count_max, int32_t* err, cudaStream_t st) {
  dim3 grid((unsigned)((F + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  dispatch_bytes(src_bytes, [&](auto tin) {
    using Tin = decltype(tin);
    dispatch_bytes(dst_bytes, [&](auto tout) {
      using Tout = decltype(tout);
      k_import<Tin, Tout><<<grid, block, 0, st>>>(src, src_layout, src_ld, F, m, reinterpret_cast<Tout*>(dst),
                                                  count_max, err);
    });
  });
  count_launch();
}

void launch_export(const void* src, int32_t bytes, int64_t F, int32_t m, int32_t* dst, cudaStream_t st) {
  dim3 grid((unsigned)((F + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_export<T><<<grid, block, 0, st>>>(reinterpret_cast<const T*>(src), F, m, dst);
  });
  count_launch();
}

void launch_fingerprint(const SysView& S, int32_t bytes, const void* data, int64_t F, uint64_t* fp0, uint64_t* fp1,
                        cudaStream_t st) {
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_fingerprint<T><<<grid_for(F), BLK, 0, st>>>(S, reinterpret_cast<const T*>(data), F, fp0, fp1);
  });
  count_launch();
}

static unsigned expand_grid(int64_t F) { return (unsigned)((F + XW * XTILE - 1) / (XW * XTILE)); }

void launch_expand(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, cudaStream_t st) {
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    if (S.delay_m > 0) {
      k_expand_delay<T><<<grid_for(L.F), BLK, 0, st>>>(S, L, O);
    } else if (!fast_expand_ok(S)) {
      k_expand_g<T><<<expand_grid(L.F), XW * 32, 0, st>>>(S, L, O);
    } else {
      const bool full = S.full8 && sizeof(T) == 1;
      const size_t smem = expand_smem_bytes<T>(full ? 256 : S.tabw);
      auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<expand_grid(L.F), XW * 32, smem, st>>>(S, L, O);
      };
      if ((full || sizeof(T) > 1) && S.tc_ok && !(S.kernel_flags & (KF_EXPAND_T | KF_NO_TC))) {
        const size_t sm = expand_tc_smem_bytes();
        auto kern = SNP_TC_WS ? k_expand_tc<true, T> : k_expand_tc<false, T>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (SNP_TC_MINB > 3) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        const int64_t nblk = (L.F + PB - 1) / PB;
        kern<<<(unsigned)((nblk + 1) / 2), TCT + (SNP_TC_WS ? 32 : 0), sm, st>>>(S, L, O);
        if (!O.classify_only) {
          k_nd_pass<T><<<grid_for(L.F), BLK, 0, st>>>(S, L, O);
          count_launch();
        }
      } else if (full && S.any_generic == 0 && S.hsg != nullptr && !(S.kernel_flags & KF_EXPAND_T)) {
        const size_t sq = expand_q_smem_bytes();
        cudaFuncSetAttribute(k_expand_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sq);
        const unsigned g = (unsigned)((L.F + QB * PB - 1) / (QB * PB));
        k_expand_q<<<g, QW * 32, sq, st>>>(S, L, O);
      } else if (full) {
        go(k_expand_t<T, true>);
      } else {
        go(k_expand_t<T, false>);
      }
    }
  });
  count_launch();
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

void launch_winners(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, unsigned long long* n_new,
                    cudaStream_t st) {
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
                    uint64_t level_ref, int insert_visited, int32_t* err, cudaStream_t st) {
  k_compact<<<grid_for(T), BLK, 0, st>>>(C, off, T, N, tb, level_ref, insert_visited, err);
  count_launch();
}

void launch_kq_off(const uint64_t* off, const uint64_t* kpos, int64_t F, uint64_t* kq_off, cudaStream_t st) {
  k_kq_off<<<grid_for(F + 1), BLK, 0, st>>>(off, kpos, F, kq_off);
  count_launch();
}

// one K-c variant, NPL (bit planes of the in-synapse count) by the largest in-degree
template <typename T, bool ES, int MWT, bool TCS, bool NARROW>
void go_materialize(const SysView& S, const LevelView& L, const ExpandOut& O, const uint64_t* kq_off,
                    const NextArrays& N, uint64_t* ovf, unsigned long long* n_ovf, uint64_t ovf_cap, size_t smem,
                    cudaStream_t st) {
  const unsigned nblk = (unsigned)((L.F + PB - 1) / PB);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<nblk, MWT * 32, smem, st>>>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap);
  };
  if (S.max_indeg < 16) go(k_materialize_bs<T, 4, ES, MWT, TCS, NARROW>);
  else if (S.max_indeg < 32) go(k_materialize_bs<T, 5, ES, MWT, TCS, NARROW>);
  else if (S.max_indeg < 64) go(k_materialize_bs<T, 6, ES, MWT, TCS, NARROW>);
  else go(k_materialize_bs<T, 8, ES, MWT, TCS, NARROW>);
}

void launch_materialize(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O,
                        const uint64_t* kq_off, const NextArrays& N, int64_t K, uint64_t* ovf,
                        unsigned long long* n_ovf, uint64_t ovf_cap, int32_t* err, cudaStream_t st) {
  if (K <= 0) return;
  if (fast_materialize_ok(S)) {
    const bool staged = materialize_stage_e(S, bytes);
    const bool tcs = materialize_tc_ok(S, bytes, staged);
    const bool narrow = materialize_narrow_ok(S, bytes);
    const int cw = kc_cta_warps(S, bytes, staged);
    const size_t smem = tcs ? materialize_tc_smem_bytes(S, staged) : materialize_smem_bytes(S, bytes, staged);
    dispatch_bytes(bytes, [&](auto tt) {
      using T = decltype(tt);
      if constexpr (sizeof(T) > 1) {
        if (narrow) {
          if (staged && cw == 8) go_materialize<T, true, 8, false, true>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
          else if (staged) go_materialize<T, true, MW, false, true>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
          else go_materialize<T, false, MW, false, true>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
        } else if (staged) {
          go_materialize<T, true, sizeof(T) == 4 ? 8 : MW, false, false>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
        } else {
          go_materialize<T, false, sizeof(T) == 4 ? 8 : MW, false, false>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
        }
      } else {
        if (tcs && staged) go_materialize<T, true, MW, true, false>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
        else if (tcs) go_materialize<T, false, MW, true, false>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
        else if (staged && cw == 8) go_materialize<T, true, 8, false, false>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
        else if (staged) go_materialize<T, true, MW, false, false>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
        else go_materialize<T, false, MW, false, false>(S, L, O, kq_off, N, ovf, n_ovf, ovf_cap, smem, st);
      }
    });
  } else {
    unsigned g = grid_for((uint64_t)K * 32, 256);
    if (g > 148u * 32u) g = 148u * 32u;
    dispatch_bytes(bytes, [&](auto tt) {
      using T = decltype(tt);
      const size_t sm = delay_smem_bytes(S.delay_m);
      if (S.delay_m > 0 && sm <= 200 * 1024) {
        cudaFuncSetAttribute(k_materialize_delay_s<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_materialize_delay_s<T><<<g, DELAY_WARPS * 32, sm, st>>>(S, L, O, N, K, err);
      } else if (S.delay_m > 0) {
        k_materialize_delay<T><<<g, 256, 0, st>>>(S, L, O, N, K, err);
      } else if ((size_t)8 * 8 * S.m <= 200 * 1024) {
        const size_t sme = (size_t)8 * 8 * S.m;
        cudaFuncSetAttribute(k_materialize_exact_s<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sme);
        k_materialize_exact_s<T><<<g, 256, sme, st>>>(S, L, O, N, K, err);
      } else {
        k_materialize_exact<T><<<g, 256, 0, st>>>(S, L, O, N, K, err);
      }
    });
  }
  count_launch();
}

void launch_aug_keys(const SysView& S, int32_t bytes, const LevelView& L, const uint64_t* off, const ExpandOut& O,
                     uint64_t T, const ChildArrays& C, int32_t* err, cudaStream_t st) {
  if (T == 0) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using TT = decltype(tt);
    k_aug_keys<TT><<<grid_for(T, 128), 128, 0, st>>>(S, L, off, O, T, C, err);
  });
  count_launch();
}

void launch_aug_fix(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const NextArrays& N,
                    int64_t K, int32_t* err, cudaStream_t st) {
  if (K <= 0) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using TT = decltype(tt);
    k_aug_fix<TT><<<grid_for(K, 128), 128, 0, st>>>(S, L, O, N, K, err);
  });
  count_launch();
}

void launch_patch(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const NextArrays& N,
                  int64_t K, int32_t* err, cudaStream_t st) {
  if (K <= 0 || !fast_materialize_ok(S)) return;  // the exact path needs no patch
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_patch<T><<<grid_for(K, 128), 128, 0, st>>>(S, L, O, N, K, err);
  });
  count_launch();
}

void launch_overflow_fix(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O,
                         const uint64_t* kq_off, const NextArrays& N, const uint64_t* ovf, uint64_t n_ovf,
                         int32_t* err, cudaStream_t st) {
  if (!n_ovf) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_overflow_fix<T><<<grid_for(n_ovf, 128), 128, 0, st>>>(S, L, O, kq_off, N, ovf, n_ovf, err);
  });
  count_launch();
}

void launch_verify_list(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, uint64_t* list,
                        unsigned long long* n_list, cudaStream_t st) {
  cudaMemsetAsync(n_list, 0, sizeof(unsigned long long), st);
  if (!T) return;
  k_verify_need<<<grid_for(T), BLK, 0, st>>>(C, T, tag_base, tb, list, n_list);
  count_launch();
}

size_t verify2_row_bytes(const SysView& S) { return (size_t)2 * S.m * ((S.small_cp ? 2 : 8) + 4); }

void launch_verify_batch(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const uint64_t* off,
                         const ChildArrays& C, const uint64_t* list, uint64_t i0, uint64_t n, uint64_t tag_base,
                         const Tables& tb, const StoredLevel* stored, void* fc, int32_t* err, cudaStream_t st) {
  if (!n) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using TT = decltype(tt);
    const unsigned gw = (unsigned)std::min<uint64_t>((n * 32 + 255) / 256, 148u * 32u);
    dim3 gc((unsigned)std::min<int64_t>((S.m + 255) / 256, 64), (unsigned)std::min<uint64_t>(n, 65535));
    uint8_t* fcb = reinterpret_cast<uint8_t*>(fc);
    if (S.small_cp) {
      k_verify_fc<TT, uint16_t><<<gw, 256, 0, st>>>(S, L, O, off, C, list, i0, n, tag_base, tb, fcb);
      k_verify_cols<TT, uint16_t><<<gc, 256, 0, st>>>(S, L, C, list, i0, n, tag_base, tb, fcb, stored, err);
    } else {
      k_verify_fc<TT, int2><<<gw, 256, 0, st>>>(S, L, O, off, C, list, i0, n, tag_base, tb, fcb);
      k_verify_cols<TT, int2><<<gc, 256, 0, st>>>(S, L, C, list, i0, n, tag_base, tb, fcb, stored, err);
    }
  });
  count_launch(2);
}

// cpT[v][s] = c | p << 8 of neuron s's first applicable rule at count v < 32
__global__ void k_build_cpT(SysView S, uint16_t* cpT) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)32 * S.m) return;
  const int32_t v = (int32_t)(i / S.m), s = (int32_t)(i % S.m);
  const int r = first_rule(S, s, v);
  cpT[i] = r >= 0 ? (uint16_t)(S.rules[r].c | (S.rules[r].p << 8)) : (uint16_t)0;
}

void launch_build_cpT(const SysView& S, uint16_t* cpT, cudaStream_t st) {
  k_build_cpT<<<grid_for((uint64_t)32 * S.m), BLK, 0, st>>>(S, cpT);
  count_launch();
}

// dedup = 0: the listed key matches, one CTA each (k_verify_m); false when the
// per-CTA rows do not fit shared memory (the batched two-pass path instead)
bool launch_verify_m(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const uint64_t* off,
                     const ChildArrays& C, const uint64_t* list, const unsigned long long* n_list, uint64_t tag_base,
                     const Tables& tb, const StoredLevel* stored, int32_t* err, cudaStream_t st) {
  if (S.delay_m > 0 || S.aug_rule >= 0 || KMAX > VM_THREADS) return false;
  const bool pk = S.small_cp != 0;
  const size_t sm = verify_m_smem_bytes(S.m, pk);
  if (sm > 200 * 1024) return false;
  const unsigned per_sm =
      (unsigned)std::max<size_t>(1, std::min<size_t>(2048 / (VM_THREADS + 32), (size_t)(220 * 1024) / (sm + 1024)));
  dispatch_bytes(bytes, [&](auto tt) {
    using TT = decltype(tt);
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<148u * per_sm, VM_THREADS + 32, sm, st>>>(S, L, O, off, C, list, n_list, tag_base, tb, stored, err);
    };
    if (pk) go(k_verify_m<TT, true>);
    else go(k_verify_m<TT, false>);
  });
  count_launch();
  return true;
}

void launch_verify(const SysView& S, int32_t bytes, const LevelView& L, const ExpandOut& O, const uint64_t* off,
                   const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, const StoredLevel* stored,
                   uint64_t* list, unsigned long long* n_list, int32_t* err, cudaStream_t st) {
  if (!T) return;
  unsigned g = grid_for(T * 32, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  dispatch_bytes(bytes, [&](auto tt) {
    using TT = decltype(tt);
    const size_t sm = verify_smem_bytes(S.m, S.small_cp ? 2 : 8);
    if (sm <= 200 * 1024 && S.delay_m == 0) {
      cudaMemsetAsync(n_list, 0, sizeof(unsigned long long), st);
      k_verify_need<<<grid_for(T), BLK, 0, st>>>(C, T, tag_base, tb, list, n_list);
      count_launch();
      const unsigned per_sm = (unsigned)std::max<size_t>(1, std::min<size_t>(8, (200u * 1024u) / sm));
      if (S.small_cp) {
        cudaFuncSetAttribute(k_verify_s<TT, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_verify_s<TT, uint16_t><<<148u * per_sm, VERIFY_WARPS * 32, sm, st>>>(S, L, O, off, C, list, n_list,
                                                                                tag_base, tb, stored, err);
      } else {
        cudaFuncSetAttribute(k_verify_s<TT, int2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_verify_s<TT, int2><<<148u * per_sm, VERIFY_WARPS * 32, sm, st>>>(S, L, O, off, C, list, n_list, tag_base,
                                                                            tb, stored, err);
      }
    } else {
      k_verify<TT><<<g, 256, 0, st>>>(S, L, O, off, C, T, tag_base, tb, stored, err);
    }
  });
  count_launch();
}

void launch_level0_compact(const uint8_t* verdict, const uint64_t* kept, const uint64_t* kpos, int64_t F0,
                           const uint64_t* fp0, const uint64_t* fp1, const NextArrays& N, uint64_t* src_index,
                           const Tables& tb, int insert_visited, int32_t* err, cudaStream_t st) {
  k_level0_compact<<<grid_for(F0), BLK, 0, st>>>(verdict, kept, kpos, F0, fp0, fp1, N, src_index, tb, insert_visited,
                                                  err);
  count_launch();
}

void launch_gather_columns(int32_t bytes, const void* src, const uint64_t* src_index, int64_t K, int32_t m, void* dst,
                           cudaStream_t st) {
  if (K <= 0) return;
  dim3 grid(grid_for(K), (unsigned)min(m, 1024));
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_gather_columns<T><<<grid, BLK, 0, st>>>(reinterpret_cast<const T*>(src), src_index, K, m,
                                              reinterpret_cast<T*>(dst));
  });
  count_launch();
}

void launch_zero_tail(int32_t bytes, void* data, int64_t F, int32_t m, cudaStream_t st) {
  if (F % PB == 0 || !data) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_zero_tail<T><<<grid_for((uint64_t)m * (PB - F % PB)), BLK, 0, st>>>(reinterpret_cast<T*>(data), F, m);
  });
  count_launch();
}

void launch_small_bfs(const SysView& S, int32_t bytes, const SmallArgs& a, cudaStream_t st) {
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    const char* e = getenv("SNP_SMALL_NT");
    const int nt = e ? atoi(e) : (a.F <= 32 ? 128 : 1024);
    if (nt == 128) k_small_bfs<T, 128><<<1, 128, 0, st>>>(S, a);
    else k_small_bfs<T, 1024><<<1, 1024, 0, st>>>(S, a);
  });
  count_launch();
}

void launch_pack_edges(const EdgeSrc* lv, int32_t nlev, int64_t max_F, int64_t* parent, uint64_t* t,
                       uint8_t* halting, uint64_t* fp2, cudaStream_t st) {
  if (nlev <= 0 || max_F <= 0) return;
  dim3 grid((unsigned)std::min<int64_t>((max_F + BLK - 1) / BLK, 4096), (unsigned)std::min(nlev, 65535));
  k_pack_edges<<<grid, BLK, 0, st>>>(lv, nlev, parent, t, halting, fp2);
  count_launch();
}

void launch_add_i64(int64_t* a, int64_t n, int64_t add, cudaStream_t st) {
  if (n <= 0 || add == 0) return;
  k_add_i64<<<grid_for((uint64_t)n), BLK, 0, st>>>(a, n, add);
  count_launch();
}

void launch_verify_level0(int32_t bytes, const void* data, int32_t m, const ChildArrays& C, uint64_t F0,
                          const Tables& tb, int32_t* err, cudaStream_t st) {
  unsigned g = grid_for(F0 * 32, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_verify_level0<T><<<g, 256, 0, st>>>(reinterpret_cast<const T*>(data), m, C, F0, tb, err);
  });
  count_launch();
}

void launch_rehash(const Slot* old_tab, uint64_t old_cap, Slot* new_tab, uint64_t new_mask, int32_t* err,
                   cudaStream_t st) {
  k_rehash<<<grid_for(old_cap), BLK, 0, st>>>(old_tab, old_cap, new_tab, new_mask, err);
  count_launch();
}

void launch_digest(const NextArrays& N, int64_t K, uint64_t level, int64_t q_offset, int64_t parent_offset,
                   unsigned long long* digest, cudaStream_t st) {
  if (K <= 0) return;
  unsigned g = grid_for(K);
  if (g > 148u * 8u) g = 148u * 8u;
  k_digest<<<g, BLK, 0, st>>>(N, K, level, q_offset, parent_offset, digest);
  count_launch();
}

void launch_owner_hist(const uint64_t* fp1, uint64_t T, uint32_t P, unsigned long long* counts, cudaStream_t st) {
  if (!T) return;
  unsigned g = grid_for(T);
  if (g > 148u * 16u) g = 148u * 16u;
  k_owner_hist<<<g, BLK, (size_t)P * 4, st>>>(fp1, T, P, counts);
  count_launch();
}

void launch_owner_pack(const uint64_t* fp0, const uint64_t* fp1, uint64_t T, uint32_t P, uint64_t tag_base,
                       unsigned long long* cursor, uint64_t* perm, uint64_t* send, cudaStream_t st) {
  if (!T) return;
  k_owner_pack<<<grid_for(T), BLK, (size_t)P * 12, st>>>(fp0, fp1, T, P, tag_base, cursor, perm, send);
  count_launch();
}

void launch_owner_dedup(const uint64_t* recv, uint64_t R, const Tables& tb, uint8_t* verdict, uint64_t* slot,
                        int32_t* err, cudaStream_t st) {
  if (!R) return;
  k_owner_dedup<<<grid_for(R), BLK, 0, st>>>(recv, R, tb, verdict, slot, err);
  count_launch();
}

void launch_owner_winners(const uint64_t* recv, uint64_t R, const Tables& tb, const uint8_t* verdict,
                          const uint64_t* slot, unsigned long long* n_new, cudaStream_t st) {
  if (!R) return;
  unsigned g = grid_for(R);
  if (g > 148u * 16u) g = 148u * 16u;
  k_owner_winners<<<g, BLK, 0, st>>>(recv, R, tb, verdict, slot, n_new);
  count_launch();
}

void launch_owner_keep(const uint64_t* recv, uint64_t R, const Tables& tb, const uint8_t* verdict,
                       const uint64_t* slot, uint64_t tau, int thin, uint8_t* out, unsigned long long* n_kept,
                       int32_t* err, cudaStream_t st) {
  if (!R) return;
  k_owner_keep<<<grid_for(R), BLK, 0, st>>>(recv, R, tb, verdict, slot, tau, thin, out, n_kept, err);
  count_launch();
}

void launch_unperm(const uint64_t* perm, const uint8_t* back, uint64_t T, uint64_t* kept, cudaStream_t st) {
  k_unperm<<<grid_for(T + 1), BLK, 0, st>>>(perm, back, T, kept);
  count_launch();
}

void launch_spiking_vectors(const SysView& S, int32_t bytes, const void* parent_data, const int64_t* parent,
                            const uint64_t* t, int64_t K, uint8_t* S_out, int32_t* err, cudaStream_t st) {
  if (K <= 0) return;
  dispatch_bytes(bytes, [&](auto tt) {
    using T = decltype(tt);
    k_spiking_vectors<T><<<grid_for(K, 128), 128, 0, st>>>(S, reinterpret_cast<const T*>(parent_data), parent, t, K,
                                                         S_out, err);
  });
  count_launch();
}

void launch_all_edges(const ChildArrays& C, uint64_t T, uint64_t tag_base, const Tables& tb, uint64_t next_ref,
                      uint64_t* ref, cudaStream_t st) {
  if (T == 0) return;
  k_all_edges<<<grid_for((int64_t)T, BLK), BLK, 0, st>>>(C, T, tag_base, tb, next_ref, ref);
  count_launch();
}

void launch_child_keys_delay(const SysView& S, int32_t bytes, const LevelView& L, const uint64_t* off,
                             const ExpandOut& O, uint64_t T, const ChildArrays& C, cudaStream_t st) {
  unsigned g = grid_for(T * 32, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  const size_t sm = delay_smem_bytes(S.delay_m);
  dispatch_bytes(bytes, [&](auto tt) {
    using TT = decltype(tt);
    if (sm <= 200 * 1024) {
      cudaFuncSetAttribute(k_child_keys_delay_s<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_child_keys_delay_s<TT><<<g, DELAY_WARPS * 32, sm, st>>>(S, L, off, O, T, C);
    } else {
      k_child_keys_delay<TT><<<g, 256, 0, st>>>(S, L, off, O, T, C);
    }
  });
  count_launch();
}

void launch_sample(const SysView& S, int64_t W, int32_t* cur, int32_t* nxt, uint64_t* fired, uint64_t seed,
                   int32_t steps, int32_t input_neuron, const int32_t* train, int32_t train_len, int32_t* halted,
                   int32_t* err, bool small_rules, cudaStream_t st) {
  const size_t smem = (size_t)S.m * 2;
  if (small_rules && smem <= 200 * 1024) {
    cudaFuncSetAttribute(k_sample_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sample_cta<<<(unsigned)W, SAMPLE_CTA, smem, st>>>(S, cur, nxt, seed, steps, input_neuron, train, train_len,
                                                        halted, err);
    count_launch();
    return;
  }
  const int64_t blocks = (W + SAMPLE_WARPS - 1) / SAMPLE_WARPS;
  k_sample<<<(unsigned)blocks, SAMPLE_WARPS * 32, 0, st>>>(S, W, cur, nxt, fired, seed, steps, input_neuron, train,
                                                           train_len, halted, err);
  count_launch();
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
