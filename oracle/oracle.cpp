// ============================================================================
// oracle.cpp — plain, slow, obviously-correct CPU oracle for the batched SNP
// transition step  C_{k+1} = C_k + S_k · M_Π  and the breadth-first
// computation tree it grows.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.  It
// shares no code, header, table or constant generator with the CUDA engine
// under paper_1104_1824_b200/ (the engine must never route through it).
//
// Source of truth: /root/reference/PAPER.md, Cabarle, Adorna, Martínez-del-Amor,
// "Simulating Spiking Neural P systems without delays using GPUs".
// Every function cites the passage it follows as PAPER.md:<line> (§, eq., alg.).
// Readings of silent / garbled passages are the A-numbered readings listed in
// DESIGN.md §3 (they follow SURVEY.md §8(c)).
//
// Arithmetic: spike counts are exact int64 (the paper's host uses unbounded
// Python ints); fingerprints are arithmetic mod 2^64 (DESIGN.md
// reading A18).  No blocking, fusion or reordering beyond the definitions.
// ============================================================================
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <string>
#include <vector>
#include <set>
#include <map>
#include <thread>
#include <unordered_map>
#include <functional>
#include <utility>
#include <algorithm>

namespace {

// Status codes (defined here independently of the engine's header).
enum {
  OR_OK = 0,
  OR_E_ARG = -1,
  OR_E_INVALID_SYSTEM = -2,
  OR_E_OVERFLOW = -3,
  OR_E_CAPACITY = -4,
};

enum { RE_EXACT = 0, RE_PERIODIC = 1, RE_UNARY = 2 };

// One rule  E/a^c -> a^p  of neuron σ (Def. 1 (b-1)); p = 0 is a
// forgetting rule ((b-2)).  The regular expression E is either
//   EXACT(k)       E = a^k          (form (b-3))
//   PERIODIC(i,j)  E = a^i (a^j)*   (the paper-simulator reading, A1)
//   UNARY(t,P)     any regular E over {a} (the paper's
//                  future work).  L(E) ⊆ a* is ultimately
//                  periodic, so it is given by its membership bits
//                  member[v] for v < t + P, with a^v ∈ L(E) for v >= t + P
//                  iff member[t + (v - t) mod P].
struct Rule {
  int64_t neuron;
  int64_t kind;
  int64_t a;  // k (EXACT), i (PERIODIC) or t (UNARY)
  int64_t b;  // j (PERIODIC), P (UNARY), unused for EXACT
  int64_t consumed;  // c >= 1
  int64_t produced;  // p >= 0
  std::vector<uint8_t> member;  // UNARY: t + P membership bits
};

struct System {
  int64_t m = 0;  // neurons
  int64_t n = 0;  // rules, in the paper's total order
  std::vector<Rule> rules;
  // M_Π (Def. 2): n rows (rules) x m columns (neurons),
  // held as a plain compressed-row list of (column, value) per rule.
  std::vector<std::vector<std::pair<int64_t, int64_t>>> M_rows;
};

// ---------------------------------------------------------------------------
// a^v ∈ L(E)?  (regex kinds per reading A1)
bool regex_matches(const Rule& r, int64_t v) {
  if (r.kind == RE_EXACT) return v == r.a;
  if (r.kind == RE_UNARY) return r.member[v < r.a + r.b ? v : r.a + (v - r.a) % r.b] != 0;
  // PERIODIC(i, j): v = i + x·j for some x >= 0  ((v - i) mod j == 0; for a
  // power-of-two j that is a mask of the low bits)
  if (v < r.a) return false;
  if ((r.b & (r.b - 1)) == 0) return ((v - r.a) & (r.b - 1)) == 0;
  return (v - r.a) % r.b == 0;
}

// Rule applicability: the neuron holds v spikes, a^v ∈ L(E) and
// v >= c.
bool applicable(const Rule& r, const std::vector<int64_t>& C) {
  int64_t v = C[r.neuron];
  return regex_matches(r, v) && v >= r.consumed;
}

// Alg. 2 step II-1 (worked example 268-294): copy of the rule
// list where every applicable rule of a neuron is marked 1, 2, 3, ... in the
// total order, and every non-applicable rule is marked 0.
std::vector<int64_t> mark_applicable(const System& sys, const std::vector<int64_t>& C) {
  std::vector<int64_t> tmp(sys.n, 0);
  std::vector<int64_t> running(sys.m, 0);
  for (int64_t r = 0; r < sys.n; ++r) {
    if (applicable(sys.rules[r], C)) {
      running[sys.rules[r].neuron] += 1;
      tmp[r] = running[sys.rules[r].neuron];
    }
  }
  return tmp;
}

// A_s for every neuron s: its applicable rules in total order, held in one
// buffer (rules are grouped by non-decreasing neuron, validate()): A[s] is a
// view with empty() / size() / operator[], A.size() = m.
class RuleSets {
 public:
  struct View {
    const int64_t* p;
    size_t n;
    bool empty() const { return n == 0; }
    size_t size() const { return n; }
    int64_t operator[](size_t i) const { return p[i]; }
  };
  explicit RuleSets(int64_t m = 0) : off_(m + 1, 0), last_(-1) {}
  void add(int64_t s, int64_t r) {  // s non-decreasing
    for (int64_t k = last_ + 1; k <= s; ++k) off_[k] = (int64_t)rules_.size();
    last_ = s;
    rules_.push_back(r);
  }
  void finish() {
    for (int64_t k = last_ + 1; k < (int64_t)off_.size(); ++k) off_[k] = (int64_t)rules_.size();
    last_ = (int64_t)off_.size() - 1;
  }
  size_t size() const { return off_.size() - 1; }
  View operator[](int64_t s) const { return View{rules_.data() + off_[s], (size_t)(off_[s + 1] - off_[s])}; }

 private:
  std::vector<int64_t> rules_, off_;
  int64_t last_;
};

// |σ_{V_i}| of eq. (8): the number of applicable rules of
// each neuron, in increasing neuron order; A_s = those rules in total order.
RuleSets applicable_rules_per_neuron(const System& sys, const std::vector<int64_t>& C) {
  RuleSets A(sys.m);
  for (int64_t r = 0; r < sys.n; ++r)
    if (applicable(sys.rules[r], C)) A.add(sys.rules[r].neuron, r);
  A.finish();
  return A;
}

// Ψ, eq. (8): product of |σ_{V_i}| over the neurons.  Reading
// A3: a neuron with no applicable rule contributes a factor 1 (it does not
// fire); reading A5: if no neuron has an applicable rule the configuration is
// halting and has no children (Ψ = 0).  Returns false if Ψ exceeds 2^62.
bool count_children(const RuleSets& A, uint64_t* psi) {
  bool any = false;
  unsigned __int128 prod = 1;
  for (int64_t s = 0; s < (int64_t)A.size(); ++s) {
    const auto As = A[s];
    if (As.empty()) continue;
    any = true;
    prod *= (unsigned __int128)As.size();
    if (prod > ((unsigned __int128)1 << 62)) return false;
  }
  *psi = any ? (uint64_t)prod : 0;
  return true;
}

// Alg. 2 steps II-2/II-3: the t-th valid spiking
// vector, t in [0, Ψ).  II-3 distributes every string of the first neuron over
// the strings of the next ones, so the first neuron with applicable rules is
// the most significant mixed-radix digit (tmp3 = ['10110','01110'],
// PAPER.md:351, 376; reading A7).  Digit x_s selects A_s[x_s]; exactly one
// rule fires per neuron with applicable rules (reading A4).
std::vector<uint8_t> spiking_vector(const System& sys, const RuleSets& A, uint64_t t) {
  std::vector<uint8_t> S(sys.n, 0);
  for (int64_t s = sys.m - 1; s >= 0; --s) {  // least significant digit last
    if (A[s].empty()) continue;
    if (A[s].size() == 1) {  // radix 1: the digit is 0 and t is unchanged (t mod 1 = 0, t / 1 = t)
      S[A[s][0]] = 1;
      continue;
    }
    uint64_t d = A[s].size();
    uint64_t x = t % d;
    t /= d;
    S[A[s][x]] = 1;
  }
  return S;
}

// Eq. (2): C_{k+1} = C_k + S_k · M_Π, as the plain row sum
// of M_Π over the rules that fire, in exact int64 arithmetic.
std::vector<int64_t> transition(const System& sys, const std::vector<int64_t>& C,
                                const std::vector<uint8_t>& S) {
  std::vector<int64_t> Cn = C;
  for (int64_t r = 0; r < sys.n; ++r) {
    if (!S[r]) continue;
    for (const auto& jv : sys.M_rows[r]) Cn[jv.first] += jv.second;
  }
  return Cn;
}

// ---- fingerprints (reading A18; used as the dedup key in mode dedup=1 and
// as the thinning key in both modes) ---------------------------------------
uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xFF51AFD7ED558CCDULL;
  k ^= k >> 33;
  k *= 0xC4CEB9FE1A85EC53ULL;
  k ^= k >> 33;
  return k;
}
// fp_ℓ(C) = Σ_j C[j]·R_ℓ[j] mod 2^64, R_ℓ[j] = splitmix64(seed_ℓ XOR j) | 1.
std::pair<uint64_t, uint64_t> fingerprint(const std::vector<int64_t>& C, uint64_t seed0, uint64_t seed1) {
  uint64_t f0 = 0, f1 = 0;
  for (size_t j = 0; j < C.size(); ++j) {
    uint64_t R0 = splitmix64(seed0 ^ (uint64_t)j) | 1ULL;
    uint64_t R1 = splitmix64(seed1 ^ (uint64_t)j) | 1ULL;
    f0 += (uint64_t)C[j] * R0;
    f1 += (uint64_t)C[j] * R1;
  }
  return {f0, f1};
}

// The same fingerprint with the weights R_ℓ[j] computed once per run instead
// of once per (configuration, neuron) — for the large runs of oracle_explore_par.
struct FpWeights {
  std::vector<uint64_t> R0, R1;
  FpWeights(int64_t m, uint64_t seed0, uint64_t seed1) : R0(m), R1(m) {
    for (int64_t j = 0; j < m; ++j) {
      R0[j] = splitmix64(seed0 ^ (uint64_t)j) | 1ULL;
      R1[j] = splitmix64(seed1 ^ (uint64_t)j) | 1ULL;
    }
  }
  std::pair<uint64_t, uint64_t> operator()(const std::vector<int64_t>& C) const {
    uint64_t f0 = 0, f1 = 0;
    for (size_t j = 0; j < C.size(); ++j) {
      f0 += (uint64_t)C[j] * R0[j];
      f1 += (uint64_t)C[j] * R1[j];
    }
    return {f0, f1};
  }
};

// ---- validation (SURVEY §8(b) list; Def. 1 and Def. 2) --------------------
std::string validate(const System& sys) {
  char buf[256];
  for (int64_t r = 0; r < sys.n; ++r) {
    const Rule& R = sys.rules[r];
    if (R.neuron < 0 || R.neuron >= sys.m) { snprintf(buf, sizeof buf, "rule %lld: neuron out of range", (long long)r); return buf; }
    if (r > 0 && R.neuron < sys.rules[r - 1].neuron) { snprintf(buf, sizeof buf, "rule %lld: rules not grouped by neuron", (long long)r); return buf; }
    if (R.kind != RE_EXACT && R.kind != RE_PERIODIC && R.kind != RE_UNARY) { snprintf(buf, sizeof buf, "rule %lld: bad regex kind", (long long)r); return buf; }
    if (R.kind == RE_UNARY && (R.b < 1 || R.a + R.b > 256 || R.member.size() != (size_t)(R.a + R.b))) { snprintf(buf, sizeof buf, "rule %lld: unary regex needs P >= 1, t + P <= 256 and its bits", (long long)r); return buf; }
    if (R.consumed < 1) { snprintf(buf, sizeof buf, "rule %lld: c < 1", (long long)r); return buf; }
    if (R.produced < 0) { snprintf(buf, sizeof buf, "rule %lld: p < 0", (long long)r); return buf; }
    if (R.a < 0) { snprintf(buf, sizeof buf, "rule %lld: regex exponent < 0", (long long)r); return buf; }
    if (R.kind == RE_PERIODIC && R.b < 1) { snprintf(buf, sizeof buf, "rule %lld: period j < 1", (long long)r); return buf; }
  }
  std::vector<int64_t> per_neuron(sys.m, 0);
  for (const Rule& R : sys.rules) per_neuron[R.neuron]++;
  for (int64_t s = 0; s < sys.m; ++s)
    if (per_neuron[s] > 255) { snprintf(buf, sizeof buf, "neuron %lld: more than 255 rules", (long long)s); return buf; }
  // Def. 2: a_{r,σ(r)} = -c ; a_{r,j} = p if (σ(r), j) ∈ syn, else 0.  All
  // spiking rules of a neuron share that neuron's synapse set.
  std::vector<std::vector<int64_t>> syn_of(sys.m);
  std::vector<int> syn_seen(sys.m, 0);
  for (int64_t r = 0; r < sys.n; ++r) {
    const Rule& R = sys.rules[r];
    bool diag = false;
    std::vector<int64_t> targets;
    for (const auto& jv : sys.M_rows[r]) {
      if (jv.first < 0 || jv.first >= sys.m) { snprintf(buf, sizeof buf, "M row %lld: column out of range", (long long)r); return buf; }
      if (jv.second == 0) continue;
      if (jv.first == R.neuron) {
        if (jv.second != -R.consumed) { snprintf(buf, sizeof buf, "M[%lld][%lld] != -c", (long long)r, (long long)jv.first); return buf; }
        diag = true;
      } else {
        if (jv.second != R.produced) { snprintf(buf, sizeof buf, "M[%lld][%lld] not in {0, p}", (long long)r, (long long)jv.first); return buf; }
        targets.push_back(jv.first);
      }
    }
    if (!diag) { snprintf(buf, sizeof buf, "M[%lld][neuron] != -c", (long long)r); return buf; }
    std::sort(targets.begin(), targets.end());
    for (size_t i = 1; i < targets.size(); ++i)
      if (targets[i] == targets[i - 1]) { snprintf(buf, sizeof buf, "M row %lld: repeated column", (long long)r); return buf; }
    if (R.produced > 0) {
      if (!syn_seen[R.neuron]) { syn_seen[R.neuron] = 1; syn_of[R.neuron] = targets; }
      else if (syn_of[R.neuron] != targets) { snprintf(buf, sizeof buf, "rule %lld: synapse set differs from neuron's other spiking rules", (long long)r); return buf; }
    }
  }
  return "";
}

struct Run {
  int status = OR_OK;
  std::string error;
  std::vector<std::vector<int64_t>> configs;   // discovery order
  std::vector<int64_t> level_offsets;          // depth_reached + 2 entries
  std::vector<int64_t> parent;                 // index within the previous level, -1 at level 0
  std::vector<uint64_t> t;                     // spiking-vector index (0 at level 0)
  std::vector<uint8_t> halting;
  std::vector<uint64_t> fp0, fp1;
  std::vector<int64_t> level_T, level_new, level_kept;  // per expanded level
  std::set<int64_t> numbers;                   // generated numbers (out_rule >= 0)
  // Reading A17 (every edge of the computation tree, Fig. 4):
  // for expanded level L, one entry per transition in (parent, t) order = the
  // global discovery index of the configuration it reached, or -1 when that
  // child was not stored (thinned, reading A19; terminal, generated numbers)
  std::vector<std::vector<int64_t>> edge_ref;
};

}  // namespace

// ============================================================================
// C ABI of the oracle (own header: oracle/oracle.h)
// ============================================================================
extern "C" {

struct oracle_system { System s; };
struct oracle_run { Run r; };

// re_bits (may be NULL): n × 4 words, bit v of rule r's row = a^v ∈ L(E_r)
// for v < 256 (read for UNARY rules only, v < t + P).
int oracle_load_unary(int64_t m, int64_t n, const int32_t* rules6, const uint64_t* re_bits, const int64_t* row_ptr,
                      const int32_t* col, const int32_t* val, oracle_system** out, char* err, int64_t errlen) {
  if (!out || m < 1 || n < 0 || (n > 0 && (!rules6 || !row_ptr))) return OR_E_ARG;
  auto* h = new oracle_system();
  System& s = h->s;
  s.m = m;
  s.n = n;
  s.rules.resize(n);
  s.M_rows.resize(n);
  for (int64_t r = 0; r < n; ++r) {
    const int32_t* q = rules6 + 6 * r;
    s.rules[r] = Rule{q[0], q[1], q[2], q[3], q[4], q[5], {}};
    if (q[1] == RE_UNARY && re_bits && q[2] >= 0 && q[3] >= 1 && q[2] + q[3] <= 256)
      for (int64_t v = 0; v < q[2] + q[3]; ++v) s.rules[r].member.push_back((re_bits[4 * r + v / 64] >> (v % 64)) & 1);
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) s.M_rows[r].push_back({col[e], val[e]});
  }
  std::string msg = validate(s);
  if (!msg.empty()) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg.c_str());
    delete h;
    return OR_E_INVALID_SYSTEM;
  }
  *out = h;
  return OR_OK;
}

int oracle_load(int64_t m, int64_t n, const int32_t* rules6, const int64_t* row_ptr, const int32_t* col,
                const int32_t* val, oracle_system** out, char* err, int64_t errlen) {
  return oracle_load_unary(m, n, rules6, nullptr, row_ptr, col, val, out, err, errlen);
}

void oracle_free(oracle_system* h) { delete h; }

// Alg. 2 II-1 marks (tmp) and |σ_{V_i}| per neuron (eq. 8).
int oracle_applicability(const oracle_system* h, const int32_t* C32, int32_t* tmp_out, int32_t* d_out) {
  const System& s = h->s;
  std::vector<int64_t> C(C32, C32 + s.m);
  auto tmp = mark_applicable(s, C);
  auto A = applicable_rules_per_neuron(s, C);
  for (int64_t r = 0; r < s.n; ++r) tmp_out[r] = (int32_t)tmp[r];
  for (int64_t j = 0; j < s.m; ++j) d_out[j] = (int32_t)A[j].size();
  return OR_OK;
}

// All children of one configuration, t = 0..Ψ-1 (Alg. 1 II + III).  Writes
// min(Ψ, cap) spiking vectors (n bytes each) and children (m int64 each).
int oracle_children(const oracle_system* h, const int32_t* C32, int64_t cap, uint8_t* S_out,
                    int64_t* C_out, uint64_t* psi_out) {
  const System& s = h->s;
  std::vector<int64_t> C(C32, C32 + s.m);
  auto A = applicable_rules_per_neuron(s, C);
  uint64_t psi = 0;
  if (!count_children(A, &psi)) return OR_E_CAPACITY;
  *psi_out = psi;
  for (uint64_t t = 0; t < psi && (int64_t)t < cap; ++t) {
    auto S = spiking_vector(s, A, t);
    auto Cn = transition(s, C, S);
    if (S_out) memcpy(S_out + t * s.n, S.data(), s.n);
    if (C_out) memcpy(C_out + t * s.m, Cn.data(), s.m * sizeof(int64_t));
  }
  return OR_OK;
}

void oracle_fingerprint(const int64_t* C, int64_t m, uint64_t seed0, uint64_t seed1, uint64_t* out2) {
  std::vector<int64_t> v(C, C + m);
  auto f = fingerprint(v, seed0, seed1);
  out2[0] = f.first;
  out2[1] = f.second;
}

uint64_t oracle_fmix64(uint64_t k) { return fmix64(k); }

// Thinning threshold of reading A19: τ = floor(F·2^64 / N_new) (exact).
uint64_t oracle_thinning_tau(int64_t F, int64_t n_new) {
  unsigned __int128 num = (unsigned __int128)(uint64_t)F << 64;
  return (uint64_t)(num / (unsigned __int128)(uint64_t)n_new);
}

// Breadth-first computation tree (Alg. 1; dedup per the
// second stopping criterion PAPER.md:229; readings A5-A7, A16-A20).
//   level0:        F0 configurations (row-major, F0 x m); duplicates keep their
//                  first occurrence (reading A20).
//   depth:         number of levels to expand; configurations of level `depth`
//                  are classified (halting) but not expanded.
//   dedup:         0 = full-configuration equality, 1 = 128-bit fingerprint.
//   count_bits:    8/16/32; a kept configuration with a count above the
//                  storage range is SNP overflow (reading A16).
//   frontier_target F: 0 = no cap; otherwise thinning (reading A19).
//   max_transitions:   per-level budget on T; 0 = unlimited (capacity error).
//
//   out_rule >= 0: the result of a computation of a
//   generating SNP system is the number of steps between the first two spikes
//   the output neuron sends to the environment (PAPER.md:89 `out`, 95-99: Π
//   "generates all numbers in N - {1}" and "this generated set is the result
//   of the computation").  An output spike at step k is the firing of rule
//   `out_rule` in S_k.  The state is augmented with A = 0 (no output spike yet)
//   or A = k - t1 >= 1 at level k (steps since the first spike at step t1), a
//   last column of every configuration (width m + 1).  A transition from
//   (C, A) by S: if A >= 1 and S fires out_rule, the computation has generated
//   the number A and ends there (the child is terminal: counted in T, not
//   stored); else A' = (A == 0 ? [S fires out_rule] : A + 1) and the child is
//   (C + S·M, A').  Dedup and halting act on the augmented state.  level0 rows
//   then have m + 1 columns.
int oracle_explore_gen(const oracle_system* h, int64_t F0, const int32_t* level0, int32_t depth,
                       int32_t dedup, int32_t count_bits, int64_t frontier_target,
                       int64_t max_transitions, uint64_t seed0, uint64_t seed1, int32_t out_rule,
                       oracle_run** out) {
  const System& s = h->s;
  if (out_rule >= s.n) return OR_E_ARG;
  const bool gen = out_rule >= 0;
  const int64_t width = s.m + (gen ? 1 : 0);
  if (!out || F0 < 1 || depth < 0 || (dedup != 0 && dedup != 1)) return OR_E_ARG;
  if (count_bits != 8 && count_bits != 16 && count_bits != 32) return OR_E_ARG;
  const int64_t cmax = count_bits == 8 ? 255 : count_bits == 16 ? 65535 : 2147483647LL;
  auto* hr = new oracle_run();
  Run& run = hr->r;
  *out = hr;

  // visited configurations (all earlier levels, reading A6) -> global index
  std::map<std::vector<int64_t>, int64_t> visited_rows;      // dedup = 0
  std::map<std::pair<uint64_t, uint64_t>, int64_t> visited_fp;  // dedup = 1
  auto seen_at = [&](const std::vector<int64_t>& C, const std::pair<uint64_t, uint64_t>& f) -> int64_t {
    if (dedup == 0) {
      auto it = visited_rows.find(C);
      return it == visited_rows.end() ? -1 : it->second;
    }
    auto it = visited_fp.find(f);
    return it == visited_fp.end() ? -1 : it->second;
  };
  auto seen = [&](const std::vector<int64_t>& C, const std::pair<uint64_t, uint64_t>& f) { return seen_at(C, f) >= 0; };
  auto insert = [&](const std::vector<int64_t>& C, const std::pair<uint64_t, uint64_t>& f) {
    const int64_t idx = (int64_t)run.configs.size();  // the index push() gives it
    if (dedup == 0) visited_rows.emplace(C, idx);
    else visited_fp.emplace(f, idx);
  };
  auto push = [&](const std::vector<int64_t>& C, const std::pair<uint64_t, uint64_t>& f,
                  int64_t parent, uint64_t t) {
    run.configs.push_back(C);
    run.parent.push_back(parent);
    run.t.push_back(t);
    run.fp0.push_back(f.first);
    run.fp1.push_back(f.second);
  };

  // Level 0 (reading A20): every distinct configuration of level0, in order.
  run.level_offsets.push_back(0);
  for (int64_t i = 0; i < F0; ++i) {
    std::vector<int64_t> C(level0 + i * width, level0 + (i + 1) * width);
    for (int64_t v : C)
      if (v < 0 || v > cmax) { run.status = OR_E_OVERFLOW; run.error = "level 0 count out of range"; return run.status; }
    auto f = fingerprint(C, seed0, seed1);
    if (seen(C, f)) continue;
    insert(C, f);
    push(C, f, -1, 0);
  }
  run.level_offsets.push_back((int64_t)run.configs.size());

  for (int32_t L = 0; L < depth; ++L) {
    const int64_t lo = run.level_offsets[L], hi = run.level_offsets[L + 1];
    if (lo == hi) break;  // stopping criterion 2: nothing new
    struct Cand { int64_t parent; uint64_t t; std::vector<int64_t> C; std::pair<uint64_t, uint64_t> f; };
    std::vector<Cand> fresh;  // new children in tag order (parent order, then t)
    std::map<std::vector<int64_t>, int64_t> level_rows;         // -> index in fresh
    std::map<std::pair<uint64_t, uint64_t>, int64_t> level_fp;
    // per transition: global index of a configuration seen earlier (>= 0), or
    // -(2 + i) for the new child fresh[i] (resolved after thinning), or -1
    std::vector<int64_t> eref;
    int64_t T = 0;
    for (int64_t i = lo; i < hi; ++i) {
      const std::vector<int64_t> Caug = run.configs[i];
      const std::vector<int64_t> C(Caug.begin(), Caug.begin() + s.m);
      auto A = applicable_rules_per_neuron(s, C);
      uint64_t psi = 0;
      if (!count_children(A, &psi)) { run.status = OR_E_CAPACITY; run.error = "psi above 2^62"; return run.status; }
      for (uint64_t t = 0; t < psi; ++t) {
        ++T;
        if (max_transitions > 0 && T > max_transitions) { run.status = OR_E_CAPACITY; run.error = "transition budget exceeded"; return run.status; }
        auto S = spiking_vector(s, A, t);
        auto Cn = transition(s, C, S);
        if (gen) {  // NEXT-1: the augmented column
          const int64_t a = Caug[s.m];
          const bool fired = S[out_rule] != 0;
          if (a >= 1 && fired) {  // second output spike: the number a is generated
            run.numbers.insert(a);
            eref.push_back(-1);
            continue;
          }
          Cn.push_back(a == 0 ? (fired ? 1 : 0) : a + 1);
        }
        auto f = fingerprint(Cn, seed0, seed1);
        const int64_t old = seen_at(Cn, f);
        if (old >= 0) {  // produced at an earlier level (A6)
          eref.push_back(old);
          continue;
        }
        const int64_t slot = (int64_t)fresh.size();
        int64_t first = slot;  // the level's first child with this key
        if (dedup == 0) {
          auto ins = level_rows.emplace(Cn, slot);
          first = ins.first->second;
        } else {
          auto ins = level_fp.emplace(f, slot);
          first = ins.first->second;
        }
        if (first != slot) {  // same-level duplicate: first (minimum) tag wins
          eref.push_back(-(2 + first));
          continue;
        }
        eref.push_back(-(2 + slot));
        fresh.push_back(Cand{i - lo, t, Cn, f});
      }
    }
    const int64_t n_new = (int64_t)fresh.size();
    int64_t kept = 0;
    const bool thin = frontier_target > 0 && n_new > frontier_target;
    const uint64_t tau = thin ? oracle_thinning_tau(frontier_target, n_new) : 0;
    std::vector<int64_t> fresh_index(fresh.size(), -1);  // global index of each kept new child
    for (size_t ci = 0; ci < fresh.size(); ++ci) {
      const Cand& c = fresh[ci];
      if (thin && !(fmix64(c.f.first) < tau)) continue;  // reading A19
      fresh_index[ci] = (int64_t)run.configs.size();
      for (int64_t v : c.C) {
        if (v < 0) { run.status = OR_E_OVERFLOW; run.error = "negative count"; return run.status; }
        if (v > cmax) { run.status = OR_E_OVERFLOW; run.error = "count above storage range"; return run.status; }
      }
      insert(c.C, c.f);
      push(c.C, c.f, c.parent, c.t);
      ++kept;
    }
    run.level_T.push_back(T);
    run.level_new.push_back(n_new);
    run.level_kept.push_back(kept);
    run.level_offsets.push_back((int64_t)run.configs.size());
    for (int64_t& r : eref)
      if (r <= -2) r = fresh_index[(size_t)(-r - 2)];
    run.edge_ref.push_back(std::move(eref));
    if (kept == 0) break;
  }
  // Halting classification of every configuration (reading A5).
  run.halting.resize(run.configs.size());
  for (size_t i = 0; i < run.configs.size(); ++i) {
    const std::vector<int64_t> C(run.configs[i].begin(), run.configs[i].begin() + s.m);
    auto A = applicable_rules_per_neuron(s, C);
    bool any = false;
    for (int64_t q = 0; q < (int64_t)A.size(); ++q) any = any || !A[q].empty();
    run.halting[i] = any ? 0 : 1;
  }
  return OR_OK;
}

int oracle_explore(const oracle_system* h, int64_t F0, const int32_t* level0, int32_t depth,
                   int32_t dedup, int32_t count_bits, int64_t frontier_target,
                   int64_t max_transitions, uint64_t seed0, uint64_t seed1, oracle_run** out) {
  return oracle_explore_gen(h, F0, level0, depth, dedup, count_bits, frontier_target, max_transitions, seed0,
                            seed1, -1, out);
}

// Single-path sampling with an input spike train (
// Def. 1 `in`; deep trees take long to explore).
// Each of W walkers follows ONE computation path: at step k a walker with
// Ψ > 0 takes the child of index t = u mod Ψ in the enumeration order of
// Alg. 2 (reading A7), u = splitmix64(splitmix64(seed XOR
// (k << 32)) XOR w) (reading A25), i.e. C <- C + S_t·M (eq. (2)); a walker
// with no applicable rule (reading A5) keeps C (no rule fires) while input
// is still to come and stops (halted_step = k) once it is not (k >=
// train_len or no input neuron).  After the transition the input neuron
// (input_neuron >= 0) receives train[k] spikes from the environment (k <
// train_len).  A count above the storage range is overflow.
// configs: W × m in/out (int32).  halted_step: W (-1 = still running).
int oracle_sample(const oracle_system* h, int64_t W, int32_t* configs, uint64_t seed, int32_t steps,
                  int32_t input_neuron, const int32_t* train, int32_t train_len, int32_t count_bits,
                  int32_t* halted_step) {
  const System& s = h->s;
  if (W < 0 || steps < 0 || input_neuron >= s.m || (count_bits != 8 && count_bits != 16 && count_bits != 32))
    return OR_E_ARG;
  const int64_t cmax = count_bits == 8 ? 255 : count_bits == 16 ? 65535 : 2147483647LL;
  for (int64_t w = 0; w < W; ++w) {
    std::vector<int64_t> C(configs + w * s.m, configs + (w + 1) * s.m);
    halted_step[w] = -1;
    for (int32_t k = 0; k < steps; ++k) {
      auto A = applicable_rules_per_neuron(s, C);
      uint64_t psi = 0;
      if (!count_children(A, &psi)) return OR_E_CAPACITY;
      const bool input_left = input_neuron >= 0 && k < train_len;
      if (psi == 0 && !input_left) { halted_step[w] = k; break; }
      if (psi > 0) {
        const uint64_t u = splitmix64(splitmix64(seed ^ ((uint64_t)k << 32)) ^ (uint64_t)w);
        auto S = spiking_vector(s, A, u % psi);
        C = transition(s, C, S);
      }
      if (input_neuron >= 0 && k < train_len) C[input_neuron] += train[k];
      for (int64_t v : C)
        if (v < 0 || v > cmax) return OR_E_OVERFLOW;
    }
    for (int64_t j = 0; j < s.m; ++j) configs[w * s.m + j] = (int32_t)C[j];
  }
  return OR_OK;
}

// ---------------------------------------------------------------------------
// SN P systems WITH delays (the paper treats systems
// without delays only, and names the delayed variant as the
// adjacent model).  Reading A26, the standard semantics of
// Ionescu-Păun-Yokomori: a rule E/a^c -> a^p; d fired at step t consumes c at
// once; with d = 0 it emits p at step t; with d >= 1 the neuron is CLOSED at
// steps t .. t+d-1 (it cannot fire and spikes sent to it are lost) and at step
// t+d it emits p and is open again (it receives the spikes sent at t+d).
// State of a neuron: (C, τ, π) = (spikes, remaining closed steps, spikes it
// will emit when it reopens); a configuration is the row
// [C_0..C_{m-1} | τ_0..τ_{m-1} | π_0..π_{m-1}] (width 3m).  One step:
//   * open neurons (τ = 0) choose their rule exactly as without delays
//     (applicability, one rule per neuron with applicable rules,
//     readings A3/A4; enumeration order of Alg. 2, reading A7);
//   * a closed neuron counts down: τ' = τ - 1, and emits π when τ' = 0;
//   * a firing open neuron loses c; d = 0: emits p now; d >= 1: τ' = d, π' = p;
//   * every neuron open after the step (τ' = 0) receives, from each in-neighbour
//     that emits, its p spikes (one per synapse, reading A11).
// Halting (reading A5 extended): no open neuron has an applicable rule and no
// neuron is closed.  With no applicable rule but a closed neuron the state has
// exactly one child (nobody fires, the clocks run).  With every d = 0 this is
// eq. (2) on the first m columns and τ = π = 0 throughout.
RuleSets applicable_open(const System& sys, const std::vector<int64_t>& X) {
  RuleSets A(sys.m);
  for (int64_t r = 0; r < sys.n; ++r) {
    const int64_t sgm = sys.rules[r].neuron;
    if (X[sys.m + sgm] == 0 && applicable(sys.rules[r], X)) A.add(sgm, r);
  }
  A.finish();
  return A;
}

// syn of Def. 1 recovered from M (Def. 2): the out-neighbours of σ are the
// nonzero off-diagonal columns of its spiking rules' rows (validate() checks
// that they agree).
std::vector<std::vector<int64_t>> synapses(const System& sys) {
  std::vector<std::vector<int64_t>> syn(sys.m);
  std::vector<int> done(sys.m, 0);
  for (int64_t r = 0; r < sys.n; ++r) {
    const Rule& R = sys.rules[r];
    if (R.produced == 0 || done[R.neuron]) continue;
    done[R.neuron] = 1;
    for (const auto& jv : sys.M_rows[r])
      if (jv.first != R.neuron && jv.second != 0) syn[R.neuron].push_back(jv.first);
  }
  return syn;
}

std::vector<int64_t> delayed_step(const System& sys, const std::vector<std::vector<int64_t>>& syn,
                                  const std::vector<int32_t>& delay, const std::vector<int64_t>& X,
                                  const std::vector<uint8_t>& S) {
  const int64_t m = sys.m;
  std::vector<int64_t> Y = X;
  std::vector<int64_t> emit(m, 0);
  for (int64_t s = 0; s < m; ++s)
    if (X[m + s] >= 1) {  // closed: the clock runs
      Y[m + s] = X[m + s] - 1;
      if (Y[m + s] == 0) { emit[s] = X[2 * m + s]; Y[2 * m + s] = 0; }
    }
  for (int64_t r = 0; r < sys.n; ++r) {
    if (!S[r]) continue;
    const Rule& R = sys.rules[r];
    Y[R.neuron] -= R.consumed;
    if (delay[r] == 0) emit[R.neuron] = R.produced;
    else { Y[m + R.neuron] = delay[r]; Y[2 * m + R.neuron] = R.produced; }
  }
  for (int64_t s = 0; s < m; ++s)
    for (int64_t j : syn[s])
      if (Y[m + j] == 0) Y[j] += emit[s];  // only open neurons receive
  return Y;
}

// All children of one delayed state (width 3m), t = 0..Ψ-1.
int oracle_children_delay(const oracle_system* h, const int32_t* delay32, const int32_t* X32, int64_t cap,
                          uint8_t* S_out, int64_t* X_out, uint64_t* psi_out) {
  const System& s = h->s;
  std::vector<int32_t> delay(delay32, delay32 + s.n);
  std::vector<int64_t> X(X32, X32 + 3 * s.m);
  const auto syn = synapses(s);
  auto A = applicable_open(s, X);
  uint64_t psi = 0;
  if (!count_children(A, &psi)) return OR_E_CAPACITY;
  bool closed = false;
  for (int64_t j = 0; j < s.m; ++j) closed = closed || X[s.m + j] != 0;
  if (psi == 0 && closed) psi = 1;
  *psi_out = psi;
  for (uint64_t t = 0; t < psi && (int64_t)t < cap; ++t) {
    auto S = spiking_vector(s, A, t);
    auto Y = delayed_step(s, syn, delay, X, S);
    if (S_out) memcpy(S_out + t * s.n, S.data(), s.n);
    if (X_out) memcpy(X_out + t * 3 * s.m, Y.data(), 3 * s.m * sizeof(int64_t));
  }
  return OR_OK;
}

// Breadth-first tree over delayed states: the BFS, dedup (readings A6, A18),
// thinning (A19) and overflow rules (A16, applied to all 3m columns) of
// oracle_explore_gen; level0 rows have 3m columns.
int oracle_explore_delay(const oracle_system* h, const int32_t* delay32, int64_t F0, const int32_t* level0,
                         int32_t depth, int32_t dedup, int32_t count_bits, int64_t frontier_target,
                         int64_t max_transitions, uint64_t seed0, uint64_t seed1, oracle_run** out) {
  const System& s = h->s;
  const int64_t width = 3 * s.m;
  if (!out || !delay32 || F0 < 1 || depth < 0 || (dedup != 0 && dedup != 1)) return OR_E_ARG;
  if (count_bits != 8 && count_bits != 16 && count_bits != 32) return OR_E_ARG;
  std::vector<int32_t> delay(delay32, delay32 + s.n);
  for (int32_t d : delay)
    if (d < 0) return OR_E_ARG;
  const auto syn = synapses(s);
  const int64_t cmax = count_bits == 8 ? 255 : count_bits == 16 ? 65535 : 2147483647LL;
  auto* hr = new oracle_run();
  Run& run = hr->r;
  *out = hr;
  std::set<std::vector<int64_t>> visited_rows;
  std::set<std::pair<uint64_t, uint64_t>> visited_fp;
  auto seen = [&](const std::vector<int64_t>& X, const std::pair<uint64_t, uint64_t>& f) {
    return dedup == 0 ? visited_rows.count(X) > 0 : visited_fp.count(f) > 0;
  };
  auto insert = [&](const std::vector<int64_t>& X, const std::pair<uint64_t, uint64_t>& f) {
    if (dedup == 0) visited_rows.insert(X);
    else visited_fp.insert(f);
  };
  auto push = [&](const std::vector<int64_t>& X, const std::pair<uint64_t, uint64_t>& f, int64_t parent, uint64_t t) {
    run.configs.push_back(X);
    run.parent.push_back(parent);
    run.t.push_back(t);
    run.fp0.push_back(f.first);
    run.fp1.push_back(f.second);
  };
  auto children_count = [&](const std::vector<int64_t>& X, RuleSets* A, uint64_t* psi) {
    *A = applicable_open(s, X);
    if (!count_children(*A, psi)) return false;
    bool closed = false;
    for (int64_t j = 0; j < s.m; ++j) closed = closed || X[s.m + j] != 0;
    if (*psi == 0 && closed) *psi = 1;
    return true;
  };
  run.level_offsets.push_back(0);
  for (int64_t i = 0; i < F0; ++i) {
    std::vector<int64_t> X(level0 + i * width, level0 + (i + 1) * width);
    for (int64_t v : X)
      if (v < 0 || v > cmax) { run.status = OR_E_OVERFLOW; run.error = "level 0 value out of range"; return run.status; }
    auto f = fingerprint(X, seed0, seed1);
    if (seen(X, f)) continue;
    insert(X, f);
    push(X, f, -1, 0);
  }
  run.level_offsets.push_back((int64_t)run.configs.size());
  for (int32_t L = 0; L < depth; ++L) {
    const int64_t lo = run.level_offsets[L], hi = run.level_offsets[L + 1];
    if (lo == hi) break;
    struct Cand { int64_t parent; uint64_t t; std::vector<int64_t> X; std::pair<uint64_t, uint64_t> f; };
    std::vector<Cand> fresh;
    std::set<std::vector<int64_t>> level_rows;
    std::set<std::pair<uint64_t, uint64_t>> level_fp;
    int64_t T = 0;
    for (int64_t i = lo; i < hi; ++i) {
      const std::vector<int64_t> X = run.configs[i];
      RuleSets A;
      uint64_t psi = 0;
      if (!children_count(X, &A, &psi)) { run.status = OR_E_CAPACITY; run.error = "psi above 2^62"; return run.status; }
      for (uint64_t t = 0; t < psi; ++t) {
        ++T;
        if (max_transitions > 0 && T > max_transitions) { run.status = OR_E_CAPACITY; run.error = "transition budget exceeded"; return run.status; }
        auto Y = delayed_step(s, syn, delay, X, spiking_vector(s, A, t));
        auto f = fingerprint(Y, seed0, seed1);
        if (seen(Y, f)) continue;
        bool dup_here = dedup == 0 ? !level_rows.insert(Y).second : !level_fp.insert(f).second;
        if (dup_here) continue;
        fresh.push_back(Cand{i - lo, t, Y, f});
      }
    }
    const int64_t n_new = (int64_t)fresh.size();
    int64_t kept = 0;
    const bool thin = frontier_target > 0 && n_new > frontier_target;
    const uint64_t tau = thin ? oracle_thinning_tau(frontier_target, n_new) : 0;
    for (const Cand& c : fresh) {
      if (thin && !(fmix64(c.f.first) < tau)) continue;
      for (int64_t v : c.X)
        if (v < 0 || v > cmax) { run.status = OR_E_OVERFLOW; run.error = "value outside the storage range"; return run.status; }
      insert(c.X, c.f);
      push(c.X, c.f, c.parent, c.t);
      ++kept;
    }
    run.level_T.push_back(T);
    run.level_new.push_back(n_new);
    run.level_kept.push_back(kept);
    run.level_offsets.push_back((int64_t)run.configs.size());
    if (kept == 0) break;
  }
  run.halting.resize(run.configs.size());
  for (size_t i = 0; i < run.configs.size(); ++i) {
    RuleSets A;
    uint64_t psi = 0;
    children_count(run.configs[i], &A, &psi);
    run.halting[i] = psi == 0 ? 1 : 0;
  }
  return OR_OK;
}

int64_t oracle_run_num_numbers(const oracle_run* h) { return (int64_t)h->r.numbers.size(); }
void oracle_run_numbers(const oracle_run* h, int64_t* out) { std::copy(h->r.numbers.begin(), h->r.numbers.end(), out); }
int oracle_run_status(const oracle_run* h) { return h->r.status; }
const char* oracle_run_error(const oracle_run* h) { return h->r.error.c_str(); }
int64_t oracle_run_num_configs(const oracle_run* h) { return (int64_t)h->r.configs.size(); }
int64_t oracle_run_num_levels(const oracle_run* h) { return (int64_t)h->r.level_offsets.size() - 1; }
int64_t oracle_run_num_expanded(const oracle_run* h) { return (int64_t)h->r.level_T.size(); }
void oracle_run_level_offsets(const oracle_run* h, int64_t* out) {
  std::copy(h->r.level_offsets.begin(), h->r.level_offsets.end(), out);
}
void oracle_run_configs(const oracle_run* h, int64_t m, int64_t* out) {
  for (size_t i = 0; i < h->r.configs.size(); ++i) std::copy(h->r.configs[i].begin(), h->r.configs[i].end(), out + i * m);
}
void oracle_run_tree(const oracle_run* h, int64_t* parent, uint64_t* t, uint8_t* halting, uint64_t* fp2) {
  const Run& r = h->r;
  for (size_t i = 0; i < r.configs.size(); ++i) {
    parent[i] = r.parent[i];
    t[i] = r.t[i];
    halting[i] = r.halting[i];
    fp2[2 * i] = r.fp0[i];
    fp2[2 * i + 1] = r.fp1[i];
  }
}
void oracle_run_counters(const oracle_run* h, int64_t* T, int64_t* n_new, int64_t* kept) {
  const Run& r = h->r;
  for (size_t i = 0; i < r.level_T.size(); ++i) { T[i] = r.level_T[i]; n_new[i] = r.level_new[i]; kept[i] = r.level_kept[i]; }
}
void oracle_run_free(oracle_run* h) { delete h; }
// reading A17: transitions of expanded level L (= T of that level) and the
// configuration each reached (global discovery index, -1 = not stored)
int64_t oracle_run_num_edges(const oracle_run* h, int64_t L) {
  return L >= 0 && L < (int64_t)h->r.edge_ref.size() ? (int64_t)h->r.edge_ref[L].size() : 0;
}
void oracle_run_edges(const oracle_run* h, int64_t L, int64_t* ref) {
  if (L >= 0 && L < (int64_t)h->r.edge_ref.size()) std::copy(h->r.edge_ref[L].begin(), h->r.edge_ref[L].end(), ref);
}

}  // extern "C"

// ============================================================================
// oracle_explore_par — the breadth-first tree of oracle_explore (dedup 0/1,
// thinning, overflow; no generated numbers) for frontiers of 10^5-10^6
// configurations (configs 3 and 5 of BASELINE.json at their stated sizes).
// Same definitions, same order of decisions:
//   * children of each parent: applicable_rules_per_neuron, count_children,
//     spiking_vector, transition, fingerprint — the functions above, called by
//     n_threads threads over disjoint ranges of parents (a child depends only
//     on its parent, Alg. 1 II-III);
//   * the dedup / thinning / insertion decisions are taken by ONE thread over
//     the children in canonical (parent, t) order, exactly as oracle_explore
//     (readings A6, A7, A16, A19, A20).
// Storage differs only in representation: visited configurations live in a
// flat arena of count_bits / 8 bytes per count (every stored count is in
// [0, 2^count_bits - 1] by the overflow check, so the slot holds it exactly), the visited set is a hash map from fp0 to arena
// indices compared row by row (dedup = 0: exact equality; dedup = 1: equality
// of (fp0, fp1)), and a new child's row is recomputed from (parent, t) when a
// comparison or the kept row needs it instead of being held for the level.
// Pinned against oracle_explore on every shape of the parity suite
// (tests/test_oracle_par.py).
// ============================================================================
namespace {

struct ParRun {
  int status = OR_OK;
  std::string error;
  int64_t m = 0;
  int64_t w = 4;                       // bytes per stored count: 1 / 2 / 4 for count_bits 8 / 16 / 32
  static constexpr int64_t CPB = 4096;  // configurations per arena chunk
  std::vector<std::vector<uint8_t>> arena;  // stored configurations, m counts of w bytes each, discovery order
  int64_t stored = 0;
  std::vector<int64_t> level_offsets;
  std::vector<int64_t> parent;
  std::vector<uint64_t> t, fp0, fp1;
  std::vector<uint8_t> halting;
  std::vector<int64_t> level_T, level_new, level_kept;
  // count j of stored configuration i (every stored count is in [0, 2^(8w) - 1], reading A16)
  int64_t at(int64_t i, int64_t j) const {
    const uint8_t* p = arena[(size_t)(i / CPB)].data() + ((size_t)(i % CPB) * (size_t)m + (size_t)j) * (size_t)w;
    if (w == 1) return p[0];
    if (w == 2) return (int64_t)p[0] | ((int64_t)p[1] << 8);
    int32_t v;
    memcpy(&v, p, 4);
    return v;
  }
  // chunks for configurations [0, n)
  void reserve(int64_t n) {
    while ((int64_t)arena.size() * CPB < n) arena.emplace_back((size_t)(CPB * m * w));
  }
  // the counts of configuration i (its chunk reserved)
  void put(int64_t i, const std::vector<int64_t>& C) {
    uint8_t* p = arena[(size_t)(i / CPB)].data() + (size_t)(i % CPB) * (size_t)(m * w);
    for (size_t j = 0; j < C.size(); ++j)
      for (int64_t b = 0; b < w; ++b) p[j * w + b] = (uint8_t)((uint64_t)C[j] >> (8 * b));
  }
  void append(const std::vector<int64_t>& C) {
    reserve(stored + 1);
    uint8_t* p = arena[(size_t)(stored / CPB)].data() + (size_t)(stored % CPB) * (size_t)(m * w);
    ++stored;
    for (size_t j = 0; j < C.size(); ++j)
      for (int64_t b = 0; b < w; ++b) p[j * w + b] = (uint8_t)((uint64_t)C[j] >> (8 * b));
  }
  void row(int64_t i, std::vector<int64_t>& r) const {
    r.resize((size_t)m);
    for (int64_t j = 0; j < m; ++j) r[j] = at(i, j);
  }
};

// run f(i) for i in [lo, hi) on n threads (contiguous ranges)
template <class F>
void parallel_for(int64_t lo, int64_t hi, int n, F f) {
  if (hi <= lo) return;
  if (n <= 1 || hi - lo < 2) {
    for (int64_t i = lo; i < hi; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  const int64_t len = hi - lo;
  for (int k = 0; k < n; ++k) {
    const int64_t a = lo + len * k / n, b = lo + len * (k + 1) / n;
    th.emplace_back([=]() { for (int64_t i = a; i < b; ++i) f(i); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

struct oracle_prun { ParRun r; };

int oracle_explore_par(const oracle_system* h, int64_t F0, const int32_t* level0, int32_t depth, int32_t dedup,
                       int32_t count_bits, int64_t frontier_target, int64_t max_transitions, uint64_t seed0,
                       uint64_t seed1, int32_t n_threads, oracle_prun** out) {
  const System& s = h->s;
  if (!out || F0 < 1 || depth < 0 || (dedup != 0 && dedup != 1)) return OR_E_ARG;
  if (count_bits != 8 && count_bits != 16 && count_bits != 32) return OR_E_ARG;
  const int64_t cmax = count_bits == 8 ? 255 : count_bits == 16 ? 65535 : 2147483647LL;
  const int64_t m = s.m;
  auto* hr = new oracle_prun();
  ParRun& run = hr->r;
  *out = hr;
  run.m = m;
  run.w = count_bits / 8;
  if (n_threads < 1) n_threads = 1;
  const FpWeights fingerprint_of(m, seed0, seed1);
  // visited: fp0 -> arena indices (dedup 0: rows compared; dedup 1: fp1 compared)
  std::unordered_multimap<uint64_t, int64_t> visited;
  auto row_equal = [&](int64_t i, const int64_t* C) {
    for (int64_t j = 0; j < m; ++j)
      if (run.at(i, j) != C[j]) return false;
    return true;
  };
  // row(): the configuration itself, materialised only when a dedup = 0
  // comparison needs it (an fp0 match)
  auto seen = [&](const std::pair<uint64_t, uint64_t>& f, const std::function<std::vector<int64_t>()>& row) {
    auto rg = visited.equal_range(f.first);
    std::vector<int64_t> C;
    for (auto it = rg.first; it != rg.second; ++it) {
      const int64_t i = it->second;
      if (dedup == 1) {
        if (run.fp1[i] == f.second) return true;
        continue;
      }
      if (C.empty()) C = row();
      if (row_equal(i, C.data())) return true;
    }
    return false;
  };
  auto push = [&](const std::vector<int64_t>& C, const std::pair<uint64_t, uint64_t>& f, int64_t parent, uint64_t t) {
    const int64_t idx = (int64_t)run.parent.size();
    run.append(C);
    run.parent.push_back(parent);
    run.t.push_back(t);
    run.fp0.push_back(f.first);
    run.fp1.push_back(f.second);
    visited.emplace(f.first, idx);
  };
  auto row_of = [&](int64_t i) {
    std::vector<int64_t> r;
    run.row(i, r);
    return r;
  };
  // Level 0 (reading A20)
  run.level_offsets.push_back(0);
  for (int64_t i = 0; i < F0; ++i) {
    std::vector<int64_t> C(level0 + i * m, level0 + (i + 1) * m);
    for (int64_t v : C)
      if (v < 0 || v > cmax) { run.status = OR_E_OVERFLOW; run.error = "level 0 count out of range"; return run.status; }
    auto f = fingerprint_of(C);
    if (seen(f, [&]() { return C; })) continue;
    push(C, f, -1, 0);
  }
  run.level_offsets.push_back((int64_t)run.parent.size());
  for (int32_t L = 0; L < depth; ++L) {
    const int64_t lo = run.level_offsets[L], hi = run.level_offsets[L + 1];
    if (lo == hi) break;
    const int64_t F = hi - lo;
    std::vector<uint64_t> psi_of(F, 0);
    struct Cand { int64_t parent; uint64_t t; std::pair<uint64_t, uint64_t> f; const int64_t* row; };
    std::vector<Cand> fresh;
    std::unordered_multimap<uint64_t, int64_t> level_keys;  // fp0 -> index in fresh
    auto child_row = [&](int64_t parent_in_level, uint64_t t) {
      const std::vector<int64_t> C = row_of(lo + parent_in_level);
      auto A = applicable_rules_per_neuron(s, C);
      return transition(s, C, spiking_vector(s, A, t));
    };
    int64_t T = 0;
    // parents in chunks; a chunk is split into n_threads contiguous ranges,
    // each producing, parent by parent, Ψ (eq. (8), readings A3-A5) and the
    // children's fingerprints — plus their rows for dedup = 0, which the
    // merge compares exactly — in canonical order (parents, then t, A7)
    const int64_t chunk = std::max<int64_t>(n_threads, dedup == 0 ? ((int64_t)1 << 23) / m : (int64_t)1 << 16);
    for (int64_t c0 = 0; c0 < F; c0 += chunk) {
      const int64_t c1 = std::min<int64_t>(F, c0 + chunk);
      struct Part {
        std::vector<std::pair<uint64_t, uint64_t>> fps;
        std::vector<int64_t> rows;
        bool cap = false;
      };
      const int nparts = (int)std::min<int64_t>(n_threads, c1 - c0);
      std::vector<Part> parts(nparts);
      std::vector<std::thread> th;
      for (int k = 0; k < nparts; ++k) {
        const int64_t a = c0 + (c1 - c0) * k / nparts, b = c0 + (c1 - c0) * (k + 1) / nparts;
        th.emplace_back([&, a, b, k]() {
          Part& P = parts[k];
          for (int64_t i = a; i < b; ++i) {
            const std::vector<int64_t> C = row_of(lo + i);
            auto A = applicable_rules_per_neuron(s, C);
            if (!count_children(A, &psi_of[i])) { P.cap = true; return; }
            for (uint64_t t = 0; t < psi_of[i]; ++t) {
              auto Cn = transition(s, C, spiking_vector(s, A, t));
              P.fps.push_back(fingerprint_of(Cn));
              if (dedup == 0) P.rows.insert(P.rows.end(), Cn.begin(), Cn.end());
            }
          }
        });
      }
      for (auto& x : th) x.join();
      for (const Part& P : parts)
        if (P.cap) { run.status = OR_E_CAPACITY; run.error = "psi above 2^62"; return run.status; }
      const size_t fresh_chunk0 = fresh.size();  // rows of fresh[fresh_chunk0..] live in `parts`
      for (int k = 0; k < nparts; ++k) {
        const int64_t a = c0 + (c1 - c0) * k / nparts, b = c0 + (c1 - c0) * (k + 1) / nparts;
        size_t pos = 0;
        for (int64_t i = a; i < b; ++i) {
          for (uint64_t t = 0; t < psi_of[i]; ++t, ++pos) {
            ++T;
            if (max_transitions > 0 && T > max_transitions) { run.status = OR_E_CAPACITY; run.error = "transition budget exceeded"; return run.status; }
            const auto& f = parts[k].fps[pos];
            const int64_t* crow = dedup == 0 ? parts[k].rows.data() + pos * (size_t)m : nullptr;
            auto cn = [&]() { return std::vector<int64_t>(crow, crow + m); };
            if (seen(f, cn)) continue;  // produced at an earlier level (A6)
            bool dup = false;
            auto rg = level_keys.equal_range(f.first);
            for (auto it = rg.first; it != rg.second && !dup; ++it) {
              const Cand& o = fresh[it->second];
              if (dedup == 1) dup = o.f.second == f.second;
              else if ((size_t)it->second >= fresh_chunk0) dup = std::equal(crow, crow + m, o.row);
              else dup = child_row(o.parent, o.t) == cn();
            }
            if (dup) continue;  // same-level duplicate: first (minimum) tag wins
            level_keys.emplace(f.first, (int64_t)fresh.size());
            fresh.push_back(Cand{i, t, f, crow});
          }
        }
      }
    }
    // halting flags of this level (reading A5: halting <=> Ψ = 0)
    for (int64_t i = 0; i < F; ++i) run.halting.push_back(psi_of[i] == 0 ? 1 : 0);
    const int64_t n_new = (int64_t)fresh.size();
    const bool thin = frontier_target > 0 && n_new > frontier_target;
    const uint64_t tau = thin ? oracle_thinning_tau(frontier_target, n_new) : 0;
    std::vector<int64_t> keep;
    for (int64_t ci = 0; ci < n_new; ++ci)
      if (!thin || fmix64(fresh[ci].f.first) < tau) keep.push_back(ci);  // reading A19
    // kept rows recomputed in parallel straight into their arena slots (the
    // next indices, tag order), then recorded in tag order; the first
    // out-of-range kept row (in tag order) is the overflow (reading A16)
    std::vector<char> bad(keep.size(), 0);
    const int64_t first = run.stored;
    run.reserve(first + (int64_t)keep.size());
    parallel_for(0, (int64_t)keep.size(), n_threads, [&](int64_t k) {
      const Cand& c = fresh[keep[k]];
      auto Cn = child_row(c.parent, c.t);
      for (int64_t v : Cn) bad[k] |= (v < 0 ? 1 : v > cmax ? 2 : 0);
      if (!bad[k]) run.put(first + k, Cn);
    });
    for (size_t k = 0; k < keep.size(); ++k) {
      if (bad[k]) { run.status = OR_E_OVERFLOW; run.error = (bad[k] & 1) ? "negative count" : "count above storage range"; return run.status; }
      const Cand& c = fresh[keep[k]];
      run.parent.push_back(c.parent);
      run.t.push_back(c.t);
      run.fp0.push_back(c.f.first);
      run.fp1.push_back(c.f.second);
      visited.emplace(c.f.first, first + (int64_t)k);
    }
    run.stored = first + (int64_t)keep.size();
    run.level_T.push_back(T);
    run.level_new.push_back(n_new);
    run.level_kept.push_back((int64_t)keep.size());
    run.level_offsets.push_back((int64_t)run.parent.size());
    if (keep.empty()) break;
  }
  // halting classification (reading A5) of the configurations of the levels
  // that were not expanded (the expanded ones got Ψ = 0 above)
  const int64_t N = (int64_t)run.parent.size();
  const int64_t classified = (int64_t)run.halting.size();
  run.halting.resize(N, 0);
  parallel_for(classified, N, n_threads, [&](int64_t i) {
    auto A = applicable_rules_per_neuron(s, row_of(i));
    bool any = false;
    for (int64_t q = 0; q < (int64_t)A.size(); ++q) any = any || !A[q].empty();
    run.halting[i] = any ? 0 : 1;
  });
  return OR_OK;
}

void oracle_prun_free(oracle_prun* h) { delete h; }
int oracle_prun_status(const oracle_prun* h) { return h->r.status; }
const char* oracle_prun_error(const oracle_prun* h) { return h->r.error.c_str(); }
int64_t oracle_prun_num_configs(const oracle_prun* h) { return (int64_t)h->r.parent.size(); }
int64_t oracle_prun_num_levels(const oracle_prun* h) { return (int64_t)h->r.level_offsets.size() - 1; }
int64_t oracle_prun_num_expanded(const oracle_prun* h) { return (int64_t)h->r.level_T.size(); }
void oracle_prun_level_offsets(const oracle_prun* h, int64_t* out) {
  std::copy(h->r.level_offsets.begin(), h->r.level_offsets.end(), out);
}
void oracle_prun_tree(const oracle_prun* h, int64_t* parent, uint64_t* t, uint8_t* halting, uint64_t* fp2) {
  const ParRun& r = h->r;
  for (size_t i = 0; i < r.parent.size(); ++i) {
    parent[i] = r.parent[i];
    t[i] = r.t[i];
    halting[i] = i < r.halting.size() ? r.halting[i] : 0;  // classified only when the run completes
    fp2[2 * i] = r.fp0[i];
    fp2[2 * i + 1] = r.fp1[i];
  }
}
void oracle_prun_counters(const oracle_prun* h, int64_t* T, int64_t* n_new, int64_t* kept) {
  const ParRun& r = h->r;
  for (size_t i = 0; i < r.level_T.size(); ++i) {
    T[i] = r.level_T[i];
    n_new[i] = r.level_new[i];
    kept[i] = r.level_kept[i];
  }
}
// rows idx[0..n) (global discovery indices) as int32
void oracle_prun_rows(const oracle_prun* h, const int64_t* idx, int64_t n, int32_t* out) {
  const ParRun& r = h->r;
  for (int64_t k = 0; k < n; ++k)
    for (int64_t j = 0; j < r.m; ++j) out[k * r.m + j] = (int32_t)r.at(idx[k], j);
}

}  // extern "C"
