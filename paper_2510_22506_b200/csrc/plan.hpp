// Host-side network bookkeeping: labels, tensor shapes, the reuse cache
// mirror and the reference FLOP meter.  No CUDA here: the same code runs
// the shape-only replay (fctn_plan_sweeps) on a CPU-only box.
//
// Labels (one int per tensor mode): physical mode of factor j is `j`; the
// bond between factors a < b is `n + tri(a, b)` with the upper-triangle
// row-major index of network.py:79-85.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <string>
#include <vector>

namespace fctn {

// Primed labels (label + PRIME) name the second copy of a bond in the
// doubled network E_j = A_(j)^T A_(j) used for the Gram of M_k.
constexpr int PRIME = 1 << 16;

struct Shape {
  int n = 0;
  std::vector<int64_t> dims;  // physical extents
  std::vector<int64_t> tri;   // rank table, strict upper triangle row-major

  int tri_index(int a, int b) const {
    if (a > b) std::swap(a, b);
    return a * (n - 1) - a * (a - 1) / 2 + (b - a - 1);
  }
  int bond_label(int a, int b) const { return n + tri_index(a, b); }
  int64_t extent(int label) const {
    if (label >= PRIME) label -= PRIME;
    return label < n ? dims[label] : tri[label - n];
  }
  bool is_phys(int label) const { return label < n; }
  // bonds-to-k labels, ascending partner (rows of M_k / columns of A_(k))
  std::vector<int> bonds_of(int k) const {
    std::vector<int> out;
    for (int j = 0; j < n; ++j)
      if (j != k) out.push_back(bond_label(j, k));
    return out;
  }
  int64_t s_of(int k) const {
    int64_t s = 1;
    for (int j = 0; j < n; ++j)
      if (j != k) s *= tri[tri_index(j, k)];
    return s;
  }
  int64_t total() const {
    int64_t t = 1;
    for (auto d : dims) t *= d;
    return t;
  }
  // slot labels of factor k in the reference's slot order (network.py:226-228)
  std::vector<int> slot_labels(int k) const {
    std::vector<int> out;
    for (int j = 0; j < n; ++j) out.push_back(j == k ? k : bond_label(j, k));
    return out;
  }
  // storage labels of factor k on device: A_(k) column-major = [k, bonds...]
  std::vector<int> factor_labels(int k) const {
    std::vector<int> out{k};
    for (int b : bonds_of(k)) out.push_back(b);
    return out;
  }
  // M_k storage labels: [phys j != k ascending..., bonds to k ascending
  // partner...]: p fastest, in X's own column order (network.py:360-371)
  std::vector<int> m_labels(int k) const {
    std::vector<int> out;
    for (int j = 0; j < n; ++j)
      if (j != k) out.push_back(j);
    for (int b : bonds_of(k)) out.push_back(b);
    return out;
  }
  // E_j = A_(j)^T A_(j): [bonds of j..., primed bonds of j...]
  std::vector<int> e_labels(int j) const {
    std::vector<int> out = bonds_of_factor(j);
    for (int b : bonds_of_factor(j)) out.push_back(b + PRIME);
    return out;
  }
  // bonds of factor j in its unfolding's column order (ascending partner)
  std::vector<int> bonds_of_factor(int j) const { return bonds_of(j); }
  // G_k layout: [bonds to k..., primed bonds to k...] (s_k x s_k, column-major)
  std::vector<int> g_labels(int k) const { return e_labels(k); }
};

// Reference FLOP meter labels (tensor.py:32-72).
struct Meter {
  int64_t mk = 0, compose = 0, gram = 0, proj = 0;
  int64_t total() const { return mk + compose + gram + proj; }
};

// A labeled tensor (first label fastest, contiguous).  `buf` is an opaque
// device allocation id owned by the executor (-1 = factor storage k when
// `factor >= 0`).
struct LTensor {
  std::vector<int> labels;
  int64_t buf = -1;   // executor buffer id, or -1
  int factor = -1;    // >= 0: this is factor storage of factor `factor`
  int64_t numel(const Shape& sh) const {
    int64_t e = 1;
    for (int l : labels) e *= sh.extent(l);
    return e;
  }
};

// One contraction emitted by the planner: out = a (*) b over shared labels,
// with out labels = a-free then b-free (network.py:249-258) unless the
// consumer asked for another order (M_k layout).
struct ContractOp {
  LTensor a, b, out;
  int64_t rows = 0, shared = 0, cols = 0;
};

class Executor;  // device side (null in dry mode)

// Reuse cache mirror of network.py:377-417, keyed by sorted factor subset,
// entries stamped with factor versions, bytes counted as the reference's
// float64 `nbytes`, lazy eviction of stale entries on lookup.
struct CacheEntry {
  std::vector<int64_t> stamps;
  LTensor t;
  int64_t ref_bytes = 0;
};

class ReuseCacheMirror {
 public:
  explicit ReuseCacheMirror(int64_t budget) : budget_(budget) {}
  int64_t hits = 0, misses = 0;
  int64_t bytes() const { return bytes_; }
  // returns true and fills `out` on hit; on a stale entry, evicts it and
  // appends its buffer to `freed`.
  bool lookup(const std::vector<int>& subset, const std::vector<int64_t>& stamps, LTensor* out,
              std::vector<int64_t>* freed);
  // returns true if kept; previously stored entry of the same subset is
  // dropped first (its buffer appended to `freed`).
  bool store(const std::vector<int>& subset, const std::vector<int64_t>& stamps, const LTensor& t,
             int64_t ref_bytes, std::vector<int64_t>* freed);
  void clear(std::vector<int64_t>* freed);
  bool holds_buffer(int64_t buf) const;

 private:
  int64_t budget_;
  int64_t bytes_ = 0;
  std::map<std::vector<int>, CacheEntry> store_;
};

// Planner of the leave-one-out partial network (network.py:426-498 for the
// accelerated variant, 281-293 for the plain one).  Executes contractions
// through `exec` (may be null: shape-only replay).
class Planner {
 public:
  Planner(const Shape& sh, int64_t budget) : sh_(sh), cache_(budget) {}
  Shape& shape() { return sh_; }
  ReuseCacheMirror& cache() { return cache_; }
  std::vector<int64_t> versions;  // per-factor version stamps
  Meter meter;
  // Optional device-side replacement of the final join M_k = left (*) right
  // (partial_cached; lseq / rseq: the factors each side contracts): when it
  // returns true it has done the work itself (formed Y_k without M_k, or M_k
  // in another association); the planner still meters the reference's join.
  std::function<bool(const LTensor&, const LTensor&, const std::vector<int>&, const std::vector<int>&)>
      final_join_hook;

  // Build M_k in the M layout into executor buffer `m_buf` (accelerated
  // variant, given visiting order).  Returns number of contractions run.
  void partial_cached(int k, const std::vector<int>& order, Executor* exec, int64_t m_buf);
  // Plain ascending chain (compose_except).  `tag_compose` counts the FLOPs
  // as "compose" instead of "mk".
  void partial_plain(int k, Executor* exec, int64_t m_buf, bool tag_compose = false);
  // FLOPs of the reference's full-chain `compose` (network.py:271-278).
  int64_t compose_chain_flops() const;
  void reset_cache(Executor* exec);

 private:
  LTensor chain(const std::vector<int>& seq, bool from_right, Executor* exec, bool final_is_m,
                int k, int64_t m_buf, bool* produced_m, bool use_cache, bool tag_compose = false);
  LTensor contract(const LTensor& a, const LTensor& b, Executor* exec, const std::vector<int>* out_labels,
                   int64_t out_buf, bool tag_compose);
  void release(const LTensor& t, Executor* exec);
  Shape sh_;
  ReuseCacheMirror cache_;
};

}  // namespace fctn
