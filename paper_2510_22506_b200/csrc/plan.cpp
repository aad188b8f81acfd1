// Planner: the leave-one-out partial network with the reuse cache
// (network.py:377-498), the plain chain (network.py:281-293) and the FLOP
// meter (tensor.py:32-72, contract's 2*rows*shared*cols at tensor.py:196).
#include "plan.hpp"

#include <algorithm>
#include <stdexcept>

#include "executor.hpp"

namespace fctn {

// ---------------------------------------------------------------- cache

bool ReuseCacheMirror::lookup(const std::vector<int>& subset, const std::vector<int64_t>& stamps,
                              LTensor* out, std::vector<int64_t>* freed) {
  auto it = store_.find(subset);
  if (it != store_.end() && it->second.stamps == stamps) {
    ++hits;
    *out = it->second.t;
    return true;
  }
  if (it != store_.end()) {  // stale: evicted lazily (network.py:404-406)
    bytes_ -= it->second.ref_bytes;
    if (freed) freed->push_back(it->second.t.buf);
    store_.erase(it);
  }
  ++misses;
  return false;
}

bool ReuseCacheMirror::store(const std::vector<int>& subset, const std::vector<int64_t>& stamps,
                             const LTensor& t, int64_t ref_bytes, std::vector<int64_t>* freed) {
  auto it = store_.find(subset);
  if (it != store_.end()) {  // network.py:410-413
    bytes_ -= it->second.ref_bytes;
    if (freed && it->second.t.buf != t.buf) freed->push_back(it->second.t.buf);
    store_.erase(it);
  }
  if (bytes_ + ref_bytes > budget_) return false;  // network.py:414-415
  store_[subset] = CacheEntry{stamps, t, ref_bytes};
  bytes_ += ref_bytes;
  return true;
}

void ReuseCacheMirror::clear(std::vector<int64_t>* freed) {
  for (auto& kv : store_)
    if (freed) freed->push_back(kv.second.t.buf);
  store_.clear();
  bytes_ = 0;
}

bool ReuseCacheMirror::holds_buffer(int64_t buf) const {
  for (auto& kv : store_)
    if (kv.second.t.buf == buf) return true;
  return false;
}

// ---------------------------------------------------------------- planner

static int64_t g_dry_ids = 1 << 30;

LTensor Planner::contract(const LTensor& a, const LTensor& b, Executor* exec,
                          const std::vector<int>* out_labels, int64_t out_buf, bool tag_compose) {
  ContractOp op;
  op.a = a;
  op.b = b;
  std::vector<int> shared, afree, bfree;
  for (int l : a.labels) {
    if (std::find(b.labels.begin(), b.labels.end(), l) != b.labels.end())
      shared.push_back(l);
    else
      afree.push_back(l);
  }
  for (int l : b.labels)
    if (std::find(a.labels.begin(), a.labels.end(), l) == a.labels.end()) bfree.push_back(l);
  if (shared.empty()) throw std::runtime_error("operands share no bond");
  op.rows = op.shared = op.cols = 1;
  for (int l : afree) op.rows *= sh_.extent(l);
  for (int l : shared) op.shared *= sh_.extent(l);
  for (int l : bfree) op.cols *= sh_.extent(l);
  int64_t fl = 2 * op.rows * op.shared * op.cols;
  if (tag_compose)
    meter.compose += fl;
  else
    meter.mk += fl;
  if (out_labels) {
    op.out.labels = *out_labels;
  } else {
    // Device layout of a partial: labels ascending = physical modes ascending,
    // then bonds.  The reference's as-built order (a-free then b-free,
    // network.py:249-258) only fixes which numbers the tensor holds, so any
    // layout is exact; this one puts the lowest physical mode first, which is
    // the fastest label of every M_k the partial later joins into, so the
    // join's gathers of it are unit-stride (join.cu) whatever the visiting
    // order.
    op.out.labels = afree;
    op.out.labels.insert(op.out.labels.end(), bfree.begin(), bfree.end());
    std::sort(op.out.labels.begin(), op.out.labels.end());
  }
  if (out_buf >= 0) {
    op.out.buf = out_buf;
  } else {
    op.out.buf = exec ? exec->alloc_labels(op.out.labels) : g_dry_ids++;
  }
  if (exec) exec->contract(op);
  return op.out;
}

void Planner::release(const LTensor& t, Executor* exec) {
  if (t.factor >= 0 || t.buf < 0) return;
  if (cache_.holds_buffer(t.buf)) return;
  if (exec && !exec->is_fixed_buffer(t.buf)) exec->free(t.buf);
}

static std::vector<int> sorted_copy(std::vector<int> v) {
  std::sort(v.begin(), v.end());
  return v;
}

LTensor Planner::chain(const std::vector<int>& seq, bool from_right, Executor* exec, bool final_is_m,
                       int k, int64_t m_buf, bool* produced_m, bool use_cache, bool tag_compose) {
  const int n = sh_.n;
  const int m = (int)seq.size();
  LTensor none;
  if (m == 0) return none;
  if (m == 1) {
    LTensor f;
    f.labels = sh_.factor_labels(seq[0]);
    f.factor = seq[0];
    return f;
  }
  // growing subsets, smallest first (network.py:449-452)
  std::vector<std::vector<int>> steps;
  if (from_right) {
    for (int i = m - 2; i >= 0; --i) steps.emplace_back(seq.begin() + i, seq.end());
  } else {
    for (int i = 0; i < m - 1; ++i) steps.emplace_back(seq.begin(), seq.begin() + i + 2);
  }
  auto stamps_of = [&](const std::vector<int>& sub) {
    std::vector<int64_t> st;
    for (int j : sorted_copy(sub)) st.push_back(versions[j]);
    return st;
  };
  LTensor arr;
  bool have = false;
  size_t start = 0;
  std::vector<int64_t> freed;
  if (use_cache) {  // largest cached intermediate first (network.py:453-461)
    for (int idx = (int)steps.size() - 1; idx >= 0; --idx) {
      LTensor got;
      if (cache_.lookup(sorted_copy(steps[idx]), stamps_of(steps[idx]), &got, &freed)) {
        arr = got;
        have = true;
        start = idx + 1;
        break;
      }
    }
  }
  for (int64_t b : freed)
    if (exec) exec->free(b);
  freed.clear();
  if (!have) {
    int j0 = from_right ? seq.back() : seq.front();
    arr.labels = sh_.factor_labels(j0);
    arr.factor = j0;
    start = 0;
  }
  for (size_t idx = start; idx < steps.size(); ++idx) {
    bool last = idx + 1 == steps.size();
    bool to_m = final_is_m && last;
    std::vector<int> mlab;
    if (to_m) mlab = sh_.m_labels(k);
    LTensor nxt;
    const int j = from_right ? steps[idx].front() : steps[idx].back();
    LTensor f;
    f.labels = sh_.factor_labels(j);
    f.factor = j;
    const LTensor& lt = from_right ? f : arr;
    const LTensor& rt = from_right ? arr : f;
    // the step that produces M_k is the final join of this side: the device
    // may form it (or Y_k) in another association (final_join_hook)
    bool hooked = false;
    if (to_m && exec && final_join_hook && !tag_compose) {
      std::vector<int> lfs(steps[idx].begin(), steps[idx].end()), rfs;
      if (from_right) {
        rfs.assign(steps[idx].begin() + 1, steps[idx].end());
        lfs.assign(1, j);
      } else {
        lfs.assign(steps[idx].begin(), steps[idx].end() - 1);
        rfs.assign(1, j);
      }
      hooked = final_join_hook(lt, rt, lfs, rfs);
    }
    nxt = contract(lt, rt, hooked ? nullptr : exec, to_m ? &mlab : nullptr, to_m ? m_buf : -1, tag_compose);
    release(arr, exec);
    arr = nxt;
    if (to_m && produced_m) *produced_m = true;
    if (use_cache && (int)steps[idx].size() < n - 1) {  // network.py:473-474
      cache_.store(sorted_copy(steps[idx]), stamps_of(steps[idx]), arr, 8 * arr.numel(sh_), &freed);
      for (int64_t b : freed)
        if (exec && b != arr.buf) exec->free(b);
      freed.clear();
    }
  }
  return arr;
}

void Planner::partial_cached(int k, const std::vector<int>& order, Executor* exec, int64_t m_buf) {
  int pos = (int)(std::find(order.begin(), order.end(), k) - order.begin());
  if (pos >= (int)order.size()) throw std::runtime_error("k not in order");
  std::vector<int> lseq(order.begin(), order.begin() + pos);
  std::vector<int> rseq(order.begin() + pos + 1, order.end());
  bool produced = false;
  LTensor left = chain(lseq, false, exec, rseq.empty(), k, m_buf, &produced, true);
  LTensor right = chain(rseq, true, exec, lseq.empty(), k, m_buf, &produced, true);
  if (lseq.empty() || rseq.empty()) {
    const LTensor& only = lseq.empty() ? right : left;
    if (!produced) {  // single factor (n == 2): relabel into M layout
      LTensor out;
      out.labels = sh_.m_labels(k);
      out.buf = m_buf;
      if (exec) exec->permute(only, out);
    }
    return;
  }
  std::vector<int> mlab = sh_.m_labels(k);
  if (exec && final_join_hook && final_join_hook(left, right, lseq, rseq))
    contract(left, right, nullptr, &mlab, m_buf, false);  // meter only (network.py:493-497)
  else
    contract(left, right, exec, &mlab, m_buf, false);  // network.py:493-497
  release(left, exec);
  release(right, exec);
}

void Planner::partial_plain(int k, Executor* exec, int64_t m_buf, bool tag_compose) {
  std::vector<int> rest;
  for (int j = 0; j < sh_.n; ++j)
    if (j != k) rest.push_back(j);
  bool produced = false;
  LTensor arr = chain(rest, false, exec, true, k, m_buf, &produced, false, tag_compose);
  if (!produced) {
    LTensor out;
    out.labels = sh_.m_labels(k);
    out.buf = m_buf;
    if (exec) exec->permute(arr, out);
  }
}

int64_t Planner::compose_chain_flops() const {
  // network.py:271-278: factor 0 then absorb 1..n-1 in index order
  const int n = sh_.n;
  std::vector<int> cur = sh_.slot_labels(0);
  int64_t fl = 0;
  for (int k = 1; k < n; ++k) {
    std::vector<int> other = sh_.slot_labels(k), nxt;
    int64_t rows = 1, shared = 1, cols = 1;
    for (int l : cur) {
      if (std::find(other.begin(), other.end(), l) != other.end())
        shared *= sh_.extent(l);
      else {
        rows *= sh_.extent(l);
        nxt.push_back(l);
      }
    }
    for (int l : other)
      if (std::find(cur.begin(), cur.end(), l) == cur.end()) {
        cols *= sh_.extent(l);
        nxt.push_back(l);
      }
    fl += 2 * rows * shared * cols;
    cur = nxt;
  }
  return fl;
}

void Planner::reset_cache(Executor* exec) {
  std::vector<int64_t> freed;
  cache_.clear(&freed);
  for (int64_t b : freed)
    if (exec) exec->free(b);
  cache_.hits = 0;
  cache_.misses = 0;
}

}  // namespace fctn
