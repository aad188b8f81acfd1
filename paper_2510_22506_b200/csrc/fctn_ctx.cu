// Context, device executor and the C ABI (include/fctn_b200.h).
//
// The context owns X (double-buffered), the mask, the factors (fp64 master
// + compute-dtype copy), the M_k buffer, the reuse-cache allocations and the
// small solve workspaces.  One sweep = one host call; the host sees only the
// few sweep scalars copied back at the end (solver.py:346-388 needs them).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fctn_b200.h"
#include "executor.hpp"
#include "kernels.cuh"
#include "plan.hpp"

namespace fctn {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(call)                                                                             \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      throw ::fctn::CudaError(std::string(#call) + " failed: " + cudaGetErrorString(_e));            \
  } while (0)

// Process-level cache of the large device blocks (>= 1 MB) a context owns:
// cudaMalloc / cudaFree of a few GB cost ~90 ms per create + close pair, a
// third of a short run(obs, cfg) call.  A closed context's blocks stay idle
// here (up to FCTN_DEVCACHE_GB, default 16; 0 disables) and the next context
// with the same extents takes them back by exact size; an allocation failure
// or fctn_trim_cache() returns them to the driver.  Contents are stale, as
// with any cudaMalloc.
struct DevCache {
  static constexpr size_t MIN_BYTES = (size_t)1 << 20;
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> idle;
  std::map<void*, std::pair<int, size_t>> live;
  size_t idle_bytes = 0, cap = 0;
  DevCache() {
    const char* e = getenv("FCTN_DEVCACHE_GB");
    cap = (size_t)((e ? atof(e) : 16.0) * (double)(1ull << 30));
  }
  cudaError_t alloc(void** p, size_t n) {
    int dev = 0;
    cudaGetDevice(&dev);
    const bool cached = cap > 0 && n >= MIN_BYTES;
    if (cached) {
      std::lock_guard<std::mutex> g(mu);
      auto it = idle.find({dev, n});
      if (it != idle.end()) {
        *p = it->second;
        idle.erase(it);
        idle_bytes -= n;
        live[*p] = {dev, n};
        return cudaSuccess;
      }
    }
    cudaError_t e = cudaMalloc(p, n);
    if (e == cudaErrorMemoryAllocation && idle_bytes > 0) {
      cudaGetLastError();
      trim();
      e = cudaMalloc(p, n);
    }
    if (e == cudaSuccess && cached) {
      std::lock_guard<std::mutex> g(mu);
      live[*p] = {dev, n};
    }
    return e;
  }
  cudaError_t release(void* p) {
    if (!p) return cudaSuccess;
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = live.find(p);
      if (it != live.end()) {
        const std::pair<int, size_t> key = it->second;
        live.erase(it);
        if (idle_bytes + key.second <= cap) {
          idle.insert({key, p});
          idle_bytes += key.second;
          return cudaSuccess;
        }
      }
    }
    return cudaFree(p);
  }
  void trim() {
    std::lock_guard<std::mutex> g(mu);
    for (auto& kv : idle) cudaFree(kv.second);
    idle.clear();
    idle_bytes = 0;
  }
};
static DevCache& dev_cache() {
  static DevCache* c = new DevCache();  // never destroyed: contexts may outlive static destruction order
  return *c;
}
// every cudaMalloc / cudaFree below this line goes through the cache
#define cudaMalloc(p, n) ::fctn::dev_cache().alloc((void**)(p), (size_t)(n))
#define cudaFree(p) ::fctn::dev_cache().release((void*)(p))

static const int64_t M_ID = 0;    // fixed executor id of the M_k buffer
static const int64_t X_ID = -10;  // the current iterate X (labels 0 .. n-1, first fastest)
static const int64_t Y_ID = -11;  // the fp64 Y_k buffer (labels [k, bonds to k])

// Collectives of the mode-0 sharded sweep: NCCL on the
// context stream (resolved at run time from the process's libnccl, so the
// library has no link-time NCCL dependency and shares torch's copy), or a
// host callback pair (tests: gloo over host memory, ranks sharing one GPU).
struct Comm {
  int kind = 0;  // 0 none, 1 NCCL, 2 host callbacks
  // NCCL
  void* nccl = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*allgather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  // host
  fctn_host_allreduce_fn h_allreduce = nullptr;
  fctn_host_allgather_fn h_allgather = nullptr;
  void* user = nullptr;
  double* hbuf = nullptr;  // pinned staging
  int64_t hcap = 0;
};

static void* nccl_lib() {
  static void* h = nullptr;
  if (!h) {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw std::runtime_error("libnccl.so.2 not found (needed for multi-GPU sharding)");
  }
  return h;
}
template <typename F>
static F nccl_sym(const char* name) {
  void* p = dlsym(nccl_lib(), name);
  if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + name);
  return reinterpret_cast<F>(p);
}

class Ctx : public Executor {
 public:
  int device = 0;
  int dtype = FCTN_F64;
  size_t esize = 8;
  Shape sh;   // execution shape (mode 0 = this rank's slab)
  Shape gsh;  // global shape: factors, solves, FLOP meter, reuse-cache budget
  std::vector<double> lam, delta;
  int sign = FCTN_SIGN_PD;
  double rho = 0.1;
  int alg = FCTN_ALG_ACCEL;
  int64_t budget = 1 << 30;
  std::string err;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::unique_ptr<Planner> planner;
  int64_t launches = 0;

  // device memory
  std::map<int64_t, void*> bufs;
  int64_t next_id = 1;
  void* X[2] = {nullptr, nullptr};
  int cur = 0;
  uint8_t* mask = nullptr;
  uint32_t* maskbits = nullptr;  // 1 bit per entry (TC compose epilogue)
  std::vector<double*> A64;
  std::vector<void*> Ac;  // compute copy (== A64 for fp64)
  double* Ascratch = nullptr;
  void* Mbuf = nullptr;
  double *Y = nullptr, *G = nullptr, *Fr = nullptr, *Fi = nullptr;
  double* ypart = nullptr;
  double* partials = nullptr;
  int64_t partial_cap = 0;
  std::vector<double*> E64;               // E_j = A_(j)^T A_(j), the doubled-network nodes
  double *epart = nullptr, *colstats = nullptr;  // colstats: one [s x 3] slot per mode
  int64_t cs_stride = 0;
  double* colstats_of(int k) const { return colstats + cs_stride * k; }
  double* gnet[2] = {nullptr, nullptr};   // doubled-network intermediates
  std::vector<DftPlan> dft;
  std::vector<double*> mu, cosT, sinT;
  std::vector<double> check_mu;
  // eigenbasis solve (eigh.cu): per-mode basis V_k (warm start across sweeps),
  // eigenvalues, the T-floor shift lam min(Lambda) + rho, a rotation scratch,
  // and the side stream the Gram network + eigendecomposition run on
  std::vector<double*> Vb;
  std::vector<double> floor_shift;
  double* phi = nullptr;
  double* Ytmp = nullptr;
  double* ework = nullptr;
  double* dft_gscr = nullptr;  // column work arrays of long-mode DFTs (I > 4266)
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fork2 = nullptr, ev_side = nullptr;
  int solve_pref = 0;  // FCTN_SOLVE: 0 auto, 1 = "chol", 2 = "eigh", 3 = "tri"
  double *tri_d = nullptr, *tri_e = nullptr;  // T of the tridiagonal form
  enum { FORM_CHOL = 0, FORM_EIGH = 1, FORM_TRI = 2 };
  // Which form solves update k.  The eigenbasis form (eigh.cu, the
  // reference's own) runs on a side stream concurrently with the Y_k pass, so
  // it is off the critical path when its single-SM Jacobi is shorter than
  // that pass.  s > 146 has no Cholesky kernel (one system no longer fits a
  // CTA's shared memory): always eigh (from global memory above s = 117).  The choice depends only on global shapes and the
  // visiting order, so every rank of a sharded run makes the same one.
  //
  // Three exact forms:
  //   chol (solve.cu) per-frequency Cholesky of G + mu_w I over all SMs --
  //                   the default for s <= 146;
  //   eigh (eigh.cu)  Jacobi eigendecomposition G = V diag(phi) V^T, the
  //                   reference's literal form: s > 146 (from global memory)
  //                   or FCTN_SOLVE=eigh;
  //   tri  (tri.cu)   G = Q T Q^T, per-frequency tridiagonal solves
  //                   (FCTN_SOLVE=tri).
  // eigh and tri decompose G once per update on the side stream, off the
  // critical path in principle, but their single-CTA FP64 kernels are
  // latency bound on B200 (c4, s = 64: Jacobi ~0.6 ms warm, tridiagonal
  // 0.28 ms) against 0.105 ms for all 1025 Cholesky systems, and the
  // update's Y_k pass does not hide them; measured sweep c4: chol 1.48 ms,
  // tri 1.86 ms, eigh 2.1 ms.
  int form_for(int k, bool long_y) const {
    (void)long_y;
    const int64_t S = gsh.s_of(k);
    if (S > 160 || !chol_solve_fits(S)) return FORM_EIGH;  // (the Cholesky CTA holds s <= 146)
    if (solve_pref == 2) return eigh_fits_smem(S) ? FORM_EIGH : FORM_CHOL;
    if (solve_pref == 3) return tridiag_fits_smem(S) ? FORM_TRI : FORM_CHOL;
    return FORM_CHOL;
  }
  bool eigh_for(int k, bool long_y) const { return form_for(k, long_y) != FORM_CHOL; }
  double* dstats = nullptr;  // [n*3 factor stats][4 sums]
  int* dstatus = nullptr;
  double* hstats = nullptr;  // pinned mirror (+ status)
  double* cscratch = nullptr;  // split-K partials of the generic contraction (fp64 Gram network)
  int64_t cscratch_cap = 0;
  bool configured = false;
  bool uploaded = false;
  // N = 3 schedule (see compute_z): Z_j = X x_j A_(j) and the A_j version it used
  void* Zb[3] = {nullptr, nullptr, nullptr};
  int64_t zver[3] = {-1, -1, -1};
  void* presplit = nullptr;     // fp32 [A hi | A lo | M hi | M lo] for the TC compose
  int64_t presplit_m_cap = 0;   // largest M_k (entries) that is pre-split
  int64_t max_is_ = 0;          // largest factor unfolding (entries), presplit layout
  int64_t ypart_cap = 0;        // doubles in ypart
  int mbuf_holds = -1;   // mode whose M_k currently sits in Mbuf (-1: none)
  bool zroute = true;    // FCTN_NO_ZROUTE=1 disables
  // Y_k without M_k (alt_join): armed per update by sweep_device
  bool alt_route = true;  // FCTN_NO_ALTJOIN=1 disables
  bool force_assoc = false;  // FCTN_FORCE_ASSOC=1 (tests): take the other associations whenever they apply
  bool alt_ok = false;
  int alt_k = -1;
  bool alt_last = false;  // alt_k is the order's last mode: the compose needs M_k or the partials
  bool assoc_ok = false;  // set around the sweep's M_k builds only (the hooks read alt_k)
  bool y_ready = false;
  // compose through the partials (compose_via_partials): the last update's
  // left / right partials are kept alive until the compose
  bool compose_alt = false;
  LTensor cp_left, cp_right;
  std::vector<int64_t> held_bufs, held_frees;
  // Three-mode sweeps have no data-dependent host decisions and no allocations,
  // so each (visiting order, X buffer parity, extrapolation) sweep is captured
  // once as a CUDA graph and replayed (FCTN_NO_GRAPH=1 disables).
  bool use_graph = true;
  std::map<std::string, std::pair<cudaGraphExec_t, int64_t>> graphs;  // -> (exec, launches)
  // mode-0 sharding: rows [slab_lo, slab_hi) of mode 0 live here
  int rank = 0, nranks = 1;
  int64_t slab_lo = 0, slab_hi = 0, slab_max = 0;
  void* Aslab = nullptr;   // rows [slab_lo, slab_hi) of A_(0), compute dtype
  double* yloc = nullptr;  // this rank's rows of Y_0 (slab_max x s_0)
  double* gbuf = nullptr;  // all-gathered rows (nranks x slab_max x s_0)
  Comm comm;
  bool sharded() const { return nranks > 1 || slab_lo != 0 || slab_hi != gsh.dims[0]; }
  const void* fac_ptr(int k) const { return (k == 0 && Aslab) ? Aslab : Ac[k]; }

  // profiling: events bracketing launch groups, accumulated per class
  struct Mark {
    int cls;
    cudaEvent_t a, b;
    double bytes;
    int64_t n;
    cudaStream_t s;
  };
  bool prof = false;
  int prof_cls = FCTN_K_MERGE;  // class of generic contractions (merge unless set)
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> evpool;
  double prof_ms[FCTN_K_COUNT] = {0};
  int64_t prof_n[FCTN_K_COUNT] = {0};
  double prof_bytes[FCTN_K_COUNT] = {0};
  cudaEvent_t tstart = nullptr, tstop = nullptr;

  cudaEvent_t take_event() {
    if (!evpool.empty()) {
      cudaEvent_t e = evpool.back();
      evpool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  int pbegin(int cls, cudaStream_t on = nullptr) {
    if (!prof) return -1;
    Mark m{cls, take_event(), take_event(), 0.0, 0, on ? on : st};
    CK(cudaEventRecord(m.a, m.s));
    marks.push_back(m);
    return (int)marks.size() - 1;
  }
  void pend(int idx, double bytes, int64_t n) {
    if (idx < 0) return;
    Mark& m = marks[idx];
    m.bytes = bytes;
    m.n = n;
    CK(cudaEventRecord(m.b, m.s));
  }
  void collect_marks() {  // after a stream sync
    for (auto& m : marks) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, m.a, m.b));
      prof_ms[m.cls] += ms;
      prof_n[m.cls] += m.n;
      prof_bytes[m.cls] += m.bytes;
      evpool.push_back(m.a);
      evpool.push_back(m.b);
    }
    marks.clear();
  }

  ~Ctx() override { release_all(); }

  // ------------------------------------------------------------ executor
  int64_t alloc_labels(const std::vector<int>& labels) override {
    int64_t numel = 1;
    for (int l : labels) numel *= sh.extent(l);
    void* p = nullptr;
    CK(cudaMallocAsync(&p, std::max<int64_t>(numel, 1) * esize, st));
    int64_t id = next_id++;
    bufs[id] = p;
    return id;
  }
  void free(int64_t id) override {
    if (id == M_ID) return;
    if (std::find(held_bufs.begin(), held_bufs.end(), id) != held_bufs.end()) {  // kept for the compose
      held_frees.push_back(id);
      return;
    }
    auto it = bufs.find(id);
    if (it == bufs.end()) return;
    CK(cudaFreeAsync(it->second, st));
    bufs.erase(it);
  }
  bool is_fixed_buffer(int64_t id) const override { return id == M_ID; }

  void* ptr_of(const LTensor& t) {
    if (t.factor >= 0) return const_cast<void*>(fac_ptr(t.factor));
    if (t.buf == M_ID) return Mbuf;
    if (t.buf == X_ID) return X[cur];
    if (t.buf == Y_ID) return Y;
    auto it = bufs.find(t.buf);
    if (it == bufs.end()) throw std::runtime_error("unknown buffer id");
    return it->second;
  }

  std::vector<int64_t> strides_of(const std::vector<int>& labels) const {
    std::vector<int64_t> s(labels.size());
    int64_t acc = 1;
    for (size_t i = 0; i < labels.size(); ++i) {
      s[i] = acc;
      acc *= sh.extent(labels[i]);
    }
    return s;
  }
  static int64_t stride_in(const std::vector<int>& labels, const std::vector<int64_t>& strides, int l) {
    for (size_t i = 0; i < labels.size(); ++i)
      if (labels[i] == l) return strides[i];
    throw std::runtime_error("label not found");
  }

  // Descriptor of out = a (*) b over shared labels for the on-device offset
  // computation (kernels.cuh ContractDesc).  Rows enumerate the operand that
  // holds the output's fastest label (coalesced stores), each group sorted
  // by output stride.
  ContractDesc desc_for(const ContractOp& op, bool* swapped) const {
    const std::vector<int>& out = op.out.labels;
    std::vector<int64_t> so = strides_of(out);
    const bool fast_in_b = std::find(op.b.labels.begin(), op.b.labels.end(), out[0]) != op.b.labels.end();
    const LTensor& ra = fast_in_b ? op.b : op.a;
    const LTensor& cb = fast_in_b ? op.a : op.b;
    std::vector<int64_t> sa = strides_of(ra.labels), sb = strides_of(cb.labels);
    std::vector<int> rfree, cfree, shared;
    for (int l : ra.labels) {
      if (std::find(cb.labels.begin(), cb.labels.end(), l) != cb.labels.end())
        shared.push_back(l);
      else
        rfree.push_back(l);
    }
    for (int l : cb.labels)
      if (std::find(ra.labels.begin(), ra.labels.end(), l) == ra.labels.end()) cfree.push_back(l);
    auto by_out_stride = [&](std::vector<int>& v) {
      std::sort(v.begin(), v.end(), [&](int x, int y) { return stride_in(out, so, x) < stride_in(out, so, y); });
    };
    by_out_stride(rfree);
    by_out_stride(cfree);
    if (rfree.size() > 12 || cfree.size() > 12 || shared.size() > 12) throw UsageError("too many modes");
    ContractDesc d;
    d.nr = (int)rfree.size();
    d.nc = (int)cfree.size();
    d.nk = (int)shared.size();
    d.rows = d.cols = d.K = 1;
    for (int q = 0; q < d.nr; ++q) {
      const int l = rfree[q];
      d.r_ext[q] = sh.extent(l);
      d.r_sa[q] = stride_in(ra.labels, sa, l);
      d.r_sc[q] = stride_in(out, so, l);
      d.rows *= d.r_ext[q];
    }
    for (int q = 0; q < d.nc; ++q) {
      const int l = cfree[q];
      d.c_ext[q] = sh.extent(l);
      d.c_sb[q] = stride_in(cb.labels, sb, l);
      d.c_sc[q] = stride_in(out, so, l);
      d.cols *= d.c_ext[q];
    }
    for (int q = 0; q < d.nk; ++q) {
      const int l = shared[q];
      d.k_ext[q] = sh.extent(l);
      d.k_sa[q] = stride_in(ra.labels, sa, l);
      d.k_sb[q] = stride_in(cb.labels, sb, l);
      d.K *= d.k_ext[q];
    }
    *swapped = fast_in_b;
    return d;
  }

  void contract(const ContractOp& op) override {
    bool sw = false;
    ContractDesc d = desc_for(op, &sw);
    int pm = pbegin(prof_cls);
    const void* ra = ptr_of(sw ? op.b : op.a);
    const void* cb = ptr_of(sw ? op.a : op.b);
    void* out = ptr_of(op.out);
    if (dtype == FCTN_F64)
      launch_contract<double>((const double*)ra, (const double*)cb, (double*)out, d, nullptr, 0, n_sm, st);
    else
      launch_contract<float>((const float*)ra, (const float*)cb, (float*)out, d, nullptr, 0, n_sm, st);
    ++launches;
    pend(pm, (double)esize * (op.out.numel(sh) + op.a.numel(sh) + op.b.numel(sh)), 1);
  }

  void permute(const LTensor& in, const LTensor& out) override {
    PermDesc pd;
    pd.nd = (int)out.labels.size();
    if (pd.nd > 16) throw std::runtime_error("too many modes");
    std::vector<int64_t> si = strides_of(in.labels);
    int64_t numel = 1;
    for (int q = 0; q < pd.nd; ++q) {
      pd.ext[q] = sh.extent(out.labels[q]);
      pd.in_stride[q] = stride_in(in.labels, si, out.labels[q]);
      numel *= pd.ext[q];
    }
    if (dtype == FCTN_F64)
      launch_permute<double>((const double*)ptr_of(in), (double*)ptr_of(out), pd, numel, st);
    else
      launch_permute<float>((const float*)ptr_of(in), (float*)ptr_of(out), pd, numel, st);
    ++launches;
  }

  // ------------------------------------------------------------ setup
  void drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.first);
    graphs.clear();
  }
  void release_shape_buffers() {
    drop_graphs();
    for (auto& kv : bufs) cudaFree(kv.second);
    bufs.clear();
    cudaFree(cscratch);
    cscratch = nullptr;
    cscratch_cap = 0;
    for (size_t k = 0; k < A64.size(); ++k) {
      cudaFree(A64[k]);
      if (dtype == FCTN_F32) cudaFree(Ac[k]);
    }
    A64.clear();
    Ac.clear();
    for (auto* p : {Ascratch, (double*)Mbuf, (double*)Zb[0], (double*)Zb[1], (double*)Zb[2], (double*)presplit,
                     (double*)Aslab, yloc, gbuf, Y, G, Fr, Fi, ypart, partials, epart, colstats, gnet[0], gnet[1]})
      cudaFree(p);
    Zb[0] = Zb[1] = Zb[2] = nullptr;
    Aslab = nullptr;
    yloc = gbuf = nullptr;
    presplit = nullptr;
    presplit_m_cap = 0;
    for (auto* p : E64) cudaFree(p);
    E64.clear();
    for (auto* p : Vb) cudaFree(p);
    Vb.clear();
    for (auto* p : {phi, Ytmp, ework, dft_gscr, tri_d, tri_e}) cudaFree(p);
    phi = Ytmp = ework = dft_gscr = tri_d = tri_e = nullptr;
    Ascratch = nullptr;
    Mbuf = nullptr;
    Y = G = Fr = Fi = ypart = partials = epart = colstats = gnet[0] = gnet[1] = nullptr;
  }
  void release_all() {
    if (st) cudaStreamSynchronize(st);
    if (comm.kind == 1 && comm.nccl && comm.destroy) comm.destroy((ncclComm_t)comm.nccl);
    if (comm.hbuf) cudaFreeHost(comm.hbuf);
    comm = Comm();
    release_shape_buffers();
    for (auto* p : mu) cudaFree(p);
    for (auto* p : cosT) cudaFree(p);
    for (auto* p : sinT) cudaFree(p);
    mu.clear();
    cosT.clear();
    sinT.clear();
    cudaFree(X[0]);
    cudaFree(X[1]);
    cudaFree(mask);
    cudaFree(maskbits);
    maskbits = nullptr;
    cudaFree(dstats);
    cudaFree(dstatus);
    if (hstats) cudaFreeHost(hstats);
    X[0] = X[1] = nullptr;
    mask = nullptr;
    dstats = nullptr;
    dstatus = nullptr;
    hstats = nullptr;
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (cudaEvent_t e : {ev_fork, ev_join, ev_fork2, ev_side})
      if (e) cudaEventDestroy(e);
    ev_fork = ev_join = ev_fork2 = ev_side = nullptr;
    if (st2) cudaStreamDestroy(st2);
    st2 = nullptr;
    if (st) cudaStreamDestroy(st);
    ev0 = ev1 = nullptr;
    st = nullptr;
  }

  int target_ctas() const { return n_sm * 4; }
  int n_sm = 148;
  bool use_tc = true;  // fp32 K2/K4 on tcgen05 (FCTN_NO_TC=1 forces the SIMT path)
  bool split3 = true;  // 3xTF32 products (FCTN_TF32=1x: one round-to-nearest TF32 pass)
  bool tc_ok(int k) const {
    if (dtype != FCTN_F32 || !use_tc) return false;
    int64_t P = 1, Q = 1;
    for (int j = 0; j < k; ++j) P *= sh.dims[j];
    for (int j = k + 1; j < sh.n; ++j) Q *= sh.dims[j];
    return tc_stream_supported(sh.dims[k], P, Q, sh.s_of(k));
  }

  void configure_shape() {
    // (re)allocate everything whose size depends on the rank table; factor,
    // solve and Gram buffers follow the global shape, X-sized ones the slab
    release_shape_buffers();
    const int n = sh.n;
    const int64_t T = sh.total();  // local
    int64_t max_is = 1, max_ss = 1, max_m = 1, max_h = 1, max_yp = 1, max_part = 1, max_ep = 1, max_s = 1;
    for (int k = 0; k < n; ++k) {
      const int64_t Ig = gsh.dims[k], S = gsh.s_of(k);
      const int64_t I = sh.dims[k], p = T / I;
      max_is = std::max(max_is, Ig * S);
      max_ss = std::max(max_ss, S * S);
      max_s = std::max(max_s, S);
      max_m = std::max(max_m, S * p);
      max_h = std::max(max_h, (Ig / 2 + 1) * S);
      StreamPlan sy = plan_stream(I, S, p, target_ctas());
      max_yp = std::max(max_yp, (int64_t)sy.nsplit * I * S);
      if (tc_ok(k)) {
        int64_t P = 1;
        for (int j = 0; j < k; ++j) P *= sh.dims[j];
        TcStreamPlan tp = plan_stream_tc(I, P, p / P, S, n_sm, split3);
        max_yp = std::max(max_yp, (tp.nsplit * I * S + 1) / 2);  // float partials in the double buffer
      }
      max_part = std::max(max_part, ((I + 63) / 64) * ((p + 63) / 64));
      max_ep = std::max(max_ep, (int64_t)fgram_splits(Ig) * S * S);
    }
    if (n == 3) {  // Y_1 partials of the Z route (split over b02)
      max_yp = std::max(max_yp, sh.tri[sh.tri_index(0, 2)] * sh.dims[1] * sh.tri[sh.tri_index(0, 1)] *
                                    sh.tri[sh.tri_index(1, 2)]);
      if (dtype == FCTN_F64) {  // the FP64 Z_0 pass stages its split partials here too (compute_z)
        const int64_t I0 = sh.dims[0], p0 = T / I0, S0 = sh.s_of(0);
        const StreamPlan sz = plan_stream(p0, S0, I0, target_ctas());
        max_yp = std::max(max_yp, (int64_t)sz.nsplit * p0 * S0);
      }
    }
    A64.assign(n, nullptr);
    Ac.assign(n, nullptr);
    E64.assign(n, nullptr);
    for (int k = 0; k < n; ++k) {
      // every fp64 factor slot has the max size: the solve output buffer is
      // swapped with the factor it replaces, so slots migrate between modes
      int64_t e = gsh.dims[k] * gsh.s_of(k);
      CK(cudaMalloc(&A64[k], max_is * sizeof(double)));
      CK(cudaMemset(A64[k], 0, max_is * sizeof(double)));
      CK(cudaMalloc(&E64[k], max_ss * sizeof(double)));
      if (dtype == FCTN_F32) {
        CK(cudaMalloc(&Ac[k], e * sizeof(float)));
      } else {
        Ac[k] = A64[k];
      }
    }
    if (sharded()) {
      const int64_t S0 = gsh.s_of(0);
      CK(cudaMalloc(&Aslab, std::max<int64_t>(1, slab_max * S0) * esize));
      CK(cudaMalloc(&yloc, std::max<int64_t>(1, slab_max * S0) * sizeof(double)));
      CK(cudaMalloc(&gbuf, std::max<int64_t>(1, nranks * slab_max * S0) * sizeof(double)));
    }
    CK(cudaMalloc(&Ascratch, max_is * sizeof(double)));
    CK(cudaMalloc(&Mbuf, max_m * esize));
    max_is_ = max_is;
    if (dtype == FCTN_F32) {
      presplit_m_cap = std::min<int64_t>(max_m, T / 4);
      CK(cudaMalloc(&presplit, (2 * max_is + 2 * presplit_m_cap) * sizeof(float)));
    }
    if (n == 3)
      for (int j = 0; j < 3; ++j)
        if (j == 0 || 4 * zsize(j) <= T) CK(cudaMalloc(&Zb[j], std::max<int64_t>(1, zsize(j)) * esize));
    z_invalidate();
    mbuf_holds = -1;
    CK(cudaMalloc(&Y, max_is * sizeof(double)));
    CK(cudaMalloc(&Ytmp, max_is * sizeof(double)));
    CK(cudaMalloc(&phi, max_s * sizeof(double)));
    CK(cudaMalloc(&tri_d, max_s * sizeof(double)));
    CK(cudaMalloc(&tri_e, max_s * sizeof(double)));
    Vb.assign(n, nullptr);
    for (int k = 0; k < n; ++k) {
      const int64_t S = gsh.s_of(k);
      CK(cudaMalloc(&Vb[k], S * S * sizeof(double)));
      launch_identity(Vb[k], S, st);  // the first eigendecomposition starts cold
    }
    {
      int64_t gs = 0;
      for (int k = 0; k < n; ++k)
        if (!dft[k].fast) gs = std::max(gs, 6 * gsh.dims[k] * gsh.s_of(k));
      if (gs) CK(cudaMalloc(&dft_gscr, gs * sizeof(double)));
    }
    if (!eigh_fits_smem(max_s)) CK(cudaMalloc(&ework, (2 * max_s * max_s + max_s) * sizeof(double)));
    CK(cudaMalloc(&G, max_ss * sizeof(double)));
    CK(cudaMalloc(&Fr, max_h * sizeof(double)));
    CK(cudaMalloc(&Fi, max_h * sizeof(double)));
    CK(cudaMalloc(&ypart, max_yp * sizeof(double)));
    ypart_cap = max_yp;
    CK(cudaMalloc(&epart, max_ep * sizeof(double)));
    cs_stride = max_s * 3;
    CK(cudaMalloc(&colstats, cs_stride * n * sizeof(double)));
    partial_cap = std::max<int64_t>(max_part, 4 * n_sm);
    CK(cudaMalloc(&partials, partial_cap * 4 * sizeof(double)));
    int64_t gcap = max_ss;
    for (int k = 0; k < n; ++k) gcap = std::max(gcap, gram_network_peak(k));
    CK(cudaMalloc(&gnet[0], gcap * sizeof(double)));
    CK(cudaMalloc(&gnet[1], gcap * sizeof(double)));
    cscratch_cap = std::max<int64_t>(std::max<int64_t>(1, 4 * gcap), (int64_t)(2 * n_sm + 8) * max_is);
    CK(cudaMalloc(&cscratch, cscratch_cap * sizeof(double)));
    // Pre-grow the stream-ordered pool that holds the reuse cache and the
    // chain intermediates (up to the cache budget, as device bytes, plus two
    // of the largest partials), so no sweep pays for a pool growth.
    if (n >= 4) {
      int64_t big = 0;
      for (int k = 0; k < n; ++k) big = std::max(big, sh.s_of(k) * (T / sh.dims[k]));
      const int64_t cache_dev = budget / 8 * (int64_t)esize;
      const int64_t want = std::min<int64_t>(cache_dev + 2 * big * (int64_t)esize, (int64_t)8 << 30);
      void* warm = nullptr;
      if (cudaMallocAsync(&warm, want, st) == cudaSuccess) CK(cudaFreeAsync(warm, st));
      else cudaGetLastError();
    }
    std::vector<int64_t> versions = planner ? planner->versions : std::vector<int64_t>(n, 0);
    planner.reset(new Planner(gsh, budget));  // the reference's chain and budget are global
    planner->versions = versions;
    planner->final_join_hook = [this](const LTensor& l, const LTensor& r, const std::vector<int>& ls,
                                      const std::vector<int>& rs) {
      return alt_join(l, r) || reassoc_join(l, r, ls, rs);
    };
  }

  // ------------------------------------------------------------ collectives
  void host_stage(int64_t n) {
    if (comm.hcap >= n) return;
    if (comm.hbuf) cudaFreeHost(comm.hbuf);
    CK(cudaMallocHost(&comm.hbuf, n * sizeof(double)));
    comm.hcap = n;
  }
  void allreduce_sum(double* d, int64_t n) {
    if (nranks == 1 && comm.kind == 0) return;
    if (comm.kind == 3) return;  // loop-back: the sum over ranks is this rank's own part
    if (comm.kind == 1) {
      if (comm.allreduce(d, d, (size_t)n, ncclFloat64, ncclSum, (ncclComm_t)comm.nccl, st) != ncclSuccess)
        throw std::runtime_error("ncclAllReduce failed");
    } else if (comm.kind == 2) {
      host_stage(n);
      CK(cudaMemcpyAsync(comm.hbuf, d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (comm.h_allreduce(comm.user, comm.hbuf, n) != 0) throw std::runtime_error("host allreduce callback failed");
      CK(cudaMemcpyAsync(d, comm.hbuf, n * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    ++launches;
  }
  void allgather(const double* send, double* recv, int64_t n) {
    if (comm.kind == 1) {
      if (comm.allgather(send, recv, (size_t)n, ncclFloat64, (ncclComm_t)comm.nccl, st) != ncclSuccess)
        throw std::runtime_error("ncclAllGather failed");
    } else if (comm.kind == 2) {
      host_stage(n * (nranks + 1));
      CK(cudaMemcpyAsync(comm.hbuf, send, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (comm.h_allgather(comm.user, comm.hbuf, comm.hbuf + n, n) != 0)
        throw std::runtime_error("host allgather callback failed");
      CK(cudaMemcpyAsync(recv, comm.hbuf + n, n * nranks * sizeof(double), cudaMemcpyHostToDevice, st));
    } else if (comm.kind == 3) {
      for (int r = 0; r < nranks; ++r)  // loop-back: every rank's block is this rank's
        CK(cudaMemcpyAsync(recv + (int64_t)r * n, send, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else {
      CK(cudaMemcpyAsync(recv, send, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    ++launches;
  }
  // rows [lo, hi) of A_(0) into the slab copy (after every update of A_0)
  void refresh_slab() {
    if (!Aslab) return;
    const int64_t S0 = gsh.s_of(0);
    launch_copy_rows(A64[0], gsh.dims[0], S0, slab_lo, slab_hi - slab_lo, Aslab, dtype == FCTN_F32, st);
    ++launches;
  }
  // finish Y_k = (sum over ranks of this rank's part) + rho A_prev
  void finish_y(int k, bool rows_local) {
    const int64_t Ig = gsh.dims[k], S = gsh.s_of(k);
    if (rows_local) {  // k == 0: this rank computed its own rows of Y_0 into yloc
      allgather(yloc, gbuf, slab_max * S);
      launch_scatter_rows(gbuf, nranks, slab_max, Ig, S, Y, st);
      ++launches;
    } else {
      allreduce_sum(Y, Ig * S);
    }
    launch_axpy(Y, A64[k], rho, Ig * S, st);
    ++launches;
  }

  // ------------------------------------------------------------ Gram of M_k
  // G_k = M_k M_k^T without forming it from M_k: the doubled network of the
  // factor Grams E_j = A_(j)^T A_(j) (j != k) contracted over every internal
  // bond and its primed twin.  Same value as sylvester.py:57-59, ~1e-16 apart;
  // cost ~ s^2 R^2 instead of 2 s^2 p_k (hard part 8).
  int64_t numel_of(const std::vector<int>& labels) const {
    int64_t e = 1;
    for (int l : labels) e *= sh.extent(l);
    return e;
  }
  static std::vector<int> contract_out_labels(const std::vector<int>& a, const std::vector<int>& b) {
    std::vector<int> out;
    for (int l : a)
      if (std::find(b.begin(), b.end(), l) == b.end()) out.push_back(l);
    for (int l : b)
      if (std::find(a.begin(), a.end(), l) == a.end()) out.push_back(l);
    return out;
  }
  int64_t gram_network_peak(int k) const {
    int64_t peak = 1;
    std::vector<int> cur;
    bool first = true;
    for (int j = 0; j < sh.n; ++j) {
      if (j == k) continue;
      if (first) {
        cur = sh.e_labels(j);
        first = false;
        continue;
      }
      cur = contract_out_labels(cur, sh.e_labels(j));
      peak = std::max(peak, numel_of(cur));
    }
    return peak;
  }
  void gram_network(int k, cudaStream_t gs) {
    std::vector<int> rest;
    for (int j = 0; j < sh.n; ++j)
      if (j != k) rest.push_back(j);
    const int64_t S = sh.s_of(k);
    if (rest.size() == 1) {  // n == 2: G_k = E_j
      CK(cudaMemcpyAsync(G, E64[rest[0]], S * S * sizeof(double), cudaMemcpyDeviceToDevice, gs));
      return;
    }
    LTensor cur;
    cur.labels = sh.e_labels(rest[0]);
    const double* cur_ptr = E64[rest[0]];
    int ping = 0;
    for (size_t q = 1; q < rest.size(); ++q) {
      ContractOp op;
      op.a = cur;
      op.b.labels = sh.e_labels(rest[q]);
      const bool last = q + 1 == rest.size();
      op.out.labels = last ? sh.g_labels(k) : contract_out_labels(op.a.labels, op.b.labels);
      double* out_ptr = last ? G : gnet[ping];
      bool sw = false;
      ContractDesc d = desc_for(op, &sw);
      const double* pa = cur_ptr;
      const double* pb = E64[rest[q]];
      launch_contract<double>(sw ? pb : pa, sw ? pa : pb, out_ptr, d, cscratch, cscratch_cap, n_sm, gs);
      ++launches;
      cur = op.out;
      cur_ptr = out_ptr;
      ping ^= 1;
    }
  }

  // factor statistics (||A - A_prev||^2, ||A||^2, tr A^T L A) and E_k for
  // factor k's current fp64 master (used after fctn_set_factors)
  void factor_refresh(int k) {
    const int64_t I = gsh.dims[k], S = gsh.s_of(k);
    const double sgn = sign == FCTN_SIGN_PD ? -1.0 : 1.0;
    launch_factor_colstats(A64[k], I, S, delta[k], sgn, colstats_of(k), st);
    launch_factor_gram(A64[k], I, S, epart, E64[k], colstats_of(k), dstats + 3 * k, st);
    launches += 3;
  }

  void configure(int dev, int dt, int n, const int64_t* dims, const int64_t* tri, const double* lm,
                 const double* dl, int sg, double r, int a, int64_t bud) {
    if (n < 2) throw UsageError("need a tensor of order >= 2");
    if (dt != FCTN_F64 && dt != FCTN_F32) throw UsageError("dtype must be FCTN_F64 or FCTN_F32");
    if (!(r > 0.0)) throw UsageError("rho must be > 0");
    device = dev;
    dtype = dt;
    esize = dt == FCTN_F64 ? 8 : 4;
    sh.n = n;
    sh.dims.assign(dims, dims + n);
    sh.tri.assign(tri, tri + n * (n - 1) / 2);
    for (auto d : sh.dims)
      if (d < 1) throw UsageError("extents must be >= 1");
    for (auto t : sh.tri)
      if (t < 1) throw UsageError("rank entries must be >= 1");
    gsh = sh;
    slab_lo = 0;
    slab_hi = sh.dims[0];
    slab_max = sh.dims[0];
    lam.assign(lm, lm + n);
    delta.assign(dl, dl + n);
    for (int k = 0; k < n; ++k) {
      if (lam[k] < 0) throw UsageError("lam must be >= 0");
      if (!(delta[k] > 0)) throw UsageError("diagonal shift delta must be > 0");
    }
    sign = sg;
    rho = r;
    alg = a;
    budget = bud;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
    {
      const char* e = getenv("FCTN_NO_TC");
      use_tc = !(e && e[0] == '1');
      const char* ng = getenv("FCTN_NO_GRAPH");
      use_graph = !(ng && ng[0] == '1');
      const char* zr = getenv("FCTN_NO_ZROUTE");
      zroute = !(zr && zr[0] == '1');
      const char* aj = getenv("FCTN_NO_ALTJOIN");
      alt_route = !(aj && aj[0] == '1');
      const char* fa = getenv("FCTN_FORCE_ASSOC");
      force_assoc = fa && fa[0] == '1';
      const char* t = getenv("FCTN_TF32");
      split3 = !(t && std::string(t) == "1x");
    }
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
    CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_fork2, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
    {
      const char* sv = getenv("FCTN_SOLVE");
      const std::string v = sv ? sv : "";
      solve_pref = v == "chol" ? 1 : v == "eigh" ? 2 : v == "tri" ? 3 : 0;
    }
    {
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t thr = UINT64_MAX;
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    const int64_t T = sh.total();
    CK(cudaMalloc(&X[0], T * esize));
    CK(cudaMalloc(&X[1], T * esize));
    CK(cudaMalloc(&mask, T));
    CK(cudaMalloc(&maskbits, ((T + 31) / 32) * sizeof(uint32_t)));
    CK(cudaMalloc(&dstats, (n * 3 + 8) * sizeof(double)));
    CK(cudaMalloc(&dstatus, sizeof(int)));
    CK(cudaMemset(dstatus, 0, sizeof(int)));
    CK(cudaMallocHost(&hstats, (n * 3 + 8) * sizeof(double) + 64));
    // spectra and DFT tables per mode (laplacian.py:46-47)
    const double sgn = sign == FCTN_SIGN_PD ? -1.0 : 1.0;
    mu.assign(n, nullptr);
    cosT.assign(n, nullptr);
    sinT.assign(n, nullptr);
    check_mu.assign(n, NAN);
    floor_shift.assign(n, 0.0);
    dft.clear();
    for (int k = 0; k < n; ++k) {
      int64_t I = sh.dims[k];
      dft.push_back(plan_dft(I));
      std::vector<double> c(I), s(I), m(I / 2 + 1);
      double lmin = INFINITY;
      for (int64_t j = 0; j < I; ++j) {
        double th = 2.0 * M_PI * (double)j / (double)I;
        c[j] = std::cos(th);
        s[j] = std::sin(th);
        double L = sgn * (-2.0 - delta[k] + 2.0 * std::cos(th));
        lmin = std::min(lmin, L);
        if (j <= I / 2) m[j] = lam[k] * L + rho;
      }
      // T-floor guard (sylvester.py:108-113): min T = lam*min(Lambda) + phi_min + rho.
      // It can only fail when lam*min(Lambda) + rho <= 1e-10 (phi >= 0 after the clamp).
      floor_shift[k] = lam[k] * lmin + rho;
      double shift = lam[k] * lmin + rho - 1e-10;
      if (shift <= 0.0) check_mu[k] = shift;
      CK(cudaMalloc(&mu[k], m.size() * sizeof(double)));
      CK(cudaMalloc(&cosT[k], I * sizeof(double)));
      CK(cudaMalloc(&sinT[k], I * sizeof(double)));
      CK(cudaMemcpy(mu[k], m.data(), m.size() * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(cosT[k], c.data(), I * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(sinT[k], s.data(), I * sizeof(double), cudaMemcpyHostToDevice));
    }
    configure_shape();
    configured = true;
  }

  // ------------------------------------------------------------ sweep pieces
  // ------------------------------------------------------------ N = 3 schedule
  // For three modes the reference's reuse cache never stores anything
  // (network.py:436-438,473) and M_k of a short mode is as large as X
  // (c4: M_2 is 268 M entries).  There Y_k is formed without M_k:
  //   Z_j = X x_j A_(j)   (one tensor-core pass over X contracting mode j;
  //                        T s_j / I_j entries),
  //   Y_k = Z_j (*) A_(l) (a small contraction over i_l and the bond (j, l),
  //                        l the third mode),
  // the same sums as X_(k) M_k^T in another association.  Z_j stays valid
  // while A_j and X are unchanged, so the sweep plans which Z to build so that
  // each one serves two consecutive updates: two passes over X per sweep for
  // the three products whatever the visiting order.  The FLOP / cache
  // counters still come from the planner's replay of the reference chain.
  int64_t zsize(int j) const { return sh.s_of(j) * (sh.total() / sh.dims[j]); }
  void z_invalidate() { zver[0] = zver[1] = zver[2] = -1; }
  // can Z_j be built on this path?
  bool z_buildable(int j) const {
    if (sh.n != 3 || !zroute || !Zb[j]) return false;
    const int64_t T = sh.total();
    if (dtype == FCTN_F64) return j == 0;
    if (!use_tc) return false;
    if (j == 0) return tc_stream_supported(T / sh.dims[0], sh.dims[0], 1, sh.s_of(0));
    if (!split3) return false;
    if (j == 1) return tc_stream_batched_supported(sh.dims[0], sh.dims[1], sh.dims[2], sh.s_of(1));
    return tc_stream_supported(sh.dims[0] * sh.dims[1], 1, sh.dims[2], sh.s_of(2));
  }
  int64_t bond_stride(int m, int partner) const {  // in A_(m)'s bond columns
    int64_t st_ = 1;
    for (int b : sh.bonds_of(m)) {
      if (b == sh.bond_label(m, partner)) return st_;
      st_ *= sh.extent(b);
    }
    return 0;
  }
  YzArgs yz_args(int j, int k) const {
    const int l = 3 - j - k;
    const int lo = std::min(k, l), hi = std::max(k, l);
    YzArgs a;
    a.long_l = (l == lo);
    a.Ir = sh.dims[lo];
    a.Io = sh.dims[hi];
    a.Rc = (int)sh.tri[sh.tri_index(j, l)];
    a.Rz = (int)sh.tri[sh.tri_index(j, k)];
    a.Ra = (int)sh.tri[sh.tri_index(k, l)];
    a.zc = bond_stride(j, l);
    a.zk = bond_stride(j, k);
    a.ac = bond_stride(l, j);
    a.aa = bond_stride(l, k);
    a.yz = bond_stride(k, j);
    a.ya = bond_stride(k, l);
    return a;
  }
  bool yz_ok(int j, int k) const {
    if (j == k || !z_buildable(j)) return false;
    const YzArgs a = yz_args(j, k);
    if (a.long_l) return a.Rc == a.Ra && a.Rc <= 8;
    return a.Ra <= 16 && (int64_t)a.Rc * a.Ir * a.Rz * a.Ra <= ypart_cap;
  }
  // route of each update in `order`: the j whose Z_j forms Y_k, -1 for the M_k stream
  std::vector<int> plan_routes(const std::vector<int>& order) const {
    std::vector<int> route(order.size(), -1);
    if (sh.n != 3 || !zroute) return route;
    const int64_t T = sh.total();
    int valid = -1;
    for (size_t t = 0; t < order.size(); ++t) {
      const int k = order[t];
      if (valid >= 0 && yz_ok(valid, k)) {
        route[t] = valid;
        continue;
      }
      const int next = t + 1 < order.size() ? order[t + 1] : -1;
      int best = -1;
      bool best_next = false;
      for (int j = 0; j < 3; ++j) {
        if (!yz_ok(j, k)) continue;
        const bool serves = next >= 0 && yz_ok(j, next);
        if (best < 0 || (serves && !best_next) || (serves == best_next && zsize(j) < zsize(best))) {
          best = j;
          best_next = serves;
        }
      }
      if (best >= 0 && !best_next) {
        // a Z for this update alone: keep the M_k stream when M_k is the cheaper operand
        const int64_t mk = sh.s_of(k) * (T / sh.dims[k]);
        const bool z_wins = dtype == FCTN_F64 ? 4 * zsize(best) <= mk : 2 * zsize(best) <= 3 * mk;
        if (!z_wins) best = -1;
      }
      route[t] = best;
      valid = best;
    }
    return route;
  }
  void compute_z(int j) {
    const int64_t T = sh.total();
    const int64_t Ij = sh.dims[j], pj = T / Ij, Sj = sh.s_of(j);
    int pm = pbegin(FCTN_K_ZPASS);
    if (dtype == FCTN_F32) {
      const float* bh = (const float*)fac_ptr(j);
      const float* bl = nullptr;
      if (split3) {  // A_(j) is tiny: split it once in HBM
        float* h = (float*)presplit;
        launch_tf32_split(bh, h, h + max_is_, Ij * Sj, st);
        bh = h;
        bl = h + max_is_;
        ++launches;
      }
      if (j == 0) {
        // the stream kernel with the roles of the modes swapped: rows = (i1, i2),
        // K = i0 (X's contiguous mode, K-major tiles), B = A_(0)
        TcStreamPlan tp = plan_stream_tc(pj, Ij, 1, Sj, n_sm, split3);
        tp.kb_per_split = tp.nkb;
        tp.nsplit = 1;
        launch_stream_tc((const float*)X[cur], bh, (float*)Zb[0], pj, Ij, 1, Sj, tp, st, bl);
      } else if (j == 1) {
        // a batch over i2 of MN-major [i0 x i1] x A_(1) products
        launch_stream_tc_batched((const float*)X[cur], bh, bl, (float*)Zb[1], sh.dims[0], sh.dims[1], sh.dims[2], Sj,
                                 n_sm, st);
      } else {
        // rows = (i0, i1) contiguous, K = i2: the k = 0 stream shape with B = A_(2)
        TcStreamPlan tp = plan_stream_tc(pj, 1, Ij, Sj, n_sm, split3);
        tp.kb_per_split = tp.nkb;
        tp.nsplit = 1;
        launch_stream_tc((const float*)X[cur], bh, (float*)Zb[2], pj, 1, Ij, Sj, tp, st, bl);
      }
    } else {
      StreamPlan sp = plan_stream(pj, Sj, Ij, target_ctas());
      if ((int64_t)sp.nsplit * pj * Sj > ypart_cap) throw std::runtime_error("split-partial buffer too small (Z pass)");
      launch_stream<double>((const double*)X[cur], (const double*)fac_ptr(0), ypart, pj, Ij, Sj, Ij, sp, st);
      launch_reduce_splits(ypart, sp.nsplit, pj * Sj, nullptr, 0.0, (double*)Zb[0], st);
      ++launches;
    }
    ++launches;
    pend(pm, (double)esize * (T + Ij * Sj + pj * Sj), 1);
    zver[j] = planner->versions[j];
  }
  void y_from_z(int j, int k) {
    const int l = 3 - j - k;
    const int64_t I = sh.dims[k], S = sh.s_of(k);
    const YzArgs a = yz_args(j, k);
    // sharded: Y_0 rows are this slab's (all-gathered), other Y_k are this slab's share (all-reduced)
    double* yout = (sharded() && k == 0) ? yloc : Y;
    int pm = pbegin(FCTN_K_YSMALL);
    // + rho A_prev (sylvester.py:106) folded into the final reduction (sharded: added after the all-reduce)
    const double* ap = sharded() ? nullptr : A64[k];
    const int nl = dtype == FCTN_F32
                       ? launch_y_from_z<float>((const float*)Zb[j], (const float*)fac_ptr(l), a, yout, ypart, ap,
                                                rho, st)
                       : launch_y_from_z<double>((const double*)Zb[j], A64[l], a, yout, ypart, ap, rho, st);
    launches += nl;
    pend(pm, (double)esize * zsize(j) + 8.0 * I * S, nl);
    if (sharded()) finish_y(k, k == 0);
  }
  // M_j of the current factors into Mbuf, outside the reference's chain (no meter)
  void build_m_direct(int k) {
    std::vector<int> rest;
    for (int j = 0; j < sh.n; ++j)
      if (j != k) rest.push_back(j);
    if (rest.size() != 2) throw std::runtime_error("direct M build is for three modes");
    ContractOp op;
    op.a.labels = sh.factor_labels(rest[0]);
    op.a.factor = rest[0];
    op.b.labels = sh.factor_labels(rest[1]);
    op.b.factor = rest[1];
    op.out.labels = sh.m_labels(k);
    op.out.buf = M_ID;
    const int cls = prof_cls;
    prof_cls = FCTN_K_MBUILD;
    contract(op);
    prof_cls = cls;
    mbuf_holds = k;
  }

  // Y_k without M_k.  The reference forms M_k = left (*) right (the final
  // join, network.py:493-497) and then Y_k = X_(k) M_k^T (sylvester.py:104).
  // When M_k is far larger than X (c3's 3-extent colour mode: |M_2| = 158 M
  // entries against T = 3.8 M) the same sums are cheaper in another
  // association: W = X (*) F over F's physical modes (F the partial whose
  // W is smaller), then Y_k = W (*) (the other partial) over the remaining
  // physical modes and the bonds between the partials.  Nothing of size M_k
  // is written (c3 mode 2: W has 9.5 M entries, 1.9 GFLOP instead of 8.9).
  // Used when M_k is not needed afterwards (k is not the order's last mode:
  // the compose reads M_last) on the FP64, unsharded path; the FLOP meter
  // still records the reference's join (plan.cpp).
  bool alt_join(const LTensor& left, const LTensor& right) {
    if (!assoc_ok || !alt_ok || !alt_route) return false;
    const int k = alt_k;
    const int n = sh.n;
    const int64_t T = sh.total(), I = sh.dims[k], S = sh.s_of(k);
    const std::vector<int> kb = sh.bonds_of(k);
    auto has = [](const std::vector<int>& v, int l) { return std::find(v.begin(), v.end(), l) != v.end(); };
    std::vector<int> shared;
    for (int l : left.labels)
      if (!sh.is_phys(l) && has(right.labels, l)) shared.push_back(l);
    int64_t rsz = 1;
    for (int l : shared) rsz *= sh.extent(l);
    auto side = [&](const LTensor& f, int64_t* psz, int64_t* ssz) {
      *psz = 1;
      *ssz = 1;
      for (int l : f.labels) {
        if (sh.is_phys(l)) *psz *= sh.extent(l);
        else if (has(kb, l)) *ssz *= sh.extent(l);
      }
    };
    int64_t pl, sl, pr, sr;
    side(left, &pl, &sl);
    side(right, &pr, &sr);
    // cost model (FP64 SIMT contractions ~15 TFLOP/s, ~4 TB/s of traffic):
    // current = join + stream with M_k written and read; alt-L / alt-R =
    // X (*) left / right first
    const double Fr_ = 15e12, Bw = 4e12;
    const double ln = (double)left.numel(sh), rn = (double)right.numel(sh);
    const double m_numel = (double)S * (double)(T / I);
    const double cur = (2.0 * (double)(pl * sl) * (double)rsz * (double)(pr * sr) + 2.0 * (double)T * S) / Fr_ +
                       8.0 * (ln + rn + 2.0 * m_numel + T) / Bw;
    const double wl = (double)(T / pl) * sl * rsz, wr = (double)(T / pr) * sr * rsz;
    const double alt_l = (2.0 * T * (double)(sl * rsz) + 2.0 * (double)(I * sl) * (double)(pr * rsz) * sr) / Fr_ +
                         8.0 * (T + ln + 2.0 * wl + rn) / Bw;
    const double alt_r = (2.0 * T * (double)(sr * rsz) + 2.0 * (double)(I * sr) * (double)(pl * rsz) * sl) / Fr_ +
                         8.0 * (T + rn + 2.0 * wr + ln) / Bw;
    const bool first_left = alt_l <= alt_r;
    const double w_numel = first_left ? wl : wr;
    double alt_cost = std::min(alt_l, alt_r), cur_cost = cur;
    if (alt_last) {
      // the compose then also runs through the partials (compose_via_partials)
      // instead of reading M_k: C = (A_k (*) F) (*) F'
      const double vl = (double)I * (double)(S / sl) * (ln / (double)sl);  // A_k (*) left
      const double vr = (double)I * (double)(S / sr) * (rn / (double)sr);  // A_k (*) right
      const double c_l = (2.0 * (double)I * S * (ln / sl) + 2.0 * (double)T * (double)(S / sl) * rsz) / Fr_ +
                         8.0 * (2.0 * vl + rn + 2.0 * T) / Bw;
      const double c_r = (2.0 * (double)I * S * (rn / sr) + 2.0 * (double)T * (double)(S / sr) * rsz) / Fr_ +
                         8.0 * (2.0 * vr + ln + 2.0 * T) / Bw;
      alt_cost += std::min(c_l, c_r);
      cur_cost += 2.0 * (double)T * S / Fr_ + 8.0 * (m_numel + 2.0 * T) / Bw;
    }
    if (alt_cost > 0.5 * cur_cost && !force_assoc) return false;  // only when clearly cheaper
    const LTensor& first = first_left ? left : right;
    const LTensor& second = first_left ? right : left;
    int pm = pbegin(FCTN_K_STREAM_Y);
    // W = X (*) first
    ContractOp op1;
    op1.a.labels.resize(n);
    for (int j = 0; j < n; ++j) op1.a.labels[j] = j;
    op1.a.buf = X_ID;
    op1.b = first;
    for (int l : op1.a.labels)
      if (!has(first.labels, l)) op1.out.labels.push_back(l);
    for (int l : first.labels)
      if (!has(op1.a.labels, l)) op1.out.labels.push_back(l);
    std::sort(op1.out.labels.begin(), op1.out.labels.end());
    ContractOp op2;
    op2.a = op1.out;
    op2.b = second;
    op2.out.labels = sh.factor_labels(k);
    op2.out.buf = Y_ID;
    // both contractions must fit the generic kernel's split-K limits
    // (kernels.cu launch_contract: K chunks <= 6144 from the scratch)
    auto feasible = [&](const ContractOp& op) {
      bool swp = false;
      const ContractDesc dd = desc_for(op, &swp);
      if (dd.K <= 6144) return true;
      const int64_t tiles = ((dd.rows + 63) / 64) * ((dd.cols + 63) / 64);
      const int64_t need = (dd.K + 6143) / 6144;
      return tiles < n_sm && need * dd.rows * dd.cols <= cscratch_cap &&
             need <= std::min<int64_t>(dd.K / 64, (2 * n_sm + tiles - 1) / tiles);
    };
    if (!feasible(op1) || !feasible(op2)) {
      pend(pm, 0.0, 0);
      return false;
    }
    op1.out.buf = alloc_labels(op1.out.labels);
    op2.a.buf = op1.out.buf;
    {
      bool sw1 = false;
      ContractDesc d1 = desc_for(op1, &sw1);
      launch_contract<double>((const double*)ptr_of(sw1 ? op1.b : op1.a), (const double*)ptr_of(sw1 ? op1.a : op1.b),
                              (double*)ptr_of(op1.out), d1, cscratch, cscratch_cap, n_sm, st);
      ++launches;
    }
    // Y_k = W (*) second, [k, bonds to k] (split-K: the reduction runs over
    // most of the tensor)
    bool sw = false;
    ContractDesc d = desc_for(op2, &sw);
    const double* pa = (const double*)ptr_of(sw ? op2.b : op2.a);
    const double* pb = (const double*)ptr_of(sw ? op2.a : op2.b);
    launch_contract<double>(pa, pb, Y, d, cscratch, cscratch_cap, n_sm, st);
    ++launches;
    free(op1.out.buf);
    launch_axpy(Y, A64[k], rho, I * S, st);  // + rho A_prev (sylvester.py:106)
    ++launches;
    pend(pm, 8.0 * (T + w_numel * 2 + ln + rn + 2.0 * I * S), 4);
    y_ready = true;
    if (alt_last) {  // keep both partials for the compose
      cp_left = left;
      cp_right = right;
      held_bufs.clear();
      for (const LTensor* t : {&left, &right})
        if (t->factor < 0 && t->buf >= 0) held_bufs.push_back(t->buf);
      compose_alt = true;
    }
    return true;
  }

  // C = A_k (*) M_k as (A_k (*) F) (*) F' from the last update's partials, then
  // the P_Omega blend and sums (solver.py:227-237,346-354): no M_k at all.
  void compose_via_partials(int k) {
    const int n = sh.n;
    const int64_t T = sh.total();
    auto has = [](const std::vector<int>& v, int l) { return std::find(v.begin(), v.end(), l) != v.end(); };
    auto out_of = [&](const std::vector<int>& a, const std::vector<int>& b) {
      std::vector<int> o;
      for (int l : a)
        if (!has(b, l)) o.push_back(l);
      for (int l : b)
        if (!has(a, l)) o.push_back(l);
      std::sort(o.begin(), o.end());
      return o;
    };
    auto numel = [&](const std::vector<int>& ls) {
      double e = 1;
      for (int l : ls) e *= (double)sh.extent(l);
      return e;
    };
    LTensor ak;
    ak.labels = sh.factor_labels(k);
    ak.factor = k;
    // absorb the side giving the smaller intermediate first
    const std::vector<int> vl = out_of(ak.labels, cp_left.labels), vr = out_of(ak.labels, cp_right.labels);
    const bool left_first = numel(vl) <= numel(vr);
    const LTensor& f1 = left_first ? cp_left : cp_right;
    const LTensor& f2 = left_first ? cp_right : cp_left;
    int pm = pbegin(FCTN_K_COMPOSE);
    ContractOp op1;
    op1.a = ak;
    op1.b = f1;
    op1.out.labels = left_first ? vl : vr;
    op1.out.buf = alloc_labels(op1.out.labels);
    contract(op1);
    ContractOp op2;
    op2.a = op1.out;
    op2.b = f2;
    op2.out.labels.resize(n);
    for (int j = 0; j < n; ++j) op2.out.labels[j] = j;  // X's own layout
    op2.out.buf = alloc_labels(op2.out.labels);
    {
      bool sw = false;
      ContractDesc d = desc_for(op2, &sw);
      launch_contract<double>((const double*)ptr_of(sw ? op2.b : op2.a), (const double*)ptr_of(sw ? op2.a : op2.b),
                              (double*)ptr_of(op2.out), d, cscratch, cscratch_cap, n_sm, st);
      ++launches;
    }
    free(op1.out.buf);
    const int nb = launch_blend((const double*)ptr_of(op2.out), (const double*)X[cur], mask, (double*)X[cur ^ 1], T,
                                rho, partials, partial_cap, st);
    launch_reduce4(partials, nb, dstats + 3 * sh.n, st);
    allreduce_sum(dstats + 3 * sh.n, 4);
    launches += 2;
    free(op2.out.buf);
    pend(pm, 8.0 * (3.0 * T + numel(op1.out.labels) * 2.0 + (double)f1.numel(sh) + (double)f2.numel(sh)) + (double)T,
         4);
    compose_alt = false;
    held_bufs.clear();
    for (int64_t id : held_frees) free(id);
    held_frees.clear();
  }

  // M_k in another association.  The reference's final join contracts two
  // partials over every bond between them (c5, middle of the order: 2 + 2
  // factors, K = 3^4 = 81 shared bonds, 20736 x 81 x 20736).  Absorbing the
  // smaller side's factors one at a time into the other partial gives the
  // same M_k with a K = 27 last step and an 81 M-entry intermediate (c5:
  // 70 -> 23 GFLOP in the 430 M-entry output step); chosen by a cost model
  // (tensor-core FLOPs at the 3xTF32 rate, bytes at HBM rate).
  bool reassoc_join(const LTensor& left, const LTensor& right, const std::vector<int>& lseq,
                    const std::vector<int>& rseq) {
    if (!assoc_ok || !alt_route || sharded()) return false;
    const bool absorb_right = rseq.size() <= lseq.size();
    const std::vector<int>& fs = absorb_right ? rseq : lseq;
    if (fs.size() != 2) return false;
    const LTensor& base = absorb_right ? left : right;
    const int k = alt_k;
    auto has = [](const std::vector<int>& v, int l) { return std::find(v.begin(), v.end(), l) != v.end(); };
    auto numel = [&](const std::vector<int>& ls) {
      double e = 1;
      for (int l : ls) e *= (double)sh.extent(l);
      return e;
    };
    auto contracted = [&](const std::vector<int>& a, const std::vector<int>& b, double* kk) {
      std::vector<int> out;
      *kk = 1;
      for (int l : a)
        if (has(b, l)) *kk *= (double)sh.extent(l);
        else out.push_back(l);
      for (int l : b)
        if (!has(a, l)) out.push_back(l);
      std::sort(out.begin(), out.end());
      return out;
    };
    const std::vector<int> mlab = sh.m_labels(k);
    const double mn = numel(mlab);
    double kjoin = 1;
    contracted(left.labels, right.labels, &kjoin);
    // pick the absorption order with the smaller intermediate
    int first = fs[0], second = fs[1];
    double k1 = 1, k1b = 1;
    std::vector<int> t1 = contracted(base.labels, sh.factor_labels(first), &k1);
    std::vector<int> t1b = contracted(base.labels, sh.factor_labels(second), &k1b);
    if (numel(t1b) < numel(t1)) {
      std::swap(first, second);
      t1 = t1b;
      k1 = k1b;
    }
    double k2 = 1;
    contracted(t1, sh.factor_labels(second), &k2);
    // join rates measured on B200 (c5 K = 27 / 81 joins: 0.48 / 1.1 ms for
    // 430 M outputs): ~75 TFLOP/s effective for the 3xTF32 join, ~10 for the
    // FP64 SIMT join; output stores at ~5 TB/s
    const double b = (double)esize, F = dtype == FCTN_F32 ? 75e12 : 10e12, B = 5e12;
    const double cur = 2.0 * mn * kjoin / F + b * mn / B;
    const double alt = (2.0 * numel(t1) * k1 + 2.0 * mn * k2) / F + b * (2.0 * numel(t1) + mn) / B;
    if ((alt > 0.8 * cur || numel(t1) > 0.5 * mn) && !force_assoc) return false;
    ContractOp op1;
    op1.a = base;
    op1.b.labels = sh.factor_labels(first);
    op1.b.factor = first;
    op1.out.labels = t1;
    op1.out.buf = alloc_labels(t1);
    contract(op1);
    ContractOp op2;
    op2.a = op1.out;
    op2.b.labels = sh.factor_labels(second);
    op2.b.factor = second;
    op2.out.labels = mlab;
    op2.out.buf = M_ID;
    contract(op2);
    free(op1.out.buf);
    return true;
  }

  void factor_update(int k, int zj, int extrap, double alpha, double beta) {
    const bool long_y = zj < 0 || zver[zj] != planner->versions[zj];
    const int form = form_for(k, long_y);
    // G_k (and, for the eigh / tri forms, its decomposition) needs only the
    // other factors' Grams E_j: the side stream forms it while this stream
    // forms Y_k; the solve joins before it reads G
    CK(cudaEventRecord(ev_fork, st));
    CK(cudaStreamWaitEvent(st2, ev_fork, 0));
    {
      const int64_t S = gsh.s_of(k);
      int pm = pbegin(FCTN_K_GRAM, st2);
      int64_t l0 = launches;
      gram_network(k, st2);
      pend(pm, 8.0 * S * S, launches - l0);
    }
    if (form != FORM_CHOL) {
      const int64_t S = gsh.s_of(k);
      int pm = pbegin(FCTN_K_EIGH, st2);
      if (form == FORM_EIGH) {
        launch_eigh(G, S, Vb[k], phi, ework, floor_shift[k], dstatus, 40, st2);
      } else {
        launch_tridiag(G, S, Vb[k], tri_d, tri_e, st2);
        if (std::isfinite(check_mu[k])) {  // T-floor test (sylvester.py:108-113): G + check_mu I must be PD
          launch_chol_solve(G, S, 0, mu[k], Fr, Fi, check_mu[k], dstatus, st2);
          ++launches;
        }
      }
      ++launches;
      pend(pm, 8.0 * 3 * S * S, 1);
    }
    CK(cudaEventRecord(ev_join, st2));
    if (zj >= 0) {
      if (zver[zj] != planner->versions[zj]) compute_z(zj);
      y_from_z(zj, k);
    } else if (y_ready) {
      y_ready = false;  // formed by alt_join during the chain
    } else {
      y_stream(k);
    }
    solve_factor(k, form, extrap, alpha, beta);
  }

  void y_stream(int k) {
    const int64_t T = sh.total();
    const int64_t I = sh.dims[k], S = sh.s_of(k), p = T / I;
    int64_t P = 1;
    for (int j = 0; j < k; ++j) P *= sh.dims[j];
    // K2: Y_k = X_(k) M_k^T + rho A_prev (sylvester.py:104-106)
    int pm = pbegin(FCTN_K_STREAM_Y);
    int nsplit = 0;
    const bool tc = tc_ok(k);
    if (tc) {
      TcStreamPlan tp = plan_stream_tc(I, P, p / P, S, n_sm, split3);
      if ((tp.nsplit * I * S + 1) / 2 > ypart_cap) throw std::runtime_error("split-partial buffer too small (stream)");
      const float* mh = (const float*)Mbuf;
      const float* ml = nullptr;
      if (split3 && S * p <= presplit_m_cap) {  // small M_k: split once in HBM, not per CTA in smem
        float* h = (float*)presplit + 2 * max_is_ + 0;
        launch_tf32_split((const float*)Mbuf, h, h + presplit_m_cap, S * p, st);
        mh = h;
        ml = h + presplit_m_cap;
        ++launches;
      }
      launch_stream_tc((const float*)X[cur], mh, (float*)ypart, I, P, p / P, S, tp, st, ml);
      nsplit = (int)tp.nsplit;
    } else {
      StreamPlan sy = plan_stream(I, S, p, target_ctas());
      if ((int64_t)sy.nsplit * I * S > ypart_cap) throw std::runtime_error("split-partial buffer too small (stream)");
      if (dtype == FCTN_F64)
        launch_stream<double>((const double*)X[cur], (const double*)Mbuf, ypart, I, P, S, p, sy, st);
      else
        launch_stream<float>((const float*)X[cur], (const float*)Mbuf, ypart, I, P, S, p, sy, st);
      nsplit = sy.nsplit;
    }
    pend(pm, (double)esize * (T + S * p), 1);
    pm = pbegin(FCTN_K_REDUCE);
    // sharded: k == 0 -> this rank's rows of Y_0 (all-gathered), k > 0 ->
    // this slab's share of Y_k (all-reduced); rho A_prev added after
    double* yout = (sharded() && k == 0) ? yloc : Y;
    const double* ap = sharded() ? nullptr : A64[k];
    if (tc)
      launch_reduce_splits_f32((const float*)ypart, nsplit, I * S, ap, rho, yout, st);
    else
      launch_reduce_splits(ypart, nsplit, I * S, ap, rho, yout, st);
    pend(pm, (tc ? 4.0 : 8.0) * nsplit * I * S + 16.0 * I * S, 1);
    if (sharded()) finish_y(k, k == 0);
  }

  void solve_factor(int k, int form, int extrap, double alpha, double beta) {
    const int64_t T = gsh.total();
    const int64_t I = gsh.dims[k], S = gsh.s_of(k), p = T / I;
    planner->meter.proj += 2 * I * p * S;   // sylvester.py:105
    planner->meter.gram += 2 * S * S * p;   // sylvester.py:58
    const DftPlan& dp = dft[k];
    const double sgn = sign == FCTN_SIGN_PD ? -1.0 : 1.0;
    int pm;
    if (form != FORM_CHOL) {
      // the reference's closed form (sylvester.py:108-116) in the basis from
      // the side stream: A = Re(F^H [(F (Y V)) / T]) V^T (eigh: T diagonal;
      // tri: V = Q, per-frequency tridiagonal solves instead of the divide)
      CK(cudaStreamWaitEvent(st, ev_join, 0));
      pm = pbegin(FCTN_K_DFT);
      launch_rotate<double>(Y, I, S, Vb[k], false, Ytmp, nullptr, 0, 0.0, 0.0, (double*)nullptr, st);
      launch_dft_fwd(Ytmp, dp, S, cosT[k], sinT[k], Fr, Fi, st, dft_gscr);
      if (form == FORM_TRI) {
        launch_thomas(tri_d, tri_e, S, dp.H1, mu[k], Fr, Fi, dstatus, st);
        ++launches;
      }
      launch_dft_inv<double>(Fr, Fi, dp, S, cosT[k], sinT[k], nullptr, Ytmp, (double*)nullptr, 0, 0.0, 0.0,
                             delta[k], sgn, nullptr, st, mu[k], form == FORM_EIGH ? phi : nullptr, dft_gscr);
      if (dtype == FCTN_F64)
        launch_rotate<double>(Ytmp, I, S, Vb[k], true, Ascratch, A64[k], extrap, alpha, beta, (double*)nullptr, st);
      else
        launch_rotate<float>(Ytmp, I, S, Vb[k], true, Ascratch, A64[k], extrap, alpha, beta, (float*)Ac[k], st);
      launch_colstats3(Ascratch, A64[k], I, S, delta[k], sgn, colstats_of(k), st);
      launches += 5;
      pend(pm, 8.0 * (6.0 * I * S + 4.0 * dp.H1 * S), 5);
    } else {
    // G_k = M_k M_k^T by the doubled network (sylvester.py:57-59) came from
    // the side stream (factor_update)
    // K3: DFT along mode k, per-frequency SPD solves, inverse DFT (sylvester.py:108-116)
    pm = pbegin(FCTN_K_DFT);
    launch_dft_fwd(Y, dp, S, cosT[k], sinT[k], Fr, Fi, st, dft_gscr);
    pend(pm, 8.0 * (I * S + 2.0 * dp.H1 * S), 1);
    CK(cudaStreamWaitEvent(st, ev_join, 0));
    pm = pbegin(FCTN_K_SOLVE);
    launch_chol_solve(G, S, dp.H1, mu[k], Fr, Fi, check_mu[k], dstatus, st);
    pend(pm, 8.0 * (S * S + 4.0 * dp.H1 * S), 1);
    pm = pbegin(FCTN_K_DFT);
    const int ninv = dtype == FCTN_F64
                         ? launch_dft_inv<double>(Fr, Fi, dp, S, cosT[k], sinT[k], A64[k], Ascratch, nullptr, extrap,
                                                  alpha, beta, delta[k], sgn, colstats_of(k), st, nullptr, nullptr,
                                                  dft_gscr)
                         : launch_dft_inv<float>(Fr, Fi, dp, S, cosT[k], sinT[k], A64[k], Ascratch, (float*)Ac[k],
                                                 extrap, alpha, beta, delta[k], sgn, colstats_of(k), st, nullptr, nullptr,
                                                 dft_gscr);
    launches += ninv - 1;
    pend(pm, 8.0 * (3.0 * I * S + 2.0 * dp.H1 * S), ninv);
    }
    if (mbuf_holds >= 0 && mbuf_holds != k) mbuf_holds = -1;  // M_j (j != k) contains A_k
    // keep every factor at a fixed address (the sweep may be replayed as a CUDA graph)
    CK(cudaMemcpyAsync(A64[k], Ascratch, I * S * sizeof(double), cudaMemcpyDeviceToDevice, st));
    // E_k = A_(k)^T A_(k) and the factor statistics are needed only by the
    // next update's Gram network (side stream) and the sweep's final stats:
    // off the critical path
    CK(cudaEventRecord(ev_fork2, st));
    CK(cudaStreamWaitEvent(st2, ev_fork2, 0));
    pm = pbegin(FCTN_K_FGRAM, st2);
    launch_factor_gram(A64[k], I, S, epart, E64[k], colstats_of(k), dstats + 3 * k, st2);
    pend(pm, 8.0 * (I * S + S * S), 2);
    launches += 7;
    planner->versions[k] += 1;  // network.py:200
    if (k == 0) refresh_slab();
  }

  void compose(int k, bool objective_only) {
    const int64_t T = sh.total();
    const int64_t I = sh.dims[k], S = sh.s_of(k), p = T / I;
    int64_t P = 1;
    for (int j = 0; j < k; ++j) P *= sh.dims[j];
    int nb;
    const bool tc = dtype == FCTN_F32 && use_tc && tc_compose_supported(I, P, p, S);
    ComposeOperands op;
    if (tc) {
      // pre-split the small operands in HBM (A_(k) always; M_k when it is at
      // most a quarter of X) so the kernel converts only what streams; timed
      // as operand preparation (MBUILD), so COMPOSE is the compose kernel
      // and its four-sum reduction
      const int ps = pbegin(FCTN_K_MBUILD);
      int nsplit = 1;
      double split_bytes = 3.0 * 4.0 * (double)(I * S);
      op.a = (const float*)fac_ptr(k);
      op.m = (const float*)Mbuf;
      float* ah = (float*)presplit;
      float* al = split3 ? ah + max_is_ : nullptr;
      launch_tf32_split(op.a, ah, al, I * S, st);
      op.a_hi = ah;
      op.a_lo = al;
      if (S * p <= presplit_m_cap) {
        float* mh = ah + 2 * max_is_;
        float* ml = split3 ? mh + presplit_m_cap : nullptr;
        launch_tf32_split(op.m, mh, ml, S * p, st);
        op.m_hi = mh;
        op.m_lo = ml;
        ++launches;
        ++nsplit;
        split_bytes += 3.0 * 4.0 * (double)(S * p);
      }
      ++launches;
      pend(ps, split_bytes, nsplit);
    }
    int pm = pbegin(FCTN_K_COMPOSE);
    if (tc) {
      nb = launch_compose_tc(op, (const float*)X[cur], maskbits, (float*)X[cur ^ 1], I, P, S, p, rho, objective_only,
                             partials, partial_cap, n_sm, split3, st);
    }
    else if (dtype == FCTN_F64)
      nb = launch_compose<double>((const double*)fac_ptr(k), (const double*)Mbuf, (const double*)X[cur], mask,
                                  (double*)X[cur ^ 1], I, P, S, p, rho, objective_only, partials, partial_cap, st);
    else
      nb = launch_compose<float>((const float*)fac_ptr(k), (const float*)Mbuf, (const float*)X[cur], mask,
                                 (float*)X[cur ^ 1], I, P, S, p, rho, objective_only, partials, partial_cap, st);
    launch_reduce4(partials, nb, dstats + 3 * sh.n, st);
    allreduce_sum(dstats + 3 * sh.n, 4);  // the four sums over all slabs
    launches += 2;
    // mask: 1 bit per entry on the tensor-core path, 1 byte on the SIMT path
    const double mask_bytes = objective_only ? 0.0 : (tc ? (double)T / 8.0 : (double)T);
    // one launch per class entry: the per-launch figure bench.py reports is
    // the compose kernel's (the 4-us reduction rides along)
    pend(pm, objective_only ? (double)esize * (S * p + T) : (double)esize * (S * p + 2 * T) + mask_bytes, 1);
  }

  void fetch_stats() {
    const int n = sh.n;
    CK(cudaMemcpyAsync(hstats, dstats, (n * 3 + 4) * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync((char*)(hstats + n * 3 + 8), dstatus, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    collect_marks();
    int status;
    std::memcpy(&status, (char*)(hstats + n * 3 + 8), sizeof(int));
    if (status) {
      CK(cudaMemsetAsync(dstatus, 0, sizeof(int), st));
      CK(cudaStreamSynchronize(st));
      if (status & 1)
        throw NumericError(
            "shifted spectrum is not strictly positive; the as-printed operator orientation cannot be "
            "inverted here");
      throw NumericError("factor subproblem matrix is not positive definite (non-finite iterate)");
    }
  }

  // all device work of one sweep (plus its host bookkeeping)
  void sweep_device(const std::vector<int>& order, int extrap, double alpha, double beta) {
    const int n = sh.n;
    const std::vector<int> route = plan_routes(order);
    compose_alt = false;
    held_bufs.clear();
    held_frees.clear();
    bool side = false;
    for (int k = 0; k < n; ++k) side |= form_for(k, true) != FORM_CHOL;
    tc_reserve_sms(side ? 1 : 0);  // one SM for the concurrent eigendecomposition
    for (size_t t = 0; t < order.size(); ++t) {
      const int k = order[t];
      const bool zr = route[t] >= 0;
      y_ready = false;
      alt_k = k;
      alt_ok = dtype == FCTN_F64 && !sharded() && n >= 4 && alg == FCTN_ALG_ACCEL;
      alt_last = k == order.back();
      assoc_ok = true;
      if (alg == FCTN_ALG_ACCEL) {
        planner->partial_cached(k, order, zr ? nullptr : this, M_ID);  // dry replay when M_k is not needed
      } else {
        planner->partial_plain(k, zr ? nullptr : this, M_ID);
      }
      alt_ok = false;
      assoc_ok = false;
      mbuf_holds = (zr || y_ready) ? -1 : k;
      factor_update(k, route[t], extrap, alpha, beta);
    }
    int k_last = order.back();
    if (alg == FCTN_ALG_ACCEL && compose_alt) {
      planner->meter.compose += 2 * (gsh.total() / gsh.dims[k_last]) * gsh.s_of(k_last) * gsh.dims[k_last];
      compose_via_partials(k_last);
    } else if (alg == FCTN_ALG_ACCEL) {
      planner->meter.compose += 2 * (gsh.total() / gsh.dims[k_last]) * gsh.s_of(k_last) * gsh.dims[k_last];
      int kc = k_last;
      if (sh.n == 3 && zroute) {
        // compose through the mode with the smallest M_j (same product, another association)
        const int64_t T = sh.total();
        for (int j = 0; j < 3; ++j)
          if (sh.s_of(j) * (T / sh.dims[j]) < sh.s_of(kc) * (T / sh.dims[kc])) kc = j;
        if (mbuf_holds != kc) build_m_direct(kc);
      }
      compose(kc, false);
    } else {
      // compose(f): the chain's FLOPs (network.py:271-278); on device the full
      // tensor is A_(n-1) times the plain partial around n-1.
      Meter keep = planner->meter;
      planner->partial_plain(n - 1, this, M_ID);
      planner->meter = keep;
      planner->meter.compose += planner->compose_chain_flops();
      compose(n - 1, false);
    }
    // rejoin the side stream (the last E_k / factor statistics) before the
    // sweep's scalars are read; also closes the fork for graph capture
    CK(cudaEventRecord(ev_side, st2));
    CK(cudaStreamWaitEvent(st, ev_side, 0));
  }

  static std::string graph_key(const std::vector<int>& order, int cur_, int extrap, double alpha, double beta) {
    std::string key;
    for (int k : order) key += std::to_string(k) + ",";
    return key + "|" + std::to_string(cur_) + "|" + std::to_string(extrap) + "|" + std::to_string(alpha) + "|" +
           std::to_string(beta);
  }
  // capture all 3! orders x both X parities up front (nothing executes; the
  // host bookkeeping of the captures is rolled back)
  void precapture(int extrap, double alpha, double beta) {
    const Meter meter0 = planner->meter;
    const std::vector<int64_t> versions0 = planner->versions;
    const int cur0 = cur, mh0 = mbuf_holds;
    int64_t zv0[3] = {zver[0], zver[1], zver[2]};
    const int64_t l0 = launches;
    struct Restore {  // also on a failed capture
      std::function<void()> f;
      ~Restore() { f(); }
    } restore{[&, meter0, versions0, cur0, mh0, l0, zv0a = zv0[0], zv0b = zv0[1], zv0c = zv0[2]] {
      planner->meter = meter0;
      planner->versions = versions0;
      cur = cur0;
      zver[0] = zv0a;
      zver[1] = zv0b;
      zver[2] = zv0c;
      mbuf_holds = mh0;
      launches = l0;
    }};
    std::vector<int> order{0, 1, 2};
    for (int parity = 0; parity < 2; ++parity) {
      do {
        cur = parity;
        z_invalidate();
        mbuf_holds = -1;
        launches = 0;
        const std::string key = graph_key(order, parity, extrap, alpha, beta);
        if (graphs.count(key)) continue;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
          sweep_device(order, extrap, alpha, beta);
        } catch (...) {
          cudaGraph_t g = nullptr;
          cudaStreamEndCapture(st, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        cudaGraph_t g;
        CK(cudaStreamEndCapture(st, &g));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphDestroy(g));
        graphs[key] = {ge, launches};
      } while (std::next_permutation(order.begin(), order.end()));
    }
  }

  // the host-side effects of sweep_device without any device work (graph replay)
  void sweep_bookkeeping(const std::vector<int>& order) {
    const int64_t T = gsh.total();
    for (int k : order) {
      if (alg == FCTN_ALG_ACCEL)
        planner->partial_cached(k, order, nullptr, M_ID);
      else
        planner->partial_plain(k, nullptr, M_ID);
      const int64_t I = gsh.dims[k], S = gsh.s_of(k), p = T / I;
      planner->meter.proj += 2 * I * p * S;  // sylvester.py:105
      planner->meter.gram += 2 * S * S * p;  // sylvester.py:58
      planner->versions[k] += 1;             // network.py:200
    }
    const int k_last = order.back();
    if (alg == FCTN_ALG_ACCEL)
      planner->meter.compose += 2 * (T / gsh.dims[k_last]) * gsh.s_of(k_last) * gsh.dims[k_last];
    else
      planner->meter.compose += planner->compose_chain_flops();
  }

  void sweep(const int32_t* order_in, int extrap, double alpha, double beta, double* stats, int64_t* counters) {
    if (!uploaded) throw UsageError("no data uploaded");
    const int n = sh.n;
    std::vector<int> order(order_in, order_in + n);
    {
      std::vector<int> chk = order;
      std::sort(chk.begin(), chk.end());
      for (int i = 0; i < n; ++i)
        if (chk[i] != i) throw UsageError("order is not a permutation of range(n)");
    }
    Meter m0 = planner->meter;
    int64_t hits0 = planner->cache().hits;
    launches = 0;
    // NCCL collectives and the loop-back copies are stream work and are captured
    // with the kernels; only the host-callback backend has to run eagerly
    const bool graphable = use_graph && sh.n == 3 && !prof && comm.kind != 2;
    const std::string key = graphable ? graph_key(order, cur, extrap, alpha, beta) : std::string();
    if (graphable && graphs.empty()) {
      if (comm.kind == 1) {
        // a communicator that cannot be captured falls back to eager sweeps
        // (same collectives in the same order on every rank)
        try {
          precapture(extrap, alpha, beta);
        } catch (const std::exception&) {
          cudaGetLastError();
          drop_graphs();
          use_graph = false;
          return sweep(order_in, extrap, alpha, beta, stats, counters);
        }
      } else {
        precapture(extrap, alpha, beta);
      }
    }
    auto it = graphable ? graphs.find(key) : graphs.end();
    if (graphable && it != graphs.end()) {
      // replay: host bookkeeping only (the reference's FLOP meter, cache,
      // versions), then the captured device work
      sweep_bookkeeping(order);
      CK(cudaEventRecord(ev0, st));
      CK(cudaGraphLaunch(it->second.first, st));
      launches = it->second.second;
    } else if (graphable) {
      CK(cudaEventRecord(ev0, st));
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        sweep_device(order, extrap, alpha, beta);
      } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      cudaGraph_t g;
      CK(cudaStreamEndCapture(st, &g));
      cudaGraphExec_t ge;
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphDestroy(g));
      graphs[key] = {ge, launches};
      CK(cudaGraphLaunch(ge, st));
    } else {
      CK(cudaEventRecord(ev0, st));
      sweep_device(order, extrap, alpha, beta);
    }
    CK(cudaEventRecord(ev1, st));
    fetch_stats();
    cur ^= 1;
    z_invalidate();  // X changed
    mbuf_holds = -1;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    double pen = 0.0, step = 0.0, fmax = 0.0;
    for (int k = 0; k < n; ++k) {
      step += hstats[3 * k + 0];
      fmax = std::max(fmax, std::sqrt(hstats[3 * k + 1]));
      pen += 0.5 * lam[k] * hstats[3 * k + 2];
    }
    const double* sums = hstats + 3 * n;
    for (int i = 0; i < FCTN_ST_COUNT; ++i) stats[i] = 0.0;
    stats[FCTN_ST_DIFF_SQ] = sums[0];
    stats[FCTN_ST_BASE_SQ] = sums[1];
    stats[FCTN_ST_DATA_SQ] = sums[2];
    stats[FCTN_ST_XNEW_SQ] = sums[3];
    stats[FCTN_ST_PENALTY] = pen;
    stats[FCTN_ST_STEP_FAC] = step;
    stats[FCTN_ST_FNORM_MAX] = fmax;
    stats[FCTN_ST_OBJECTIVE] = 0.5 * sums[2] + pen;
    stats[FCTN_ST_DEVICE_MS] = ms;
    if (counters) {
      for (int i = 0; i < FCTN_CT_COUNT; ++i) counters[i] = 0;
      const Meter& m1 = planner->meter;
      counters[FCTN_CT_FLOPS] = m1.total() - m0.total();
      counters[FCTN_CT_MK] = m1.mk - m0.mk;
      counters[FCTN_CT_COMPOSE] = m1.compose - m0.compose;
      counters[FCTN_CT_HITS] = planner->cache().hits - hits0;
      counters[FCTN_CT_LAUNCHES] = launches;
    }
  }

  double objective(int64_t* counters) {
    if (!uploaded) throw UsageError("no data uploaded");
    const int n = sh.n;
    Meter keep = planner->meter;
    planner->partial_plain(0, this, M_ID);
    planner->meter = keep;
    mbuf_holds = -1;
    compose(0, true);
    fetch_stats();
    double val = 0.5 * hstats[3 * n + 2];
    for (int k = 0; k < n; ++k) val += 0.5 * lam[k] * hstats[3 * k + 2];
    if (counters) {
      for (int i = 0; i < FCTN_CT_COUNT; ++i) counters[i] = 0;
      int64_t c = planner->compose_chain_flops();
      counters[FCTN_CT_FLOPS] = c;
      counters[FCTN_CT_COMPOSE] = c;
    }
    return val;
  }
};

static thread_local std::string g_err;

template <typename F>
static int guarded(Ctx* c, F&& f) {
  try {
    // every call runs on its context's device (several contexts / devices per process)
    if (c && c->configured) CK(cudaSetDevice(c->device));
    f();
    return 0;
  } catch (const UsageError& e) {
    (c ? c->err : g_err) = e.what();
    return 1;
  } catch (const NumericError& e) {
    (c ? c->err : g_err) = e.what();
    return 2;
  } catch (const std::exception& e) {
    (c ? c->err : g_err) = e.what();
    return 3;
  }
}

}  // namespace fctn

using fctn::Ctx;

struct fctn_ctx {
  Ctx impl;
};

extern "C" {

int fctn_create(int device, int dtype, int n, const int64_t* dims, const int64_t* rank_tri, const double* lam,
                const double* delta, int lap_sign, double rho, int algorithm, int64_t cache_budget, fctn_ctx** out) {
  *out = nullptr;
  fctn_ctx* c = new fctn_ctx();
  int rc = fctn::guarded(nullptr, [&] {
    c->impl.configure(device, dtype, n, dims, rank_tri, lam, delta, lap_sign, rho, algorithm, cache_budget);
  });
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return 0;
}

int fctn_upload(fctn_ctx* c, const void* x_F, const uint8_t* mask_F) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    const int64_t T = x.sh.total();
    CK(cudaMemcpyAsync(x.X[0], x_F, T * x.esize, cudaMemcpyHostToDevice, x.st));
    CK(cudaMemcpyAsync(x.mask, mask_F, T, cudaMemcpyHostToDevice, x.st));
    fctn::launch_pack_mask(x.mask, T, x.maskbits, x.st);
    CK(cudaStreamSynchronize(x.st));
    x.cur = 0;
    x.uploaded = true;
    x.z_invalidate();
    x.mbuf_holds = -1;
  });
}

}  // extern "C"

namespace fctn {
// Page-lock a caller buffer for the duration of one large transfer (the
// pageable path stages through the driver at a fraction of the PCIe/C2C
// rate).  Falls back to pageable if registration fails.
struct HostPin {
  void* p = nullptr;
  HostPin(const void* ptr, size_t bytes) {
    if (bytes < ((size_t)64 << 20) || getenv("FCTN_NO_PIN")) return;
    if (cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterDefault) == cudaSuccess)
      p = const_cast<void*>(ptr);
    else
      cudaGetLastError();
  }
  ~HostPin() {
    if (p) cudaHostUnregister(p);
  }
};

// Large host <-> device transfers through a ring of pinned 32 MB chunks:
// several host threads copy a chunk between the caller's (pageable) buffer
// and a pinned buffer while the DMA engine moves the previous one.  Measured
// alternative: page-locking the caller's 2 GB buffer (cudaHostRegister)
// costs more than the copy itself and the pageable driver path runs at
// ~8 GB/s.  Synchronous with respect to the host on return.
struct Stager {
  static constexpr size_t CH = (size_t)32 << 20;
  static constexpr int NB = 3;
  void* buf[NB] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev[NB] = {nullptr, nullptr, nullptr};
  int nthr = 1;
  Stager() {
    for (int b = 0; b < NB; ++b) {
      CK(cudaMallocHost(&buf[b], CH));
      CK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    const unsigned hc = std::thread::hardware_concurrency();
    // one copy thread per host core up to 16 (measured with the fp64 <-> fp32
    // conversion on these threads: 8 -> 16 threads, upload 54 -> 43 ms, download 64 -> 46 ms at c4)
    nthr = (int)std::max(1u, std::min(16u, hc ? hc : 1u));
    if (const char* e = getenv("FCTN_STAGE_THREADS")) nthr = std::max(1, atoi(e));
  }
  ~Stager() {
    for (int b = 0; b < NB; ++b) {
      if (buf[b]) cudaFreeHost(buf[b]);
      if (ev[b]) cudaEventDestroy(ev[b]);
    }
  }
  void pcopy(void* dst, const void* src, size_t n) const {  // parallel memcpy
    if (nthr <= 1 || n < ((size_t)4 << 20)) {
      std::memcpy(dst, src, n);
      return;
    }
    const size_t part = ((n + nthr - 1) / nthr + 4095) & ~(size_t)4095;
    std::vector<std::thread> th;
    for (int t = 1; t < nthr; ++t) {
      const size_t o = (size_t)t * part;
      if (o >= n) break;
      th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, std::min(part, n - o)); });
    }
    std::memcpy(dst, src, std::min(part, n));
    for (auto& x : th) x.join();
  }
  void h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
    size_t c = 0;
    for (size_t o = 0; o < n; o += CH, ++c) {
      const int b = (int)(c % NB);
      const size_t m = std::min(CH, n - o);
      CK(cudaEventSynchronize(ev[b]));  // the DMA that last read buf[b] is done
      pcopy(buf[b], (const char*)src + o, m);
      CK(cudaMemcpyAsync((char*)dst + o, buf[b], m, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(ev[b], st));
    }
    CK(cudaStreamSynchronize(st));
  }
  // f(lo, hi) over [0, n) on the copy threads
  template <typename F>
  void pfor(size_t n, F&& f) const {
    if (nthr <= 1 || n < ((size_t)1 << 20)) {
      f((size_t)0, n);
      return;
    }
    const size_t part = ((n + nthr - 1) / nthr + 1023) & ~(size_t)1023;
    std::vector<std::thread> th;
    for (int t = 1; t < nthr; ++t) {
      const size_t o = (size_t)t * part;
      if (o >= n) break;
      th.emplace_back([=] { f(o, std::min(n, o + part)); });
    }
    f((size_t)0, std::min(part, n));
    for (auto& x : th) x.join();
  }
  // fp64 host tensor -> fp32 device tensor: the copy threads round to fp32
  // (round-to-nearest-even, the bits of the device's own conversion) while
  // they fill the pinned ring, so half the bytes cross PCIe and the ring
  void h2d_f64_to_f32(float* dst, const double* src, size_t count, cudaStream_t st) {
    const size_t CE = CH / 4;  // floats per ring buffer
    size_t c = 0;
    for (size_t o = 0; o < count; o += CE, ++c) {
      const int b = (int)(c % NB);
      const size_t m = std::min(CE, count - o);
      CK(cudaEventSynchronize(ev[b]));
      float* stage = (float*)buf[b];
      const double* from = src + o;
      pfor(m, [=](size_t lo, size_t hi) {
        for (size_t e = lo; e < hi; ++e) stage[e] = (float)from[e];
      });
      CK(cudaMemcpyAsync(dst + o, stage, m * 4, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(ev[b], st));
    }
    CK(cudaStreamSynchronize(st));
  }
  // fp32 device tensor -> fp64 host tensor, widened by the copy threads
  void d2h_f32_to_f64(double* dst, const float* src, size_t count, cudaStream_t st) {
    const size_t CE = CH / 4;
    const size_t nc = (count + CE - 1) / CE;
    for (size_t c = 0; c <= nc; ++c) {
      if (c < nc) {
        const int b = (int)(c % NB);
        const size_t o = c * CE, m = std::min(CE, count - o);
        CK(cudaEventSynchronize(ev[b]));
        CK(cudaMemcpyAsync(buf[b], src + o, m * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ev[b], st));
      }
      if (c >= 1) {
        const size_t pc = c - 1;
        const int pb = (int)(pc % NB);
        const size_t o = pc * CE, m = std::min(CE, count - o);
        CK(cudaEventSynchronize(ev[pb]));
        const float* stage = (const float*)buf[pb];
        double* to = dst + o;
        pfor(m, [=](size_t lo, size_t hi) {
          for (size_t e = lo; e < hi; ++e) to[e] = (double)stage[e];
        });
      }
    }
    CK(cudaStreamSynchronize(st));
  }
  // D2H of n bytes produced chunk by chunk: `produce(o, m)` enqueues on `st`
  // whatever must run before chunk [o, o+m) of `src` is ready (may be empty)
  template <typename Produce>
  void d2h(void* dst, const void* src, size_t n, cudaStream_t st, Produce&& produce) {
    const size_t nc = (n + CH - 1) / CH;
    for (size_t c = 0; c <= nc; ++c) {
      if (c < nc) {
        const int b = (int)(c % NB);
        const size_t o = c * CH, m = std::min(CH, n - o);
        produce(o, m, b);
        CK(cudaMemcpyAsync(buf[b], (const char*)src + o, m, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ev[b], st));
      }
      if (c >= 1) {  // drain the previous chunk while this one moves
        const size_t pc = c - 1;
        const int pb = (int)(pc % NB);
        const size_t o = pc * CH, m = std::min(CH, n - o);
        CK(cudaEventSynchronize(ev[pb]));
        pcopy((char*)dst + o, buf[pb], m);
      }
    }
  }
};

// One ring per device, leased under that device's mutex for a whole
// transfer: contexts on different devices never share pinned buffers or
// events (events belong to the device current at creation), and two threads
// driving two contexts on one device take turns instead of sharing a slot.
struct StagerLease {
  std::unique_lock<std::mutex> lock;
  Stager* s;
  Stager* operator->() const { return s; }
};
static StagerLease stager() {
  static std::mutex map_mu;
  static std::map<int, std::pair<std::unique_ptr<std::mutex>, Stager*>> rings;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::mutex* mu;
  {
    std::lock_guard<std::mutex> g(map_mu);
    auto& slot = rings[dev];
    if (!slot.first) {
      slot.first.reset(new std::mutex());
      slot.second = new Stager();  // created with `dev` current: its events live there
    }
    mu = slot.first.get();
  }
  StagerLease l{std::unique_lock<std::mutex>(*mu), nullptr};
  std::lock_guard<std::mutex> g(map_mu);
  l.s = rings[dev].second;
  return l;
}
// stream-ordered device scratch released on every exit path
struct DevScratch {
  void* p = nullptr;
  cudaStream_t st;
  DevScratch(size_t bytes, cudaStream_t s) : st(s) { CK(cudaMallocAsync(&p, bytes, st)); }
  ~DevScratch() {
    if (p) cudaFreeAsync(p, st);
  }
};
static bool use_stager(size_t bytes) {
  if (getenv("FCTN_NO_STAGE")) return false;
  const char* m = getenv("FCTN_STAGE_MIN_BYTES");  // tests lower it to exercise the ring on small tensors
  const size_t lo = m ? (size_t)std::strtoull(m, nullptr, 10) : ((size_t)64 << 20);
  return bytes >= lo;
}
}  // namespace fctn

extern "C" {

int fctn_upload_f64(fctn_ctx* c, const double* x_F, const uint8_t* mask_F) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    const int64_t T = x.sh.total();
    const bool stage = fctn::use_stager((size_t)T * 8);
    fctn::HostPin pin_x(stage ? nullptr : x_F, stage ? 0 : (size_t)T * 8), pin_m(stage ? nullptr : mask_F, stage ? 0 : (size_t)T);
    if (x.dtype == FCTN_F64) {
      if (stage) fctn::stager()->h2d(x.X[0], x_F, (size_t)T * 8, x.st);
      else CK(cudaMemcpyAsync(x.X[0], x_F, T * 8, cudaMemcpyHostToDevice, x.st));
    } else if (stage) {  // fp64 host data, fp32 context: rounded by the ring's copy threads
      fctn::stager()->h2d_f64_to_f32((float*)x.X[0], x_F, (size_t)T, x.st);
    } else {  // small tensors: convert on the device, in chunks
      const int64_t chunk = std::min<int64_t>(T, (int64_t)1 << 26);
      fctn::DevScratch scratch(chunk * 8, x.st);
      double* tmp = (double*)scratch.p;
      for (int64_t o = 0; o < T; o += chunk) {
        const int64_t n = std::min(chunk, T - o);
        if (stage) fctn::stager()->h2d(tmp, x_F + o, (size_t)n * 8, x.st);
        else CK(cudaMemcpyAsync(tmp, x_F + o, n * 8, cudaMemcpyHostToDevice, x.st));
        fctn::launch_convert_f64_f32(tmp, (float*)x.X[0] + o, n, x.st);
      }
    }
    if (stage) fctn::stager()->h2d(x.mask, mask_F, (size_t)T, x.st);
    else CK(cudaMemcpyAsync(x.mask, mask_F, T, cudaMemcpyHostToDevice, x.st));
    fctn::launch_pack_mask(x.mask, T, x.maskbits, x.st);
    CK(cudaStreamSynchronize(x.st));
    x.cur = 0;
    x.uploaded = true;
    x.z_invalidate();
    x.mbuf_holds = -1;
  });
}

int fctn_trim_cache(void) {
  fctn::dev_cache().trim();
  return 0;
}

int fctn_get_x_f64(fctn_ctx* c, double* x_F) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    const int64_t T = x.sh.total();
    if (fctn::use_stager((size_t)T * 8)) {
      fctn::StagerLease lease = fctn::stager();
      fctn::Stager& sg = *lease.s;
      if (x.dtype == FCTN_F64) {
        sg.d2h(x_F, x.X[x.cur], (size_t)T * 8, x.st, [](size_t, size_t, int) {});
      } else {  // fp32 over PCIe, widened to fp64 by the ring's copy threads
        sg.d2h_f32_to_f64(x_F, (const float*)x.X[x.cur], (size_t)T, x.st);
      }
      CK(cudaStreamSynchronize(x.st));
      return;
    }
    fctn::HostPin pin_x(x_F, (size_t)T * 8);
    if (x.dtype == FCTN_F64) {
      CK(cudaMemcpyAsync(x_F, x.X[x.cur], T * 8, cudaMemcpyDeviceToHost, x.st));
    } else {
      const int64_t chunk = std::min<int64_t>(T, (int64_t)1 << 26);
      double* tmp = nullptr;
      CK(cudaMallocAsync((void**)&tmp, chunk * 8, x.st));
      for (int64_t o = 0; o < T; o += chunk) {
        const int64_t n = std::min(chunk, T - o);
        fctn::launch_convert_f32_f64((const float*)x.X[x.cur] + o, tmp, n, x.st);
        CK(cudaMemcpyAsync(x_F + o, tmp, n * 8, cudaMemcpyDeviceToHost, x.st));
      }
      CK(cudaFreeAsync(tmp, x.st));
    }
    CK(cudaStreamSynchronize(x.st));
  });
}

int fctn_set_factors(fctn_ctx* c, const double* const* a_unf, const int64_t* versions, int reset_cache) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    for (int k = 0; k < x.gsh.n; ++k) {
      int64_t e = x.gsh.dims[k] * x.gsh.s_of(k);
      CK(cudaMemcpyAsync(x.A64[k], a_unf[k], e * sizeof(double), cudaMemcpyHostToDevice, x.st));
      if (x.dtype == FCTN_F32) fctn::launch_convert_f64_f32(x.A64[k], (float*)x.Ac[k], e, x.st);
      if (versions) x.planner->versions[k] = versions[k];
    }
    for (int k = 0; k < x.gsh.n; ++k) x.factor_refresh(k);
    x.refresh_slab();
    x.z_invalidate();
    x.mbuf_holds = -1;
    if (reset_cache) x.planner->reset_cache(&x);
    CK(cudaStreamSynchronize(x.st));
  });
}

int fctn_set_rank(fctn_ctx* c, const int64_t* rank_tri) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    CK(cudaStreamSynchronize(x.st));
    for (int i = 0; i < x.sh.n * (x.sh.n - 1) / 2; ++i)
      if (rank_tri[i] < 1) throw fctn::UsageError("rank entries must be >= 1");
    x.sh.tri.assign(rank_tri, rank_tri + x.sh.n * (x.sh.n - 1) / 2);
    x.gsh.tri = x.sh.tri;
    x.configure_shape();
  });
}

int fctn_get_factors(fctn_ctx* c, double* const* a_unf) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    for (int k = 0; k < x.gsh.n; ++k) {
      int64_t e = x.gsh.dims[k] * x.gsh.s_of(k);
      CK(cudaMemcpyAsync(a_unf[k], x.A64[k], e * sizeof(double), cudaMemcpyDeviceToHost, x.st));
    }
    CK(cudaStreamSynchronize(x.st));
  });
}

int fctn_get_x(fctn_ctx* c, void* x_F) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    CK(cudaMemcpyAsync(x_F, x.X[x.cur], x.sh.total() * x.esize, cudaMemcpyDeviceToHost, x.st));
    CK(cudaStreamSynchronize(x.st));
  });
}

int fctn_objective(fctn_ctx* c, double* out, int64_t* counters) {
  return fctn::guarded(&c->impl, [&] { *out = c->impl.objective(counters); });
}

int fctn_sweep(fctn_ctx* c, const int32_t* order, int extrap, double alpha, double beta, double* stats,
               int64_t* counters) {
  return fctn::guarded(&c->impl, [&] { c->impl.sweep(order, extrap, alpha, beta, stats, counters); });
}

int fctn_plan_sweeps(int n, const int64_t* dims, const int64_t* rank_tri, int algorithm, int64_t cache_budget,
                     int n_sweeps, const int32_t* orders, int64_t* counters) {
  return fctn::guarded(nullptr, [&] {
    fctn::Shape sh;
    sh.n = n;
    sh.dims.assign(dims, dims + n);
    sh.tri.assign(rank_tri, rank_tri + n * (n - 1) / 2);
    fctn::Planner pl(sh, cache_budget);
    pl.versions.assign(n, 0);
    for (int t = 0; t < n_sweeps; ++t) {
      std::vector<int> order(orders + (int64_t)t * n, orders + (int64_t)(t + 1) * n);
      fctn::Meter m0 = pl.meter;
      int64_t h0 = pl.cache().hits;
      const int64_t T = sh.total();
      for (int k : order) {
        if (algorithm == FCTN_ALG_ACCEL)
          pl.partial_cached(k, order, nullptr, 0);
        else
          pl.partial_plain(k, nullptr, 0);
        int64_t I = sh.dims[k], S = sh.s_of(k), p = T / I;
        pl.meter.proj += 2 * I * p * S;
        pl.meter.gram += 2 * S * S * p;
        pl.versions[k] += 1;
      }
      int kl = order.back();
      if (algorithm == FCTN_ALG_ACCEL)
        pl.meter.compose += 2 * (T / sh.dims[kl]) * sh.s_of(kl) * sh.dims[kl];
      else
        pl.meter.compose += pl.compose_chain_flops();
      int64_t* ct = counters + (int64_t)t * FCTN_CT_COUNT;
      for (int i = 0; i < FCTN_CT_COUNT; ++i) ct[i] = 0;
      ct[FCTN_CT_FLOPS] = pl.meter.total() - m0.total();
      ct[FCTN_CT_MK] = pl.meter.mk - m0.mk;
      ct[FCTN_CT_COMPOSE] = pl.meter.compose - m0.compose;
      ct[FCTN_CT_HITS] = pl.cache().hits - h0;
    }
  });
}

int fctn_nccl_unique_id(uint8_t* id128) {
  return fctn::guarded(nullptr, [&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    auto get = fctn::nccl_sym<ncclResult_t (*)(ncclUniqueId*)>("ncclGetUniqueId");
    ncclUniqueId id;
    if (get(&id) != ncclSuccess) throw std::runtime_error("ncclGetUniqueId failed");
    std::memcpy(id128, &id, 128);
  });
}

namespace fctn {
// standard partition of mode 0 over ranks; reshape the context to the slab
static void shard_to(Ctx& x, int rank, int nranks, int64_t lo, int64_t hi) {
  if (x.uploaded) throw UsageError("set the communicator before uploading data");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw UsageError("bad rank / nranks");
  const int64_t I0 = x.gsh.dims[0];
  if (lo != rank * I0 / nranks || hi != (rank + 1) * I0 / nranks)
    throw UsageError("slab must be the standard partition [r*I0/n, (r+1)*I0/n)");
  if (hi <= lo) throw UsageError("empty slab: more ranks than rows of mode 0");
  x.rank = rank;
  x.nranks = nranks;
  x.slab_lo = lo;
  x.slab_hi = hi;
  x.slab_max = (I0 + nranks - 1) / nranks;
  x.sh.dims[0] = hi - lo;
  const int64_t T = x.sh.total();
  cudaFree(x.X[0]);
  cudaFree(x.X[1]);
  cudaFree(x.mask);
  cudaFree(x.maskbits);
  CK(cudaMalloc(&x.X[0], T * x.esize));
  CK(cudaMalloc(&x.X[1], T * x.esize));
  CK(cudaMalloc(&x.mask, T));
  CK(cudaMalloc(&x.maskbits, ((T + 31) / 32) * sizeof(uint32_t)));
  x.configure_shape();
}
}  // namespace fctn

int fctn_set_comm(fctn_ctx* c, const uint8_t* id128, int rank, int nranks, int64_t slab_lo, int64_t slab_hi) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    fctn::shard_to(x, rank, nranks, slab_lo, slab_hi);
    if (nranks > 1 || id128) {
      using InitFn = ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int);
      auto init = fctn::nccl_sym<InitFn>("ncclCommInitRank");
      x.comm.allreduce = fctn::nccl_sym<decltype(x.comm.allreduce)>("ncclAllReduce");
      x.comm.allgather = fctn::nccl_sym<decltype(x.comm.allgather)>("ncclAllGather");
      x.comm.destroy = fctn::nccl_sym<decltype(x.comm.destroy)>("ncclCommDestroy");
      ncclUniqueId id;
      if (!id128) throw fctn::UsageError("an NCCL unique id is required");
      std::memcpy(&id, id128, 128);
      ncclComm_t comm;
      CK(cudaSetDevice(x.device));
      if (init(&comm, nranks, id, rank) != ncclSuccess) throw std::runtime_error("ncclCommInitRank failed");
      x.comm.nccl = comm;
      x.comm.kind = 1;
      // both collectives once outside any capture (NCCL sets up its channels
      // and buffers lazily, per collective), at a size of the sweep's own
      // messages
      const size_t wn = 1 << 14;
      double* w = nullptr;
      CK(cudaMalloc(&w, wn * (size_t)(nranks + 1) * sizeof(double)));
      CK(cudaMemsetAsync(w, 0, wn * (size_t)(nranks + 1) * sizeof(double), x.st));
      const ncclResult_t r1 = x.comm.allreduce(w, w, wn, ncclFloat64, ncclSum, comm, x.st);
      const ncclResult_t r2 = x.comm.allgather(w, w + wn, wn, ncclFloat64, comm, x.st);
      CK(cudaStreamSynchronize(x.st));
      cudaFree(w);
      if (r1 != ncclSuccess || r2 != ncclSuccess) throw std::runtime_error("NCCL warm-up collectives failed");
    }
  });
}

int fctn_set_comm_loopback(fctn_ctx* c, int rank, int nranks, int64_t slab_lo, int64_t slab_hi) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    fctn::shard_to(x, rank, nranks, slab_lo, slab_hi);
    x.comm.kind = 3;
  });
}

int fctn_set_comm_host(fctn_ctx* c, fctn_host_allreduce_fn allreduce, fctn_host_allgather_fn allgather, void* user,
                       int rank, int nranks, int64_t slab_lo, int64_t slab_hi) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    if (!allreduce || !allgather) throw fctn::UsageError("both host callbacks are required");
    fctn::shard_to(x, rank, nranks, slab_lo, slab_hi);
    x.comm.h_allreduce = allreduce;
    x.comm.h_allgather = allgather;
    x.comm.user = user;
    x.comm.kind = 2;
  });
}

int fctn_timer(fctn_ctx* c, int op, double* ms) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    if (!x.tstart) {
      CK(cudaEventCreate(&x.tstart));
      CK(cudaEventCreate(&x.tstop));
    }
    if (op == 0) {
      CK(cudaEventRecord(x.tstart, x.st));
    } else {
      CK(cudaEventRecord(x.tstop, x.st));
      CK(cudaEventSynchronize(x.tstop));
      float f = 0.f;
      CK(cudaEventElapsedTime(&f, x.tstart, x.tstop));
      if (ms) *ms = f;
    }
  });
}

int fctn_set_profiling(fctn_ctx* c, int on) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    x.prof = on != 0;
    for (int i = 0; i < FCTN_K_COUNT; ++i) {
      x.prof_ms[i] = 0;
      x.prof_n[i] = 0;
      x.prof_bytes[i] = 0;
    }
  });
}

int fctn_get_profile(fctn_ctx* c, double* ms, int64_t* launches, double* bytes) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    for (int i = 0; i < FCTN_K_COUNT; ++i) {
      ms[i] = x.prof_ms[i];
      launches[i] = x.prof_n[i];
      bytes[i] = x.prof_bytes[i];
    }
  });
}

int fctn_selftest_stream(int device, int dtype, int use_tc, int64_t I, int64_t P, int64_t Q, int64_t S,
                         const void* x, const void* m, double* y) {
  return fctn::guarded(nullptr, [&] {
    CK(cudaSetDevice(device));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    const size_t es = dtype == FCTN_F64 ? 8 : 4;
    const int64_t T = I * P * Q, p = P * Q;
    void *dx, *dm;
    double *part, *dy;
    int nsm = 148;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    CK(cudaMalloc(&dx, T * es));
    CK(cudaMalloc(&dm, p * S * es));
    CK(cudaMalloc(&dy, I * S * sizeof(double)));
    CK(cudaMemcpy(dx, x, T * es, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dm, m, p * S * es, cudaMemcpyHostToDevice));
    if (use_tc && dtype == FCTN_F32 && fctn::tc_stream_supported(I, P, Q, S)) {
      fctn::TcStreamPlan tp = fctn::plan_stream_tc(I, P, Q, S, nsm, !(getenv("FCTN_TF32") && std::string(getenv("FCTN_TF32")) == "1x"));
      CK(cudaMalloc(&part, tp.nsplit * I * S * sizeof(float)));
      fctn::launch_stream_tc((const float*)dx, (const float*)dm, (float*)part, I, P, Q, S, tp, st);
      fctn::launch_reduce_splits_f32((const float*)part, (int)tp.nsplit, I * S, nullptr, 0.0, dy, st);
    } else {
      fctn::StreamPlan sp = fctn::plan_stream(I, S, p, nsm * 4);
      CK(cudaMalloc(&part, (int64_t)sp.nsplit * I * S * sizeof(double)));
      if (dtype == FCTN_F64)
        fctn::launch_stream<double>((const double*)dx, (const double*)dm, part, I, P, S, p, sp, st);
      else
        fctn::launch_stream<float>((const float*)dx, (const float*)dm, part, I, P, S, p, sp, st);
      fctn::launch_reduce_splits(part, sp.nsplit, I * S, nullptr, 0.0, dy, st);
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(y, dy, I * S * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(dx);
    cudaFree(dm);
    cudaFree(dy);
    cudaFree(part);
    cudaStreamDestroy(st);
  });
}

int fctn_selftest_eigh(int device, int64_t S, const double* G, double* V, double* phi, int reps,
                       double* ms_per_launch, int* sweeps) {
  return fctn::guarded(nullptr, [&] {
    CK(cudaSetDevice(device));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    double *dG, *dV0, *dV, *dphi, *work = nullptr;
    int *dstat, *dsw;
    CK(cudaMalloc(&dG, S * S * 8));
    CK(cudaMalloc(&dV0, S * S * 8));
    CK(cudaMalloc(&dV, S * S * 8));
    CK(cudaMalloc(&dphi, S * 8));
    CK(cudaMalloc(&dstat, 4));
    CK(cudaMalloc(&dsw, 4));
    if (!fctn::eigh_fits_smem(S)) CK(cudaMalloc(&work, (2 * S * S + S) * 8));
    CK(cudaMemset(dstat, 0, 4));
    CK(cudaMemcpy(dG, G, S * S * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dV0, V, S * S * 8, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < std::max(reps, 1); ++r) {
      CK(cudaMemcpyAsync(dV, dV0, S * S * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaEventRecord(a, st));
      fctn::launch_eigh(dG, S, dV, dphi, work, 1.0, dstat, 40, st, dsw);
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    CK(cudaMemcpy(V, dV, S * S * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(phi, dphi, S * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sweeps, dsw, 4, cudaMemcpyDeviceToHost));
    *ms_per_launch = best;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    for (void* p : {(void*)dG, (void*)dV0, (void*)dV, (void*)dphi, (void*)dstat, (void*)dsw, (void*)work}) cudaFree(p);
    cudaStreamDestroy(st);
  });
}

int fctn_selftest_chol(int device, int64_t S, int64_t H1, const double* G, const double* mu, double* Fr,
                       double* Fi, int reps, double* ms_per_launch) {
  return fctn::guarded(nullptr, [&] {
    CK(cudaSetDevice(device));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    double *dG, *dmu, *dFr, *dFi, *wFr, *wFi;
    int* dstat;
    CK(cudaMalloc(&dG, S * S * 8));
    CK(cudaMalloc(&dmu, H1 * 8));
    CK(cudaMalloc(&dFr, H1 * S * 8));
    CK(cudaMalloc(&dFi, H1 * S * 8));
    CK(cudaMalloc(&wFr, H1 * S * 8));
    CK(cudaMalloc(&wFi, H1 * S * 8));
    CK(cudaMalloc(&dstat, 4));
    CK(cudaMemset(dstat, 0, 4));
    CK(cudaMemcpy(dG, G, S * S * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dmu, mu, H1 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dFr, Fr, H1 * S * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dFi, Fi, H1 * S * 8, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < std::max(reps, 1); ++r) {
      CK(cudaMemcpyAsync(wFr, dFr, H1 * S * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(wFi, dFi, H1 * S * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaEventRecord(a, st));
      fctn::launch_chol_solve(dG, S, H1, dmu, wFr, wFi, NAN, dstat, st);
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    if (ms_per_launch) *ms_per_launch = best;
    CK(cudaMemcpy(Fr, wFr, H1 * S * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(Fi, wFi, H1 * S * 8, cudaMemcpyDeviceToHost));
    int status = 0;
    CK(cudaMemcpy(&status, dstat, 4, cudaMemcpyDeviceToHost));
    for (auto* p : {dG, dmu, dFr, dFi, wFr, wFi}) cudaFree(p);
    cudaFree(dstat);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    if (status) throw fctn::NumericError("factorisation failed");
  });
}

}  // extern "C"

namespace fctn {
// Both metric passes over device-resident est / truth; `reduce` sums the
// per-slice partials over ranks (identity on one GPU).  out: FCTN_Q_COUNT.
template <typename TE, typename TT, typename R>
static void quality_passes(int64_t hw_local, int64_t hw_global, int64_t nslices, int n_sm, const TE* e, const TT* t,
                           const uint8_t* mask, double peak, R&& reduce, double* out, cudaStream_t st) {
  const QualityPlan p = quality_plan(hw_local, nslices, n_sm);
  const double inv_hw = 1.0 / (double)hw_global;
  double* scratch = nullptr;
  const int64_t nd = p.part_doubles + p.sums_doubles + QUALITY_OUT;
  CK(cudaMallocAsync((void**)&scratch, nd * sizeof(double), st));
  double* part = scratch;
  double* s1 = part + p.part_doubles;
  double* s2 = s1 + nslices * QUALITY_S1;
  double* dout = s2 + nslices * QUALITY_S2;
  launch_quality_pass1<TE, TT>(p, e, t, mask, part, s1, st);
  reduce(s1, nslices * QUALITY_S1);
  launch_quality_pass2<TE, TT>(p, e, t, s1, inv_hw, part, s2, st);
  reduce(s2, nslices * QUALITY_S2);
  launch_quality_final(p, s1, s2, inv_hw, peak, dout, st);
  CK(cudaGetLastError());
  double h[QUALITY_OUT];
  CK(cudaMemcpyAsync(h, dout, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(scratch, st));
  CK(cudaStreamSynchronize(st));
  for (int q = 0; q < FCTN_Q_COUNT; ++q) out[q] = q < QUALITY_OUT ? h[q] : 0.0;
}

template <typename R>
static void quality_dispatch(int te, int tt, int64_t hw_local, int64_t hw_global, int64_t nslices, int n_sm,
                             const void* e, const void* t, const uint8_t* mask, double peak, R&& reduce, double* out,
                             cudaStream_t st) {
  if (te == FCTN_F64 && tt == FCTN_F64)
    quality_passes(hw_local, hw_global, nslices, n_sm, (const double*)e, (const double*)t, mask, peak, reduce, out, st);
  else if (te == FCTN_F32 && tt == FCTN_F32)
    quality_passes(hw_local, hw_global, nslices, n_sm, (const float*)e, (const float*)t, mask, peak, reduce, out, st);
  else if (te == FCTN_F32 && tt == FCTN_F64)
    quality_passes(hw_local, hw_global, nslices, n_sm, (const float*)e, (const double*)t, mask, peak, reduce, out, st);
  else
    quality_passes(hw_local, hw_global, nslices, n_sm, (const double*)e, (const float*)t, mask, peak, reduce, out, st);
}

static void quality_check(int n, double peak, int dtype) {
  if (n < 2) throw UsageError("need at least two modes");
  if (!(peak > 0)) throw UsageError("peak must be > 0");
  if (dtype != FCTN_F64 && dtype != FCTN_F32) throw UsageError("dtype must be FCTN_F64 or FCTN_F32");
}
}  // namespace fctn

extern "C" {

int fctn_quality(int device, int dtype, int n, const int64_t* dims, const void* est_F, const void* truth_F,
                 const uint8_t* mask_F, double peak, double* out) {
  return fctn::guarded(nullptr, [&] {
    fctn::quality_check(n, peak, dtype);
    int64_t T = 1;
    for (int k = 0; k < n; ++k) {
      if (dims[k] < 1) throw fctn::UsageError("extents must be >= 1");
      T *= dims[k];
    }
    const int64_t hw = dims[0] * dims[1];
    const size_t es = dtype == FCTN_F64 ? 8 : 4;
    CK(cudaSetDevice(device));
    int n_sm = 148;
    CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    void *de = nullptr, *dt = nullptr;
    uint8_t* dm = nullptr;
    CK(cudaMallocAsync(&de, T * es, st));
    CK(cudaMallocAsync(&dt, T * es, st));
    if (mask_F) CK(cudaMallocAsync((void**)&dm, T, st));
    auto up = [&](void* d, const void* h, size_t n) {
      if (fctn::use_stager(n)) fctn::stager()->h2d(d, h, n, st);
      else CK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, st));
    };
    up(de, est_F, T * es);
    up(dt, truth_F, T * es);
    if (mask_F) up(dm, mask_F, T);
    fctn::quality_dispatch(dtype, dtype, hw, hw, T / hw, n_sm, de, dt, dm, peak, [](double*, int64_t) {}, out, st);
    CK(cudaFreeAsync(de, st));
    CK(cudaFreeAsync(dt, st));
    if (dm) CK(cudaFreeAsync(dm, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fctn_quality_ctx(fctn_ctx* c, const void* truth_F, int truth_dtype, int mask_mode, double peak, double* out) {
  return fctn::guarded(&c->impl, [&] {
    Ctx& x = c->impl;
    fctn::quality_check(x.gsh.n, peak, truth_dtype);
    if (!x.uploaded) throw fctn::UsageError("no data uploaded");
    if (mask_mode != 0 && mask_mode != 1) throw fctn::UsageError("mask_mode must be 0 or 1");
    const int64_t T = x.sh.total();
    const size_t es = truth_dtype == FCTN_F64 ? 8 : 4;
    const int64_t hw_local = x.sh.dims[0] * x.sh.dims[1];
    const int64_t hw_global = x.gsh.dims[0] * x.gsh.dims[1];
    void* dt = nullptr;
    CK(cudaMallocAsync(&dt, T * es, x.st));
    if (fctn::use_stager(T * es)) fctn::stager()->h2d(dt, truth_F, T * es, x.st);
    else CK(cudaMemcpyAsync(dt, truth_F, T * es, cudaMemcpyHostToDevice, x.st));
    fctn::quality_dispatch(x.dtype, truth_dtype, hw_local, hw_global, T / hw_local, x.n_sm, x.X[x.cur], dt,
                           mask_mode ? x.mask : nullptr, peak,
                           [&](double* d, int64_t nd) { x.allreduce_sum(d, nd); }, out, x.st);
    CK(cudaFreeAsync(dt, x.st));
    CK(cudaStreamSynchronize(x.st));
  });
}

int fctn_sync(fctn_ctx* c) {
  return fctn::guarded(&c->impl, [&] { CK(cudaStreamSynchronize(c->impl.st)); });
}

const char* fctn_last_error(fctn_ctx* c) { return c ? c->impl.err.c_str() : fctn::g_err.c_str(); }

const char* fctn_version(void) { return "fctn_b200 0.1.0 (sm_100a)"; }

void fctn_destroy(fctn_ctx* c) { delete c; }

}  // extern "C"
