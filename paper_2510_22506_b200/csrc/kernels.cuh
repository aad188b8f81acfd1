// Kernel launch wrappers (sm_100a).  All launches go on the caller's stream;
// every reduction runs in a fixed order (no floating-point atomics).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fctn {

// ---------------------------------------------------------------- K1 merge
// Generic labeled contraction (network.py:249-258, tensor.py:156-200):
// C[rc(r)+cc(c)] = sum_k A[ra(r)+ka(k)] * B[cb(c)+kb(k)], each offset a
// mixed-radix multi-index over the labels (up to 12 per group).
struct ContractDesc {
  int nr = 0, nc = 0, nk = 0;
  int64_t r_ext[12], r_sa[12], r_sc[12];
  int64_t c_ext[12], c_sb[12], c_sc[12];
  int64_t k_ext[12], k_sa[12], k_sb[12];
  int64_t rows = 1, cols = 1, K = 1;
};
// scratch: split-K partials (may be null: no split); returns nothing
template <typename T>
void launch_contract(const T* A, const T* B, T* C, const ContractDesc& d, T* scratch, int64_t scratch_cap, int n_sm,
                     cudaStream_t st);
int64_t contract_split_scratch(const ContractDesc& d, int n_sm);
// large-output contractions (join.cu): register-tiled, cp.async-staged
bool join_applicable(const ContractDesc& d, size_t esize);
template <typename T>
void launch_join(const T* A, const T* B, T* C, const ContractDesc& d, int n_sm, cudaStream_t st);
// fp32 large-output contractions on the tensor cores (join_tc.cu, 3xTF32)
bool tc_join_applicable(const ContractDesc& d);
void launch_join_tc(const float* A, const float* B, float* C, const ContractDesc& d, int n_sm, cudaStream_t st);

// generic permutation: out[o] = in[sum_d digit_d(o) * in_stride[d]]
struct PermDesc {
  int nd;
  int64_t ext[16];
  int64_t in_stride[16];
};
template <typename T>
void launch_permute(const T* in, T* out, const PermDesc& d, int64_t numel, cudaStream_t st);

void launch_convert_f64_f32(const double* in, float* out, int64_t n, cudaStream_t st);
void launch_convert_f32_f64(const float* in, double* out, int64_t n, cudaStream_t st);
// N = 3 schedule: Y_k = Z_j (*) A_(l) with Z_j = X x_j A_(j) = [r, o, b_j.., b_j..]
// (rows: the two other modes, the lower one fastest; then the bonds of j in
// A_(j)'s column order) and l the third mode.  Strides are in units of the
// row extents: Z bond (j,l) zc, bond (j,k) zk; A_(l) bond (l,j) ac, (l,k) aa;
// Y_k bond (k,j) yz, (k,l) ya.  long_l: l is the fast row mode (r = i_l,
// o = i_k), otherwise k is (r = i_k, o = i_l).  Y fp64 (I_k x s_k).
struct YzArgs {
  int64_t Ir, Io;
  int Rc, Rz, Ra;
  int64_t zc, zk, ac, aa, yz, ya;
  bool long_l;
};
template <typename T>
// + rho * aprev when aprev != null (sylvester.py:106); returns the launches
int launch_y_from_z(const T* Z, const T* Al, const YzArgs& a, double* Y, double* part, const double* aprev, double rho,
                    cudaStream_t st);
// mode-0 sharding helpers (fctn_set_comm)
void launch_copy_rows(const double* A, int64_t I, int64_t S, int64_t lo, int64_t rows, void* out, bool f32,
                      cudaStream_t st);
void launch_scatter_rows(const double* g, int nranks, int64_t slab_max, int64_t I, int64_t S, double* Y,
                         cudaStream_t st);
void launch_axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st);

// ---------------------------------------------------------------- K2 stream
// part[split][i + I*s] = sum_{p in split} X(i,p) * M[p + p_total*s]
// with X(i,p) = X[(p%P) + P*i + P*I*(p/P)] (the mode-k view of an F-order
// tensor; P = product of extents before mode k).
struct StreamPlan {
  int ts;        // padded s tile (16, 32, 64, 128)
  int ri;        // rows of mode k per thread (1 or 4)
  int ti;        // i tile
  int n_itiles;
  int nsplit;
  int64_t chunk; // p per split
};
StreamPlan plan_stream(int64_t I, int64_t S, int64_t p, int target_ctas);
template <typename T>
void launch_stream(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S, int64_t p,
                   const StreamPlan& sp, cudaStream_t st);
// out[e] = sum_split part[split*n+e] + rho*aprev[e] (aprev may be null)   (sylvester.py:104-106)
void launch_reduce_splits(const double* part, int nsplit, int64_t n, const double* aprev, double rho,
                          double* out, cudaStream_t st);
void launch_reduce_splits_f32(const float* part, int nsplit, int64_t n, const double* aprev, double rho,
                              double* out, cudaStream_t st);

// tcgen05 TF32 path (stream_tc.cu): fp32 partials part[split][i + I*s]
struct TcStreamPlan {
  int nt;              // UMMA N (bond tile, padded S)
  int64_t n_mtiles;    // 128-row tiles of mode k
  int64_t npb;         // 32-wide K blocks per run of the fastest mode (1 when P == 1)
  int64_t nkb;         // K blocks in total
  int64_t kb_per_split;
  int64_t nsplit;
  bool split3;         // 3xTF32 (hi/lo split) instead of round-to-nearest TF32
};
bool tc_stream_supported(int64_t I, int64_t P, int64_t Q, int64_t S);
TcStreamPlan plan_stream_tc(int64_t I, int64_t P, int64_t Q, int64_t S, int n_sm, bool split3);
// Mlo: optional pre-split low part of M (then M holds rn_tf32 hi); with
// split3 only the streamed X tile is split in shared memory
void launch_stream_tc(const float* X, const float* M, float* part, int64_t I, int64_t P, int64_t Q, int64_t S,
                      const TcStreamPlan& tp, cudaStream_t st, const float* Mlo = nullptr);
bool tc_stream_batched_supported(int64_t R, int64_t Q, int64_t NB, int64_t S);
// persistent tensor-core passes leave n SMs free (side-stream work)
void tc_reserve_sms(int n);
void launch_stream_tc_batched(const float* X, const float* Bh, const float* Bl, float* out, int64_t R, int64_t Q,
                              int64_t NB, int64_t S, int n_sm, cudaStream_t st);

// ---------------------------------------------------------------- K3 solve
struct DftPlan {
  int64_t I, H1, I1, I2;
  size_t smem;
  bool fast;
};
DftPlan plan_dft(int64_t I);
// F[w + H1*s] = sum_j Y[j + I*s] exp(-2 pi i w j / I), w < H1  (laplacian.py:75-81)
// (modes with p.fast == false run from `gscr`: 6 I doubles per column)
void launch_dft_fwd(const double* Y, const DftPlan& p, int64_t S, const double* cosT, const double* sinT,
                    double* Fr, double* Fi, cudaStream_t st, double* gscr = nullptr);
// per-frequency Cholesky solves of (G + mu_w I) a_w = F_w; extra check CTA
// when check_mu is finite (T-floor test, sylvester.py:108-113)
bool chol_solve_fits(int64_t S);  // one system's factor + panel buffers fit shared memory (s <= 146)
void launch_chol_solve(const double* G, int64_t S, int64_t H1, const double* mu, double* Fr, double* Fi,
                       double check_mu, int* status, cudaStream_t st);
// inverse DFT + extrapolation + factor write + per-column stats
// (solver.py:240-243,330-333; laplacian.py:59-71)
template <typename T>
int launch_dft_inv(const double* Fr, const double* Fi, const DftPlan& p, int64_t S, const double* cosT,
                    const double* sinT, const double* Aold, double* Anew, T* Acompute, int extrap, double alpha,
                    double beta, double delta, double sgn, double* colstats, cudaStream_t st,
                    const double* mu = nullptr, const double* phi = nullptr, double* gscr = nullptr);
// eigenbasis form of the solve (eigh.cu; sylvester.py:51-61,98-116):
// G = V diag(phi) V^T by one-sided Jacobi (V in: warm start, out: basis);
// status |= 1 when floor_shift + min(phi) <= 1e-10 (T floor), 2 if non-finite
size_t eigh_smem_bytes(int64_t S);
bool eigh_fits_smem(int64_t S);
void launch_eigh(const double* G, int64_t S, double* V, double* phi, double* work, double floor_shift, int* status,
                 int max_sweeps, cudaStream_t st, int* nsweeps = nullptr);
// out = A W, W = V or V^T (A: I x S); with aold: extrapolation epilogue and the
// compute-dtype copy acomp
template <typename T>
void launch_rotate(const double* A, int64_t I, int64_t S, const double* V, bool trans, double* out,
                   const double* aold, int extrap, double alpha, double beta, T* acomp, cudaStream_t st);
void launch_identity(double* V, int64_t S, cudaStream_t st);
// tridiagonal form of the solve (tri.cu): G = Q T Q^T (d: diagonal, e:
// sub-diagonal of T) in one CTA; per-frequency Thomas solves of
// (T + mu_w I) x = F_w in place on (Fr, Fi) (status |= 2 on a non-positive pivot)
size_t tridiag_smem_bytes(int64_t S);
bool tridiag_fits_smem(int64_t S);
void launch_tridiag(const double* G, int64_t S, double* Q, double* d, double* e, cudaStream_t st);
void launch_thomas(const double* d, const double* e, int64_t S, int64_t H1, const double* mu, double* Fr, double* Fi,
                   int* status, cudaStream_t st);
// [||a - a_old||^2, ||a||^2, a.(L a)] per column
void launch_colstats3(const double* A, const double* Aold, int64_t I, int64_t S, double delta, double sgn,
                      double* colstats, cudaStream_t st);
// per-column [0, ||a||^2, a.(L a)] without a previous iterate
void launch_factor_colstats(const double* A, int64_t I, int64_t S, double delta, double sgn, double* colstats,
                            cudaStream_t st);
// E = A^T A (s x s) and the fold of colstats (S x 3) into stats3
int fgram_splits(int64_t I);
void launch_factor_gram(const double* A, int64_t I, int64_t S, double* part, double* E, const double* colstats,
                        double* stats3, cudaStream_t st);

// ---------------------------------------------------------------- K4 compose
// C = A_(k) M (network.py:313-332) fused with the P_Omega blend
// (solver.py:227-237) and the four sweep reductions (solver.py:220,346-354,382).
// objective_only: no X_new write; sums (X - C)^2 into slot 2.
template <typename T>
int launch_compose(const T* A, const T* M, const T* Xold, const uint8_t* mask, T* Xnew, int64_t I,
                   int64_t P, int64_t S, int64_t p, double rho, bool objective_only, double* partials,
                   int64_t partial_cap, cudaStream_t st);
// tcgen05 TF32 path (compose_tc.cu); returns the number of partial rows written
bool tc_compose_supported(int64_t I, int64_t P, int64_t p, int64_t S);
// operands: A_(k) [I, S] and M_k [p, S] fp32; optional pre-split copies
// (hi = rn_tf32, lo = rest) skip the in-kernel conversion of that operand
struct ComposeOperands {
  const float* a = nullptr;
  const float* m = nullptr;
  const float *a_hi = nullptr, *a_lo = nullptr, *m_hi = nullptr, *m_lo = nullptr;
};
int launch_compose_tc(const ComposeOperands& op, const float* Xo, const uint32_t* maskbits, float* Xn, int64_t I,
                      int64_t P, int64_t S, int64_t p, double rho, bool objective_only, double* partials,
                      int64_t partial_cap, int n_sm, bool split3, cudaStream_t st);
// hi = rn_tf32(x), lo = x - hi (lo may be null)
void launch_tf32_split(const float* x, float* hi, float* lo, int64_t n, cudaStream_t st);
void launch_pack_mask(const uint8_t* mask, int64_t T, uint32_t* bits, cudaStream_t st);
// fixed-order final reduction of n x 4 partials into out[0..3]
void launch_reduce4(const double* partials, int64_t n, double* out, cudaStream_t st);
// the blend + sums of K4 for an already formed C (T entries, fp64)
int launch_blend(const double* C, const double* Xo, const uint8_t* mask, double* Xn, int64_t T, double rho,
                 double* partials, int64_t partial_cap, cudaStream_t st);

// ---------------------------------------------------------------- quality metrics (metrics.cu)
// psnr / ssim / rel_err of metrics.py:33-105 over F-order slices of hw entries
struct QualityPlan {
  int64_t hw = 0, nslices = 0, seglen = 0;
  int nseg = 0;
  int64_t part_doubles = 0;  // segment partials scratch
  int64_t sums_doubles = 0;  // per-slice sums (pass 1 then pass 2)
};
QualityPlan quality_plan(int64_t hw, int64_t nslices, int n_sm);
static constexpr int QUALITY_S1 = 7, QUALITY_S2 = 3, QUALITY_OUT = 7;
// per-slice [sum e, sum t, sum d^2, sum t^2, off-mask sum d^2, sum t^2, count]
template <typename TE, typename TT>
void launch_quality_pass1(const QualityPlan& p, const TE* est, const TT* truth, const uint8_t* mask, double* part,
                          double* sums1, cudaStream_t st);
// per-slice centred [sum (e-mu)^2, sum (t-mu)^2, sum (e-mu)(t-mu)]; inv_hw = 1/(global H*W)
template <typename TE, typename TT>
void launch_quality_pass2(const QualityPlan& p, const TE* est, const TT* truth, const double* sums1, double inv_hw,
                          double* part, double* sums2, cudaStream_t st);
// out[QUALITY_OUT] = [mean psnr, mean ssim, ||e-t||^2, ||t||^2, off-mask ||e-t||^2, ||t||^2, count]
void launch_quality_final(const QualityPlan& p, const double* sums1, const double* sums2, double inv_hw, double peak,
                          double* out, cudaStream_t st);

}  // namespace fctn
