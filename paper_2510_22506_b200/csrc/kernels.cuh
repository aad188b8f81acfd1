// Kernel launch wrappers (sm_100a).  All launches go on the caller's stream;
// every reduction runs in a fixed order (no floating-point atomics).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fctn {

// K1: generic labeled contraction via offset tables (network.py:249-258,
// tensor.py:156-200).  C[rowC[r]+colC[c]] = sum_k A[rowA[r]+kA[k]] * B[colB[c]+kB[k]].
template <typename T>
void launch_contract(const T* A, const T* B, T* C, const int64_t* rowA, const int64_t* rowC,
                     const int64_t* colB, const int64_t* colC, const int64_t* kA, const int64_t* kB,
                     int64_t rows, int64_t cols, int64_t K, cudaStream_t st);

// generic permutation: out[o] = in[sum_d digit_d(o) * in_stride[d]]
struct PermDesc {
  int nd;
  int64_t ext[16];
  int64_t in_stride[16];
};
template <typename T>
void launch_permute(const T* in, T* out, const PermDesc& d, int64_t numel, cudaStream_t st);

// K2: split-K streaming products over the long reduction axis p.
//   part[split][i + I*s] = sum_{p in split} X(i,p) * M[s + S*p]
// with X(i,p) = X[(p%P) + P*i + P*I*(p/P)] (the mode-k view of an F-order
// tensor; P = product of extents before mode k).  With X := M, I := S, P := 1
// the same kernel yields the Gram partials.
struct StreamPlan {
  int ts;        // padded s tile (16, 32, 64, 128)
  int ti;        // i tile (4096 / ts)
  int n_itiles;
  int nsplit;
  int64_t chunk; // p per split
};
StreamPlan plan_stream(int64_t I, int64_t S, int64_t p, int target_ctas);
template <typename T>
void launch_stream(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S, int64_t p,
                   const StreamPlan& sp, cudaStream_t st);
// Y[i+I*s] = sum_split part + rho * Aprev[i+I*s]   (sylvester.py:104-106)
void launch_reduce_y(const double* part, int nsplit, int64_t I, int64_t S, const double* aprev,
                     double rho, double* Y, cudaStream_t st);
// G = sym(sum_split part)   (sylvester.py:57-59)
void launch_reduce_g(const double* part, int nsplit, int64_t S, double* G, cudaStream_t st);

// K3: the factor subproblem (sylvester.py:98-116) by real DFT along mode k
// (L is circulant, laplacian.py:46-47,75-81) and one Cholesky solve of
// (G + (lam*Lambda_w + rho) I) per frequency pair.
void launch_dft_fwd(const double* Y, int64_t I, int64_t S, const double* cosT, const double* sinT,
                    double* Fr, double* Fi, cudaStream_t st);
// per-frequency solves; extra check CTA when check_mu is finite:
// Cholesky of G + check_mu I must succeed (T-floor test, sylvester.py:108-113)
void launch_chol_solve(const double* G, int64_t S, int64_t H1, const double* mu, double* Fr, double* Fi,
                       double check_mu, int* status, cudaStream_t st);
// inverse DFT + extrapolation + factor write (solver.py:240-243,330-333)
template <typename T>
void launch_dft_inv(const double* Fr, const double* Fi, int64_t I, int64_t S, const double* cosT,
                    const double* sinT, const double* Aold, double* Anew, T* Acompute, int extrap,
                    double alpha, double beta, cudaStream_t st);
// ||A_new - A_old||^2, ||A_new||^2, tr(A^T L A) (laplacian.py:59-71) into out[0..2]
void launch_factor_stats(const double* Anew, const double* Aold, int64_t I, int64_t S, double delta,
                         double sgn, double* out, cudaStream_t st);

// K4: C = A_(k) M (network.py:313-332) fused with the P_Omega blend
// (solver.py:227-237) and the four sweep reductions (solver.py:220,346-354,382).
// objective_only: no X_new write; sums (X - C)^2 into slot 2.
template <typename T>
int launch_compose(const T* A, const T* M, const T* Xold, const uint8_t* mask, T* Xnew, int64_t I,
                   int64_t P, int64_t S, int64_t p, double rho, bool objective_only, double* partials,
                   int64_t partial_cap, cudaStream_t st);
// fixed-order final reduction of n x 4 partials into out[0..3]
void launch_reduce4(const double* partials, int64_t n, double* out, cudaStream_t st);

void launch_convert_f64_f32(const double* in, float* out, int64_t n, cudaStream_t st);

}  // namespace fctn
