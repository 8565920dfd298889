// internal.h — host/device structures shared by the kernels and the C-ABI layer.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>
#include <utility>

#include "common.cuh"

namespace fcgno {

// State of one batched FCG solve (all device pointers).  Passed by value to every kernel.
struct FcgDev {
  int n, B, N, nblk;          // grid, batch, n*n, CTAs per system (ceil(N / kTile))
  int m, maxit, schedule;
  double tol, scale;          // scale = (n+1)^2
  const double* k;            // [B][N]
  int kfast;                  // problem's k all in [2^-400, 2^400] (branch-free face division)
  int vec32;                  // r, w, ring_p, ring_s stored as float (opts.vec_fp32, reading R21);
                              // the double* fields below then point at float arrays
  double* r64;                // vec32 with a NO: fp64 copy of r (the NO's input), else nullptr
  const double* f;            // [B][N]
  double* u;                  // [B][N]  caller's iterate
  double* r;                  // [B][N]  residual
  const double* w;            // [B][N]  preconditioned residual (== r for identity)
  double* ring_p;             // [m+1][B][N]
  double* ring_s;             // [m+1][B][N]
  double* gamma;              // [m+1][B]   (p_k, s_k)
  double* beta;               // [B][kMmax]
  double* alpha;              // [B]
  double* rr;                 // [B]        (r_i, r_i)
  double* rho0;               // [B]
  dd* part_win;               // [B][nblk][kMmax]
  dd* part_step;              // [B][nblk][2]
  dd* part_rr;                // [B][nblk]
  unsigned* cnt;              // [3][B] last-CTA counters
  int* flags;                 // [B]
  int* status;                // [B] caller
  int* iters;                 // [B] caller
  double* hist;               // [B][maxit+1] caller or nullptr
  int* iter;                  // global iteration counter
  int* active;                // systems still running (set by init, then by the last update CTA)
  unsigned* gcnt;             // [2] systems arrived in this update / of them still running
  // classical preconditioner (fcgno_fcg_solve_stationary): kind 1 Jacobi, 2 red-black SGS, 0 none
  int st_kind, st_sweeps;
  double *st_xa, *st_xb;      // [B][N] sweep iterates
  // Theorem-1 diagnostics (fcgno_fcg_solve_diag; all nullptr otherwise)
  const double* dg_ustar;     // [B][N] reference solution u*
  double* dg_eps;             // [B][maxit] eps_i = ||w_i - e_i||_A / ||e_i||_A
  double* dg_erra;            // [B][maxit] ||e_i||_A, e_i = u* - u_i
  double *dg_e, *dg_d, *dg_Ae, *dg_Ad;   // [B][N] scratch
  double* dg_sc;              // [2][B] (e, A e), (d, A d)
  dd* dg_part;                // [B][nblk] dot partials
  unsigned* dg_cnt;           // [B] dot counters
};

// Packed NO weights (element offsets into the packed array of T; complex = 2 T).
struct NoLayout {
  int w;
  size_t W1E, b1, A0, A1, A2;          // layer 1 with the lift folded in
  size_t W[2], b[2], R[2];             // layers 2 and 3: W [o][c], b [o], R [kappa][c][o] complex
  size_t Q, dw, cst;                   // layer 4 folded with the projection
  size_t total;                        // elements of T
};
NoLayout no_layout(int w);

// Device view of the NO for one launch sequence.
template <typename T>
struct NoDev {
  int n, B, N, w;
  int use_gelu;
  int k0;                     // mode index of a constant field (Fourier kappa = 0: 210; Chebyshev k = 0: 0)
  const double* k;            // [B][N] nodal k (fp64, the problem's)
  const T* pk;                // packed weights
  NoLayout L;
  const T* F;                 // twiddles [n][kModes] complex: exp(-2 pi i kappa j / n)
  const T* khat;              // [B][400] complex DFT_M(k)
  T* rpart;                   // [B][ngroups][400] complex partial DFT_M(r/s)
  double* rinv;               // [B] 1/||r|| (written by the input DFT; tensor-core path)
  int ngroups;                // row groups of the input DFT
  T* v0;                      // [B][w][N]
  T* v1;                      // [B][w][N]
  T* chat;                    // [400][B][w] complex
  T* ghat;                    // [B][w][400] complex
  unsigned char* vb0;         // tensor-core path: activation blobs (ping-pong), px_layout.cuh
  unsigned char* vb1;
  unsigned char* Gb;          // G rows (y-synthesised spectral term)
  float* Tb;                  // T rows (x-analysed activations)
  unsigned char* cst;         // constant operand blobs (twiddles, layer weights, mixing weights)
  float* p3;                  // [B][n][n] layer-3 projection bypass term (tensor-core path)
  int tc;                     // 1: fp32 layers on tcgen05 (no_px_kernels.cu)
};

// Tensor-core (pixel-major) SNO path, no_px_kernels.cu.
struct PxLayerHost {
  int n, w, B, layer, use_gelu;              // layer 0, 1, 2 = SNO layers 1-3
  const double *r, *rr, *k;                  // layer 1 inputs (rr: 1/||r|| per system, from the input DFT)
  const unsigned char* vin;                  // V blobs (layers 2, 3)
  unsigned char* vout;                       // V blobs written (layers 1, 2)
  const unsigned char* G;                    // G rows (y-synthesised spectral term)
  float* T;                                  // T rows (x-analysed activations)
  const unsigned char* cst;                  // constant operand blobs (launch_px_prep)
  const float *bias, *w1e, *dw;              // [w]; layer 1: W1 E [w][2]; layer 3: D W4 [w]
  float* p3;                                 // layer 3: projection bypass term [B][n][n]
  const int* status;
};
bool px_supported_shape(int n, int w);       // geometry and shared-memory budget (no device query)
bool px_supported(int n, int w);             // ... and the device's opt-in shared memory allows it
size_t px_const_bytes(int n, int w);
size_t px_v_bytes(int n, int w, int B);
size_t px_g_bytes(int n, int w, int B);
size_t px_t_floats(int n, int w, int B);
size_t px_mx_offset(int n, int w, int mix);
cudaError_t prepare_px_kernels();
cudaError_t launch_px_prep(int n, int w, const float* W2, const float* W3, const float* R2, const float* R3,
                           const float* Q, const float* F, unsigned char* out, cudaStream_t s);
cudaError_t launch_px_layer(const PxLayerHost& h, cudaStream_t s);
cudaError_t launch_px_ysyn(const float* ghat, const unsigned char* cst, unsigned char* Gb, int n, int w, int B,
                           const int* status, cudaStream_t s);
cudaError_t launch_px_yan(const float* T, const unsigned char* cst, float* chat, int n, int w, int B, const int* status,
                          cudaStream_t s);
cudaError_t px_trace_read(unsigned long long* host, int count);
cudaError_t launch_mix_px(int mix, const float* chat, const unsigned char* cst, float* ghat, int n, int w, int B,
                          float inv_n2, const int* status, cudaStream_t s);

// In-graph profiling hook: begin/end record CUDA events around launches of a kernel class.
enum ProfClass : int { PROF_NO_LAYER = 0, PROF_NO_MIX, PROF_NO_OUT, PROF_NO_INPUT, PROF_WINDOW, PROF_PFORM,
                       PROF_STENCIL, PROF_UPDATE, PROF_FINALIZE, PROF_NO_YDIR, PROF_NCLASS };
struct ProfHook {
  virtual ~ProfHook() = default;
  virtual void begin(int cls, cudaStream_t s) = 0;
  virtual void end(int cls, cudaStream_t s) = 0;
};

// Launch helpers (defined in fcg_kernels.cu / no_kernels.cu).  All return cudaGetLastError().
cudaError_t launch_apply_A(const double* k, const double* x, double* y, int n, int B, bool kfast, cudaStream_t s);
cudaError_t launch_dot(const double* x, const double* y, double* out, dd* part, unsigned* cnt, int n, int B,
                       cudaStream_t s);
cudaError_t launch_check_k(const double* k, size_t count, int* bad, cudaStream_t s);
cudaError_t launch_init_residual(const FcgDev& d, cudaStream_t s);
cudaError_t launch_window_dots(const FcgDev& d, cudaStream_t s);
// classical preconditioners (kind 1 = Jacobi, 2 = red-black SGS); z, w of the FCG vector type (v32)
cudaError_t launch_stationary(const double* k, const void* z, double* xa, double* xb, void* w, bool v32, int n, int B,
                              bool kfast, int kind, int sweeps, const int* status, cudaStream_t s);
cudaError_t launch_pform_stencil(const FcgDev& d, cudaStream_t s);
cudaError_t launch_update(const FcgDev& d, cudaStream_t s);
cudaError_t launch_flush_x(const FcgDev& d, cudaStream_t s);
cudaError_t launch_loop_cond(const int* active, cudaGraphConditionalHandle h, cudaStream_t s);

cudaError_t launch_twiddles(float* F32, double* F64, int n, int basis, cudaStream_t s);
template <typename T>
cudaError_t launch_khat(const double* k, const T* F, T* part, T* khat, int n, int B, int ngroups,
                        cudaStream_t s);
// NO forward; when fcg != nullptr the output kernel also computes the FCG window dots and
// freezes converged systems; otherwise w = NO(r) standalone (rr must hold (r,r)).
template <typename T>
cudaError_t launch_no_forward(const NoDev<T>& no, const double* r, const double* rr, double* w,
                              const FcgDev* fcg, const int* status, cudaStream_t s, int* nlaunch,
                              ProfHook* prof = nullptr);
template <typename T>
cudaError_t prepare_no_kernels();
cudaError_t prepare_no_constants(const NoDev<float>& no, cudaStream_t s);
template <typename T>
size_t no_max_smem(int n, int w);   // largest dynamic smem any NO kernel needs for (n, w)

// SNO training (train_kernels.cu).  Batched strided fp32 GEMM:
// C[z](m,n) = alpha sum_k A[z](m,k) B[z](k,n) + beta C[z](m,n) (+ bias[n]; GELU copy to aux), z = b0 nb1 + b1.
enum : int { TR_EPI_STORE = 0, TR_EPI_BIAS = 1, TR_EPI_BIAS_GELU = 2 };
struct TrGemm {
  int M, N, K, nb0, nb1;
  const float* A; long long sAm, sAk, sA0, sA1;
  const float* B; long long sBk, sBn, sB0, sB1;
  float* C; long long sCm, sCn, sC0, sC1;
  float alpha, beta;
  int epi; const float* bias; float* aux;
};
cudaError_t launch_tr_gemm(const TrGemm& g, cudaStream_t s);
cudaError_t launch_tr_reduce(const float* part, int S, int M, int N, float* out, long long sOm, long long sOn,
                             cudaStream_t s);
cudaError_t launch_tr_twiddles(int n, float* Fj, float* Fi, float* Gi, float* Gj, float* one, cudaStream_t s);
cudaError_t launch_tr_gather(const double* k, const double* r, const double* e, const int* perm, const int* ksys, int N,
                             int B, double* kg, double* rg, double* eg, cudaStream_t s);
cudaError_t launch_tr_lift(const double* rg, const double* kg, const double* rr, const float* E, const float* bE, int N,
                           int B, int w, float* X2, float* v0, cudaStream_t s);
cudaError_t launch_tr_proj(const float* v4, const float* D, const float* bD, const double* rr, const double* eg, int N,
                           int B, int w, double* wout, double* d, cudaStream_t s);
cudaError_t launch_tr_loss(const double* dd, const double* ee, const double* rr, int B, int Bmean, double* loss,
                           double* coef, cudaStream_t s);
cudaError_t launch_tr_dout(const double* gvec, const double* coef, const float* D, int N, int B, int w, float* dout,
                           float* dv, cudaStream_t s);
cudaError_t launch_tr_gelu_bwd(float* dv, const float* z, size_t count, cudaStream_t s);
size_t tr_mix_smem(int B, int w, bool bwd);
cudaError_t prepare_tr_kernels();
cudaError_t launch_tr_mix_fwd(const float* C, const float* R, int B, int w, float* G, cudaStream_t s);
cudaError_t launch_tr_mix_bwd(const float* C, const float* dG, const float* R, int B, int w, float* dR, float* dC,
                              cudaStream_t s);
cudaError_t launch_tr_adamw(size_t count, float* th, const float* g, float* m, float* v, double lr, double b1, double b2,
                            double eps, double wd, int t, cudaStream_t s);
cudaError_t launch_tr_pair(const double* f, const double* Au, const double* ustar, const double* u, size_t count,
                           double e_scale, double* r, double* e, cudaStream_t s);

uint64_t& launch_counter();

// Persistent single-kernel solve of small identity-preconditioned systems (fcg_small.cu).
bool fcg_small_applies(int n, int m);
cudaError_t launch_fcg_small(const FcgDev& d, cudaStream_t s);

// Theorem-1 / Notay diagnostics (diag_kernels.cu)
cudaError_t launch_notay_form(const double* w, const double* e, const double* c, double* d, int n, int B, cudaStream_t s);
cudaError_t launch_notay_coef(const double* wAe, const double* wAw, double* c, int B, cudaStream_t s);
cudaError_t launch_notay_final(const double* dAd, const double* eAe, double* eps, double* err_a, const int* iter,
                               size_t stride, const int* status, int B, cudaStream_t s);
int enqueue_diag(const FcgDev& d, cudaStream_t s);

// Launch with programmatic stream serialization (PDL), unless FCGNO_PDL=0.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace fcgno
