// api.cu — the extern "C" boundary of libfcgno.so (declared in include/fcgno.h).
//
// Host-side responsibilities only: argument validation, workspace carving (the caller owns all
// device memory), weight folding/packing, and the solve driver, which captures one FCG
// iteration into a CUDA graph and replays it, polling an on-device "systems still running"
// counter every check_every iterations (Algorithm 1 runs entirely in kernels).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fcgno.h"
#include "internal.h"

using namespace fcgno;

struct fcgno_problem {
  int n, B;
  const double* k;
  float* F32[2];       // [basis] twiddles [n][20] complex (fcgno_basis: Fourier, Chebyshev)
  double* F64[2];
  float* khat32[2];    // [basis] transform of k per system [B][400] complex
  double* khat64[2];
  bool no_ok;
  bool kfast;   // every k in [2^-400, 2^400]: stencil faces by the branch-free division (fcg_device.cuh)
};

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(FCGNO_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}
#define CK(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

// Bump allocator over a caller workspace (256-byte aligned regions).  With base == nullptr it
// only measures.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
  size_t bytes() const { return (off + 255) & ~size_t(255); }
};

bool aligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 255u) == 0; }
int ngroups_of(int n) { return (n + dft_rows(n) - 1) / dft_rows(n); }
int nblk_of(int n) { return part_cap(n); }   // partial-array capacity per system
bool no_grid_ok(int n) { return n >= kModes && n <= FCGNO_NO_NMAX; }

struct ProblemWs {
  float* F32[2]; double* F64[2]; float* khat32[2]; double* khat64[2]; double* part; int* bad;
};
ProblemWs carve_problem(Carver& c, int n, int B) {
  ProblemWs w{};
  w.bad = c.take<int>(1);
  for (int bs = 0; bs < 2; ++bs) {
    w.F32[bs] = c.take<float>((size_t)n * kModes * 2);
    w.F64[bs] = c.take<double>((size_t)n * kModes * 2);
  }
  if (no_grid_ok(n)) {
    for (int bs = 0; bs < 2; ++bs) {
      w.khat32[bs] = c.take<float>((size_t)B * kModes2 * 2);
      w.khat64[bs] = c.take<double>((size_t)B * kModes2 * 2);
    }
    w.part = c.take<double>((size_t)B * ngroups_of(n) * kModes2 * 2);
  }
  return w;
}

// FCGNO_TC=0 in the environment forces the FFMA layer kernel (A/B comparisons, fallbacks).
bool tc_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FCGNO_TC");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// The fp32 NO runs its operator layers on the tensor cores (no_px_kernels.cu) for these shapes; the
// workspace then holds the tensor-core blobs and no FFMA activations (the carve decides the path).
bool use_px(int n, int w, bool fp32) { return fp32 && tc_enabled() && px_supported_shape(n, w); }

template <typename T>
struct NoWs {
  T *rpart, *v0, *v1, *chat, *ghat;
  unsigned char *vb0, *vb1, *Gb, *cst;   // tensor-core path blobs (fp32 NO only)
  float *Tb, *p3;
  double* rinv;
  size_t vb_bytes, gb_bytes;
};
template <typename T>
NoWs<T> carve_no(Carver& c, int n, int B, int w) {
  NoWs<T> r{};
  const size_t N = (size_t)n * n;
  r.rpart = c.take<T>((size_t)B * ngroups_of(n) * kModes2 * 2);
  const size_t wp = (size_t)((w + 3) & ~3);   // tensor-core path: mode-major spectra rows padded to 32 bytes
  r.ghat = c.take<T>((size_t)B * wp * kModes2 * 2);
  if (use_px(n, w, sizeof(T) == sizeof(float))) {
    r.rinv = c.take<double>(B);
    r.chat = c.take<T>((size_t)kModes2 * B * wp * 2);
    r.vb_bytes = px_v_bytes(n, w, B);
    r.gb_bytes = px_g_bytes(n, w, B);
    r.vb0 = c.take<unsigned char>(r.vb_bytes);
    r.vb1 = c.take<unsigned char>(r.vb_bytes);
    r.Gb = c.take<unsigned char>(r.gb_bytes);
    r.Tb = c.take<float>(px_t_floats(n, w, B));
    r.cst = c.take<unsigned char>(px_const_bytes(n, w));
    r.p3 = c.take<float>((size_t)B * N);
  } else {
    r.v0 = c.take<T>((size_t)B * w * N);
    r.v1 = c.take<T>((size_t)B * w * N);
    r.chat = c.take<T>((size_t)kRowSplitMax * kModes2 * B * w * 2);   // row-split partials (FFMA layer)
  }
  return r;
}

void carve_no_any(Carver& c, int n, int B, const fcgno_no_desc& d, NoWs<float>* f32, NoWs<double>* f64) {
  if (d.precision == FCGNO_FP64) *f64 = carve_no<double>(c, n, B, d.width);
  else *f32 = carve_no<float>(c, n, B, d.width);
}

int check_desc(const fcgno_no_desc& d) {
  if (d.width < 1 || d.width > 1024) return fail(FCGNO_EINVAL, "NO width %d out of range", d.width);
  if (d.precision != FCGNO_FP32 && d.precision != FCGNO_FP64) return fail(FCGNO_EINVAL, "bad NO precision");
  if (d.basis != FCGNO_BASIS_FOURIER && d.basis != FCGNO_BASIS_CHEBYSHEV) return fail(FCGNO_EINVAL, "bad NO basis");
  return FCGNO_OK;
}

template <typename T>
NoDev<T> make_nodev(const fcgno_problem* p, const fcgno_no_desc& d, const void* packed, const NoWs<T>& w,
                    const T* F, const T* khat) {
  NoDev<T> no{};
  no.n = p->n; no.B = p->B; no.N = p->n * p->n; no.w = d.width; no.use_gelu = d.use_gelu;
  no.k = p->k; no.pk = static_cast<const T*>(packed); no.L = no_layout(d.width);
  no.k0 = d.basis == FCGNO_BASIS_CHEBYSHEV ? 0 : (kModes / 2) * kModes + kModes / 2;   // mode of a constant
  no.F = F; no.khat = khat; no.rpart = w.rpart; no.ngroups = ngroups_of(p->n);
  no.v0 = w.v0; no.v1 = w.v1; no.chat = w.chat; no.ghat = w.ghat;
  no.vb0 = w.vb0; no.vb1 = w.vb1; no.Gb = w.Gb; no.Tb = w.Tb; no.cst = w.cst; no.p3 = w.p3; no.rinv = w.rinv;
  no.tc = (sizeof(T) == sizeof(float)) && w.Gb != nullptr;
  return no;
}

int check_no_smem(const fcgno_no_desc& d, int n) {
  if (use_px(n, d.width, d.precision == FCGNO_FP32)) {
    if (!px_supported(n, d.width)) return fail(FCGNO_EUNSUPPORTED, "tensor-core NO needs 227 KB of shared memory per CTA");
    return FCGNO_OK;
  }
  const size_t need = d.precision == FCGNO_FP64 ? no_max_smem<double>(n, d.width) : no_max_smem<float>(n, d.width);
  if (need > 227 * 1024)
    return fail(FCGNO_EUNSUPPORTED, "NO width %d at n=%d needs %zu B of shared memory per CTA", d.width, n, need);
  return FCGNO_OK;
}

}  // namespace

namespace fcgno {
NoLayout no_layout(int w) {
  NoLayout L{};
  L.w = w;
  size_t o = 0;
  auto take = [&](size_t count) {
    o = (o + 3) & ~size_t(3);
    const size_t at = o;
    o += count;
    return at;
  };
  L.W1E = take((size_t)2 * w);
  L.b1 = take(w);
  L.A0 = take((size_t)kModes2 * w * 2);
  L.A1 = take((size_t)kModes2 * w * 2);
  L.A2 = take((size_t)w * 2);
  for (int l = 0; l < 2; ++l) {
    L.W[l] = take((size_t)w * w);
    L.b[l] = take(w);
    L.R[l] = take((size_t)kModes2 * w * w * 2);
  }
  L.Q = take((size_t)kModes2 * w * 2);
  L.dw = take(w);
  L.cst = take(1);
  L.total = (o + 3) & ~size_t(3);
  return L;
}
}  // namespace fcgno

extern "C" {

const char* fcgno_last_error(void) { return g_err.c_str(); }
int fcgno_abi_version(void) { return FCGNO_ABI_VERSION; }
uint64_t fcgno_kernel_launches(void) { return launch_counter(); }

// ------------------------------------------------------------------ problem
size_t fcgno_problem_workspace_bytes(fcgno_grid g) {
  if (g.n < 2 || g.batch < 1) return 0;
  Carver c(nullptr);
  carve_problem(c, g.n, g.batch);
  return c.bytes();
}

int fcgno_assemble(fcgno_grid g, const double* k, void* ws, size_t ws_bytes, void* stream, fcgno_problem** out) {
  if (!out || !k || !ws) return fail(FCGNO_EINVAL, "assemble: NULL argument");
  *out = nullptr;
  if (g.n < 2 || g.batch < 1 || (long long)g.n * g.n > (1LL << 26)) return fail(FCGNO_EINVAL, "assemble: bad grid n=%d B=%d", g.n, g.batch);
  if (!aligned(ws) || ws_bytes < fcgno_problem_workspace_bytes(g)) return fail(FCGNO_EWORKSPACE, "assemble: workspace too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  ProblemWs w = carve_problem(c, g.n, g.batch);
  CK(cudaMemsetAsync(w.bad, 0, sizeof(int), s));
  CK(launch_check_k(k, (size_t)g.batch * g.n * g.n, w.bad, s));
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, w.bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad & 1) return fail(FCGNO_ENONPOS_K, "assemble: k has a non-positive or non-finite entry");
  const bool no_ok = no_grid_ok(g.n);
  for (int bs = 0; bs < 2; ++bs) {
    CK(launch_twiddles(w.F32[bs], w.F64[bs], g.n, bs, s));
    if (no_ok) {
      CK(launch_khat<double>(k, w.F64[bs], w.part, w.khat64[bs], g.n, g.batch, ngroups_of(g.n), s));
      CK(launch_khat<float>(k, w.F32[bs], reinterpret_cast<float*>(w.part), w.khat32[bs], g.n, g.batch, ngroups_of(g.n), s));
    }
  }
  fcgno_problem* p = new fcgno_problem{g.n, g.batch, k, {w.F32[0], w.F32[1]}, {w.F64[0], w.F64[1]},
                                       {w.khat32[0], w.khat32[1]}, {w.khat64[0], w.khat64[1]}, no_ok, (bad & 2) == 0};
  *out = p;
  return FCGNO_OK;
}

void fcgno_problem_destroy(fcgno_problem* p) { delete p; }

int fcgno_apply_A(const fcgno_problem* p, const double* x, double* y, void* stream) {
  if (!p || !x || !y) return fail(FCGNO_EINVAL, "apply_A: NULL argument");
  if (x == y) return fail(FCGNO_EINVAL, "apply_A: y must not alias x");
  CK(launch_apply_A(p->k, x, y, p->n, p->B, p->kfast, static_cast<cudaStream_t>(stream)));
  return FCGNO_OK;
}

size_t fcgno_dot_workspace_bytes(fcgno_grid g) {
  if (g.n < 2 || g.batch < 1) return 0;
  Carver c(nullptr);
  c.take<dd>((size_t)g.batch * nblk_of(g.n));
  c.take<unsigned>(g.batch);
  return c.bytes();
}

int fcgno_batched_dot(const fcgno_problem* p, const double* x, const double* y, double* out, void* ws, size_t ws_bytes,
                      void* stream) {
  if (!p || !x || !y || !out || !ws) return fail(FCGNO_EINVAL, "batched_dot: NULL argument");
  fcgno_grid g{p->n, p->B};
  if (!aligned(ws) || ws_bytes < fcgno_dot_workspace_bytes(g)) return fail(FCGNO_EWORKSPACE, "batched_dot: workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  dd* part = c.take<dd>((size_t)p->B * nblk_of(p->n));
  unsigned* cnt = c.take<unsigned>(p->B);
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * p->B, s));
  CK(launch_dot(x, y, out, part, cnt, p->n, p->B, s));
  return FCGNO_OK;
}

// ------------------------------------------------------------------ NO weights
size_t fcgno_no_packed_bytes(fcgno_no_desc d) {
  if (check_desc(d) != FCGNO_OK) return 0;
  const size_t tsz = d.precision == FCGNO_FP64 ? sizeof(double) : sizeof(float);
  return no_layout(d.width).total * tsz;
}

int fcgno_no_pack(fcgno_no_desc d, const double* blob, void* packed, void* stream) {
  if (int e = check_desc(d)) return e;
  if (!blob || !packed) return fail(FCGNO_EINVAL, "no_pack: NULL argument");
  const int w = d.width, K2 = kModes2;
  using cd = std::complex<double>;
  // unpack the canonical blob (include/fcgno.h)
  size_t pos = 0;
  auto take = [&](size_t count) { const double* at = blob + pos; pos += count; return at; };
  const double* E = take((size_t)w * 2);
  const double* bE = take(w);
  const double *W[4], *b[4], *R[4];
  for (int l = 0; l < 4; ++l) {
    W[l] = take((size_t)w * w);
    b[l] = take(w);
    R[l] = take((size_t)w * w * K2 * 2);
  }
  const double* D = take(w);
  const double bD = *take(1);
  for (size_t t = 0; t < pos; ++t)
    if (!std::isfinite(blob[t])) return fail(FCGNO_EINVAL, "no_pack: non-finite weight at %zu", t);
  // Chebyshev basis (R25): real mixing (imaginary parts unused) and the analysis weights D^-1 folded in
  // per mode, so the kernels' 1/n^2 synthesis scale applies to both bases
  const bool cheb = d.basis == FCGNO_BASIS_CHEBYSHEV;
  auto Rc = [&](int l, int c, int o, int kk) {
    const double* q = R[l] + (((size_t)c * w + o) * K2 + kk) * 2;
    if (!cheb) return cd(q[0], q[1]);
    const double f = (kk / kModes == 0 ? 1.0 : 2.0) * (kk % kModes == 0 ? 1.0 : 2.0);
    return cd(q[0] * f, 0.0);
  };
  const NoLayout L = no_layout(w);
  std::vector<double> P(L.total, 0.0);
  // layer 1 with the lift folded in: W1 (E x + bE) + b1 = (W1 E) x + (W1 bE + b1)
  for (int o = 0; o < w; ++o) {
    double a0 = 0, a1 = 0, bb = b[0][o];
    for (int c = 0; c < w; ++c) {
      a0 += W[0][(size_t)o * w + c] * E[c * 2 + 0];
      a1 += W[0][(size_t)o * w + c] * E[c * 2 + 1];
      bb += W[0][(size_t)o * w + c] * bE[c];
    }
    P[L.W1E + o * 2 + 0] = a0;
    P[L.W1E + o * 2 + 1] = a1;
    P[L.b1 + o] = bb;
  }
  // spectral term of layer 1: sum_c R1[c][o] DFT(E[c,0] r^ + E[c,1] k + bE[c])
  const int k0 = cheb ? 0 : (kModes / 2) * kModes + kModes / 2;   // mode of a constant field
  for (int kk = 0; kk < K2; ++kk)
    for (int o = 0; o < w; ++o) {
      cd a0 = 0, a1 = 0;
      for (int c = 0; c < w; ++c) {
        a0 += Rc(0, c, o, kk) * E[c * 2 + 0];
        a1 += Rc(0, c, o, kk) * E[c * 2 + 1];
      }
      P[L.A0 + ((size_t)kk * w + o) * 2 + 0] = a0.real(); P[L.A0 + ((size_t)kk * w + o) * 2 + 1] = a0.imag();
      P[L.A1 + ((size_t)kk * w + o) * 2 + 0] = a1.real(); P[L.A1 + ((size_t)kk * w + o) * 2 + 1] = a1.imag();
    }
  for (int o = 0; o < w; ++o) {
    cd a2 = 0;
    for (int c = 0; c < w; ++c) a2 += Rc(0, c, o, k0) * bE[c];
    P[L.A2 + o * 2 + 0] = a2.real(); P[L.A2 + o * 2 + 1] = a2.imag();
  }
  // layers 2, 3 as they are (R re-laid out mode-major)
  for (int l = 1; l <= 2; ++l) {
    for (size_t t = 0; t < (size_t)w * w; ++t) P[L.W[l - 1] + t] = W[l][t];
    for (int o = 0; o < w; ++o) P[L.b[l - 1] + o] = b[l][o];
    for (int kk = 0; kk < K2; ++kk)
      for (int c = 0; c < w; ++c)
        for (int o = 0; o < w; ++o) {
          const cd v = Rc(l, c, o, kk);
          const size_t at = L.R[l - 1] + (((size_t)kk * w + c) * w + o) * 2;
          P[at] = v.real(); P[at + 1] = v.imag();
        }
  }
  // layer 4 folded with the projection: out = (D W4) v3 + (D b4 + bD) + S(sum_c (R4 D)[c] c3[c])
  double cst = bD;
  for (int o = 0; o < w; ++o) cst += D[o] * b[3][o];
  for (int c = 0; c < w; ++c) {
    double a = 0;
    for (int o = 0; o < w; ++o) a += D[o] * W[3][(size_t)o * w + c];
    P[L.dw + c] = a;
  }
  for (int kk = 0; kk < K2; ++kk)
    for (int c = 0; c < w; ++c) {
      cd q = 0;
      for (int o = 0; o < w; ++o) q += Rc(3, c, o, kk) * D[o];
      P[L.Q + ((size_t)kk * w + c) * 2 + 0] = q.real();
      P[L.Q + ((size_t)kk * w + c) * 2 + 1] = q.imag();
    }
  P[L.cst] = cst;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (d.precision == FCGNO_FP64) {
    CK(cudaMemcpyAsync(packed, P.data(), P.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  } else {
    std::vector<float> Pf(P.size());
    for (size_t t = 0; t < P.size(); ++t) Pf[t] = (float)P[t];
    CK(cudaMemcpyAsync(packed, Pf.data(), Pf.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  return FCGNO_OK;
}

int fcgno_no_uses_tensor_cores(fcgno_grid g, fcgno_no_desc d) {
  if (check_desc(d) != FCGNO_OK || g.n < 2 || g.batch < 1) return 0;
  return (use_px(g.n, d.width, d.precision == FCGNO_FP32) && px_supported(g.n, d.width)) ? 1 : 0;
}

// ------------------------------------------------------------------ apply_NO
size_t fcgno_apply_no_workspace_bytes(fcgno_grid g, fcgno_no_desc d) {
  if (g.n < 2 || g.batch < 1 || check_desc(d) != FCGNO_OK) return 0;
  Carver c(nullptr);
  c.take<double>(g.batch);
  c.take<dd>((size_t)g.batch * nblk_of(g.n));
  c.take<unsigned>(g.batch);
  NoWs<float> a; NoWs<double> b;
  carve_no_any(c, g.n, g.batch, d, &a, &b);
  return c.bytes();
}

int fcgno_apply_NO(const fcgno_problem* p, fcgno_no_desc d, const void* packed, const double* r, double* w, void* ws,
                   size_t ws_bytes, void* stream) {
  if (!p || !packed || !r || !w || !ws) return fail(FCGNO_EINVAL, "apply_NO: NULL argument");
  if (r == w) return fail(FCGNO_EINVAL, "apply_NO: w must not alias r");
  if (int e = check_desc(d)) return e;
  if (!p->no_ok) return fail(FCGNO_EUNSUPPORTED, "apply_NO: needs %d <= n <= %d (n=%d)", kModes, FCGNO_NO_NMAX, p->n);
  if (int e = check_no_smem(d, p->n)) return e;
  fcgno_grid g{p->n, p->B};
  if (!aligned(ws) || ws_bytes < fcgno_apply_no_workspace_bytes(g, d)) return fail(FCGNO_EWORKSPACE, "apply_NO: workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  double* rr = c.take<double>(p->B);
  dd* part = c.take<dd>((size_t)p->B * nblk_of(p->n));
  unsigned* cnt = c.take<unsigned>(p->B);
  NoWs<float> w32{}; NoWs<double> w64{};
  carve_no_any(c, p->n, p->B, d, &w32, &w64);
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * p->B, s));
  CK(launch_dot(r, r, rr, part, cnt, p->n, p->B, s));
  if (d.precision == FCGNO_FP64) {
    CK(prepare_no_kernels<double>());
    NoDev<double> no = make_nodev<double>(p, d, packed, w64, p->F64[d.basis], p->khat64[d.basis]);
    CK(launch_no_forward<double>(no, r, rr, w, nullptr, nullptr, s, nullptr));
  } else {
    CK(prepare_no_kernels<float>());
    CK(prepare_px_kernels());
    NoDev<float> no = make_nodev<float>(p, d, packed, w32, p->F32[d.basis], p->khat32[d.basis]);
    CK(prepare_no_constants(no, s));
    CK(launch_no_forward<float>(no, r, rr, w, nullptr, nullptr, s, nullptr));
  }
  return FCGNO_OK;
}

// ------------------------------------------------------------------ Notay ratio (Theorem-1 diagnostic)
size_t fcgno_notay_workspace_bytes(fcgno_grid g, const fcgno_no_desc* nd) {
  if (g.n < 2 || g.batch < 1 || (nd && check_desc(*nd) != FCGNO_OK)) return 0;
  Carver c(nullptr);
  const size_t BN = (size_t)g.batch * g.n * g.n;
  for (int t = 0; t < 5; ++t) c.take<double>(BN);
  c.take<double>((size_t)5 * g.batch);
  c.take<dd>((size_t)g.batch * nblk_of(g.n));
  c.take<unsigned>(g.batch);
  if (nd) c.take<unsigned char>(fcgno_apply_no_workspace_bytes(g, *nd));
  return c.bytes();
}

int fcgno_notay_ratio(const fcgno_problem* p, const fcgno_no_desc* nd, const void* packed, const double* r,
                      const double* e, int optimal_scale, double* eps, void* ws, size_t ws_bytes, void* stream) {
  if (!p || !r || !e || !eps || !ws || (nd && !packed)) return fail(FCGNO_EINVAL, "notay_ratio: NULL argument");
  fcgno_grid g{p->n, p->B};
  if (!aligned(ws) || ws_bytes < fcgno_notay_workspace_bytes(g, nd)) return fail(FCGNO_EWORKSPACE, "notay_ratio: workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  const size_t BN = (size_t)p->B * p->n * p->n;
  double* wv = c.take<double>(BN);
  double* Ae = c.take<double>(BN);
  double* Aw = c.take<double>(BN);
  double* dv = c.take<double>(BN);
  double* Ad = c.take<double>(BN);
  double* sc = c.take<double>((size_t)5 * p->B);   // (e,Ae), (w,Aw), (w,Ae), c, (d,Ad)
  dd* part = c.take<dd>((size_t)p->B * nblk_of(p->n));
  unsigned* cnt = c.take<unsigned>(p->B);
  const int B = p->B, n = p->n;
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * B, s));
  const double* w = r;                               // identity: B(r) = r
  if (nd) {
    const size_t nb = fcgno_apply_no_workspace_bytes(g, *nd);
    unsigned char* nws = c.take<unsigned char>(nb);
    if (int rc = fcgno_apply_NO(p, *nd, packed, r, wv, nws, nb, stream)) return rc;
    w = wv;
  }
  CK(launch_apply_A(p->k, e, Ae, n, B, p->kfast, s));
  CK(launch_dot(e, Ae, sc, part, cnt, n, B, s));
  const double* coef = nullptr;
  if (optimal_scale) {   // c* = (w, A e) / (w, A w)
    CK(launch_apply_A(p->k, w, Aw, n, B, p->kfast, s));
    CK(launch_dot(w, Aw, sc + B, part, cnt, n, B, s));
    CK(launch_dot(w, Ae, sc + 2 * B, part, cnt, n, B, s));
    CK(launch_notay_coef(sc + 2 * B, sc + B, sc + 3 * B, B, s));
    coef = sc + 3 * B;
  }
  CK(launch_notay_form(w, e, coef, dv, n, B, s));
  CK(launch_apply_A(p->k, dv, Ad, n, B, p->kfast, s));
  CK(launch_dot(dv, Ad, sc + 4 * B, part, cnt, n, B, s));
  CK(launch_notay_final(sc + 4 * B, sc, eps, nullptr, nullptr, 1, nullptr, B, s));
  return FCGNO_OK;
}

// ------------------------------------------------------------------ fcg_solve
namespace {
struct SolveWs {
  FcgDev d;
  NoWs<float> n32;
  NoWs<double> n64;
  double* wvec;
};

SolveWs carve_solve(Carver& c, int n, int B, const fcgno_no_desc* nd, const fcgno_solve_opts& o, bool diag = false,
                    bool stationary = false) {
  SolveWs s{};
  const size_t N = (size_t)n * n;
  const int nblk = nblk_of(n);
  FcgDev& d = s.d;
  // r, w and the ring in fp64, or fp32 with opts.vec_fp32 (reading R21; the FcgDev fields then
  // point at float arrays), plus an fp64 copy of r for the NO input
  const size_t es = o.vec_fp32 ? sizeof(float) : sizeof(double);
  d.vec32 = o.vec_fp32 ? 1 : 0;
  d.r = reinterpret_cast<double*>(c.take<unsigned char>(es * B * N));
  s.wvec = (nd || stationary) ? reinterpret_cast<double*>(c.take<unsigned char>(es * B * N)) : nullptr;
  if (stationary) {   // classical preconditioner sweep iterates (fp64)
    d.st_xa = c.take<double>(B * N);
    d.st_xb = c.take<double>(B * N);
  }
  d.r64 = (nd && o.vec_fp32) ? c.take<double>(B * N) : nullptr;
  d.ring_p = reinterpret_cast<double*>(c.take<unsigned char>(es * (o.m + 1) * B * N));
  d.ring_s = reinterpret_cast<double*>(c.take<unsigned char>(es * (o.m + 1) * B * N));
  d.gamma = c.take<double>((size_t)(o.m + 1) * B);
  d.beta = c.take<double>((size_t)B * kMmax);
  d.alpha = c.take<double>(B);
  d.rr = c.take<double>(B);
  d.rho0 = c.take<double>(B);
  d.part_win = c.take<dd>((size_t)B * nblk * kMmax);
  d.part_step = c.take<dd>((size_t)B * nblk * 2);
  d.part_rr = c.take<dd>((size_t)B * nblk);
  d.cnt = c.take<unsigned>((size_t)3 * B + 2);
  d.gcnt = d.cnt + (size_t)3 * B;
  d.flags = c.take<int>(B);
  d.iter = c.take<int>(2);
  d.active = d.iter + 1;
  if (nd) carve_no_any(c, n, B, *nd, &s.n32, &s.n64);
  if (diag) {   // Theorem-1 diagnostics scratch (fcgno_fcg_solve_diag)
    d.dg_e = c.take<double>(B * N);
    d.dg_d = c.take<double>(B * N);
    d.dg_Ae = c.take<double>(B * N);
    d.dg_Ad = c.take<double>(B * N);
    d.dg_sc = c.take<double>((size_t)2 * B);
    d.dg_part = c.take<dd>((size_t)B * nblk);
    d.dg_cnt = c.take<unsigned>(B);
  }
  return s;
}

int check_opts(const fcgno_solve_opts& o) {
  if (o.m < 1 || o.m > FCGNO_MMAX) return fail(FCGNO_EINVAL, "m=%d outside [1, %d]", o.m, FCGNO_MMAX);
  if (o.maxit < 0) return fail(FCGNO_EINVAL, "maxit < 0");
  if (o.schedule != FCGNO_SCHEDULE_PAPER && o.schedule != FCGNO_SCHEDULE_SLIDING) return fail(FCGNO_EINVAL, "bad schedule");
  if (o.vec_fp32 != 0 && o.vec_fp32 != 1) return fail(FCGNO_EINVAL, "vec_fp32 must be 0 or 1");
  if (!(o.tol >= 0.0) && !std::isnan(o.tol)) return fail(FCGNO_EINVAL, "tol < 0");
  return FCGNO_OK;
}

// Lanes: the batch is split into up to kMaxLanes groups of independent systems whose iterations
// are captured as parallel branches of one graph.  Every kernel of this path is latency-bound at
// the paper's batch sizes, so two concurrent chains fill the SMs' idle issue and
// memory slots.  Per-system arithmetic is unchanged (systems never interact), so results are
// bitwise independent of the split.  Opt-in (FCGNO_LANES=2): measured +4% at B = 64 on B200, not
// yet the default.
constexpr int kMaxLanes = 2;
int solve_lanes(int B) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FCGNO_LANES");
    v = e ? std::max(1, std::min(kMaxLanes, atoi(e))) : 1;
  }
  return std::max(1, std::min(v, B / 32));   // lanes of at least 32 systems
}
struct LaneSplit { int b0[kMaxLanes], nb[kMaxLanes], n; };
LaneSplit lane_split(int B) {
  LaneSplit L{};
  L.n = solve_lanes(B);
  int b0 = 0;
  for (int l = 0; l < L.n; ++l) {
    L.b0[l] = b0;
    L.nb[l] = B / L.n + (l < B % L.n ? 1 : 0);
    b0 += L.nb[l];
  }
  return L;
}

// In-graph CUDA-event profiler: one (start, end) event pair per instrumented launch of every
// unrolled iteration of a chunk graph; read back after the chunk completes.
struct Profiler : ProfHook {
  int mask = 0;
  struct Rec { int cls; cudaEvent_t a, b; cudaStream_t s; };
  std::vector<Rec> recs;          // of the chunk being captured
  std::vector<Rec> pending;       // open begin() per class
  bool failed = false;
  void begin(int cls, cudaStream_t s) override {
    if (!(mask >> cls & 1)) return;
    Rec r{cls, nullptr, nullptr, s};
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) { failed = true; return; }
    if (cudaEventRecordWithFlags(r.a, s, cudaEventRecordExternal) != cudaSuccess) failed = true;
    pending.push_back(r);
  }
  void end(int cls, cudaStream_t s) override {
    if (!(mask >> cls & 1)) return;
    for (size_t t = pending.size(); t-- > 0;)
      if (pending[t].cls == cls && pending[t].s == s) {
        Rec r = pending[t];
        pending.erase(pending.begin() + t);
        if (cudaEventRecordWithFlags(r.b, s, cudaEventRecordExternal) != cudaSuccess) failed = true;
        recs.push_back(r);
        return;
      }
  }
};

struct ProfTotals { double ms[PROF_NCLASS]; int64_t n[PROF_NCLASS]; };
ProfTotals& prof_totals() { static ProfTotals t{}; return t; }

// One FCG iteration (the graph body).  Returns the number of kernels enqueued or -1.
int enqueue_iteration(const FcgDev& d, const fcgno_no_desc* nd, const void* packed, const fcgno_problem* p,
                      const SolveWs& sw, cudaStream_t s, ProfHook* prof) {
  auto pb = [&](int c) { if (prof) prof->begin(c, s); };
  auto pe = [&](int c) { if (prof) prof->end(c, s); };
  int count = 0;
  if (nd) {
    int nl = 0;
    cudaError_t e;
    if (nd->precision == FCGNO_FP64) {
      NoDev<double> no = make_nodev<double>(p, *nd, packed, sw.n64, p->F64[nd->basis], p->khat64[nd->basis]);
      e = launch_no_forward<double>(no, d.vec32 ? d.r64 : d.r, d.rr, sw.wvec, &d, d.status, s, &nl, prof);
    } else {
      NoDev<float> no = make_nodev<float>(p, *nd, packed, sw.n32, p->F32[nd->basis], p->khat32[nd->basis]);
      e = launch_no_forward<float>(no, d.vec32 ? d.r64 : d.r, d.rr, sw.wvec, &d, d.status, s, &nl, prof);
    }
    if (e != cudaSuccess) return -1;
    count += nl;
  } else {
    if (d.st_kind) {   // w = Jacobi(k) / SGS(k) r, then the window dots of w
      if (launch_stationary(d.k, d.r, d.st_xa, d.st_xb, const_cast<double*>(d.w), d.vec32 != 0, d.n, d.B, d.kfast != 0,
                            d.st_kind, d.st_sweeps, d.status, s) != cudaSuccess)
        return -1;
      count += d.st_kind == FCGNO_PRECOND_JACOBI ? d.st_sweeps : 4 * d.st_sweeps;
    }
    pb(PROF_WINDOW);
    if (launch_window_dots(d, s) != cudaSuccess) return -1;
    pe(PROF_WINDOW);
    ++count;
  }
  if (d.dg_ustar) {   // Theorem-1 diagnostics of w_i = B(r_i) (fcgno_fcg_solve_diag)
    const int nd_l = enqueue_diag(d, s);
    if (nd_l < 0) return -1;
    count += nd_l;
  }
  pb(PROF_STENCIL);
  if (launch_pform_stencil(d, s) != cudaSuccess) return -1;
  pe(PROF_STENCIL);
  pb(PROF_UPDATE);
  if (launch_update(d, s) != cudaSuccess) return -1;
  pe(PROF_UPDATE);
  return count + 2;
}

// A CUDA graph replaying `iters` unrolled FCG iterations (+ its profiling events).
struct Chunk {
  int iters = 0, kernels = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<Profiler::Rec> recs;
  void destroy() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (auto& r : recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    exec = nullptr; graph = nullptr; recs.clear();
  }
  // Accumulate the event timings of the last replay into the process-wide totals.
  void harvest() {
    for (auto& r : recs) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
        prof_totals().ms[r.cls] += ms;
        prof_totals().n[r.cls] += 1;
      } else {
        (void)cudaGetLastError();  // never leave a stale error for the caller's runtime
      }
    }
  }
};

struct Lane {
  fcgno_problem p;   // view of the lane's systems
  SolveWs sw;
};

int build_chunk(Chunk& c, int iters, int mask, const fcgno_no_desc* nd, const void* packed, const Lane* lanes,
                int nlanes, cudaStream_t* st, cudaEvent_t* ev) {
  Profiler prof;
  prof.mask = mask;
  c.iters = iters;
  cudaStream_t s = st[0];
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_fail(e, "graph capture");
  const uint64_t before = launch_counter();
  int per_iter = 0, total = 0;
  if (nlanes > 1) {   // fork the side lanes off the capture origin
    e = cudaEventRecord(ev[0], s);
    for (int l = 1; l < nlanes && e == cudaSuccess; ++l) e = cudaStreamWaitEvent(st[l], ev[0], 0);
  }
  // events only in the first unrolled iteration: the profiled solve keeps PDL overlap and its
  // timing in the other iterations (per-launch averages are what the profile reports)
  for (int t = 0; t < iters && per_iter >= 0 && e == cudaSuccess; ++t)
    for (int l = 0; l < nlanes && per_iter >= 0; ++l) {
      per_iter = enqueue_iteration(lanes[l].sw.d, nd, packed, &lanes[l].p, lanes[l].sw, st[l],
                                   (mask && t == 0) ? &prof : nullptr);
      total += per_iter;
    }
  for (int l = 1; l < nlanes && e == cudaSuccess; ++l) {   // join
    e = cudaEventRecord(ev[l], st[l]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[l], 0);
  }
  launch_counter() = before;  // captured, not launched
  const cudaError_t e2 = cudaStreamEndCapture(s, &c.graph);
  if (e == cudaSuccess) e = e2;
  c.recs = prof.recs;
  for (auto& r : prof.pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  if (per_iter < 0 || e != cudaSuccess || prof.failed)
    return cuda_fail(e != cudaSuccess ? e : cudaGetLastError(), "iteration capture");
  c.kernels = total;
  e = cudaGraphInstantiate(&c.exec, c.graph, 0);
  if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
  return FCGNO_OK;
}
// Device-side iteration loop: one graph whose WHILE node replays a body of `chunk` unrolled
// iterations followed by k_loop_cond (condition: a system is still running), so a solve is one
// graph launch and the GPU never waits for the host.  Returns FCGNO_OK, or -1 when the graph could
// not be built (the caller then uses the host-polled chunk loop).
struct DeviceLoop {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int kernels = 0;   // kernels of one body replay
  void destroy() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr; graph = nullptr;
  }
};

int build_device_loop(DeviceLoop& L, int chunk, const fcgno_no_desc* nd, const void* packed, const Lane& ln,
                      cudaStream_t s) {
  const uint64_t before = launch_counter();
  cudaGraphConditionalHandle h;
  cudaGraphNode_t node;
  cudaGraphNodeParams np{};
  if (cudaGraphCreate(&L.graph, 0) != cudaSuccess) return -1;
  if (cudaGraphConditionalHandleCreate(&h, L.graph, 1, cudaGraphCondAssignDefault) != cudaSuccess) return -1;
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  if (cudaGraphAddNode(&node, L.graph, nullptr, 0, &np) != cudaSuccess) return -1;
  cudaGraph_t body = np.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return -1;
  int per = 0, total = 0;
  for (int t = 0; t < chunk && per >= 0; ++t) {
    per = enqueue_iteration(ln.sw.d, nd, packed, &ln.p, ln.sw, s, nullptr);
    total += per;
  }
  const cudaError_t ec = (per >= 0) ? launch_loop_cond(ln.sw.d.active, h, s) : cudaErrorUnknown;
  cudaGraph_t out = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(s, &out);
  launch_counter() = before;   // captured, not launched
  if (per < 0 || ec != cudaSuccess || ee != cudaSuccess) {
    (void)cudaGetLastError();
    return -1;
  }
  L.kernels = total + 1;
  if (cudaGraphInstantiate(&L.exec, L.graph, 0) != cudaSuccess) {
    (void)cudaGetLastError();
    return -1;
  }
  return FCGNO_OK;
}

// Instantiated device-loop graphs, reused across solves whose captured kernel arguments are
// identical (same problem arrays, workspace carve, NO weights, options): a repeated solve is then
// one graph launch with no capture / instantiation on the host.  Kernel arguments are captured by
// value, so an identical key means an identical graph whatever allocation the pointers belong to.
struct LoopKey {
  FcgDev d;
  fcgno_no_desc nd;
  int has_nd, chunk;
  const void* packed;
  const void* pf[8];
  int n, B, no_ok, kfast;   // the NO buffers are carved from the workspace after d.r (d) at
};                          // offsets fixed by (n, B, nd, m): covered by the fields above
struct LoopEntry { LoopKey key; DeviceLoop loop; uint64_t used; };
std::vector<LoopEntry>& loop_cache() { static std::vector<LoopEntry> c; return c; }
std::mutex& loop_cache_mutex() { static std::mutex m; return m; }   // held from lookup to launch
// (an evicted exec still in flight is freed by CUDA when it completes)
constexpr size_t kLoopCacheMax = 4;

LoopKey loop_key(const Lane& ln, const fcgno_no_desc* nd, const void* packed, int chunk) {
  LoopKey k;
  std::memset(&k, 0, sizeof(k));   // padding bytes too: the key is compared with memcmp
  k.d = ln.sw.d;
  if (nd) { k.nd = *nd; k.has_nd = 1; }
  k.chunk = chunk;
  k.packed = packed;
  for (int bs = 0; bs < 2; ++bs) {
    k.pf[4 * bs + 0] = ln.p.F32[bs]; k.pf[4 * bs + 1] = ln.p.F64[bs];
    k.pf[4 * bs + 2] = ln.p.khat32[bs]; k.pf[4 * bs + 3] = ln.p.khat64[bs];
  }
  k.n = ln.p.n; k.B = ln.p.B; k.no_ok = ln.p.no_ok; k.kfast = ln.p.kfast;
  return k;
}

bool host_loop_forced() {
  const char* e = getenv("FCGNO_HOSTLOOP");
  return e && e[0] == '1';
}
}  // namespace

namespace {
struct DiagArgs { const double* u_star; double* eps; double* err_a; };
struct StationaryArgs { int kind, sweeps; };

size_t solve_ws_bytes(fcgno_grid g, const fcgno_no_desc* nd, const fcgno_solve_opts& o, bool diag, bool stationary = false) {
  if (g.n < 2 || g.batch < 1 || check_opts(o) != FCGNO_OK) return 0;
  if (nd && check_desc(*nd) != FCGNO_OK) return 0;
  Carver c(nullptr);
  const LaneSplit L = lane_split(g.batch);
  for (int l = 0; l < L.n; ++l) carve_solve(c, g.n, L.nb[l], nd, o, diag, stationary);
  return c.bytes();
}

int solve_impl(const fcgno_problem* p, const fcgno_no_desc* nd, const void* packed, const double* f, double* u,
               fcgno_solve_opts o, int32_t* iters, int32_t* status, double* history, const DiagArgs* dg, void* ws,
               size_t ws_bytes, void* stream, const StationaryArgs* st = nullptr);

int check_stationary(int kind, int sweeps) {
  if (kind != FCGNO_PRECOND_JACOBI && kind != FCGNO_PRECOND_SGS_RB) return fail(FCGNO_EINVAL, "unknown classical preconditioner %d", kind);
  if (sweeps < 1 || sweeps > 64) return fail(FCGNO_EINVAL, "sweeps=%d outside [1, 64]", sweeps);
  return FCGNO_OK;
}
}  // namespace

size_t fcgno_solve_stationary_workspace_bytes(fcgno_grid g, fcgno_solve_opts o) {
  return solve_ws_bytes(g, nullptr, o, false, true);
}

int fcgno_fcg_solve_stationary(const fcgno_problem* p, int kind, int sweeps, const double* f, double* u,
                               fcgno_solve_opts o, int32_t* iters, int32_t* status, double* history, void* ws,
                               size_t ws_bytes, void* stream) {
  if (int e = check_stationary(kind, sweeps)) return e;
  const StationaryArgs st{kind, sweeps};
  return solve_impl(p, nullptr, nullptr, f, u, o, iters, status, history, nullptr, ws, ws_bytes, stream, &st);
}

size_t fcgno_stationary_workspace_bytes(fcgno_grid g) {
  if (g.n < 2 || g.batch < 1) return 0;
  Carver c(nullptr);
  c.take<double>((size_t)g.batch * g.n * g.n);
  c.take<double>((size_t)g.batch * g.n * g.n);
  return c.bytes();
}

int fcgno_apply_stationary(const fcgno_problem* p, int kind, int sweeps, const double* r, double* w, void* ws,
                           size_t ws_bytes, void* stream) {
  if (!p || !r || !w || !ws) return fail(FCGNO_EINVAL, "apply_stationary: NULL argument");
  if (r == w) return fail(FCGNO_EINVAL, "apply_stationary: w must not alias r");
  if (int e = check_stationary(kind, sweeps)) return e;
  fcgno_grid g{p->n, p->B};
  if (!aligned(ws) || ws_bytes < fcgno_stationary_workspace_bytes(g)) return fail(FCGNO_EWORKSPACE, "apply_stationary: workspace");
  Carver c(ws);
  double* xa = c.take<double>((size_t)p->B * p->n * p->n);
  double* xb = c.take<double>((size_t)p->B * p->n * p->n);
  CK(launch_stationary(p->k, r, xa, xb, w, false, p->n, p->B, p->kfast, kind, sweeps, nullptr,
                       static_cast<cudaStream_t>(stream)));
  return FCGNO_OK;
}

size_t fcgno_solve_workspace_bytes(fcgno_grid g, const fcgno_no_desc* nd, fcgno_solve_opts o) {
  return solve_ws_bytes(g, nd, o, false);
}

size_t fcgno_solve_diag_workspace_bytes(fcgno_grid g, const fcgno_no_desc* nd, fcgno_solve_opts o) {
  return solve_ws_bytes(g, nd, o, true);
}

int fcgno_fcg_solve(const fcgno_problem* p, const fcgno_no_desc* nd, const void* packed, const double* f, double* u,
                    fcgno_solve_opts o, int32_t* iters, int32_t* status, double* history, void* ws, size_t ws_bytes,
                    void* stream) {
  return solve_impl(p, nd, packed, f, u, o, iters, status, history, nullptr, ws, ws_bytes, stream);
}

int fcgno_fcg_solve_diag(const fcgno_problem* p, const fcgno_no_desc* nd, const void* packed, const double* f,
                         double* u, fcgno_solve_opts o, int32_t* iters, int32_t* status, double* history,
                         const double* u_star, double* eps, double* err_a, void* ws, size_t ws_bytes, void* stream) {
  if (!u_star || (!eps && !err_a)) return fail(FCGNO_EINVAL, "fcg_solve_diag: u_star and eps or err_a are required");
  if (o.profile_mask) return fail(FCGNO_EINVAL, "fcg_solve_diag: profiling is not available with diagnostics");
  const DiagArgs dg{u_star, eps, err_a};
  return solve_impl(p, nd, packed, f, u, o, iters, status, history, &dg, ws, ws_bytes, stream);
}

namespace {
int solve_impl(const fcgno_problem* p, const fcgno_no_desc* nd, const void* packed, const double* f, double* u,
               fcgno_solve_opts o, int32_t* iters, int32_t* status, double* history, const DiagArgs* dg, void* ws,
               size_t ws_bytes, void* stream, const StationaryArgs* sta) {
  if (!p || !f || !u || !iters || !status || !ws) return fail(FCGNO_EINVAL, "fcg_solve: NULL argument");
  if (int e = check_opts(o)) return e;
  if (nd) {
    if (int e = check_desc(*nd)) return e;
    if (!packed) return fail(FCGNO_EINVAL, "fcg_solve: NO descriptor without packed weights");
    if (!p->no_ok) return fail(FCGNO_EUNSUPPORTED, "fcg_solve: the NO needs %d <= n <= %d (n=%d)", kModes, FCGNO_NO_NMAX, p->n);
    if (int e = check_no_smem(*nd, p->n)) return e;
  }
  fcgno_grid g{p->n, p->B};
  if (!aligned(ws) || ws_bytes < solve_ws_bytes(g, nd, o, dg != nullptr, sta != nullptr)) return fail(FCGNO_EWORKSPACE, "fcg_solve: workspace");
  if (!nd && !sta && !dg && !o.vec_fp32 && !o.profile_mask && fcg_small_applies(p->n, o.m)) {
    // small systems, identity preconditioner: the whole solve in one persistent kernel (fcg_small.cu), one
    // CTA per system, on the caller's stream; same arithmetic as the launch-per-step path below
    FcgDev d{};
    d.n = p->n; d.B = p->B; d.N = p->n * p->n;
    d.m = o.m; d.maxit = o.maxit; d.schedule = o.schedule; d.tol = o.tol;
    d.scale = double(p->n + 1) * double(p->n + 1);
    d.k = p->k; d.f = f; d.u = u; d.status = status; d.iters = iters; d.hist = history;
    CK(launch_fcg_small(d, static_cast<cudaStream_t>(stream)));
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));   // the entry's contract: complete on return
    return FCGNO_OK;
  }
  if (nd) {
    if (nd->precision == FCGNO_FP64) CK(prepare_no_kernels<double>());
    else { CK(prepare_no_kernels<float>()); CK(prepare_px_kernels()); }
  }
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  const LaneSplit LS = lane_split(p->B);
  const int nl = LS.n;
  const size_t N = (size_t)p->n * p->n;
  Lane lanes[kMaxLanes];
  for (int l = 0; l < nl; ++l) {
    const int b0 = LS.b0[l], nb = LS.nb[l];
    Lane& ln = lanes[l];
    ln.p = *p;
    ln.p.B = nb;
    ln.p.k = p->k + b0 * N;
    for (int bs = 0; bs < 2; ++bs) {
      if (p->khat32[bs]) ln.p.khat32[bs] = p->khat32[bs] + (size_t)b0 * kModes2 * 2;
      if (p->khat64[bs]) ln.p.khat64[bs] = p->khat64[bs] + (size_t)b0 * kModes2 * 2;
    }
    ln.sw = carve_solve(c, p->n, nb, nd, o, dg != nullptr, sta != nullptr);
    FcgDev& d = ln.sw.d;
    d.n = p->n; d.B = nb; d.N = p->n * p->n; d.nblk = nblk_of(p->n);
    d.m = o.m; d.maxit = o.maxit; d.schedule = o.schedule; d.tol = o.tol;
    d.scale = double(p->n + 1) * double(p->n + 1);
    d.k = ln.p.k; d.kfast = p->kfast ? 1 : 0; d.f = f + b0 * N; d.u = u + b0 * N; d.w = (nd || sta) ? ln.sw.wvec : d.r;
    if (sta) { d.st_kind = sta->kind; d.st_sweeps = sta->sweeps; }
    d.status = status + b0; d.iters = iters + b0;
    d.hist = history ? history + (size_t)b0 * (o.maxit + 1) : nullptr;
    if (dg) {
      d.dg_ustar = dg->u_star + b0 * N;
      d.dg_eps = dg->eps ? dg->eps + (size_t)b0 * o.maxit : nullptr;
      d.dg_erra = dg->err_a ? dg->err_a + (size_t)b0 * o.maxit : nullptr;
    }
  }

  // Private streams (graph capture is not allowed on the legacy default stream), ordered after
  // everything already enqueued on the caller's stream.  Owned by `res`, whose destructor releases
  // whatever was created, on every return path.
  struct SolveResources {
    cudaStream_t st[kMaxLanes] = {};
    cudaEvent_t ev_in = nullptr, ev_poll[2] = {}, ev_fj[kMaxLanes] = {};
    int* h_active = nullptr;
    Chunk full[2], tail;
    ~SolveResources() {
      full[0].destroy(); full[1].destroy(); tail.destroy();
      if (h_active) cudaFreeHost(h_active);
      if (ev_in) cudaEventDestroy(ev_in);
      for (cudaEvent_t e : ev_poll) if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : ev_fj) if (e) cudaEventDestroy(e);
      for (cudaStream_t q : st) if (q) cudaStreamDestroy(q);
    }
  } res;
  cudaStream_t* st = res.st;
  cudaEvent_t* ev_poll = res.ev_poll;
  cudaEvent_t* ev_fj = res.ev_fj;
  for (int l = 0; l < nl; ++l) CK(cudaStreamCreateWithFlags(&st[l], cudaStreamNonBlocking));
  cudaStream_t s = st[0];
  CK(cudaEventCreateWithFlags(&res.ev_in, cudaEventDisableTiming));
  cudaEvent_t ev_in = res.ev_in;
  CK(cudaEventCreateWithFlags(&ev_poll[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev_poll[1], cudaEventDisableTiming));
  for (int l = 0; l < nl; ++l) CK(cudaEventCreateWithFlags(&ev_fj[l], cudaEventDisableTiming));
  CK(cudaEventRecord(ev_in, caller));
  CK(cudaStreamWaitEvent(s, ev_in, 0));
  CK(cudaHostAlloc(&res.h_active, 2 * kMaxLanes * sizeof(int), cudaHostAllocDefault));
  int* h_active = res.h_active;
  int rc = FCGNO_OK;
  Chunk* full = res.full;
  Chunk& tail = res.tail;
  do {
    cudaError_t e = cudaSuccess;
    for (int l = 0; l < nl && rc == FCGNO_OK; ++l) {
      const FcgDev& d = lanes[l].sw.d;
      const SolveWs& sw = lanes[l].sw;
      if ((e = cudaMemsetAsync(d.cnt, 0, sizeof(unsigned) * (3 * d.B + 2), s)) != cudaSuccess) { rc = cuda_fail(e, "memset"); break; }
      if ((e = cudaMemsetAsync(d.iter, 0, 2 * sizeof(int), s)) != cudaSuccess) { rc = cuda_fail(e, "memset"); break; }
      if (d.dg_cnt && (e = cudaMemsetAsync(d.dg_cnt, 0, sizeof(unsigned) * d.B, s)) != cudaSuccess) { rc = cuda_fail(e, "memset"); break; }
      if (nd && sw.n32.Gb) {   // tensor-core constant operands (every blob byte the kernels read is written by them)
        NoDev<float> no = make_nodev<float>(&lanes[l].p, *nd, packed, sw.n32, p->F32[nd->basis], lanes[l].p.khat32[nd->basis]);
        if ((e = prepare_no_constants(no, s)) != cudaSuccess) { rc = cuda_fail(e, "tc constants"); break; }
      }
      if ((e = launch_init_residual(d, s)) != cudaSuccess) { rc = cuda_fail(e, "init_residual"); break; }
    }
    if (rc != FCGNO_OK || o.maxit == 0) break;
    const int chunk = std::min(o.check_every > 0 ? o.check_every : 16, o.maxit);
    const int mask = o.profile_mask & ((1 << PROF_NCLASS) - 1);
    // two replicas of the full chunk when profiling, so a replay never overwrites events that
    // have not been read yet (the host reads chunk k-1 while chunk k runs)
    if ((rc = build_chunk(full[0], chunk, mask, nd, packed, lanes, nl, st, ev_fj)) != FCGNO_OK) break;
    if (mask && (rc = build_chunk(full[1], chunk, mask, nd, packed, lanes, nl, st, ev_fj)) != FCGNO_OK) break;
    if (o.maxit % chunk && (rc = build_chunk(tail, o.maxit % chunk, mask, nd, packed, lanes, nl, st, ev_fj)) != FCGNO_OK) break;
    // default: the whole iteration loop on the device (one graph launch); the host-polled chunk
    // loop below is kept for in-graph profiling (event nodes are not allowed in conditional
    // bodies), batch lanes, and as a fallback
    DeviceLoop* dlp = nullptr;
    std::unique_lock<std::mutex> cache_lock(loop_cache_mutex(), std::defer_lock);
    if (nl == 1 && mask == 0 && !host_loop_forced()) {
      cache_lock.lock();
      static uint64_t tick = 0;
      const LoopKey key = loop_key(lanes[0], nd, packed, chunk);
      auto& cache = loop_cache();
      for (auto& ent : cache)
        if (std::memcmp(&ent.key, &key, sizeof(key)) == 0) { dlp = &ent.loop; ent.used = ++tick; break; }
      if (!dlp) {
        DeviceLoop dl;
        if (build_device_loop(dl, chunk, nd, packed, lanes[0], s) == FCGNO_OK) {
          if (cache.size() >= kLoopCacheMax) {   // evict the least recently used
            size_t victim = 0;
            for (size_t t = 1; t < cache.size(); ++t) if (cache[t].used < cache[victim].used) victim = t;
            cache[victim].loop.destroy();
            cache.erase(cache.begin() + victim);
          }
          cache.push_back(LoopEntry{key, dl, ++tick});
          dlp = &cache.back().loop;
        } else {
          dl.destroy();
        }
      }
    }
    if (dlp) {
      DeviceLoop& dl = *dlp;
      if ((e = cudaGraphLaunch(dl.exec, s)) != cudaSuccess) rc = cuda_fail(e, "graph launch");
      const int kernels = dl.kernels;
      cache_lock.unlock();
      int it = 0;
      if (rc == FCGNO_OK && (e = cudaMemcpyAsync(h_active, lanes[0].sw.d.iter, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        rc = cuda_fail(e, "iteration count");
      if (rc == FCGNO_OK && (e = cudaStreamSynchronize(s)) != cudaSuccess) rc = cuda_fail(e, "solve");
      if (rc == FCGNO_OK) {
        it = h_active[0];
        launch_counter() += (uint64_t)kernels * (uint64_t)((it + chunk - 1) / chunk > 0 ? (it + chunk - 1) / chunk : 1);
      }
      if (rc == FCGNO_OK && (e = launch_flush_x(lanes[0].sw.d, s)) != cudaSuccess) rc = cuda_fail(e, "flush_x");
      break;
    }
    int launched = 0, k = 0;
    Chunk* prev = nullptr;
    while (launched < o.maxit) {
      Chunk* c = (o.maxit - launched >= chunk) ? &full[mask ? (k & 1) : 0] : &tail;
      if ((e = cudaGraphLaunch(c->exec, s)) != cudaSuccess) { rc = cuda_fail(e, "graph launch"); break; }
      launch_counter() += (uint64_t)c->kernels;
      launched += c->iters;
      int* hk = h_active + (k & 1) * kMaxLanes;
      for (int l = 0; l < nl && e == cudaSuccess; ++l)
        e = cudaMemcpyAsync(hk + l, lanes[l].sw.d.active, sizeof(int), cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) { rc = cuda_fail(e, "poll copy"); break; }
      if ((e = cudaEventRecord(ev_poll[k & 1], s)) != cudaSuccess) { rc = cuda_fail(e, "poll event"); break; }
      bool done = false;
      if (k > 0) {
        if ((e = cudaEventSynchronize(ev_poll[(k - 1) & 1])) != cudaSuccess) { rc = cuda_fail(e, "poll sync"); break; }
        if (mask && prev) prev->harvest();
        const int* hp = h_active + ((k - 1) & 1) * kMaxLanes;
        done = true;
        for (int l = 0; l < nl; ++l) done = done && hp[l] == 0;
      }
      prev = c;
      ++k;
      if (done) break;
    }
    if (rc == FCGNO_OK && (e = cudaStreamSynchronize(s)) == cudaSuccess && mask && prev) prev->harvest();
    for (int l = 0; l < nl && rc == FCGNO_OK; ++l)   // last lazy x update of the stopped systems
      if ((e = launch_flush_x(lanes[l].sw.d, s)) != cudaSuccess) rc = cuda_fail(e, "flush_x");
  } while (false);
  cudaError_t e_end = cudaStreamSynchronize(s);
  for (int l = 1; l < nl; ++l) {
    const cudaError_t el = cudaStreamSynchronize(st[l]);
    if (e_end == cudaSuccess) e_end = el;
  }
  if (rc == FCGNO_OK && e_end != cudaSuccess) rc = cuda_fail(e_end, "solve");
  if (rc == FCGNO_OK) (void)cudaGetLastError();
  // order the caller's stream after the solve (resources are released by `res`)
  if (cudaEventRecord(ev_in, s) == cudaSuccess) cudaStreamWaitEvent(caller, ev_in, 0);
  return rc;
}
}  // namespace

int fcgno_debug_px_trace(uint64_t* host, int count) {
  if (!host || count < 0) return fail(FCGNO_EINVAL, "debug_px_trace: bad arguments");
  CK(px_trace_read(reinterpret_cast<unsigned long long*>(host), count));
  return FCGNO_OK;
}

int fcgno_profile_get(int cls, double* total_ms, int64_t* launches) {
  if (cls < 0 || cls >= PROF_NCLASS || !total_ms || !launches) return fail(FCGNO_EINVAL, "profile_get: bad class");
  *total_ms = prof_totals().ms[cls];
  *launches = prof_totals().n[cls];
  return FCGNO_OK;
}

void fcgno_profile_reset(void) { prof_totals() = ProfTotals{}; }

const char* fcgno_profile_name(int cls) {
  static const char* names[PROF_NCLASS] = {"k_no_layer", "k_mix", "k_no_out", "k_dft_rows+k_lift_mix",
                                           "k_window_dots", "(unused 5)", "k_pform_stencil", "k_update", "(unused 8)",
                                           "k_yan+k_ysyn"};
  return (cls >= 0 && cls < PROF_NCLASS) ? names[cls] : "";
}

// ------------------------------------------------------------------ host-buffer end-to-end entry point
size_t fcgno_solve_host_workspace_bytes(fcgno_grid g, const fcgno_no_desc* nd, fcgno_solve_opts o) {
  const size_t sb = fcgno_solve_workspace_bytes(g, nd, o);
  if (!sb) return 0;
  Carver c(nullptr);
  const size_t BN = (size_t)g.batch * g.n * g.n;
  c.take<double>(BN); c.take<double>(BN); c.take<double>(BN);
  c.take<int32_t>(g.batch); c.take<int32_t>(g.batch);
  c.take<double>((size_t)g.batch * (o.maxit + 1));
  c.take<char>(fcgno_problem_workspace_bytes(g));
  c.take<char>(sb);
  return c.bytes();
}

int fcgno_solve_host(fcgno_grid g, const double* k_host, const double* f_host, double* u_host,
                     const fcgno_no_desc* nd, const void* packed, fcgno_solve_opts o, int32_t* iters_host,
                     int32_t* status_host, double* history_host, void* dev_ws, size_t ws_bytes, void* stream) {
  if (!k_host || !f_host || !u_host || !iters_host || !status_host || !dev_ws) return fail(FCGNO_EINVAL, "solve_host: NULL argument");
  const size_t need = fcgno_solve_host_workspace_bytes(g, nd, o);
  if (!need) return fail(FCGNO_EINVAL, "solve_host: bad grid or options");
  if (!aligned(dev_ws) || ws_bytes < need) return fail(FCGNO_EWORKSPACE, "solve_host: workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(dev_ws);
  const size_t BN = (size_t)g.batch * g.n * g.n;
  double* k = c.take<double>(BN);
  double* f = c.take<double>(BN);
  double* u = c.take<double>(BN);
  int32_t* it = c.take<int32_t>(g.batch);
  int32_t* st = c.take<int32_t>(g.batch);
  double* hist = c.take<double>((size_t)g.batch * (o.maxit + 1));
  const size_t pb = fcgno_problem_workspace_bytes(g);
  void* pws = c.take<char>(pb);
  const size_t sb = fcgno_solve_workspace_bytes(g, nd, o);
  void* sws = c.take<char>(sb);
  CK(cudaMemcpyAsync(k, k_host, BN * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(f, f_host, BN * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(u, u_host, BN * sizeof(double), cudaMemcpyHostToDevice, s));
  fcgno_problem* p = nullptr;
  if (int e = fcgno_assemble(g, k, pws, pb, stream, &p)) return e;
  int rc = fcgno_fcg_solve(p, nd, packed, f, u, o, it, st, history_host ? hist : nullptr, sws, sb, stream);
  fcgno_problem_destroy(p);
  if (rc) return rc;
  CK(cudaMemcpyAsync(u_host, u, BN * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(iters_host, it, g.batch * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(status_host, st, g.batch * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  if (history_host)
    CK(cudaMemcpyAsync(history_host, hist, (size_t)g.batch * (o.maxit + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return FCGNO_OK;
}

}  // extern "C"

// ================================================================== SNO training
namespace {

using ll = long long;

struct TrWs {
  float *Fj, *Fi, *Gi, *Gj, *one;
  double *kg, *rg, *eg, *d, *Ad, *Ae, *rr, *dAd, *eAe, *coef;
  dd* part;
  unsigned* cnt;            // [3][B] last-CTA counters of the three dots
  float *X2, *V[5], *Z[3], *Cs[4], *T, *G, *DV, *DV2, *DG, *DC, *dout, *partials;
};
constexpr int kTrSplit = 256;     // split-K target of the weight-gradient GEMMs

int check_train_desc(fcgno_train_desc d) {
  if (d.n < kModes || d.n > 256) return fail(FCGNO_EUNSUPPORTED, "train: needs %d <= n <= 256 (n=%d)", kModes, d.n);
  if (d.width < 1 || d.width > 128) return fail(FCGNO_EINVAL, "train: width %d outside 1..128", d.width);
  if (d.batch < 1 || (size_t)d.batch * d.n > 65535) return fail(FCGNO_EINVAL, "train: batch %d", d.batch);
  if (d.loss != FCGNO_LOSS_NOTAY && d.loss != FCGNO_LOSS_L2) return fail(FCGNO_EINVAL, "train: loss kind %d", d.loss);
  if (tr_mix_smem(d.batch, d.width, true) > 227 * 1024)
    return fail(FCGNO_EUNSUPPORTED, "train: batch x width too large for the per-mode mixing kernel");
  return FCGNO_OK;
}

TrWs carve_train(Carver& c, fcgno_train_desc d) {
  const int n = d.n, w = d.width, B = d.batch;
  const size_t N = (size_t)n * n, BN = (size_t)B * N, act = BN * w, spec = (size_t)B * 2 * kModes2 * w;
  TrWs t{};
  t.Fj = c.take<float>((size_t)2 * kModes * n);
  t.Fi = c.take<float>((size_t)2 * kModes * 2 * n);
  t.Gi = c.take<float>((size_t)2 * n * 2 * kModes);
  t.Gj = c.take<float>((size_t)n * 2 * kModes);
  t.one = c.take<float>(1);
  t.kg = c.take<double>(BN); t.rg = c.take<double>(BN); t.eg = c.take<double>(BN);
  t.d = c.take<double>(BN); t.Ad = c.take<double>(BN); t.Ae = c.take<double>(BN);
  t.rr = c.take<double>(B); t.dAd = c.take<double>(B); t.eAe = c.take<double>(B); t.coef = c.take<double>(B);
  t.part = c.take<dd>((size_t)B * part_cap(n));
  t.cnt = c.take<unsigned>((size_t)3 * B);
  t.X2 = c.take<float>(2 * BN);
  for (auto& v : t.V) v = c.take<float>(act);
  for (auto& z : t.Z) z = c.take<float>(act);
  for (auto& s : t.Cs) s = c.take<float>(spec);
  t.T = c.take<float>((size_t)B * n * 2 * kModes * w);
  t.G = c.take<float>(spec);
  t.DV = c.take<float>(act); t.DV2 = c.take<float>(act);
  t.DG = c.take<float>(spec); t.DC = c.take<float>(spec);
  t.dout = c.take<float>(BN);
  t.partials = c.take<float>((size_t)kTrSplit * 2 * std::max(w * w, 2 * w));
  return t;
}

// Blocks of the canonical weight blob (include/fcgno.h), as element offsets.
struct TrOff {
  size_t E, bE, W[4], b[4], R[4], D, bD, total;
};
TrOff tr_offsets(int w) {
  TrOff o{};
  size_t pos = 0;
  o.E = pos; pos += 2 * (size_t)w;
  o.bE = pos; pos += w;
  for (int l = 0; l < 4; ++l) {
    o.W[l] = pos; pos += (size_t)w * w;
    o.b[l] = pos; pos += w;
    o.R[l] = pos; pos += (size_t)w * w * kModes2 * 2;
  }
  o.D = pos; pos += w;
  o.bD = pos; pos += 1;
  o.total = pos;
  return o;
}

// Smallest divisor of K that is >= K / target (the split-K chunk; every chunk has the same length).
int split_chunk(int K, int target) {
  int c = std::max(1, (K + target - 1) / target);
  while (K % c) ++c;
  return c;
}

TrGemm gemm0() {
  TrGemm g{};
  g.nb0 = g.nb1 = 1;
  g.alpha = 1.f;
  return g;
}

// Truncated analysis X[b][i][j][c] -> C[b][part][kappa1][kappa2][c], times alpha (two GEMMs).
cudaError_t tr_analysis(const TrWs& t, const float* X, float* Cout, int n, int B, int w, float alpha, cudaStream_t s) {
  TrGemm g = gemm0();
  g.M = 2 * kModes; g.N = w; g.K = n; g.nb0 = B; g.nb1 = n;
  g.A = t.Fj; g.sAm = n; g.sAk = 1;
  g.B = X; g.sBk = w; g.sBn = 1; g.sB0 = (ll)n * n * w; g.sB1 = (ll)n * w;
  g.C = t.T; g.sCm = w; g.sCn = 1; g.sC0 = (ll)n * 2 * kModes * w; g.sC1 = (ll)2 * kModes * w;
  cudaError_t e = launch_tr_gemm(g, s);
  if (e != cudaSuccess) return e;
  TrGemm h = gemm0();
  h.M = 2 * kModes; h.N = kModes * w; h.K = 2 * n; h.nb0 = B;
  h.A = t.Fi; h.sAm = 2 * n; h.sAk = 1;
  h.B = t.T; h.sBk = (ll)kModes * w; h.sBn = 1; h.sB0 = (ll)n * 2 * kModes * w;
  h.C = Cout; h.sCm = (ll)kModes * w; h.sCn = 1; h.sC0 = (ll)2 * kModes2 * w;
  h.alpha = alpha;
  return launch_tr_gemm(h, s);
}

// Truncated synthesis x = alpha Re sum_M G e^{+i theta} (+ beta x), G[b][part][kappa1][kappa2][o] -> x[b][i][j][o].
cudaError_t tr_synthesis(const TrWs& t, const float* G, float* X, int n, int B, int w, float alpha, float beta,
                         cudaStream_t s) {
  TrGemm g = gemm0();
  g.M = 2 * n; g.N = kModes * w; g.K = 2 * kModes; g.nb0 = B;
  g.A = t.Gi; g.sAm = 2 * kModes; g.sAk = 1;
  g.B = G; g.sBk = (ll)kModes * w; g.sBn = 1; g.sB0 = (ll)2 * kModes2 * w;
  g.C = t.T; g.sCm = (ll)kModes * w; g.sCn = 1; g.sC0 = (ll)n * 2 * kModes * w;
  cudaError_t e = launch_tr_gemm(g, s);
  if (e != cudaSuccess) return e;
  TrGemm h = gemm0();
  h.M = n; h.N = w; h.K = 2 * kModes; h.nb0 = B; h.nb1 = n;
  h.A = t.Gj; h.sAm = 2 * kModes; h.sAk = 1;
  h.B = t.T; h.sBk = w; h.sBn = 1; h.sB0 = (ll)n * 2 * kModes * w; h.sB1 = (ll)2 * kModes * w;
  h.C = X; h.sCm = w; h.sCn = 1; h.sC0 = (ll)n * n * w; h.sC1 = (ll)n * w;
  h.alpha = alpha; h.beta = beta;
  return launch_tr_gemm(h, s);
}

// out(m, n) = sum_p A(m, p) B(p, n) over p < K, as kTrSplit-way split-K partials reduced in order.
cudaError_t tr_wgrad(const TrWs& t, int M, int N, int K, const float* A, ll sAm, ll sAk, const float* Bm, ll sBk, ll sBn,
                     float* out, ll sOm, ll sOn, cudaStream_t s) {
  const int chunk = split_chunk(K, kTrSplit), S = K / chunk;
  TrGemm g = gemm0();
  g.M = M; g.N = N; g.K = chunk; g.nb0 = S;
  g.A = A; g.sAm = sAm; g.sAk = sAk; g.sA0 = chunk * sAk;
  g.B = Bm; g.sBk = sBk; g.sBn = sBn; g.sB0 = chunk * sBk;
  g.C = t.partials; g.sCm = N; g.sCn = 1; g.sC0 = (ll)M * N;
  cudaError_t e = launch_tr_gemm(g, s);
  if (e != cudaSuccess) return e;
  return launch_tr_reduce(t.partials, S, M, N, out, sOm, sOn, s);
}

#define CKE(call)                                  \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return e_;              \
  } while (0)

// One minibatch: forward, loss, and (grad != nullptr) the full gradient of the mean loss.
cudaError_t tr_loss_grad(const TrWs& t, fcgno_train_desc d, int B, const float* P, const double* k, const double* r,
                         const double* e, const int* perm, const int* ksys, double* loss, float* grad, cudaStream_t s) {
  const int n = d.n, w = d.width, N = n * n, BP = B * N;
  const TrOff o = tr_offsets(w);
  const size_t act = (size_t)BP * w;
  CKE(launch_tr_twiddles(n, t.Fj, t.Fi, t.Gi, t.Gj, t.one, s));
  CKE(launch_tr_gather(k, r, e, perm, ksys, N, B, t.kg, t.rg, t.eg, s));
  CKE(cudaMemsetAsync(t.cnt, 0, sizeof(unsigned) * 3 * B, s));
  CKE(launch_dot(t.rg, t.rg, t.rr, t.part, t.cnt, n, B, s));
  // ---- forward (R10): lift, 4 layers, projection
  CKE(launch_tr_lift(t.rg, t.kg, t.rr, P + o.E, P + o.bE, N, B, w, t.X2, t.V[0], s));
  for (int l = 0; l < 4; ++l) {
    float* zout = l < 3 ? t.Z[l] : t.V[4];
    CKE(tr_analysis(t, t.V[l], t.Cs[l], n, B, w, 1.f, s));
    CKE(launch_tr_mix_fwd(t.Cs[l], P + o.R[l], B, w, t.G, s));
    CKE(tr_synthesis(t, t.G, zout, n, B, w, 1.f / float(N), 0.f, s));
    TrGemm g = gemm0();          // z = v W^T + b + S L A v;  v' = GELU(z) (layers 1-3)
    g.M = BP; g.N = w; g.K = w;
    g.A = t.V[l]; g.sAm = w; g.sAk = 1;
    g.B = P + o.W[l]; g.sBk = 1; g.sBn = w;
    g.C = zout; g.sCm = w; g.sCn = 1;
    g.beta = 1.f;
    g.epi = l < 3 ? TR_EPI_BIAS_GELU : TR_EPI_BIAS;
    g.bias = P + o.b[l];
    g.aux = l < 3 ? t.V[l + 1] : nullptr;
    CKE(launch_tr_gemm(g, s));
  }
  CKE(launch_tr_proj(t.V[4], P + o.D, P + o.bD, t.rr, t.eg, N, B, w, nullptr, t.d, s));
  // ---- loss
  const double* gvec = t.d;
  if (d.loss == FCGNO_LOSS_NOTAY) {
    CKE(launch_apply_A(t.kg, t.d, t.Ad, n, B, false, s));
    CKE(launch_apply_A(t.kg, t.eg, t.Ae, n, B, false, s));
    CKE(launch_dot(t.d, t.Ad, t.dAd, t.part, t.cnt + B, n, B, s));
    CKE(launch_dot(t.eg, t.Ae, t.eAe, t.part, t.cnt + 2 * B, n, B, s));
    gvec = t.Ad;
  } else {
    CKE(launch_dot(t.d, t.d, t.dAd, t.part, t.cnt + B, n, B, s));
    CKE(launch_dot(t.eg, t.eg, t.eAe, t.part, t.cnt + 2 * B, n, B, s));
  }
  CKE(launch_tr_loss(t.dAd, t.eAe, t.rr, B, B, loss, t.coef, s));
  if (!grad) return cudaSuccess;
  // ---- backward (oracle/train.py no_backward)
  CKE(launch_tr_dout(gvec, t.coef, P + o.D, N, B, w, t.dout, t.DV, s));
  CKE(tr_wgrad(t, 1, w, BP, t.dout, 0, 1, t.V[4], w, 1, grad + o.D, 0, 1, s));          // dD
  CKE(tr_wgrad(t, 1, 1, BP, t.dout, 0, 1, t.one, 0, 0, grad + o.bD, 0, 0, s));           // dbD
  float *DV = t.DV, *DV2 = t.DV2;
  for (int l = 3; l >= 0; --l) {
    if (l < 3) CKE(launch_tr_gelu_bwd(DV, t.Z[l], act, s));                              // dz (in place)
    CKE(tr_wgrad(t, w, w, BP, DV, 1, w, t.V[l], w, 1, grad + o.W[l], w, 1, s));          // dW[o][c]
    CKE(tr_wgrad(t, 1, w, BP, t.one, 0, 0, DV, w, 1, grad + o.b[l], 0, 1, s));           // db
    CKE(tr_analysis(t, DV, t.DG, n, B, w, 1.f / float(N), s));                           // dg = A(dz)/n^2
    CKE(launch_tr_mix_bwd(t.Cs[l], t.DG, P + o.R[l], B, w, grad + o.R[l], t.DC, s));     // dR, dc
    CKE(tr_synthesis(t, t.DC, DV2, n, B, w, 1.f, 0.f, s));                               // dv = n^2 S(dc)
    TrGemm g = gemm0();                                                                   // dv += dz W
    g.M = BP; g.N = w; g.K = w;
    g.A = DV; g.sAm = w; g.sAk = 1;
    g.B = P + o.W[l]; g.sBk = w; g.sBn = 1;
    g.C = DV2; g.sCm = w; g.sCn = 1;
    g.beta = 1.f;
    CKE(launch_tr_gemm(g, s));
    std::swap(DV, DV2);
  }
  CKE(tr_wgrad(t, 2, w, BP, t.X2, 1, 2, DV, w, 1, grad + o.E, 1, 2, s));                // dE[c][i]
  CKE(tr_wgrad(t, 1, w, BP, t.one, 0, 0, DV, w, 1, grad + o.bE, 0, 1, s));              // dbE
  return cudaSuccess;
}
#undef CKE

}  // namespace

extern "C" {

size_t fcgno_train_param_count(int32_t width) { return width >= 1 ? tr_offsets(width).total : 0; }

size_t fcgno_train_workspace_bytes(fcgno_train_desc d) {
  if (check_train_desc(d) != FCGNO_OK) return 0;
  Carver c(nullptr);
  carve_train(c, d);
  return c.bytes();
}

int fcgno_train_loss_grad(fcgno_train_desc d, int32_t count, const float* params, const double* k, const double* r,
                          const double* e, const int32_t* perm, const int32_t* ksys, double* loss, float* grad,
                          void* ws, size_t ws_bytes, void* stream) {
  if (int rc = check_train_desc(d)) return rc;
  if (!params || !k || !r || !e || !ws) return fail(FCGNO_EINVAL, "train_loss_grad: NULL argument");
  if (count < 1 || count > d.batch) return fail(FCGNO_EINVAL, "train_loss_grad: count %d outside 1..%d", count, d.batch);
  if (!aligned(ws) || ws_bytes < fcgno_train_workspace_bytes(d)) return fail(FCGNO_EWORKSPACE, "train_loss_grad: workspace");
  CK(prepare_tr_kernels());
  Carver c(ws);
  const TrWs t = carve_train(c, d);
  CK(tr_loss_grad(t, d, count, params, k, r, e, perm, ksys, loss, grad, static_cast<cudaStream_t>(stream)));
  return FCGNO_OK;
}

int fcgno_adamw_step(size_t count, float* params, const float* grad, float* m, float* v, int32_t t, fcgno_adamw_opts o,
                     void* stream) {
  if (!params || !grad || !m || !v) return fail(FCGNO_EINVAL, "adamw_step: NULL argument");
  if (t < 1 || !(o.lr >= 0) || !(o.beta1 >= 0 && o.beta1 < 1) || !(o.beta2 >= 0 && o.beta2 < 1) || !(o.eps > 0))
    return fail(FCGNO_EINVAL, "adamw_step: bad step or hyperparameters");
  if (count == 0) return FCGNO_OK;
  CK(launch_tr_adamw(count, params, grad, m, v, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay, t,
                     static_cast<cudaStream_t>(stream)));
  return FCGNO_OK;
}

int fcgno_train_epoch(fcgno_train_desc d, int32_t nsamples, float* params, float* grad, float* m, float* v,
                      int32_t* t_host, fcgno_adamw_opts o, const double* k, const double* r, const double* e,
                      const int32_t* perm, const int32_t* ksys, double* loss, void* ws, size_t ws_bytes,
                      void* stream) {
  if (int rc = check_train_desc(d)) return rc;
  if (!params || !grad || !m || !v || !t_host || !k || !r || !e || !perm || !ws)
    return fail(FCGNO_EINVAL, "train_epoch: NULL argument");
  if (nsamples < 1) return fail(FCGNO_EINVAL, "train_epoch: nsamples %d", nsamples);
  if (!aligned(ws) || ws_bytes < fcgno_train_workspace_bytes(d)) return fail(FCGNO_EWORKSPACE, "train_epoch: workspace");
  CK(prepare_tr_kernels());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  const TrWs t = carve_train(c, d);
  const size_t P = tr_offsets(d.width).total;
  for (int s0 = 0; s0 < nsamples; s0 += d.batch) {
    const int cnt = std::min(d.batch, nsamples - s0);
    CK(tr_loss_grad(t, d, cnt, params, k, r, e, perm + s0, ksys, loss ? loss + s0 : nullptr, grad, s));
    const int step = ++*t_host;
    CK(launch_tr_adamw(P, params, grad, m, v, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay, step, s));
  }
  return FCGNO_OK;
}

int fcgno_krylov_pair(const fcgno_problem* p, const double* f, const double* u_star, const double* u, double e_scale,
                      double* r, double* e, void* stream) {
  if (!p || !f || !u_star || !u || !r || !e) return fail(FCGNO_EINVAL, "krylov_pair: NULL argument");
  if (!(e_scale > 0.0) || !std::isfinite(e_scale)) return fail(FCGNO_EINVAL, "krylov_pair: e_scale must be positive and finite");
  if (r == u || r == f || e == u || e == u_star || r == e) return fail(FCGNO_EINVAL, "krylov_pair: outputs alias inputs");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(launch_apply_A(p->k, u, r, p->n, p->B, p->kfast, s));
  CK(launch_tr_pair(f, r, u_star, u, (size_t)p->B * p->n * p->n, e_scale, r, e, s));
  return FCGNO_OK;
}

}  // extern "C"
