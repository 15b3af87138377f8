#include <stdlib.h>
// Test-only C-ABI exports: single kernels on caller-owned device buffers (sd_api.h, last section).
#include "api_common.h"
#include "common.cuh"
#include "kernels.h"
#include "kernels_ew.h"

namespace sd {
std::atomic<long long> g_launches{0};
static thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }
}  // namespace sd

static int g_dbg_splits = 0;  // split-K of sd_debug_conv3x3 (0 = the production rule)
static int g_dbg_f16 = 0;     // sd_debug_set_f16: fp16 instead of bf16 operands in the GEMM / conv / norm exports

extern "C" sd_status sd_debug_set_f16(int32_t on) {
  g_dbg_f16 = on ? 1 : 0;
  return SD_OK;
}

extern "C" const char* sd_last_error(void) { return sd::g_err.c_str(); }

extern "C" const char* sd_status_str(sd_status s) {
  switch (s) {
    case SD_OK: return "SD_OK";
    case SD_E_INVAL: return "SD_E_INVAL";
    case SD_E_NOMEM: return "SD_E_NOMEM";
    case SD_E_CUDA: return "SD_E_CUDA";
    case SD_E_AGAIN: return "SD_E_AGAIN";
    case SD_E_STATE: return "SD_E_STATE";
    case SD_E_NOTSUP: return "SD_E_NOTSUP";
  }
  return "SD_E_UNKNOWN";
}

extern "C" sd_status sd_debug_gemm(const void* A, const void* B, const float* bias, void* D, int32_t M, int32_t N,
                                   int32_t K, int32_t out_f32, int32_t act, void* stream) {
  SD_REQUIRE(A && B && D && M > 0 && N > 0 && K > 0, "sd_debug_gemm: bad arguments");
  SD_REQUIRE(K % 8 == 0, "sd_debug_gemm: K must be a multiple of 8");
  SD_API_BEGIN
  sd::GemmDesc d;
  d.mode = sd::GEMM_DENSE;
  d.A = static_cast<const bf16*>(A);
  d.M = M;
  d.K = K;
  d.lda = K;
  d.Bw[0] = static_cast<const bf16*>(B);
  d.N = N;
  d.ldb = K;
  d.out = D;
  d.ldo = act == sd::ACT_GEGLU ? N / 2 : N;
  d.out_f32 = out_f32;
  d.bias = bias;
  d.act = act;
  d.f16 = g_dbg_f16;
  sd::gemm(d, static_cast<cudaStream_t>(stream));
  SD_API_END
}

extern "C" sd_status sd_debug_gemm_res(const void* A, const void* B, const float* bias, const void* res, int32_t ldr,
                                       void* D, int32_t M, int32_t N, int32_t K, void* stream) {
  SD_REQUIRE(A && B && D && res && M > 0 && N > 0 && K > 0 && ldr >= N, "sd_debug_gemm_res: bad arguments");
  SD_REQUIRE(K % 8 == 0, "sd_debug_gemm_res: K must be a multiple of 8");
  SD_API_BEGIN
  sd::GemmDesc d;
  d.mode = sd::GEMM_DENSE;
  d.A = static_cast<const bf16*>(A);
  d.M = M;
  d.K = K;
  d.lda = K;
  d.Bw[0] = static_cast<const bf16*>(B);
  d.N = N;
  d.ldb = K;
  d.out = D;
  d.ldo = N;
  d.bias = bias;
  d.res = static_cast<const bf16*>(res);
  d.ldr = ldr;
  d.f16 = g_dbg_f16;
  d.splits = g_dbg_splits > 1 ? g_dbg_splits : 0;  // dense split-K only when forced (sd_debug_set_conv_splits)
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  d.split_ws_bytes = sd::gemm_split_ws_bytes(d);
  if (d.split_ws_bytes) SD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d.split_ws), d.split_ws_bytes, st));
  sd::gemm(d, st);
  if (d.split_ws) SD_CUDA(cudaFreeAsync(d.split_ws, st));
  SD_API_END
}

extern "C" sd_status sd_debug_conv3x3(const void* x, int32_t cin, const void* x2, int32_t cin2, const void* w,
                                      const void* w2, const float* bias, const float* temb, const void* res, void* y,
                                      int32_t nb, int32_t h, int32_t wd, int32_t cout, void* stream) {
  SD_REQUIRE(x && w && y && cin > 0 && cout > 0 && nb > 0 && h > 0 && wd > 0, "sd_debug_conv3x3: bad arguments");
  SD_REQUIRE(!x2 || (w2 && cin2 > 0), "sd_debug_conv3x3: second source needs weights");
  SD_API_BEGIN
  sd::GemmDesc d;
  d.mode = sd::GEMM_CONV3;
  d.nsrc = x2 ? 2 : 1;
  d.xs[0] = static_cast<const bf16*>(x);
  d.cs[0] = cin;
  d.xs[1] = static_cast<const bf16*>(x2);
  d.cs[1] = cin2;
  d.Bw[0] = static_cast<const bf16*>(w);
  d.Bw[1] = static_cast<const bf16*>(w2);
  d.B = nb;
  d.H = h;
  d.W = wd;
  d.N = cout;
  d.out = y;
  d.ldo = cout;
  d.bias = bias;
  d.temb = temb;
  d.ld_temb = cout;
  d.res = static_cast<const bf16*>(res);
  d.ldr = cout;
  d.splits = g_dbg_splits;
  d.f16 = g_dbg_f16;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  d.split_ws_bytes = sd::gemm_split_ws_bytes(d);
  if (d.split_ws_bytes) SD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d.split_ws), d.split_ws_bytes, st));
  sd::gemm(d, st);
  if (d.split_ws) SD_CUDA(cudaFreeAsync(d.split_ws, st));
  SD_API_END
}

extern "C" sd_status sd_debug_conv3x3_s2(const void* x, int32_t cin, const void* w, const float* bias, void* y,
                                         int32_t nb, int32_t h_in, int32_t w_in, int32_t cout, void* stream) {
  SD_REQUIRE(x && w && y && cin > 0 && cout > 0 && nb > 0 && h_in > 0 && w_in > 0 && h_in % 2 == 0 && w_in % 2 == 0,
             "sd_debug_conv3x3_s2: bad arguments");
  SD_API_BEGIN
  sd::GemmDesc d;
  d.mode = sd::GEMM_CONV3;
  d.stride = 2;
  d.xs[0] = static_cast<const bf16*>(x);
  d.cs[0] = cin;
  d.Bw[0] = static_cast<const bf16*>(w);
  d.B = nb;
  d.H = h_in / 2;
  d.W = w_in / 2;
  d.N = cout;
  d.out = y;
  d.ldo = cout;
  d.bias = bias;
  d.splits = 1;
  d.f16 = g_dbg_f16;
  sd::gemm(d, static_cast<cudaStream_t>(stream));
  SD_API_END
}

extern "C" sd_status sd_debug_set_conv_splits(int32_t splits) {
  SD_REQUIRE(splits >= 0 && splits <= 8, "sd_debug_set_conv_splits: 0 (auto), 1 (off) or 2..8");
  g_dbg_splits = splits;
  return SD_OK;
}

extern "C" sd_status sd_debug_set_gemm_cg(int32_t cg) {
  SD_REQUIRE(cg >= 0 && cg <= 2, "sd_debug_set_gemm_cg: 0 (heuristic), 1 or 2");
  sd::g_cg_override = cg;
  return SD_OK;
}

extern "C" sd_status sd_debug_attention(const void* q, const void* k, const void* v, void* o, int32_t rows,
                                        int32_t heads, int32_t d, int32_t Lq, int32_t Lk, void* stream) {
  SD_REQUIRE(q && k && v && o && rows > 0 && heads > 0 && d > 0 && d % 8 == 0 && Lq > 0 && Lk > 0,
             "sd_debug_attention: bad arguments");
  SD_API_BEGIN
  const int C = heads * d;
  sd::AttnDesc a{};
  a.Q = static_cast<const bf16*>(q);
  a.ldq = C;
  a.q_bstride = (long)Lq * C;
  a.K = static_cast<const bf16*>(k);
  a.V = static_cast<const bf16*>(v);
  a.ldk = C;
  a.kv_bstride = (long)Lk * C;
  a.O = static_cast<bf16*>(o);
  a.ldo = C;
  a.o_bstride = (long)Lq * C;
  a.rows = rows;
  a.heads = heads;
  a.d = d;
  a.Lq = Lq;
  a.Lk = Lk;
  sd::attention(a, static_cast<cudaStream_t>(stream));
  SD_API_END
}

extern "C" sd_status sd_debug_attention_tc(const void* qk, const void* vt, void* o, int32_t rows, int32_t heads,
                                           int32_t d, int32_t P, int32_t use_f16, void* stream) {
  SD_REQUIRE(qk && vt && o && rows > 0 && heads > 0, "sd_debug_attention_tc: bad arguments");
  SD_REQUIRE(sd::attention_tc_supported(d, P, heads * d), "sd_debug_attention_tc: d in {40,64,80,160}, P % 8 == 0");
  SD_API_BEGIN
  if (use_f16)
    sd::attention_tc(static_cast<const f16*>(qk), static_cast<const f16*>(vt), static_cast<f16*>(o), rows, heads, d,
                     heads * d, P, static_cast<cudaStream_t>(stream));
  else
    sd::attention_tc(static_cast<const bf16*>(qk), static_cast<const bf16*>(vt), static_cast<bf16*>(o), rows, heads,
                     d, heads * d, P, static_cast<cudaStream_t>(stream));
  SD_API_END
}

extern "C" sd_status sd_debug_xattention_tc(const void* q, const void* kc, int32_t ldk, int32_t n_slots, int32_t kcol,
                                            const void* vtc, int32_t vt_rows, int32_t ld_keys, int32_t vrow,
                                            const int32_t* kv_index, int32_t Lk, void* o, int32_t rows, int32_t heads,
                                            int32_t d, int32_t P, int32_t use_f16, void* stream) {
  SD_REQUIRE(q && kc && vtc && kv_index && o && rows > 0 && heads > 0 && Lk > 0 && n_slots > 0,
             "sd_debug_xattention_tc: bad arguments");
  SD_REQUIRE(sd::attention_tc_supported(d, 128, heads * d) && ldk % 8 == 0 && ld_keys % 8 == 0,
             "sd_debug_xattention_tc: d in {40,64,80,160}, ldk and ld_keys multiples of 8");
  SD_API_BEGIN
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* v2 = getenv("SD_XATTN_TC2");  // SD_XATTN_TC2=0: the general tcgen05 kernel
  if (!(v2 && v2[0] == '0') && sd::xattention_tc2_supported(d, Lk)) {
    if (use_f16)
      sd::xattention_tc2(static_cast<const f16*>(q), static_cast<const f16*>(kc), ldk, n_slots, kcol,
                         static_cast<const f16*>(vtc), vt_rows, ld_keys, vrow, kv_index, Lk, static_cast<f16*>(o),
                         rows, heads, d, heads * d, P, st);
    else
      sd::xattention_tc2(static_cast<const bf16*>(q), static_cast<const bf16*>(kc), ldk, n_slots, kcol,
                         static_cast<const bf16*>(vtc), vt_rows, ld_keys, vrow, kv_index, Lk, static_cast<bf16*>(o),
                         rows, heads, d, heads * d, P, st);
  } else if (use_f16)
    sd::xattention_tc(static_cast<const f16*>(q), static_cast<const f16*>(kc), ldk, n_slots, kcol,
                      static_cast<const f16*>(vtc), vt_rows, ld_keys, vrow, kv_index, Lk, static_cast<f16*>(o), rows,
                      heads, d, heads * d, P, st);
  else
    sd::xattention_tc(static_cast<const bf16*>(q), static_cast<const bf16*>(kc), ldk, n_slots, kcol,
                      static_cast<const bf16*>(vtc), vt_rows, ld_keys, vrow, kv_index, Lk, static_cast<bf16*>(o), rows,
                      heads, d, heads * d, P, st);
  SD_API_END
}

extern "C" sd_status sd_debug_groupnorm(const void* x, void* y, int32_t nb, int32_t P, int32_t C, int32_t G,
                                        const float* gamma, const float* beta, float eps, int32_t silu, void* stream) {
  SD_REQUIRE(x && y && gamma && beta && nb > 0 && P > 0 && C > 0 && G > 0 && C % G == 0 && C % 8 == 0,
             "sd_debug_groupnorm: bad arguments");
  SD_API_BEGIN
  void* ws = nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SD_CUDA(cudaMallocAsync(&ws, sd::gn_workspace_bytes(nb, P, G, C), st));
  if (g_dbg_f16)
    sd::group_norm(static_cast<const f16*>(x), static_cast<f16*>(y), nb, P, C, G, gamma, beta, eps, silu != 0, ws, st);
  else
    sd::group_norm(static_cast<const bf16*>(x), static_cast<bf16*>(y), nb, P, C, G, gamma, beta, eps, silu != 0, ws,
                   st);
  SD_CUDA(cudaFreeAsync(ws, st));
  SD_API_END
}

extern "C" sd_status sd_debug_conv3x3_gn(const void* x, int32_t cin, const void* w, const float* bias, const void* res,
                                         void* y, int32_t nb, int32_t h, int32_t wd, int32_t cout, float* gn_part,
                                         void* stream) {
  SD_REQUIRE(x && w && y && gn_part && cin > 0 && cout > 0 && nb > 0 && h > 0 && wd > 0,
             "sd_debug_conv3x3_gn: bad arguments");
  SD_API_BEGIN
  sd::GemmDesc d;
  d.mode = sd::GEMM_CONV3;
  d.xs[0] = static_cast<const bf16*>(x);
  d.cs[0] = cin;
  d.Bw[0] = static_cast<const bf16*>(w);
  d.B = nb;
  d.H = h;
  d.W = wd;
  d.N = cout;
  d.out = y;
  d.ldo = cout;
  d.bias = bias;
  d.res = static_cast<const bf16*>(res);
  d.ldr = cout;
  d.splits = 1;
  d.f16 = g_dbg_f16;
  d.gn_part = reinterpret_cast<float2*>(gn_part);
  if (!sd::gemm_gn_ok(d)) throw std::invalid_argument("sd_debug_conv3x3_gn: launch cannot emit GroupNorm statistics");
  sd::gemm(d, static_cast<cudaStream_t>(stream));
  SD_API_END
}

extern "C" sd_status sd_debug_gemm_gn(const void* A, const void* B, const float* bias, const void* res, void* D,
                                      int32_t M, int32_t N, int32_t K, int32_t P, float* gn_part, void* stream) {
  SD_REQUIRE(A && B && D && gn_part && M > 0 && N > 0 && K > 0 && K % 8 == 0 && P > 0,
             "sd_debug_gemm_gn: bad arguments");
  SD_API_BEGIN
  sd::GemmDesc d;
  d.A = static_cast<const bf16*>(A);
  d.M = M;
  d.K = K;
  d.lda = K;
  d.Bw[0] = static_cast<const bf16*>(B);
  d.N = N;
  d.ldb = K;
  d.out = D;
  d.ldo = N;
  d.bias = bias;
  d.res = static_cast<const bf16*>(res);
  d.ldr = N;
  d.f16 = g_dbg_f16;
  d.gn_part = reinterpret_cast<float2*>(gn_part);
  d.gn_P = P;
  if (!sd::gemm_gn_ok(d)) throw std::invalid_argument("sd_debug_gemm_gn: launch cannot emit GroupNorm statistics");
  sd::gemm(d, static_cast<cudaStream_t>(stream));
  SD_API_END
}

extern "C" sd_status sd_debug_groupnorm_parts(const void* x0, int32_t C0, const float* part0, const void* x1,
                                              int32_t C1, const float* part1, void* y, int32_t nb, int32_t P,
                                              int32_t G, const float* gamma, const float* beta, float eps,
                                              int32_t silu, void* stream) {
  SD_REQUIRE(x0 && part0 && y && gamma && beta && nb > 0 && P > 0 && P % 32 == 0 && C0 > 0 && G > 0,
             "sd_debug_groupnorm_parts: bad arguments");
  SD_REQUIRE(!x1 || (part1 && C1 > 0), "sd_debug_groupnorm_parts: second source needs its statistics");
  SD_API_BEGIN
  const int C = C0 + (x1 ? C1 : 0);
  void* ws = nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SD_CUDA(cudaMallocAsync(&ws, sd::gn_workspace_bytes(nb, P, G, C), st));
  const float2* p0 = reinterpret_cast<const float2*>(part0);
  const float2* p1 = reinterpret_cast<const float2*>(part1);
  if (g_dbg_f16)
    sd::group_norm_parts(static_cast<const f16*>(x0), C0, p0, static_cast<const f16*>(x1), C1, p1,
                         static_cast<f16*>(y), nb, P, G, gamma, beta, eps, silu != 0, ws, st);
  else
    sd::group_norm_parts(static_cast<const bf16*>(x0), C0, p0, static_cast<const bf16*>(x1), C1, p1,
                         static_cast<bf16*>(y), nb, P, G, gamma, beta, eps, silu != 0, ws, st);
  SD_CUDA(cudaFreeAsync(ws, st));
  SD_API_END
}

namespace {
template <class T>
void gemm_ln_impl(const void* x, int32_t T_, const void* W, int32_t Nw, int32_t K, const float* gamma,
                  const float* beta, const float* bias, void* D, float eps, int32_t cols, int32_t act,
                  cudaStream_t st) {
  float2* stat = nullptr;
  T* Wf = nullptr;
  float *wbar = nullptr, *bf = nullptr;
  SD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&stat), (size_t)T_ * sizeof(float2), st));
  SD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&Wf), (size_t)Nw * K * sizeof(T), st));
  SD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wbar), (size_t)Nw * sizeof(float), st));
  SD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bf), (size_t)Nw * sizeof(float), st));
  sd::ln_stats(static_cast<const T*>(x), T_, K, eps, stat, st);
  sd::ln_fold(static_cast<const T*>(W), Nw, K, gamma, beta, bias, Wf, wbar, bf, st);
  sd::GemmDescT<T> d;
  d.mode = sd::GEMM_DENSE;
  d.K = K;
  d.lda = K;
  d.ldb = K;
  d.ln_stat = stat;
  d.ln_wbar = wbar;
  d.ln_cols = cols;
  d.bias = bf;
  d.out = D;
  if (!cols) {  // D[T][Nw] = LN(x)·Wᵀ + b
    d.A = static_cast<const T*>(x);
    d.M = T_;
    d.Bw[0] = Wf;
    d.N = Nw;
    d.act = act;
    d.ldo = act == sd::ACT_GEGLU ? Nw / 2 : Nw;
  } else {  // D[Nw][T] = W·LN(x)ᵀ + b (bias per row)
    d.A = Wf;
    d.M = Nw;
    d.Bw[0] = static_cast<const T*>(x);
    d.N = T_;
    d.bias_per_row = 1;
    d.ldo = T_;
  }
  sd::gemm(d, st);
  SD_CUDA(cudaFreeAsync(stat, st));
  SD_CUDA(cudaFreeAsync(Wf, st));
  SD_CUDA(cudaFreeAsync(wbar, st));
  SD_CUDA(cudaFreeAsync(bf, st));
}
}  // namespace

extern "C" sd_status sd_debug_gemm_ln(const void* x, int32_t T, const void* W, int32_t N, int32_t K, const float* gamma,
                                      const float* beta, const float* bias, void* D, float eps, int32_t cols,
                                      int32_t act, void* stream) {
  SD_REQUIRE(x && W && gamma && beta && D && T > 0 && N > 0 && K > 0 && K % 8 == 0 && (act == 0 || act == 2) &&
                 (!cols || act == 0),
             "sd_debug_gemm_ln: bad arguments");
  SD_API_BEGIN
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (g_dbg_f16)
    gemm_ln_impl<f16>(x, T, W, N, K, gamma, beta, bias, D, eps, cols, act, st);
  else
    gemm_ln_impl<bf16>(x, T, W, N, K, gamma, beta, bias, D, eps, cols, act, st);
  SD_API_END
}

extern "C" sd_status sd_debug_layernorm(const void* x, void* y, int32_t T, int32_t C, const float* gamma,
                                        const float* beta, float eps, void* stream) {
  SD_REQUIRE(x && y && gamma && beta && T > 0 && C > 0 && C % 8 == 0, "sd_debug_layernorm: bad arguments");
  SD_API_BEGIN
  if (g_dbg_f16)
    sd::layer_norm(static_cast<const f16*>(x), static_cast<f16*>(y), T, C, gamma, beta, eps,
                   static_cast<cudaStream_t>(stream));
  else
    sd::layer_norm(static_cast<const bf16*>(x), static_cast<bf16*>(y), T, C, gamma, beta, eps,
                   static_cast<cudaStream_t>(stream));
  SD_API_END
}
