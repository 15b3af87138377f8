// Internal interface of the non-GEMM kernels (norms, attention, elementwise, weight init).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stddef.h>
#include <stdint.h>

typedef __nv_bfloat16 bf16;
typedef __half f16;

namespace sd {

// ---- norms (norm.cu) ----  bf16 activations (the product path) and fp32 (parity mode, R19); both
// element types share the kernels, the workspace layout and the fixed reduction order
size_t gn_workspace_bytes(int B, int P, int G, int C);  // C = the largest channel count normalised
int gn_chunk_px(int C);  // pixels per statistics chunk (divides 128)
// x, y: [B][P][C]
template <class T>
void group_norm(const T* x, T* y, int B, int P, int C, int G, const float* gamma, const float* beta, float eps,
                bool silu, void* ws, cudaStream_t st);
// GroupNorm over the channel concat [x0 (C0 channels) | x1 (C1 channels)] of two [B][P][·] tensors,
// written to y [B][P][C0 + C1] — the up-block concat is never materialised
template <class T>
void group_norm2(const T* x0, int C0, const T* x1, int C1, T* y, int B, int P, int G, const float* gamma,
                 const float* beta, float eps, bool silu, void* ws, cudaStream_t st);
// pixel ranges [p0, p1) must be multiples of 128 (or end at P)
template <class T>
void gn_stats_range(const T* x, int P, int C, int G, int p0, int p1, void* ws, cudaStream_t st);
template <class T>
void gn_apply_range(const T* x, T* y, int P, int C, int G, int p0, int p1, const float* gamma, const float* beta,
                    float eps, bool silu, void* ws, cudaStream_t st);
// GroupNorm whose statistics came from the producers' GEMM / conv epilogues (GemmDescT::gn_part):
// part0 / part1 = [B][P/32][C0] / [B][P/32][C1] (Σy, Σy²) per 32-pixel slot and channel (P % 32 == 0).
// One finalize launch + the apply: no statistics pass over x.
template <class T>
void group_norm_parts(const T* x0, int C0, const float2* part0, const T* x1, int C1, const float2* part1, T* y, int B,
                      int P, int G, const float* gamma, const float* beta, float eps, bool silu, void* ws,
                      cudaStream_t st);
// banded apply (B = 1) from producer statistics; the finalize runs with the first band (p0 == 0)
template <class T>
void gn_apply_range_parts(const T* x, T* y, int P, int C, int G, int p0, int p1, const float2* part, const float* gamma,
                          const float* beta, float eps, bool silu, void* ws, cudaStream_t st);
// LayerNorm folded into the consumer GEMM (norm.cu; gemm.cu ln_stat epilogue): per-token (μ, rstd), and
// the folded weights W′ = W·diag(γ) (16-bit), w̄ = row sums of W′, b′ = b + W·β (bias may be null)
template <class T>
void ln_stats(const T* x, int T_, int C, float eps, float2* st, cudaStream_t s);
template <class T>
void ln_fold(const T* W, int N, int K, const float* gamma, const float* beta, const float* bias, T* Wf, float* wbar,
             float* bf, cudaStream_t s);
template <class T>
void layer_norm(const T* x, T* y, int T_, int C, const float* gamma, const float* beta, float eps, cudaStream_t st);

// ---- attention (attention.cu): O = softmax(Q Kᵀ/√d) V per (batch row, head) ----
template <class T>
struct AttnDescT {
  const T* Q;
  int ldq;           // elements between consecutive tokens
  long q_bstride;    // elements between batch rows
  const T* K;
  const T* V;
  int ldk;
  long kv_bstride;
  const int* kv_index;  // optional per-row batch index for K/V (cross-attention ctx slots)
  T* O;
  int ldo;
  long o_bstride;
  int rows, heads, d, Lq, Lk;
};
using AttnDesc = AttnDescT<bf16>;
void attention(const AttnDesc& a, cudaStream_t st);
// fp32 parity mode (fp32.cu): one warp per query, fp32 online softmax; any d ≤ 512
void attention(const AttnDescT<float>& a, cudaStream_t st);
void attention(const AttnDescT<f16>& a, cudaStream_t st);  // SD_PREC_FP16 (mma.sync .f16)

// tcgen05 flash attention (attention_tc.cu): qk [rows·P][2C] (q | k), vt [C][rows·P], O [rows·P][C]
bool attention_tc_supported(int d, int P, int C);
void attention_tc(const bf16* qk, const bf16* vt, bf16* O, int rows, int heads, int d, int C, int P, cudaStream_t st);
void attention_tc(const f16* qk, const f16* vt, f16* O, int rows, int heads, int d, int C, int P, cudaStream_t st);
// tcgen05 cross-attention over cached text tokens (K7): q [rows·P][C]; kc [n_slots·Lk][ldk] (this layer's K at
// column kcol); vtc [vt_rows][ld_keys] (this layer's Vᵀ at row vrow; key j of slot s at column s·⌈Lk⌉₈ + j);
// kv_index [rows] slot per batch row (device); O [rows·P][C]. d ∈ {40, 64, 80, 160}.
void xattention_tc(const bf16* q, const bf16* kc, int ldk, long n_slots, int kcol, const bf16* vtc, long vt_rows,
                   long ld_keys, int vrow, const int* kv_index, int Lk, bf16* O, int rows, int heads, int d, int C, int P,
                   cudaStream_t st);
void xattention_tc(const f16* q, const f16* kc, int ldk, long n_slots, int kcol, const f16* vtc, long vt_rows,
                   long ld_keys, int vrow, const int* kv_index, int Lk, f16* O, int rows, int heads, int d, int C, int P,
                   cudaStream_t st);
// the same layouts on the persistent variant (xattention_tc.cu): one CTA per (row, head) run of query tiles
// with K / Vᵀ resident; d ∈ {40, 64, 80}, Lk ≤ 128
bool xattention_tc2_supported(int d, int Lk);
void xattention_tc2(const bf16* q, const bf16* kc, int ldk, long n_slots, int kcol, const bf16* vtc, long vt_rows,
                    long ld_keys, int vrow, const int* kv_index, int Lk, bf16* O, int rows, int heads, int d, int C,
                    int P, cudaStream_t st);
void xattention_tc2(const f16* q, const f16* kc, int ldk, long n_slots, int kcol, const f16* vtc, long vt_rows,
                    long ld_keys, int vrow, const int* kv_index, int Lk, f16* O, int rows, int heads, int d, int C,
                    int P, cudaStream_t st);

// row softmax for the VAE attention path: P[r][:] = softmax(S[r][:]) (S fp32, P bf16)
void softmax_rows(const float* S, bf16* P, int rows, int cols, cudaStream_t st);
void softmax_rows(const float* S, f16* P, int rows, int cols, cudaStream_t st);

// ---- elementwise (elementwise.cu) ----
struct RowMap {                 // device-side per-step metadata (uploaded once per call)
  const float* const* latents;  // [n_req] fp32 [4][h][w]
  const float* c_in;            // [n_req]
  const float* t_row;           // [rows]
  const int* row_req;           // [rows] request index of each UNet row
  const int* unc_row;           // [n_req] row index of the uncond row or -1
  const float* guidance;        // [n_req]
  const float* coef_a;          // [n_req] x ← a·x + b·ε̃
  const float* coef_b;          // [n_req]
};
template <class T>
void gather_rows(const RowMap& m, int rows, int hw, int cpad, T* out, cudaStream_t st);
void combine_update(const RowMap& m, int n_req, int hw, const float* eps, int ld_eps, float* const* latents_dev,
                    cudaStream_t st);
template <class T>
void timestep_sinusoid(const float* t_row, int rows, int dim, T* out, cudaStream_t st);
template <class T>
void upsample2x(const T* x, T* y, int B, int H, int W, int C, cudaStream_t st);
template <class T>
void im2col_s2(const T* x, T* y, int B, int H, int W, int C, cudaStream_t st);  // 3x3 stride 2 pad 1
template <class T>
void concat_channels(const T* a, int ca, const T* b, int cb, T* y, long P, cudaStream_t st);
void f32_to_bf16(const float* x, bf16* y, long n, cudaStream_t st);
inline void f32_to_act(const float* x, bf16* y, long n, cudaStream_t st) { f32_to_bf16(x, y, n, st); }
void f32_to_act(const float* x, float* y, long n, cudaStream_t st);  // device copy
void f32_to_act(const float* x, f16* y, long n, cudaStream_t st);
void gather_rows_f32(const float* src, const int* idx, int rows, int n, float* dst, cudaStream_t st);
// VAE head input: z fp32 [4][h][w] → NHWC [h][w][cpad] of z·scale (zeros in channels ≥ 4)
template <class T>
void latent_to_nhwc(const float* z, int hw, float scale, int cpad, T* out, cudaStream_t st);
// image NHWC fp32 [P][ld] (first 3 channels) → NCHW fp32 [3][P]
void nhwc_to_nchw3(const float* x, int ld, long P, float* y, cudaStream_t st);

// ---- weight init (weights.cu) — counter-based generator shared in spec with synth/ ----
enum { WL_PLAIN = 0, WL_CONV3 = 1, WL_GEGLU = 2, WL_ROWS = 4 };  // WL_ROWS: [O][I] into rows of Ipad
enum { WK_UNIFORM = 0, WK_GAMMA = 1, WK_BETA = 2 };
struct WeightInit {
  uint64_t tseed;      // tensor_seed(global_seed, name)
  int kind;            // WK_*
  float bound;         // fl32(1/sqrt(fan_in)) (uniform kind)
  int layout;          // WL_*
  long n;              // canonical element count
  int O, I, I1;        // conv3: O out channels, I in channels, I1 split (first source channels)
  int Ipad;            // conv3 destination channels of source 0 (≥ I1) when no split
  int F;               // GEGLU: half width (rows are [value F | gate F])
  void* dst0;
  void* dst1;
  int out_bf16;        // 0 fp32, 1 bf16, 2 fp16 (SD_PREC_FP16)
  const float* src;    // nullptr: generate; else canonical fp32 values (sd_engine_set_weight)
};
void init_weight(const WeightInit& w, cudaStream_t st);

}  // namespace sd
