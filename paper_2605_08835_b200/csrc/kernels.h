// Internal (C++) interface of the sm_100a kernels. Not part of the C ABI (include/sd_api.h).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

typedef __nv_bfloat16 bf16;
typedef __half f16;

namespace sd {

enum { ACT_NONE = 0, ACT_SILU = 1, ACT_GEGLU = 2 };
enum { GEMM_DENSE = 0, GEMM_CONV3 = 1 };

// One tcgen05 GEMM launch: D[M][N] = A[M][K] · B[N][K]ᵀ, fp32 accumulate in TMEM, fused epilogue.
//  mode GEMM_DENSE : A row-major [M][K] (row stride lda elements), B [N][K] (ldb = K).
//  mode GEMM_CONV3 : implicit 3x3 / stride 1 / pad 1 convolution over NHWC bf16 inputs.
//                    A = im2col(concat(xs[0], xs[1])) is never materialised: every K block is one
//                    TMA box of 128 output pixels × 64 input channels shifted by the tap (dy,dx);
//                    out-of-image rows/cols are zero-filled by TMA (= the conv padding).
//                    B = weights [N][9][cs[s]] per source (tap-major, channel-minor).
// Epilogue: v = alpha·acc + bias[n] (or bias[m] if bias_per_row) + temb[img][n];
//           act (SiLU, or GEGLU over column pairs (c, c+64) of every 128-column group);
//           + res[m][n]; stored bf16 or fp32 at out[m·ldo + col_off + n].
// GemmDescT<bf16> drives the tcgen05 kernel (gemm.cu); GemmDescT<float> the fp32 parity-mode SIMT
// kernel (fp32.cu, R19 "fp32 mode"), which has the same operand layouts and epilogue. In the fp32
// kernel m_tile_begin / m_tile_count count output PIXELS (rows of image 0) instead of 128-row boxes.
template <class T>
struct GemmDescT {
  int mode = GEMM_DENSE;
  const T* A = nullptr;
  int M = 0, K = 0, lda = 0;
  int nsrc = 1;             // conv3: two sources = implicit channel concat; dense: A = [xs[0] | xs[1]]
  const T* xs[2] = {nullptr, nullptr};
  int cs[2] = {0, 0};
  int B = 0, H = 0, W = 0;   // conv3: batch and OUTPUT spatial size
  int stride = 1;            // conv3: 1, or 2 (input 2H×2W, pad 1: the UNet downsamplers) — tcgen05 kernel only;
                             // the taps are read by TMA boxes with element strides 2 (no im2col)
  const T* Bw[2] = {nullptr, nullptr};
  int N = 0, ldb = 0;
  void* out = nullptr;
  int ldo = 0, col_off = 0, out_f32 = 0;
  const float* bias = nullptr;
  int bias_per_row = 0;
  float alpha = 1.f;
  const float* temb = nullptr;
  int ld_temb = 0;
  int rows_per_img = 1;       // dense mode: image index = m / rows_per_img (for temb)
  const T* res = nullptr;
  int ldr = 0;
  int act = ACT_NONE;
  int m_tile_begin = 0, m_tile_count = -1;  // restrict to a contiguous range of M tiles (bands)
  int bn = 0;                 // N tile (64/128/160/256), 0 = auto
  // split-K (deterministic: fp32 partials per split, summed in split order by a reduce kernel).
  // 0 = auto (conv3 layers of ≤ 64 pixels with ≥ 90 K blocks — a function of the layer only, so
  // results stay batch-invariant), 1 = off. Needs split_ws of gemm_split_ws_bytes(d) bytes, else off.
  int splits = 0;
  float* split_ws = nullptr;
  size_t split_ws_bytes = 0;
  int f16 = 0;                // fp16 instead of bf16 (set by the GemmDescT<f16> overloads)
  // GroupNorm statistics of the stored output for a consumer GroupNorm (gemm.cu gn_colstats): per
  // 32-pixel quarter slot and channel, (Σy, Σy²) → gn_part[(img·(P/32) + slot)·N + n]. Needs
  // gemm_gn_ok(d); gn_P = pixels per image (dense mode; conv3 uses H·W).
  float2* gn_part = nullptr;
  int gn_P = 0;
  // LayerNorm folded into this GEMM (dense; norm.cu ln_fold / ln_stats): the weights are W′ = W·diag(γ) and
  // the bias b′; the epilogue applies v = rstd·(acc − μ·w̄) before the bias, with (μ, rstd) = ln_stat[row]
  // and w̄ = ln_wbar[column] — or, with ln_cols (the LN output is the B operand: Vᵀ = W·LN(h)ᵀ), (μ, rstd) =
  // ln_stat[column] and w̄ = ln_wbar[row]. Never split.
  const float2* ln_stat = nullptr;
  const float* ln_wbar = nullptr;
  int ln_cols = 0;
};

using GemmDesc = GemmDescT<bf16>;
using GemmDescF = GemmDescT<float>;

void gemm(const GemmDesc& d, cudaStream_t st);
void gemm(const GemmDescF& d, cudaStream_t st);  // fp32 parity mode (fp32.cu)
inline size_t gemm_split_ws_bytes(const GemmDescF&) { return 0; }
int gemm_splits(const GemmDesc& d);              // the split count gemm() will use given a workspace
size_t gemm_split_ws_bytes(const GemmDesc& d);   // workspace bytes (0 when not split)
void gemm(const GemmDescT<f16>& d, cudaStream_t st);  // SD_PREC_FP16: fp16 operands / outputs
int gemm_splits(const GemmDescT<f16>& d);
// whether gemm() can emit the GroupNorm statistics of this launch's output (16-bit TMA-stored output,
// N % 32 == 0, whole 32-pixel quarters inside one image, no split-K)
bool gemm_gn_ok(const GemmDesc& d);
bool gemm_gn_ok(const GemmDescT<f16>& d);
inline bool gemm_gn_ok(const GemmDescF&) { return false; }
size_t gemm_split_ws_bytes(const GemmDescT<f16>& d);
// M tiles of a conv3 launch whose output rows lie in [y0, y1) of image 0 (used for bands).
void conv3_tile_geometry(int B, int H, int W, int* wt, int* ht, int* bt);
int num_sms();
// SMs a kernel launched on `st` can use: the partition's count for an SM-partition stream (smpart.cpp,
// green contexts), else num_sms(). Persistent and cooperative grids are sized by it.
int stream_sms(cudaStream_t st);
struct Partition;
Partition* partition_create(int device, int vae_sms);
void partition_destroy(Partition* p);
cudaStream_t partition_stream(Partition* p, int i);  // 0 = the vae_sms group, 1 = the rest
extern int g_cg_override;

}  // namespace sd
