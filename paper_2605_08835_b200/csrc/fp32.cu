// fp32 parity-mode kernels (§8(c) R19 "fp32 mode: everything fp32"; the north
// star's "≤ 1e-4 in an fp32 GPU mode"). SD_PREC_FP32 engines run the same UNet / VAE graph as the
// bf16 product path with fp32 weights and activations. The bf16 tensor cores cannot reach 1e-4, so
// the contractions here are SIMT FP32 FMA kernels: correctness first, used for parity runs only.
//
//   gemm(GemmDescF)      dense GEMM and implicit 3×3 conv (stride 1, pad 1, NHWC) with the same
//                        operand layouts and fused epilogue as the tcgen05 kernel (kernels.h):
//                        v = α·acc + bias + temb[img]; SiLU | GEGLU; + residual.
//                        64×64 output tiles, K slabs of 16 staged in shared memory, 4×4 per thread.
//   attention(AttnDescT<float>)  one warp per (query, head, row); fp32 online softmax (R28); d ≤ 512.
#include <float.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "kernels_ew.h"

namespace sd {

namespace {

constexpr int FBM = 64, FBN = 64, FBK = 16;

struct F32GemmArgs {
  int mode;
  const float* A;
  int lda;
  const float* x;  // conv input NHWC [B][H][W][Cin]
  int Cin, B, H, W;
  const float* Bw;
  int ldb;
  int M, N, K;       // N = accumulator columns (8C for GEGLU), K = reduction length
  int m0, m_end;     // output rows [m0, m_end)
  float* out;
  int ldo, col_off;
  const float* bias;
  int bias_per_row;
  float alpha;
  const float* temb;
  int ld_temb, rows_per_img;
  const float* res;
  int ldr;
  int act;
};

__device__ __forceinline__ float a_elem(const F32GemmArgs& g, int m, int k) {
  if (m >= g.m_end || k >= g.K) return 0.f;
  if (g.mode == GEMM_DENSE) return g.A[(long)m * g.lda + k];
  const int tap = k / g.Cin, c = k - tap * g.Cin;
  const int hw = g.H * g.W;
  const int b = m / hw, p = m - b * hw;
  const int y = p / g.W + tap / 3 - 1, x = p % g.W + tap % 3 - 1;
  if (y < 0 || y >= g.H || x < 0 || x >= g.W) return 0.f;  // zero padding
  return g.x[(((long)b * g.H + y) * g.W + x) * g.Cin + c];
}

// GEGLU: output column j reads accumulator columns value(j) and value(j) + 64 (kernels.h layout:
// rows of the projection are interleaved per 64 as [value 64 | gate 64])
__device__ __forceinline__ int geglu_value_col(int j) { return (j / 64) * 128 + (j % 64); }

template <bool GEGLU>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const F32GemmArgs g) {
  pdl_wait();
  constexpr int NB = GEGLU ? 2 : 1;  // B row sets per tile: value (+ gate)
  __shared__ float As[FBK][FBM + 4];
  __shared__ float Bs[NB][FBK][FBN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int mb = g.m0 + blockIdx.x * FBM;
  const int nb = blockIdx.y * FBN;  // output column base (GEGLU: of the N/2 outputs)
  const int n_out = GEGLU ? g.N / 2 : g.N;
  float acc[NB][4][4];
#pragma unroll
  for (int s = 0; s < NB; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[s][i][j] = 0.f;
  for (int k0 = 0; k0 < g.K; k0 += FBK) {
    for (int e = threadIdx.x; e < FBM * FBK; e += 256) {
      const int r = e / FBK, kk = e % FBK;
      As[kk][r] = a_elem(g, mb + r, k0 + kk);
    }
    for (int e = threadIdx.x; e < NB * FBN * FBK; e += 256) {
      const int s = e / (FBN * FBK), r = (e / FBK) % FBN, kk = e % FBK;
      const int j = nb + r;
      int n = j;
      if (GEGLU) n = geglu_value_col(j) + 64 * s;
      const int k = k0 + kk;
      Bs[s][kk][r] = (j < n_out && n < g.N && k < g.K) ? g.Bw[(long)n * g.ldb + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < FBK; ++kk) {
      float a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        float b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[s][kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[s][i][j] = fmaf(a[i], b[j], acc[s][i][j]);
      }
    }
    __syncthreads();
  }
  // fused epilogue (same order as the tcgen05 kernel: α, bias, temb, act, residual)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = mb + ty * 4 + i;
    if (m >= g.m_end) continue;
    const int img = g.mode == GEMM_DENSE ? m / g.rows_per_img : m / (g.H * g.W);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = nb + tx * 4 + j;
      if (col >= n_out) continue;
      float o;
      if (GEGLU) {
        const int vc = geglu_value_col(col);
        float v = acc[0][i][j] * g.alpha, gt = acc[NB - 1][i][j] * g.alpha;
        if (g.bias) {
          v += g.bias[vc];
          gt += g.bias[vc + 64];
        }
        o = v * gelu_f(gt);
      } else {
        o = acc[0][i][j] * g.alpha;
        if (g.bias) o += g.bias_per_row ? g.bias[m] : g.bias[col];
        if (g.temb) o += g.temb[(long)img * g.ld_temb + col];
        if (g.act == ACT_SILU) o = silu_f(o);
      }
      if (g.res) o += g.res[(long)m * g.ldr + col];
      g.out[(long)m * g.ldo + g.col_off + col] = o;
    }
  }
}

// O = softmax(Q·Kᵀ/√d)·V for one query per warp; lane l holds head channels l, l+32, … (NPL each)
template <int NPL>
__global__ void __launch_bounds__(128) attn_f32_kernel(const AttnDescT<float> a, float scale) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * 4 + warp, head = blockIdx.y, row = blockIdx.z;
  if (q >= a.Lq) return;
  const int d = a.d;
  const int kvb = a.kv_index ? a.kv_index[row] : row;
  const float* Qp = a.Q + (long)row * a.q_bstride + (long)q * a.ldq + (long)head * d;
  const float* Kp = a.K + (long)kvb * a.kv_bstride + (long)head * d;
  const float* Vp = a.V + (long)kvb * a.kv_bstride + (long)head * d;
  float qv[NPL], acc[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int c = lane + 32 * i;
    qv[i] = c < d ? Qp[c] : 0.f;
    acc[i] = 0.f;
  }
  float mx = -FLT_MAX, l = 0.f;
  for (int key = 0; key < a.Lk; ++key) {
    const float* kr = Kp + (long)key * a.ldk;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int c = lane + 32 * i;
      if (c < d) s = fmaf(qv[i], kr[c], s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    s *= scale;
    const float mn = fmaxf(mx, s);
    const float corr = expf(mx - mn), p = expf(s - mn);
    l = l * corr + p;
    const float* vr = Vp + (long)key * a.ldk;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int c = lane + 32 * i;
      acc[i] = acc[i] * corr + (c < d ? p * vr[c] : 0.f);
    }
    mx = mn;
  }
  float* Op = a.O + (long)row * a.o_bstride + (long)q * a.ldo + (long)head * d;
  const float inv = 1.f / l;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int c = lane + 32 * i;
    if (c < d) Op[c] = acc[i] * inv;
  }
}

}  // namespace

void gemm(const GemmDescF& d, cudaStream_t st) {
  F32GemmArgs g{};
  g.mode = d.mode;
  g.N = d.N;
  if (d.mode == GEMM_DENSE) {
    g.A = d.A;
    g.lda = d.lda;
    g.M = d.M;
    g.K = d.K;
    g.ldb = d.ldb ? d.ldb : d.K;
  } else {
    if (d.nsrc != 1 || d.stride != 1) throw CudaError("fp32 conv3: one source, stride 1");
    g.x = d.xs[0];
    g.Cin = d.cs[0];
    g.B = d.B;
    g.H = d.H;
    g.W = d.W;
    g.M = d.B * d.H * d.W;
    g.K = 9 * d.cs[0];
    g.ldb = 9 * d.cs[0];
  }
  g.Bw = d.Bw[0];
  // m_tile_begin / m_tile_count are output rows (pixels) in the fp32 kernel (kernels.h)
  g.m0 = d.m_tile_begin;
  g.m_end = d.m_tile_count >= 0 ? std::min(g.M, d.m_tile_begin + d.m_tile_count) : g.M;
  g.out = static_cast<float*>(d.out);
  g.ldo = d.ldo;
  g.col_off = d.col_off;
  g.bias = d.bias;
  g.bias_per_row = d.bias_per_row;
  g.alpha = d.alpha;
  g.temb = d.temb;
  g.ld_temb = d.ld_temb;
  g.rows_per_img = d.rows_per_img > 0 ? d.rows_per_img : 1;
  g.res = d.res;
  g.ldr = d.ldr;
  g.act = d.act;
  if (g.m_end <= g.m0 || d.N <= 0) return;
  const int n_out = d.act == ACT_GEGLU ? d.N / 2 : d.N;
  const dim3 grid(cdiv(g.m_end - g.m0, FBM), cdiv(n_out, FBN));
  if (d.act == ACT_GEGLU)
    launch_k(gemm_f32_kernel<true>, grid, 256, 0, st, g);
  else
    launch_k(gemm_f32_kernel<false>, grid, 256, 0, st, g);
  SD_CHECK_LAUNCH();
}

void attention(const AttnDescT<float>& a, cudaStream_t st) {
  if (a.d > 512 || a.d <= 0) throw CudaError("fp32 attention: d must be in [1, 512]");
  const dim3 grid(cdiv(a.Lq, 4), a.heads, a.rows);
  const float scale = 1.f / sqrtf((float)a.d);
  const int npl = cdiv(a.d, 32);
  if (npl <= 1)
    launch_k(attn_f32_kernel<1>, grid, 128, 0, st, a, scale);
  else if (npl <= 2)
    launch_k(attn_f32_kernel<2>, grid, 128, 0, st, a, scale);
  else if (npl <= 4)
    launch_k(attn_f32_kernel<4>, grid, 128, 0, st, a, scale);
  else if (npl <= 8)
    launch_k(attn_f32_kernel<8>, grid, 128, 0, st, a, scale);
  else
    launch_k(attn_f32_kernel<16>, grid, 128, 0, st, a, scale);
  SD_CHECK_LAUNCH();
}

}  // namespace sd
