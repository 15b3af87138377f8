// GroupNorm (+SiLU) and LayerNorm on NHWC / token-major bf16 activations.
//
// GroupNorm is two launches: `gn_stats` writes deterministic per-(image, pixel-chunk, group)
// partials (mean, M2) from fp32 register sums; `gn_apply` merges the partials of its image in fixed
// chunk order (Chan et al.), then normalises, applies γ/β (+SiLU) and writes bf16 with 16-byte
// vector accesses. Thread (v, r) of a block always owns channel vector v, so the reduction order
// is fixed and never depends on the batch (batch invariance, I5) or on banding (I6).
// Chunk size adapts to C (≈ 32 K elements per chunk) so every block has enough loads in flight.
#include "common.cuh"
#include "kernels_ew.h"

namespace sd {

struct GNPart {
  float mean, m2;
};

int gn_chunk_px(int C) { return C <= 256 ? 128 : C <= 512 ? 64 : C <= 1024 ? 32 : 16; }

static dim3 gn_block(int C) {
  const int V = C / 8;
  int R = 512 / V;
  if (R < 1) R = 1;
  return dim3(V, R);
}

// block (V, R): V = C/8 vector lanes, R pixel rows; grid (chunks in range, B)
__global__ void gn_stats_kernel(const bf16* __restrict__ x, int P, int C, int G, int chunk_px, int c_base,
                                int nch_total, GNPart* __restrict__ part) {
  extern __shared__ float sh[];  // [R][V][8] sums, then sumsq
  const int V = blockDim.x, R = blockDim.y;
  const int v = threadIdx.x, ry = threadIdx.y;
  const int b = blockIdx.y, ch = blockIdx.x + c_base;
  const int p0 = ch * chunk_px, p1 = min(P, p0 + chunk_px);
  float s[8], q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] = q[i] = 0.f;
  const bf16* xb = x + (long)b * P * C + v * 8;
  int p = p0 + ry;
  for (; p + 3 * R < p1; p += 4 * R) {  // 4 independent 16-byte loads in flight
    uint4 u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = *reinterpret_cast<const uint4*>(xb + (long)(p + k * R) * C);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bf16* e = reinterpret_cast<const bf16*>(&u[k]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float f = __bfloat162float(e[i]);
        s[i] += f;
        q[i] += f * f;
      }
    }
  }
  for (; p < p1; p += R) {
    const uint4 u = *reinterpret_cast<const uint4*>(xb + (long)p * C);
    const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float f = __bfloat162float(e[i]);
      s[i] += f;
      q[i] += f * f;
    }
  }
  float* ss = sh;
  float* sq = sh + R * V * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ss[(ry * V + v) * 8 + i] = s[i];
    sq[(ry * V + v) * 8 + i] = q[i];
  }
  __syncthreads();
  // one thread per group reduces in fixed order (rows, then channels)
  const int cg = C / G;
  const int tid = ry * V + v;
  for (int g = tid; g < G; g += V * R) {
    float S = 0.f, Q = 0.f;
    for (int r = 0; r < R; ++r)
      for (int c = g * cg; c < (g + 1) * cg; ++c) {
        S += ss[(r * V + c / 8) * 8 + c % 8];
        Q += sq[(r * V + c / 8) * 8 + c % 8];
      }
    const float n = (float)(p1 - p0) * cg;
    const float mean = S / n;
    GNPart pp;
    pp.mean = mean;
    pp.m2 = fmaxf(Q - S * mean, 0.f);
    part[((long)b * nch_total + ch) * G + g] = pp;
  }
}

__global__ void gn_apply_kernel(const bf16* __restrict__ x, int P, int C, int G, int chunk_px, int c_base,
                                int nchunks, const GNPart* __restrict__ part, const float* __restrict__ gamma,
                                const float* __restrict__ beta, float eps, int silu, bf16* __restrict__ y) {
  __shared__ float s_mean[64], s_rstd[64];
  const int V = blockDim.x, R = blockDim.y;
  const int v = threadIdx.x, ry = threadIdx.y;
  const int b = blockIdx.y, ch = blockIdx.x + c_base;
  const int cg = C / G;
  const int tid = ry * V + v;
  for (int g = tid; g < G; g += V * R) {
    float n = 0.f, mean = 0.f, m2 = 0.f;
    for (int k = 0; k < nchunks; ++k) {
      const GNPart pp = part[((long)b * nchunks + k) * G + g];
      const float nb = (float)(min(P, (k + 1) * chunk_px) - k * chunk_px) * cg;
      const float tot = n + nb;
      const float d = pp.mean - mean;
      mean += d * (nb / tot);
      m2 += pp.m2 + d * d * (n * nb / tot);
      n = tot;
    }
    s_mean[g] = mean;
    s_rstd[g] = rsqrtf(m2 / n + eps);
  }
  __syncthreads();
  const int p0 = ch * chunk_px, p1 = min(P, p0 + chunk_px);
  float ga[8], be[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = v * 8 + i;
    const float rs = s_rstd[c / cg];
    ga[i] = gamma[c] * rs;                      // y = x·(γ·rstd) + (β − mean·γ·rstd)
    be[i] = beta[c] - s_mean[c / cg] * ga[i];
  }
  const long base = (long)b * P * C + v * 8;
  int p = p0 + ry;
  for (; p + R < p1; p += 2 * R) {
    uint4 u[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) u[k] = *reinterpret_cast<const uint4*>(x + base + (long)(p + k * R) * C);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const bf16* e = reinterpret_cast<const bf16*>(&u[k]);
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float f = __bfloat162float(e[i]) * ga[i] + be[i];
        o[i] = silu ? silu_f(f) : f;
      }
      *reinterpret_cast<uint4*>(y + base + (long)(p + k * R) * C) =
          make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
    }
  }
  for (; p < p1; p += R) {
    const uint4 u = *reinterpret_cast<const uint4*>(x + base + (long)p * C);
    const bf16* e = reinterpret_cast<const bf16*>(&u);
    float o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float f = __bfloat162float(e[i]) * ga[i] + be[i];
      o[i] = silu ? silu_f(f) : f;
    }
    *reinterpret_cast<uint4*>(y + base + (long)p * C) =
        make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
  }
}

size_t gn_workspace_bytes(int B, int P, int G) { return (size_t)B * cdiv(P, 16) * G * sizeof(GNPart) + 256; }

static void check_gn(int C, int G) {
  if (C % 8 || C / 8 > 1024 || G > 64 || C % G) throw CudaError("group_norm: unsupported C/G");
}

// band-restricted halves of group_norm (B = 1) over pixels [p0, p1) (multiples of 128): stats of the
// chunks in the range; normalisation of the chunks in the range with ALL chunk partials merged in
// fixed order — a banded GN is bitwise equal to the whole-tensor GN (R7 V1).
void gn_stats_range(const bf16* x, int P, int C, int G, int p0, int p1, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const int cp = gn_chunk_px(C);
  const dim3 blk = gn_block(C);
  const size_t sh = (size_t)blk.x * blk.y * 8 * 2 * sizeof(float);
  gn_stats_kernel<<<dim3(cdiv(p1, cp) - p0 / cp, 1), blk, sh, st>>>(x, P, C, G, cp, p0 / cp, cdiv(P, cp),
                                                                     reinterpret_cast<GNPart*>(ws));
  SD_CHECK_LAUNCH();
}
void gn_apply_range(const bf16* x, bf16* y, int P, int C, int G, int p0, int p1, const float* gamma, const float* beta,
                    float eps, bool silu, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const int cp = gn_chunk_px(C);
  const dim3 blk = gn_block(C);
  gn_apply_kernel<<<dim3(cdiv(p1, cp) - p0 / cp, 1), blk, 0, st>>>(x, P, C, G, cp, p0 / cp, cdiv(P, cp),
                                                                    reinterpret_cast<const GNPart*>(ws), gamma, beta,
                                                                    eps, silu ? 1 : 0, y);
  SD_CHECK_LAUNCH();
}

void group_norm(const bf16* x, bf16* y, int B, int P, int C, int G, const float* gamma, const float* beta, float eps,
                bool silu, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const dim3 blk = gn_block(C);
  const int cp = gn_chunk_px(C);
  const int nch = cdiv(P, cp);
  GNPart* part = reinterpret_cast<GNPart*>(ws);
  const size_t sh = (size_t)blk.x * blk.y * 8 * 2 * sizeof(float);
  gn_stats_kernel<<<dim3(nch, B), blk, sh, st>>>(x, P, C, G, cp, 0, nch, part);
  SD_CHECK_LAUNCH();
  gn_apply_kernel<<<dim3(nch, B), blk, 0, st>>>(x, P, C, G, cp, 0, nch, part, gamma, beta, eps, silu ? 1 : 0, y);
  SD_CHECK_LAUNCH();
}

// ---- LayerNorm: one warp per token, two-pass in registers ---------------------------------------
template <int NV>  // vectors (of 8) per lane, ceil(C/8/32)
__global__ void layer_norm_kernel(const bf16* __restrict__ x, int T, int C, const float* __restrict__ gamma,
                                  const float* __restrict__ beta, float eps, bf16* __restrict__ y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T) return;
  const int V = C / 8;
  const bf16* xr = x + (long)warp * C;
  float f[NV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = lane + 32 * k;
    if (vi < V) {
      uint4 u = *reinterpret_cast<const uint4*>(xr + vi * 8);
      const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        f[k][i] = __bfloat162float(e[i]);
        s += f[k][i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[k][i] = 0.f;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float mean = s / C;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (lane + 32 * k < V)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = f[k][i] - mean;
        q += d * d;
      }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  const float rstd = rsqrtf(q / C + eps);
  bf16* yr = y + (long)warp * C;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = lane + 32 * k;
    if (vi < V) {
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (f[k][i] - mean) * rstd * gamma[vi * 8 + i] + beta[vi * 8 + i];
      *reinterpret_cast<uint4*>(yr + vi * 8) =
          make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
    }
  }
}

void layer_norm(const bf16* x, bf16* y, int T, int C, const float* gamma, const float* beta, float eps,
                cudaStream_t st) {
  if (C % 8) throw CudaError("layer_norm: C % 8");
  const int nv = cdiv(C / 8, 32);
  const int threads = 256;
  const int blocks = cdiv((long)T * 32, threads);
  switch (nv) {
    case 1: layer_norm_kernel<1><<<blocks, threads, 0, st>>>(x, T, C, gamma, beta, eps, y); break;
    case 2: layer_norm_kernel<2><<<blocks, threads, 0, st>>>(x, T, C, gamma, beta, eps, y); break;
    case 3: layer_norm_kernel<3><<<blocks, threads, 0, st>>>(x, T, C, gamma, beta, eps, y); break;
    case 4: layer_norm_kernel<4><<<blocks, threads, 0, st>>>(x, T, C, gamma, beta, eps, y); break;
    case 5: layer_norm_kernel<5><<<blocks, threads, 0, st>>>(x, T, C, gamma, beta, eps, y); break;
    case 8: layer_norm_kernel<8><<<blocks, threads, 0, st>>>(x, T, C, gamma, beta, eps, y); break;
    default: throw CudaError("layer_norm: C too large");
  }
  SD_CHECK_LAUNCH();
}

}  // namespace sd
