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

int gn_chunk_px(int C) { return C <= 512 ? 128 : C <= 1024 ? 64 : C <= 2048 ? 32 : 16; }

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

// finalize: one warp per (image, group): lane l merges chunks l, l+32, … sequentially, then a fixed
// butterfly (Chan) — deterministic; writes (mean, rstd) for the apply kernels
__global__ void gn_finalize_kernel(int P, int C, int G, int chunk_px, int nchunks, const GNPart* __restrict__ part,
                                   float eps, float2* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b = blockIdx.y;
  if (g >= G) return;
  const int cg = C / G;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  for (int k = lane; k < nchunks; k += 32) {
    const GNPart pp = part[((long)b * nchunks + k) * G + g];
    const float nb = (float)(min(P, (k + 1) * chunk_px) - k * chunk_px) * cg;
    const float tot = n + nb;
    const float d = pp.mean - mean;
    mean += d * (nb / tot);
    m2 += pp.m2 + d * d * (n * nb / tot);
    n = tot;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float n2 = __shfl_xor_sync(0xffffffff, n, o);
    const float mu2 = __shfl_xor_sync(0xffffffff, mean, o);
    const float q2 = __shfl_xor_sync(0xffffffff, m2, o);
    const bool lo = (lane & o) == 0;  // lower lane first: both partners compute the identical value
    const float na = lo ? n : n2, ma = lo ? mean : mu2, qa = lo ? m2 : q2;
    const float nb = lo ? n2 : n, mb = lo ? mu2 : mean, qb = lo ? q2 : m2;
    const float tot = na + nb;
    if (tot > 0.f) {
      const float d = mb - ma;
      mean = ma + d * (nb / tot);
      m2 = qa + qb + d * d * (na * nb / tot);
    } else {
      mean = 0.f;
      m2 = 0.f;
    }
    n = tot;
  }
  if (lane == 0) stats[(long)b * G + g] = make_float2(mean, rsqrtf(m2 / n + eps));
}

__global__ void gn_apply_kernel(const bf16* __restrict__ x, int P, int C, int G, int chunk_px, int c_base,
                                const float2* __restrict__ stats, const float* __restrict__ gamma,
                                const float* __restrict__ beta, int silu, bf16* __restrict__ y) {
  const int R = blockDim.y;
  const int v = threadIdx.x, ry = threadIdx.y;
  const int b = blockIdx.y, ch = blockIdx.x + c_base;
  const int cg = C / G;
  __shared__ float s_mean[64], s_rstd[64];
  const int tid = ry * blockDim.x + v;
  if (tid < G) {
    const float2 st = stats[(long)b * G + tid];
    s_mean[tid] = st.x;
    s_rstd[tid] = st.y;
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

static size_t gn_part_bytes(int B, int P, int G) {
  return ((size_t)B * cdiv(P, 16) * G * sizeof(GNPart) + 255) & ~size_t(255);
}
size_t gn_workspace_bytes(int B, int P, int G) { return gn_part_bytes(B, P, G) + (size_t)B * G * sizeof(float2) + 256; }

static void gn_finalize(int B, int P, int C, int G, int cp, void* ws, float eps, cudaStream_t st) {
  const int wpb = 4;  // warps per block
  gn_finalize_kernel<<<dim3(cdiv(G, wpb), B), 32 * wpb, 0, st>>>(
      P, C, G, cp, cdiv(P, cp), reinterpret_cast<const GNPart*>(ws), eps,
      reinterpret_cast<float2*>(reinterpret_cast<char*>(ws) + gn_part_bytes(B, P, G)));
  SD_CHECK_LAUNCH();
}

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
  if (p0 == 0) gn_finalize(1, P, C, G, cp, ws, eps, st);  // bands run in order: finalize before band 0
  gn_apply_kernel<<<dim3(cdiv(p1, cp) - p0 / cp, 1), blk, 0, st>>>(
      x, P, C, G, cp, p0 / cp, reinterpret_cast<const float2*>(reinterpret_cast<char*>(ws) + gn_part_bytes(1, P, G)),
      gamma, beta, silu ? 1 : 0, y);
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
  gn_finalize(B, P, C, G, cp, ws, eps, st);
  gn_apply_kernel<<<dim3(nch, B), blk, 0, st>>>(
      x, P, C, G, cp, 0, reinterpret_cast<const float2*>(reinterpret_cast<char*>(ws) + gn_part_bytes(B, P, G)), gamma,
      beta, silu ? 1 : 0, y);
  SD_CHECK_LAUNCH();
}

// ---- LayerNorm: LANES lanes per token (NV 16-byte vectors each), two-pass in registers ----------
// C = 320/640/1280 → 8/16/32 lanes × 5 vectors: every lane issues all its loads up front and a warp
// serves 4/2/1 tokens, so the per-token reduction is short and the loads are balanced.
template <int NV, int LANES>
__global__ void layer_norm_kernel(const bf16* __restrict__ x, int T, int C, const float* __restrict__ gamma,
                                  const float* __restrict__ beta, float eps, bf16* __restrict__ y) {
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int tok = gtid / LANES, l = gtid % LANES;
  if (tok >= T) return;  // LANES divides 32, so whole lane groups exit together
  const int V = C / 8;
  const bf16* xr = x + (long)tok * C;
  float f[NV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = l + LANES * k;
    if (vi < V) {
      const uint4 u = *reinterpret_cast<const uint4*>(xr + vi * 8);
      const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
      for (int i = 0; i < 8; ++i) f[k][i] = __bfloat162float(e[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[k][i] = 0.f;
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) s += f[k][i];
#pragma unroll
  for (int o = LANES / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float mean = s / C;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (l + LANES * k < V)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = f[k][i] - mean;
        q += d * d;
      }
#pragma unroll
  for (int o = LANES / 2; o; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  const float rstd = rsqrtf(q / C + eps);
  bf16* yr = y + (long)tok * C;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = l + LANES * k;
    if (vi < V) {
      const float4 g0 = *reinterpret_cast<const float4*>(gamma + vi * 8);
      const float4 g1 = *reinterpret_cast<const float4*>(gamma + vi * 8 + 4);
      const float4 b0 = *reinterpret_cast<const float4*>(beta + vi * 8);
      const float4 b1 = *reinterpret_cast<const float4*>(beta + vi * 8 + 4);
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (f[k][i] - mean) * rstd * gg[i] + bb[i];
      *reinterpret_cast<uint4*>(yr + vi * 8) =
          make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
    }
  }
}

template <int NV, int LANES>
static void ln_launch(const bf16* x, bf16* y, int T, int C, const float* g, const float* b, float eps,
                      cudaStream_t st) {
  const int threads = 256;
  const long total = (long)T * LANES;
  layer_norm_kernel<NV, LANES><<<cdiv(total, threads), threads, 0, st>>>(x, T, C, g, b, eps, y);
  SD_CHECK_LAUNCH();
}

void layer_norm(const bf16* x, bf16* y, int T, int C, const float* gamma, const float* beta, float eps,
                cudaStream_t st) {
  if (C % 8) throw CudaError("layer_norm: C % 8");
  const int V = C / 8;
  if (V == 40) return ln_launch<5, 8>(x, y, T, C, gamma, beta, eps, st);
  if (V == 80) return ln_launch<5, 16>(x, y, T, C, gamma, beta, eps, st);
  if (V == 160) return ln_launch<5, 32>(x, y, T, C, gamma, beta, eps, st);
  if (V <= 4) return ln_launch<1, 4>(x, y, T, C, gamma, beta, eps, st);
  if (V <= 8) return ln_launch<1, 8>(x, y, T, C, gamma, beta, eps, st);
  if (V <= 16) return ln_launch<1, 16>(x, y, T, C, gamma, beta, eps, st);
  if (V <= 32) return ln_launch<1, 32>(x, y, T, C, gamma, beta, eps, st);
  if (V <= 64) return ln_launch<2, 32>(x, y, T, C, gamma, beta, eps, st);
  if (V <= 128) return ln_launch<4, 32>(x, y, T, C, gamma, beta, eps, st);
  if (V <= 256) return ln_launch<8, 32>(x, y, T, C, gamma, beta, eps, st);
  throw CudaError("layer_norm: C too large");
}

}  // namespace sd
