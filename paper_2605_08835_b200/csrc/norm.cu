// GroupNorm (+SiLU) and LayerNorm on NHWC / token-major bf16 activations.
//
// GroupNorm is two launches: `gn_stats` writes deterministic per-(image, pixel-chunk, group)
// partials (mean, M2) from fp32 register sums (one warp per group reduces the block's rows and
// channels); `gn_apply` merges the partials of its image in fixed chunk order (Chan et al.; a
// separate finalize launch instead when an image has more than 128 chunks), then normalises, applies γ/β (+SiLU) and writes bf16 with 16-byte
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
template <class T>
__global__ void gn_stats_kernel(const T* __restrict__ x, int P, int C, int G, int chunk_px, int c_base,
                                int nch_total, GNPart* __restrict__ part) {
  extern __shared__ float sh[];  // [R][V][8] sums, then sumsq
  const int V = blockDim.x, R = blockDim.y;
  const int v = threadIdx.x, ry = threadIdx.y;
  const int b = blockIdx.y, ch = blockIdx.x + c_base;
  const int p0 = ch * chunk_px, p1 = min(P, p0 + chunk_px);
  float s[8], q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] = q[i] = 0.f;
  const T* xb = x + (long)b * P * C + v * 8;
  int p = p0 + ry;
  for (; p + 3 * R < p1; p += 4 * R) {  // 4 independent vector loads in flight
    float f[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k) load8(xb + (long)(p + k * R) * C, f[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s[i] += f[k][i];
        q[i] += f[k][i] * f[k][i];
      }
  }
  for (; p < p1; p += R) {
    float f[8];
    load8(xb + (long)p * C, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s[i] += f[i];
      q[i] += f[i] * f[i];
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
  // one warp per group: lanes stride the R × cg (row, channel) partials in a fixed order, then a
  // xor butterfly (both partners add the same two values, so every lane holds the same bits)
  const int cg = C / G;
  const int tid = ry * V + v, lane = tid & 31, nw = (V * R) >> 5;
  const int ne = R * cg;
  for (int g = tid >> 5; g < G; g += nw) {
    float S = 0.f, Q = 0.f;
    for (int e = lane; e < ne; e += 32) {
      const int r = e / cg, c = g * cg + e % cg;
      S += ss[r * V * 8 + c];
      Q += sq[r * V * 8 + c];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      S += __shfl_xor_sync(0xffffffff, S, o);
      Q += __shfl_xor_sync(0xffffffff, Q, o);
    }
    if (lane == 0) {
      const float n = (float)(p1 - p0) * cg;
      const float mean = S / n;
      GNPart pp;
      pp.mean = mean;
      pp.m2 = fmaxf(Q - S * mean, 0.f);
      part[((long)b * nch_total + ch) * G + g] = pp;
    }
  }
}

// finalize: one warp per (image, group): lane l merges chunks l, l+32, … sequentially, then a fixed
// butterfly (Chan) — deterministic; writes (mean, rstd) for the apply kernels
// (the same function serves the separate finalize kernel and the in-block merge of gn_apply, so
// both produce identical bits)
__device__ __forceinline__ float2 gn_merge(int P, int C, int G, int chunk_px, int nchunks,
                                           const GNPart* __restrict__ part, float eps, int b, int g, int lane) {
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
  return make_float2(mean, rsqrtf(m2 / n + eps));
}

__global__ void gn_finalize_kernel(int P, int C, int G, int chunk_px, int nchunks, const GNPart* __restrict__ part,
                                   float eps, float2* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b = blockIdx.y;
  if (g >= G) return;
  const float2 r = gn_merge(P, C, G, chunk_px, nchunks, part, eps, b, g, lane);
  if (lane == 0) stats[(long)b * G + g] = r;
}

template <class T>
__global__ void gn_apply_kernel(const T* __restrict__ x, int P, int C, int G, int chunk_px, int c_base,
                                const float2* __restrict__ stats, const GNPart* __restrict__ part, int nchunks,
                                float eps, const float* __restrict__ gamma, const float* __restrict__ beta, int silu,
                                T* __restrict__ y) {
  const int R = blockDim.y;
  const int v = threadIdx.x, ry = threadIdx.y;
  const int b = blockIdx.y, ch = blockIdx.x + c_base;
  const int cg = C / G;
  __shared__ float s_mean[64], s_rstd[64];
  const int tid = ry * blockDim.x + v;
  if (part) {
    // few partials: every block merges its image's chunk partials itself (no finalize launch)
    const int nw = (blockDim.x * R) >> 5;
    for (int g = tid >> 5; g < G; g += nw) {
      const float2 st = gn_merge(P, C, G, chunk_px, nchunks, part, eps, b, g, tid & 31);
      if ((tid & 31) == 0) {
        s_mean[g] = st.x;
        s_rstd[g] = st.y;
      }
    }
  } else if (tid < G) {
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
    float u[2][8];
#pragma unroll
    for (int k = 0; k < 2; ++k) load8(x + base + (long)(p + k * R) * C, u[k]);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float f = u[k][i] * ga[i] + be[i];
        o[i] = silu ? silu_f(f) : f;
      }
      store8(y + base + (long)(p + k * R) * C, o);
    }
  }
  for (; p < p1; p += R) {
    float u[8];
    load8(x + base + (long)p * C, u);
    float o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float f = u[i] * ga[i] + be[i];
      o[i] = silu ? silu_f(f) : f;
    }
    store8(y + base + (long)p * C, o);
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
template <class T>
void gn_stats_range(const T* x, int P, int C, int G, int p0, int p1, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const int cp = gn_chunk_px(C);
  const dim3 blk = gn_block(C);
  const size_t sh = (size_t)blk.x * blk.y * 8 * 2 * sizeof(float);
  gn_stats_kernel<<<dim3(cdiv(p1, cp) - p0 / cp, 1), blk, sh, st>>>(x, P, C, G, cp, p0 / cp, cdiv(P, cp),
                                                                     reinterpret_cast<GNPart*>(ws));
  SD_CHECK_LAUNCH();
}
template <class T>
void gn_apply_range(const T* x, T* y, int P, int C, int G, int p0, int p1, const float* gamma, const float* beta,
                    float eps, bool silu, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const int cp = gn_chunk_px(C);
  const dim3 blk = gn_block(C);
  if (p0 == 0) gn_finalize(1, P, C, G, cp, ws, eps, st);  // bands run in order: finalize before band 0
  gn_apply_kernel<<<dim3(cdiv(p1, cp) - p0 / cp, 1), blk, 0, st>>>(
      x, P, C, G, cp, p0 / cp, reinterpret_cast<const float2*>(reinterpret_cast<char*>(ws) + gn_part_bytes(1, P, G)),
      nullptr, 0, eps, gamma, beta, silu ? 1 : 0, y);
  SD_CHECK_LAUNCH();
}

template <class T>
void group_norm(const T* x, T* y, int B, int P, int C, int G, const float* gamma, const float* beta, float eps,
                bool silu, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const dim3 blk = gn_block(C);
  const int cp = gn_chunk_px(C);
  const int nch = cdiv(P, cp);
  GNPart* part = reinterpret_cast<GNPart*>(ws);
  const size_t sh = (size_t)blk.x * blk.y * 8 * 2 * sizeof(float);
  gn_stats_kernel<<<dim3(nch, B), blk, sh, st>>>(x, P, C, G, cp, 0, nch, part);
  SD_CHECK_LAUNCH();
  // ≤ 128 chunk partials per (image, group) (every UNet GN up to a 128×128 latent): merged inside the
  // apply blocks; more (the VAE's large images): one finalize launch first
  const bool inline_merge = nch <= 128;
  if (!inline_merge) gn_finalize(B, P, C, G, cp, ws, eps, st);
  gn_apply_kernel<<<dim3(nch, B), blk, 0, st>>>(
      x, P, C, G, cp, 0, reinterpret_cast<const float2*>(reinterpret_cast<char*>(ws) + gn_part_bytes(B, P, G)),
      inline_merge ? part : nullptr, nch, eps, gamma, beta, silu ? 1 : 0, y);
  SD_CHECK_LAUNCH();
}

// ---- LayerNorm: LANES lanes per token (NV 16-byte vectors each), two-pass in registers ----------
// C = 320/640/1280 → 8/16/32 lanes × 5 vectors: every lane issues all its loads up front and a warp
// serves 4/2/1 tokens, so the per-token reduction is short and the loads are balanced.
template <int NV, int LANES, class E>
__global__ void layer_norm_kernel(const E* __restrict__ x, int T, int C, const float* __restrict__ gamma,
                                  const float* __restrict__ beta, float eps, E* __restrict__ y) {
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int tok = gtid / LANES, l = gtid % LANES;
  if (tok >= T) return;  // LANES divides 32, so whole lane groups exit together
  const int V = C / 8;
  const E* xr = x + (long)tok * C;
  float f[NV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = l + LANES * k;
    if (vi < V) {
      load8(xr + vi * 8, f[k]);
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
  E* yr = y + (long)tok * C;
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
      store8(yr + vi * 8, o);
    }
  }
}

template <int NV, int LANES, class E>
static void ln_launch(const E* x, E* y, int T, int C, const float* g, const float* b, float eps,
                      cudaStream_t st) {
  const int threads = 256;
  const long total = (long)T * LANES;
  layer_norm_kernel<NV, LANES, E><<<cdiv(total, threads), threads, 0, st>>>(x, T, C, g, b, eps, y);
  SD_CHECK_LAUNCH();
}

template <class E>
void layer_norm(const E* x, E* y, int T, int C, const float* gamma, const float* beta, float eps,
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

#define SD_NORM_INST(T)                                                                                      \
  template void group_norm<T>(const T*, T*, int, int, int, int, const float*, const float*, float, bool, void*, \
                              cudaStream_t);                                                                 \
  template void gn_stats_range<T>(const T*, int, int, int, int, int, void*, cudaStream_t);                   \
  template void gn_apply_range<T>(const T*, T*, int, int, int, int, int, const float*, const float*, float, bool, \
                                  void*, cudaStream_t);                                                      \
  template void layer_norm<T>(const T*, T*, int, int, const float*, const float*, float, cudaStream_t);
SD_NORM_INST(bf16)
SD_NORM_INST(float)

}  // namespace sd
