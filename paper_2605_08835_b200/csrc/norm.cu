// GroupNorm (+SiLU) and LayerNorm on NHWC / token-major activations;
// bf16 on the product path, fp32 in the parity mode (R19).
//
// GroupNorm is three launches:
//   gn_stats     deterministic per-(image, pixel-chunk, group) partials (mean, M2) from fp32 register
//                sums: thread (v, r) of a block always owns channel vector v and issues 8 independent
//                16-byte loads per batch; one warp per group then reduces the block's rows and
//                channels in a fixed order.
//   merge        one warp per (image, group) merges the chunk partials in fixed order (Chan et al.)
//                and writes the per-(image, channel) affine table scale = γ·rstd, shift = β − μ·scale;
//                (gn_finalize launch).
//   gn_apply     y = x·scale + shift (+SiLU): each thread owns one channel vector (its table entries
//                stay in registers), 4 pixel rows in flight per thread, grid-stride.
// The reduction order depends only on (P, C, G) — never on the batch (I5) or on banding (I6).
// Chunk size adapts to C (≈ 40 K elements per chunk).
#include <algorithm>
#include <mutex>
#include <map>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "kernels_ew.h"

namespace sd {

struct GNPart {
  float mean, m2;
};

int gn_chunk_px(int C) { return C <= 512 ? 128 : C <= 1024 ? 64 : C <= 2048 ? 32 : 16; }

static dim3 gn_stats_block(int C) {
  const int V = C / 8;
  int R = 256 / V;
  if (R < 1) R = 1;
  if (V * R < 32) R = cdiv(32, V);
  return dim3(V, R);
}

// raw 8-element vectors: loads stay in flight without conversion registers
template <class T>
struct Raw8;
template <>
struct Raw8<bf16> {
  uint4 u;
  __device__ __forceinline__ void ld(const bf16* p) { u = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void get(float (&f)[8]) const {
    const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(e[i]);
  }
};
template <>
struct Raw8<f16> {
  uint4 u;
  __device__ __forceinline__ void ld(const f16* p) { u = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void get(float (&f)[8]) const {
    const f16* e = reinterpret_cast<const f16*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __half2float(e[i]);
  }
};
template <>
struct Raw8<float> {
  float4 a, b;
  __device__ __forceinline__ void ld(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  __device__ __forceinline__ void get(float (&f)[8]) const {
    f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
  }
};

// Chan merge of one (image, group)'s chunk partials by one warp (weights by the fast MUFU division:
// the merge is a latency chain, and every path uses this same function, so results stay bitwise
// consistent across batch sizes, bands and launch paths): lane l merges chunks l, l+32, …
// sequentially, then a fixed butterfly in which both partners compute the identical value —
// deterministic, independent of which block runs it. Writes the group's affine table entries
// (scale = γ·rstd, shift = β − μ·scale). Partials are read through L2 (written by other SMs).
// `ld(k)` returns chunk k's partial (global through L2, or a shared-memory copy); `tab` = the image's
// C table entries.
template <class LD>
__device__ __forceinline__ void gn_merge_group(int P, int C, int G, int chunk_px, int nchunks, LD ld, float eps,
                                               const float* __restrict__ gamma, const float* __restrict__ beta,
                                               float2* __restrict__ tab, int g, int lane) {
  const int cg = C / G;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  for (int k = lane; k < nchunks; k += 32) {
    const float2 pp = ld(k);
    const float nb = (float)(min(P, (k + 1) * chunk_px) - k * chunk_px) * cg;
    const float tot = n + nb;
    const float d = pp.x - mean;
    const float w = __fdividef(nb, tot);
    mean += d * w;
    m2 += pp.y + d * d * (n * w);
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
      const float w = __fdividef(nb, tot);
      mean = ma + d * w;
      m2 = qa + qb + d * d * (na * w);
    } else {
      mean = 0.f;
      m2 = 0.f;
    }
    n = tot;
  }
  const float rstd = rsqrtf(m2 / n + eps);
  for (int c = g * cg + lane; c < (g + 1) * cg; c += 32) {
    const float sc = gamma[c] * rstd;  // y = x·(γ·rstd) + (β − mean·γ·rstd)
    tab[c] = make_float2(sc, beta[c] - mean * sc);
  }
}

// block (V, R): V = C/8 vector lanes, R pixel rows; grid (chunks in range, B)
// (measured: merging in the last-arriving stats block instead of a finalize launch serialises the
// 32 group merges on one block — 2.1 vs 1.8 ms of GN per 16-row SD-1.5 step; merging redundantly in
// every apply block — partials staged in smem, one launch fewer — costs 2.0-2.3 vs 1.9 ms: the
// per-block merge prologue outweighs the saved launch)
// Two sources (x1 != nullptr): the channels are the concat [x (V0 vectors) | x1 (V − V0 vectors)], each
// source contiguous in its own [B][P][channels] layout — the up-block concat is never materialised.
template <class T>
__device__ __forceinline__ const T* gn_src(const T* x, const T* x1, int V0, int V, int b, int P, int v, int& ld) {
  if (!x1 || v < V0) {
    ld = (x1 ? V0 : V) * 8;
    return x + (long)b * P * ld + v * 8;
  }
  ld = (V - V0) * 8;
  return x1 + (long)b * P * ld + (v - V0) * 8;
}

// partials of one (image b, pixel chunk ch) by one block (V, R); sh = [R][C] sums then [R][C] squares
template <class T>
__device__ __forceinline__ void gn_stats_item(const T* __restrict__ x, const T* __restrict__ x1, int V0, int P, int C,
                                              int G, int chunk_px, int b, int ch, int nch_total,
                                              GNPart* __restrict__ part, float* sh) {
  const int V = blockDim.x, R = blockDim.y;
  const int v = threadIdx.x, ry = threadIdx.y;
  const int p0 = ch * chunk_px, p1 = min(P, p0 + chunk_px);
  float s[8], q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] = q[i] = 0.f;
  int ld;
  const T* xb = gn_src(x, x1, V0, V, b, P, v, ld);
  for (int p = p0 + ry; p < p1; p += 8 * R) {
    // unconditional loads from clamped rows (the compiler keeps all 8 in flight); rows past the
    // chunk are masked out afterwards
    Raw8<T> u[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) u[k].ld(xb + (long)min(p + k * R, p1 - 1) * ld);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (p + k * R < p1) {
        float f[8];
        u[k].get(f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          s[i] += f[i];
          q[i] += f[i] * f[i];
        }
      }
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
  const int tid = ry * V + v, lane = tid & 31, nw = (V * R) >> 5;  // full warps only (V·R ≥ 32)
  const int ne = R * cg;
  for (int g = tid >> 5; g < G && (tid >> 5) < nw; g += nw) {
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

template <class T>
__global__ void __launch_bounds__(512) gn_stats_kernel(const T* __restrict__ x, const T* __restrict__ x1, int V0, int P,
                                                       int C, int G, int chunk_px, int c_base, int nch_total,
                                                       GNPart* __restrict__ part) {
  pdl_wait();
  extern __shared__ float sh[];  // [R][C] sums, then [R][C] sums of squares
  gn_stats_item(x, x1, V0, P, C, G, chunk_px, blockIdx.y, blockIdx.x + c_base, nch_total, part, sh);
}

// finalize: one warp per (image, group)
__global__ void gn_finalize_kernel(int P, int C, int G, int chunk_px, int nchunks, const GNPart* __restrict__ part,
                                   float eps, const float* __restrict__ gamma, const float* __restrict__ beta,
                                   float2* __restrict__ tab) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b = blockIdx.y;
  if (g >= G) return;
  const GNPart* pb = part + (long)b * nchunks * G + g;
  gn_merge_group(
      P, C, G, chunk_px, nchunks, [&](int k) { return __ldcg(reinterpret_cast<const float2*>(pb + (long)k * G)); },
      eps, gamma, beta, tab + (long)b * C, g, lane);
}

// ---- finalize from the producer's epilogue statistics (gemm.cu gn_colstats) --------------------
// part[(b·ns + s)·C_src + c] = (Σy, Σy²) of channel c over the 32 pixels of slot s of image b (ns = P/32
// slots per image). One block of NT threads per (group, image); the group's ns·cg (slot, channel) items
// (cg = C/G) are each the (Σ, Σ²) of 32 values: thread t merges items t, t+NT, … sequentially (Chan et
// al.), then a fixed xor butterfly per warp and one across the warps' results. The order depends only on
// (P, C, G) — NT is a function of them — never on the batch or on banding (I5, I6). Two sources:
// channels [0, C0) from part0 (stride C0), [C0, C) from part1 (stride C − C0) — a group may straddle the
// concat boundary, and the two producers' slots need not cover the same pixels: (Σy, Σy²) are additive
// over any partition of the group's values.
__device__ __forceinline__ void chan_butterfly(float& n, float& mean, float& m2, int lane) {
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
      const float w = __fdividef(nb, tot);
      mean = ma + d * w;
      m2 = qa + qb + d * d * (na * w);
    } else {
      mean = 0.f;
      m2 = 0.f;
    }
    n = tot;
  }
}

__global__ void __launch_bounds__(1024) gn_finalize_cols_kernel(int ns, int C, int C0, int G,
                                                                const float2* __restrict__ part0,
                                                                const float2* __restrict__ part1, float eps,
                                                                const float* __restrict__ gamma,
                                                                const float* __restrict__ beta,
                                                                float2* __restrict__ tab) {
  pdl_wait();
  __shared__ float sh[32][3];
  const int g = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nt = blockDim.x, nw = nt >> 5;
  const int cg = C / G, c0 = g * cg, C1 = C - C0;
  // items i = (slot i / cg, channel c0 + i mod cg): consecutive threads read consecutive channels of a
  // slot; each item is the (Σ, Σ²) of 32 values — its (mean, M2) merged sequentially per thread (Chan
  // et al.), 4 items' loads in flight at a time
  const int items = ns * cg;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  auto ld = [&](int i) {
    const int s = i / cg, c = c0 + (i - s * cg);
    const long row = (long)b * ns + s;
    return c < C0 ? __ldcg(part0 + row * C0 + c) : __ldcg(part1 + row * C1 + (c - C0));
  };
  auto merge = [&](float2 p) {
    const float ms = p.x * (1.f / 32.f);
    const float qs = fmaxf(p.y - p.x * ms, 0.f);
    const float tot = n + 32.f;
    const float d = ms - mean;
    const float w = __fdividef(32.f, tot);
    mean += d * w;
    m2 += qs + d * d * (n * w);
    n = tot;
  };
  int i = tid;
  for (; i + 3 * nt < items; i += 4 * nt) {
    const float2 p0 = ld(i), p1 = ld(i + nt), p2 = ld(i + 2 * nt), p3 = ld(i + 3 * nt);
    merge(p0);
    merge(p1);
    merge(p2);
    merge(p3);
  }
  for (; i < items; i += nt) merge(ld(i));
  chan_butterfly(n, mean, m2, lane);
  if (nw > 1) {
    if (lane == 0) {
      sh[wid][0] = n;
      sh[wid][1] = mean;
      sh[wid][2] = m2;
    }
    __syncthreads();
    if (wid) return;
    n = lane < nw ? sh[lane][0] : 0.f;
    mean = lane < nw ? sh[lane][1] : 0.f;
    m2 = lane < nw ? sh[lane][2] : 0.f;
    chan_butterfly(n, mean, m2, lane);
  }
  const float rstd = rsqrtf(m2 / n + eps);
  float2* tb = tab + (long)b * C;
  for (int c = c0 + lane; c < c0 + cg; c += 32) {
    const float sc = gamma[c] * rstd;
    tb[c] = make_float2(sc, beta[c] - mean * sc);
  }
}

// threads per (group, image) block: ~8 items each, 32 … 1024 (a function of the layer only)
static int gn_cols_threads(int items) { return std::min(1024, std::max(32, (items / 8 + 31) / 32 * 32)); }

// SiLU(x) = x·σ(x) = ½x + ½x·tanh(x/2) on MUFU tanh.approx: absolute error ≤ ½|x|·2^-10.9 — about one
// bf16 ulp for x > 0, but up to ~10 % relative for x ≈ −6 where SiLU is near 0 (bf16 path only; measured
// effect on the SD-1.5 parity tests: none, DESIGN R33; 16-bit outputs only)
__device__ __forceinline__ float silu_tanh(float x) {
  const float hx = 0.5f * x;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(hx));
  return fmaf(hx, t, hx);
}

// apply over pixels [p_begin, p_end) of x viewed as [B·P][V vectors of 8]: block (V, R); thread
// (v, r) always owns channel vector v, so its 8 (scale, shift) pairs stay in registers (reloaded
// only when its pixel crosses into the next image); U pixel rows per thread per iteration, all
// loads issued before any math; grid-stride over blocks of R·U pixels.
template <class T>
__device__ __forceinline__ void gn_apply_dev(const T* __restrict__ x, const T* __restrict__ x1, int V0, long p_begin,
                                             long p_end, int P, int V, const float2* __restrict__ tab, int silu,
                                             T* __restrict__ y) {
  constexpr int U = 4;
  const int v = threadIdx.x, R = blockDim.y;
  // source of this thread's channel vector; pixel p of the flat [B·P] range sits at row p of it
  const bool second = x1 && v >= V0;
  const T* xs = second ? x1 : x;
  const int ldv = x1 ? (second ? V - V0 : V0) : V;  // vectors per pixel row of the source
  const int vs = second ? v - V0 : v;
  int b_cur = -1;
  float sc[8], sf[8];
  for (long pb = p_begin + (long)blockIdx.x * R * U + threadIdx.y; pb < p_end; pb += (long)gridDim.x * R * U) {
    Raw8<T> u[U];
#pragma unroll
    for (int k = 0; k < U; ++k) u[k].ld(xs + (min(pb + (long)k * R, p_end - 1) * ldv + vs) * 8);
    // image of each row without a division per row: one per iteration, then step across image ends
    int b = (int)((unsigned)pb / (unsigned)P);  // < 2^31 pixels (checked on the host)
    long b_end = (long)(b + 1) * P;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long p = pb + (long)k * R;
      if (p >= p_end) break;
      while (p >= b_end) {
        ++b;
        b_end += P;
      }
      if (b != b_cur) {
        const float4* t4 = reinterpret_cast<const float4*>(tab + ((long)b * V + v) * 8);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 t = __ldg(t4 + j);
          sc[2 * j] = t.x, sf[2 * j] = t.y, sc[2 * j + 1] = t.z, sf[2 * j + 1] = t.w;
        }
        b_cur = b;
      }
      float f[8], o[8];
      u[k].get(f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float a = f[j] * sc[j] + sf[j];
        o[j] = silu == 2 ? silu_tanh(a) : silu ? silu_f(a) : a;
      }
      store8(y + (p * V + v) * 8, o);
    }
  }
}

template <class T>
__global__ void __launch_bounds__(512, 2) gn_apply_kernel(const T* __restrict__ x, const T* __restrict__ x1, int V0,
                                                       long p_begin, long p_end, int P, int V,
                                                       const float2* __restrict__ tab, int silu, T* __restrict__ y) {
  pdl_wait();
  gn_apply_dev(x, x1, V0, p_begin, p_end, P, V, tab, silu, y);
}

// TMA-staged apply (single source): the pixel rows [p_begin, p_end) of x are contiguous, so a block moves
// whole chunks of CP rows × C channels with one bulk copy each (cp.async.bulk, mbarrier completion) into a
// 2-deep shared-memory ring, its threads normalise the chunk in place, and one bulk copy stores it back —
// the memory pipeline no longer depends on how many loads each thread keeps in flight (the register-bound
// apply held 4 × 16 B per thread). Thread t keeps channel vector t mod V (its 8 table entries in registers);
// arithmetic identical to gn_apply_dev, so the results are bitwise the same.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

template <class T>
__global__ void __launch_bounds__(512) gn_apply_bulk_kernel(const T* __restrict__ x, const T* __restrict__ x1, int V0,
                                                           long p_begin, long p_end, int P, int V, int CP,
                                                           const float2* __restrict__ tab, int silu,
                                                           T* __restrict__ y) {
  // stage layout: [in0: CP × C0][in1: CP × C1 (two sources)][out: CP × C (two sources; else in place)]
  extern __shared__ __align__(128) uint8_t gsm[];
  const int nt = blockDim.x, tid = threadIdx.x;
  const int C = V * 8, C0 = (x1 ? V0 : V) * 8, C1 = C - C0;
  const long in0_b = (long)CP * C0 * sizeof(T), in1_b = (long)CP * C1 * sizeof(T);
  const long stage_b = in0_b + in1_b + (x1 ? (long)CP * C * sizeof(T) : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + 2 * stage_b);
  const long npix = p_end - p_begin;
  const int nchunks = (int)((npix + CP - 1) / CP);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  auto in0 = [&](int st_) { return reinterpret_cast<T*>(gsm + st_ * stage_b); };
  auto in1 = [&](int st_) { return reinterpret_cast<T*>(gsm + st_ * stage_b + in0_b); };
  auto outb = [&](int st_) { return x1 ? reinterpret_cast<T*>(gsm + st_ * stage_b + in0_b + in1_b) : in0(st_); };
  auto issue = [&](int c, int s) {
    const long q0 = p_begin + (long)c * CP;
    const int n = (int)min((long)CP, p_end - q0);
    mbar_expect_tx(&full[s], (uint32_t)(n * C * sizeof(T)));
    bulk_g2s(in0(s), x + q0 * C0, (uint32_t)(n * C0 * sizeof(T)), &full[s]);
    if (x1) bulk_g2s(in1(s), x1 + q0 * C1, (uint32_t)(n * C1 * sizeof(T)), &full[s]);
  };
  if (tid == 0) {
    if ((int)blockIdx.x < nchunks) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < nchunks) issue(blockIdx.x + gridDim.x, 1);
  }
  const int v = tid % V, r0 = tid / V, rstep = nt / V;  // nt is a multiple of V
  const bool second = x1 && v >= V0;
  int b_cur = -1;
  float sc[8], sf[8];
  int it = 0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int s = it & 1;
    mbar_wait(&full[s], (it >> 1) & 1);
    const long q0 = p_begin + (long)c * CP;
    const int n = (int)min((long)CP, p_end - q0);
    const T* src = second ? in1(s) + (v - V0) * 8 : in0(s) + v * 8;
    const int lds = second ? C1 : C0;
    T* dst = outb(s) + v * 8;
    for (int r = r0; r < n; r += rstep) {
      const long p = q0 + r;
      const int b = (int)((unsigned)p / (unsigned)P);
      if (b != b_cur) {
        const float4* t4 = reinterpret_cast<const float4*>(tab + ((long)b * V + v) * 8);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 t = __ldg(t4 + j);
          sc[2 * j] = t.x, sf[2 * j] = t.y, sc[2 * j + 1] = t.z, sf[2 * j + 1] = t.w;
        }
        b_cur = b;
      }
      float f[8], o[8];
      load8(src + (long)r * lds, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float a = f[j] * sc[j] + sf[j];
        o[j] = silu == 2 ? silu_tanh(a) : silu ? silu_f(a) : a;
      }
      store8(dst + (long)r * C, o);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes → the bulk store
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(y + q0 * C, outb(s), (uint32_t)(n * C * sizeof(T)));
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      const int cn = c + 2 * gridDim.x;
      if (cn < nchunks) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the store has read stage s
        issue(cn, s);
      }
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// GroupNorm in ONE cooperative launch (the whole-tensor path, group_norm / group_norm2): the three
// phases of the three-kernel path, separated by grid-wide barriers instead of kernel boundaries —
//   1. partials of every (image, chunk) item, block-strided (gn_stats_item),
//   2. one warp per (image, group): gn_merge_group → the affine table,
//   3. the apply, grid-stride (gn_apply_dev; x is re-read, mostly from L2).
// Identical arithmetic and reduction order to the three-kernel path (bitwise equal results); 2 launch
// boundaries fewer per GroupNorm. Needs every block co-resident (cooperative launch, grid ≤ occupancy).
template <class T>
__global__ void __launch_bounds__(512) gn_fused_kernel(const T* __restrict__ x, const T* __restrict__ x1, int V0,
                                                       int B, int P, int C, int G, int chunk_px, int nchunks,
                                                       GNPart* __restrict__ part, float2* __restrict__ tab,
                                                       const float* __restrict__ gamma, const float* __restrict__ beta,
                                                       float eps, int silu, T* __restrict__ y) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ float sh[];
  pdl_wait();
  const int items = nchunks * B;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    gn_stats_item(x, x1, V0, P, C, G, chunk_px, it / nchunks, it % nchunks, nchunks, part, sh);
    __syncthreads();  // the shared partial sums are rewritten by the next item
  }
  __threadfence();
  grid.sync();
  {
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, lane = tid & 31;
    const int nwf = (blockDim.x * blockDim.y) >> 5;  // full warps of the block
    if ((tid >> 5) < nwf) {
      for (int pr = blockIdx.x * nwf + (tid >> 5); pr < B * G; pr += gridDim.x * nwf) {
        const int b = pr / G, g = pr % G;
        const GNPart* pb = part + (long)b * nchunks * G + g;
        gn_merge_group(
            P, C, G, chunk_px, nchunks,
            [&](int k) { return __ldcg(reinterpret_cast<const float2*>(pb + (long)k * G)); }, eps, gamma, beta,
            tab + (long)b * C, g, lane);
      }
    }
  }
  __threadfence();
  grid.sync();
  gn_apply_dev(x, x1, V0, 0L, (long)B * P, P, C / 8, tab, silu, y);
}

// workspace: [partials] [affine table]
static size_t gn_part_bytes(int B, int P, int G) {
  return ((size_t)B * cdiv(P, 16) * G * sizeof(GNPart) + 255) & ~size_t(255);
}
size_t gn_workspace_bytes(int B, int P, int G, int C) {
  return gn_part_bytes(B, P, G) + (size_t)B * C * sizeof(float2) + 256;
}
static GNPart* gn_parts(void* ws) { return reinterpret_cast<GNPart*>(ws); }
static float2* gn_tab(void* ws, int B, int P, int G) {
  return reinterpret_cast<float2*>(reinterpret_cast<char*>(ws) + gn_part_bytes(B, P, G));
}

static void gn_finalize(int B, int P, int C, int G, int cp, void* ws, float eps, const float* gamma, const float* beta,
                        cudaStream_t st) {
  const int wpb = 4;  // warps per block
  launch_k(gn_finalize_kernel, dim3(cdiv(G, wpb), B), 32 * wpb, 0, st, P, C, G, cp, cdiv(P, cp), gn_parts(ws), eps, gamma,
                                                                  beta, gn_tab(ws, B, P, G));
  SD_CHECK_LAUNCH();
}

// SiLU form of the apply: 0 none, 1 ex2 + rcp, 2 one MUFU tanh (bf16 only; SD_SILU_TANH=0 disables)
template <class T>
static int gn_silu_mode(bool silu) {
  static int st_env = -1;
  if (st_env < 0) {
    const char* e = getenv("SD_SILU_TANH");
    st_env = e ? atoi(e) : 1;
  }
  // 16-bit outputs (bf16 and fp16): one MUFU tanh; fp32 (the 1e-4 parity mode): ex2 + rcp. For fp16 the
  // measured SD-scale errors are unchanged (per-row ε 1.18e-3, images 2.38e-3 with either form) and GN per
  // bench step drops 98 → 92 ms
  return !silu ? 0 : (!std::is_same<T, float>::value && st_env) ? 2 : 1;
}

// SD_GN_FUSED=1: the single cooperative launch for whole tensors. Off by default — measured slower than the
// three launches it replaces (B200: [16, 4096, 320] 49 vs 35 µs, [16, 256, 1280] 24 vs 16 µs; GN per bench
// step 133 vs 99 ms): the two grid-wide barriers of a co-resident grid cost more than two launch gaps
// inside a CUDA graph with programmatic dependent launch, and the co-residency limit caps its grid
static bool gn_fused_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_GN_FUSED");
    v = e && e[0] == '1';
  }
  return v != 0;
}

template <class T>
static void gn_fused(const T* x, const T* x1, int C0, T* y, int B, int P, int C, int G, int cp, void* ws,
                     const float* gamma, const float* beta, float eps, bool silu, cudaStream_t st) {
  const dim3 blk = gn_stats_block(C);
  const size_t sh = (size_t)blk.x * blk.y * 8 * 2 * sizeof(float);
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> occ;  // (block threads, smem) → co-resident blocks per SM
  int per_sm;
  {
    std::lock_guard<std::mutex> g(mu);
    auto key = std::make_pair((int)(blk.x * blk.y), (int)sh);
    auto it = occ.find(key);
    if (it == occ.end()) {
      int n = 0;
      SD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gn_fused_kernel<T>, blk.x * blk.y, sh));
      it = occ.emplace(key, std::max(n, 1)).first;
    }
    per_sm = it->second;
  }
  const int sms = stream_sms(st);  // cooperative: every block co-resident on the stream's SMs
  const int nchunks = cdiv(P, cp);
  const long rows = (long)blk.y * 4;
  const long want = std::max<long>((long)nchunks * B, ((long)B * P + rows - 1) / rows);
  const int grid = (int)std::min<long>(want, (long)sms * per_sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = blk;
  cfg.dynamicSmemBytes = sh;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SD_CUDA(cudaLaunchKernelEx(&cfg, gn_fused_kernel<T>, x, x1, C0 / 8, B, P, C, G, cp, nchunks, gn_parts(ws),
                             gn_tab(ws, B, P, G), gamma, beta, eps, gn_silu_mode<T>(silu), y));
  SD_CHECK_LAUNCH();
}

// SD_GN_BULK=0: the register-pipelined apply for single-source tensors too
static bool gn_bulk_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_GN_BULK");
    v = !(e && e[0] == '0');
  }
  return v != 0;
}

template <class T>
static void gn_apply(const T* x, const T* x1, int C0, T* y, long p0, long p1, int B, int P, int C, const float2* tab,
                     bool silu, cudaStream_t st) {
  if (p1 <= p0) return;
  if (p1 >= (1L << 31)) throw CudaError("group_norm: tensor too large");
  if (gn_bulk_on() && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                        reinterpret_cast<uintptr_t>(x1)) & 15) == 0) {
    const int V = C / 8;
    const int k = std::max(1, 256 / V);        // pixel rows per pass; threads = V·k (≤ 512)
    const int nt = V * k;
    const long row_bytes = (long)C * sizeof(T) * (x1 ? 2 : 1);  // two sources: in0 | in1 | out per row
    static long stage_kb = -1;  // SD_GN_CHUNK_KB: stage size (experiments)
    if (stage_kb < 0) {
      const char* e = getenv("SD_GN_CHUNK_KB");
      stage_kb = e ? std::max(4, atoi(e)) : 24;
    }
    int CP = (int)std::max<long>(k, (stage_kb * 1024 / row_bytes) / k * k);  // ~24 KB stages, whole passes
    const size_t smem = 2 * (size_t)CP * row_bytes + 64;
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, int> occ;
    int per_sm;
    {
      std::lock_guard<std::mutex> g(mu);
      auto key = std::make_pair(nt, smem);
      auto it = occ.find(key);
      if (it == occ.end()) {
        if (smem > 48 * 1024)
          SD_CUDA(cudaFuncSetAttribute(gn_apply_bulk_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int n = 0;
        SD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gn_apply_bulk_kernel<T>, nt, smem));
        it = occ.emplace(key, std::max(n, 1)).first;
      }
      per_sm = it->second;
    }
    static int sms = 0;
    if (!sms) SD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long nchunks = (p1 - p0 + CP - 1) / CP;
    const int grid = (int)std::min<long>(nchunks, (long)sms * per_sm);
    launch_k(gn_apply_bulk_kernel<T>, grid, nt, smem, st, x, x1, C0 / 8, p0, p1, P, V, CP, tab, gn_silu_mode<T>(silu),
             y);
    SD_CHECK_LAUNCH();
    (void)B;
    return;
  }
  const dim3 blk = gn_stats_block(C);
  const long rows = (long)blk.y * 4;
  static int sms = 0;
  if (!sms) SD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // resident blocks per SM of this block shape (registers bound it: ncu showed 2 of the assumed 8 blocks
  // of 240 threads at 85 registers — 16 warps per SM; ≤ 64 registers now)
  static std::mutex mu;
  static std::map<int, int> occ;
  int per_sm;
  {
    std::lock_guard<std::mutex> g(mu);
    const int nt = (int)(blk.x * blk.y);
    auto it = occ.find(nt);
    if (it == occ.end()) {
      int n = 0;
      SD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gn_apply_kernel<T>, nt, 0));
      it = occ.emplace(nt, std::max(n, 1)).first;
    }
    per_sm = it->second;
  }
  const long want = (p1 - p0 + rows - 1) / rows;
  const int grid = (int)std::min<long>(want, (long)sms * per_sm);
  // 16-bit outputs: SiLU through one MUFU tanh instead of ex2 + rcp (the apply pass was partly
  // MUFU-bound: 2 MUFU ops per element); fp32 outputs keep the exact form.
  const int sm = gn_silu_mode<T>(silu);
  launch_k(gn_apply_kernel<T>, grid, blk, 0, st, x, x1, C0 / 8, p0, p1, P, C / 8, tab, sm, y);
  SD_CHECK_LAUNCH();
  (void)B;
}

static void check_gn(int C, int G) {
  if (C % 8 || C / 8 > 512 || G > 64 || C % G) throw CudaError("group_norm: unsupported C/G");
}

template <class T>
static void gn_stats(const T* x, const T* x1, int C0, int B, int P, int C, int G, int c0, int c1, void* ws,
                     cudaStream_t st) {
  const int cp = gn_chunk_px(C);
  const dim3 blk = gn_stats_block(C);
  const size_t sh = (size_t)blk.x * blk.y * 8 * 2 * sizeof(float);
  launch_k(gn_stats_kernel<T>, dim3(c1 - c0, B), blk, sh, st, x, x1, C0 / 8, P, C, G, cp, c0, cdiv(P, cp), gn_parts(ws));
  SD_CHECK_LAUNCH();
}

// band-restricted halves of group_norm (B = 1) over pixels [p0, p1) (multiples of 128): stats of the
// chunks in the range; normalisation of the pixels in the range with ALL chunk partials merged in
// fixed order — a banded GN is bitwise equal to the whole-tensor GN (R7 V1).
template <class T>
void gn_stats_range(const T* x, int P, int C, int G, int p0, int p1, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const int cp = gn_chunk_px(C);
  gn_stats(x, (const T*)nullptr, C, 1, P, C, G, p0 / cp, cdiv(p1, cp), ws, st);
}
template <class T>
void gn_apply_range(const T* x, T* y, int P, int C, int G, int p0, int p1, const float* gamma, const float* beta,
                    float eps, bool silu, void* ws, cudaStream_t st) {
  check_gn(C, G);
  const int cp = gn_chunk_px(C);
  if (p0 == 0) gn_finalize(1, P, C, G, cp, ws, eps, gamma, beta, st);  // bands run in order
  gn_apply(x, (const T*)nullptr, C, y, p0, p1, 1, P, C, gn_tab(ws, 1, P, G), silu, st);
}

template <class T>
void group_norm(const T* x, T* y, int B, int P, int C, int G, const float* gamma, const float* beta, float eps,
                bool silu, void* ws, cudaStream_t st) {
  group_norm2(x, C, (const T*)nullptr, 0, y, B, P, G, gamma, beta, eps, silu, ws, st);
}

template <class T>
void group_norm2(const T* x0, int C0, const T* x1, int C1, T* y, int B, int P, int G, const float* gamma,
                 const float* beta, float eps, bool silu, void* ws, cudaStream_t st) {
  const int C = C0 + C1;
  check_gn(C, G);
  if (x1 && (C0 % 8 || C1 % 8)) throw CudaError("group_norm2: source channels must be multiples of 8");
  const int cp = gn_chunk_px(C);
  if (gn_fused_on() && (long)B * P < (1L << 31)) {
    gn_fused(x0, x1, C0, y, B, P, C, G, cp, ws, gamma, beta, eps, silu, st);
    return;
  }
  gn_stats(x0, x1, C0, B, P, C, G, 0, cdiv(P, cp), ws, st);
  gn_finalize(B, P, C, G, cp, ws, eps, gamma, beta, st);
  gn_apply(x0, x1, C0, y, 0, (long)B * P, B, P, C, gn_tab(ws, B, P, G), silu, st);
}

static void gn_finalize_cols(int B, int P, int C0, const float2* part0, int C1, const float2* part1, int G, void* ws,
                             float eps, const float* gamma, const float* beta, cudaStream_t st) {
  const int C = C0 + C1;
  check_gn(C, G);
  if (P % 32) throw CudaError("group_norm_parts: P must be a multiple of 32");
  const int ns = P / 32;
  launch_k(gn_finalize_cols_kernel, dim3(G, B), gn_cols_threads(ns * (C / G)), 0, st, ns, C, C0, G, part0, part1, eps, gamma,
           beta, gn_tab(ws, B, P, G));
  SD_CHECK_LAUNCH();
}

template <class T>
void group_norm_parts(const T* x0, int C0, const float2* part0, const T* x1, int C1, const float2* part1, T* y, int B,
                      int P, int G, const float* gamma, const float* beta, float eps, bool silu, void* ws,
                      cudaStream_t st) {
  if (x1 && (C0 % 8 || C1 % 8)) throw CudaError("group_norm_parts: source channels must be multiples of 8");
  gn_finalize_cols(B, P, C0, part0, x1 ? C1 : 0, part1, G, ws, eps, gamma, beta, st);
  gn_apply(x0, x1, C0, y, 0, (long)B * P, B, P, C0 + (x1 ? C1 : 0), gn_tab(ws, B, P, G), silu, st);
}

template <class T>
void gn_apply_range_parts(const T* x, T* y, int P, int C, int G, int p0, int p1, const float2* part, const float* gamma,
                          const float* beta, float eps, bool silu, void* ws, cudaStream_t st) {
  if (p0 == 0) gn_finalize_cols(1, P, C, part, 0, nullptr, G, ws, eps, gamma, beta, st);  // bands run in order
  gn_apply(x, (const T*)nullptr, C, y, p0, p1, 1, P, C, gn_tab(ws, 1, P, G), silu, st);
}

// ---- LayerNorm: LANES lanes per token (NV 16-byte vectors each), two-pass in registers ----------
// C = 320/640/1280 → 8/16/32 lanes × 5 vectors: every lane issues all its loads up front and a warp
// serves 4/2/1 tokens, so the per-token reduction is short and the loads are balanced.
template <int NV, int LANES, class E>
__global__ void layer_norm_kernel(const E* __restrict__ x, int T, int C, const float* __restrict__ gamma,
                                  const float* __restrict__ beta, float eps, E* __restrict__ y) {
  pdl_wait();
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
  launch_k(layer_norm_kernel<NV, LANES, E>, cdiv(total, threads), threads, 0, st, x, T, C, g, b, eps, y);
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

// ---- LayerNorm folded into its consumer GEMMs (the algebraic form; gemm.cu ln_stat epilogue) ----------
// LN(h)·Wᵀ + b = rstd_m·(h·W′ᵀ − μ_m·w̄) + b′ with W′ = W·diag(γ), w̄_n = Σ_k W′_nk, b′ = b + W·β: the GEMM reads
// the raw hidden state h and its epilogue applies (μ_m, rstd_m) per row (or per column when h is the B
// operand, the Vᵀ projection). ln_stats: the same two-pass register arithmetic as layer_norm_kernel, only
// the per-token (μ, rstd) written (8 bytes per token instead of the normalised row).
template <int NV, int LANES, class E>
__global__ void ln_stats_kernel(const E* __restrict__ x, int T, int C, float eps, float2* __restrict__ st) {
  pdl_wait();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int tok = gtid / LANES, l = gtid % LANES;
  if (tok >= T) return;
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
  if (l == 0) st[tok] = make_float2(mean, rsqrtf(q / C + eps));
}

template <int NV, int LANES, class E>
static void lns_launch(const E* x, int T, int C, float eps, float2* st, cudaStream_t s) {
  const long total = (long)T * LANES;
  launch_k(ln_stats_kernel<NV, LANES, E>, cdiv(total, 256), 256, 0, s, x, T, C, eps, st);
  SD_CHECK_LAUNCH();
}

template <class E>
void ln_stats(const E* x, int T, int C, float eps, float2* st, cudaStream_t s) {
  if (C % 8) throw CudaError("ln_stats: C % 8");
  const int V = C / 8;
  if (V == 40) return lns_launch<5, 8>(x, T, C, eps, st, s);
  if (V == 80) return lns_launch<5, 16>(x, T, C, eps, st, s);
  if (V == 160) return lns_launch<5, 32>(x, T, C, eps, st, s);
  if (V <= 4) return lns_launch<1, 4>(x, T, C, eps, st, s);
  if (V <= 8) return lns_launch<1, 8>(x, T, C, eps, st, s);
  if (V <= 16) return lns_launch<1, 16>(x, T, C, eps, st, s);
  if (V <= 32) return lns_launch<1, 32>(x, T, C, eps, st, s);
  if (V <= 64) return lns_launch<2, 32>(x, T, C, eps, st, s);
  if (V <= 128) return lns_launch<4, 32>(x, T, C, eps, st, s);
  if (V <= 256) return lns_launch<8, 32>(x, T, C, eps, st, s);
  throw CudaError("ln_stats: C too large");
}

// one warp per weight row n: W′[n][k] = 16-bit(W[n][k]·γ[k]); w̄[n] = Σ_k W′[n][k] (of the rounded values the
// MMA multiplies, so the μ term cancels exactly up to fp32 accumulation); b′[n] = b[n] + Σ_k W[n][k]·β[k].
// Fixed lane-strided order and xor butterfly: deterministic.
template <class E>
__global__ void ln_fold_kernel(const E* __restrict__ W, int N, int K, const float* __restrict__ gamma,
                               const float* __restrict__ beta, const float* __restrict__ bias, E* __restrict__ Wf,
                               float* __restrict__ wbar, float* __restrict__ bf) {
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (n >= N) return;
  const E* wr = W + (long)n * K;
  E* fr = Wf + (long)n * K;
  float sw = 0.f, sb = 0.f;
  for (int k = lane; k < K; k += 32) {
    const float w = act_ld(wr + k);
    E wf;
    act_st(&wf, w * gamma[k]);
    fr[k] = wf;
    sw += act_ld(&wf);
    sb = fmaf(w, beta[k], sb);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sw += __shfl_xor_sync(0xffffffff, sw, o);
    sb += __shfl_xor_sync(0xffffffff, sb, o);
  }
  if (lane == 0) {
    wbar[n] = sw;
    bf[n] = (bias ? bias[n] : 0.f) + sb;
  }
}

template <class E>
void ln_fold(const E* W, int N, int K, const float* gamma, const float* beta, const float* bias, E* Wf, float* wbar,
             float* bf, cudaStream_t s) {
  launch_k(ln_fold_kernel<E>, cdiv(N, 8), 256, 0, s, W, N, K, gamma, beta, bias, Wf, wbar, bf);
  SD_CHECK_LAUNCH();
}

#define SD_NORM_INST(T)                                                                                      \
  template void group_norm<T>(const T*, T*, int, int, int, int, const float*, const float*, float, bool, void*, \
                              cudaStream_t);                                                                 \
  template void gn_stats_range<T>(const T*, int, int, int, int, int, void*, cudaStream_t);                   \
  template void gn_apply_range<T>(const T*, T*, int, int, int, int, int, const float*, const float*, float, bool, \
                                  void*, cudaStream_t);                                                      \
  template void layer_norm<T>(const T*, T*, int, int, const float*, const float*, float, cudaStream_t);   \
  template void group_norm2<T>(const T*, int, const T*, int, T*, int, int, int, const float*, const float*, float, \
                               bool, void*, cudaStream_t);                                                   \
  template void ln_stats<T>(const T*, int, int, float, float2*, cudaStream_t);                               \
  template void ln_fold<T>(const T*, int, int, const float*, const float*, const float*, T*, float*, float*,  \
                           cudaStream_t);                                                                    \
  template void group_norm_parts<T>(const T*, int, const float2*, const T*, int, const float2*, T*, int, int, int, \
                                    const float*, const float*, float, bool, void*, cudaStream_t);           \
  template void gn_apply_range_parts<T>(const T*, T*, int, int, int, int, int, const float2*, const float*,     \
                                        const float*, float, bool, void*, cudaStream_t);
SD_NORM_INST(bf16)
SD_NORM_INST(f16)
SD_NORM_INST(float)

}  // namespace sd
