// Fused multi-head attention O = softmax(Q Kᵀ / √d) V (SURVEY.md §2.4 K6 self-attention, K7
// cross-attention to the cached text K/V). Flash-style: the L×L score matrix never leaves the SM;
// running row max / row sum in fp32 (R28); exp2 with the log2(e)/√d scale folded in.
//
// Round-1 implementation: bf16 mma.sync.m16n8k16 tensor-core tiles (4 warps × 16 query rows,
// 64-key tiles, cp.async double buffering, ldmatrix fragments). The tcgen05/TMEM version (S and O
// in TMEM, softmax warps, polynomial exp2 offload) is the planned replacement — see DESIGN.md.
#include <float.h>

#include <stdlib.h>

#include <algorithm>

#include <string.h>

#include "common.cuh"
#include "kernels_ew.h"

namespace sd {

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  const uint32_t d = smem_u32(dst);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
template <bool F16>  // fp16 operands (SD_PREC_FP16) or bf16
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  if (F16)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int D>  // padded head dim (multiple of 16)
struct AttnSmem {
  static constexpr int BM = 64, BN = 64, LD = D + 8;  // +16 B row pad against bank conflicts
  static constexpr int Q_ELEMS = BM * LD, KV_ELEMS = BN * LD;
  static constexpr int BYTES = (Q_ELEMS + 4 * KV_ELEMS) * 2;
};

template <int D, bool F16>
__global__ void __launch_bounds__(128) attn_kernel(const AttnDesc a, float scale_log2) {
  pdl_wait();
  using S = AttnSmem<D>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sK = sQ + S::Q_ELEMS;           // [2][BN][LD]
  bf16* sV = sK + 2 * S::KV_ELEMS;      // [2][BN][LD]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qt = blockIdx.x, head = blockIdx.y, row = blockIdx.z;
  const int d = a.d;
  const int q0 = qt * S::BM;
  const int kvb = a.kv_index ? a.kv_index[row] : row;
  const bf16* Qg = a.Q + (long)row * a.q_bstride + (long)head * d;
  const bf16* Kg = a.K + (long)kvb * a.kv_bstride + (long)head * d;
  const bf16* Vg = a.V + (long)kvb * a.kv_bstride + (long)head * d;
  const int nchunk = d / 8;  // 16-byte chunks per row (d multiple of 8)

  // zero the pad columns [d, D) of every tile (never written by cp.async)
  if (d < D) {
    for (int i = tid; i < (S::BM + 4 * S::BN) * (D - d); i += 128) {
      const int r = i / (D - d), c = d + i % (D - d);
      sQ[r * S::LD + c] = __float2bfloat16(0.f);
    }
  }
  // Q tile
  for (int i = tid; i < S::BM * nchunk; i += 128) {
    const int r = i / nchunk, c = (i % nchunk) * 8;
    const bool ok = q0 + r < a.Lq;
    cp_async16(sQ + r * S::LD + c, Qg + (long)(ok ? q0 + r : 0) * a.ldq + c, ok);
  }
  auto load_kv = [&](int tile, int buf) {
    const int k0 = tile * S::BN;
    bf16* dk = sK + buf * S::KV_ELEMS;
    bf16* dv = sV + buf * S::KV_ELEMS;
    for (int i = tid; i < S::BN * nchunk; i += 128) {
      const int r = i / nchunk, c = (i % nchunk) * 8;
      const bool ok = k0 + r < a.Lk;
      const long off = (long)(ok ? k0 + r : 0) * a.ldk + c;
      cp_async16(dk + r * S::LD + c, Kg + off, ok);
      cp_async16(dv + r * S::LD + c, Vg + off, ok);
    }
  };
  const int ntiles = (a.Lk + S::BN - 1) / S::BN;
  load_kv(0, 0);
  cp_async_commit();

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-FLT_MAX, -FLT_MAX}, lrow[2] = {0.f, 0.f};
  const int g = lane >> 2, t4 = lane & 3;

  for (int j = 0; j < ntiles; ++j) {
    if (j + 1 < ntiles) load_kv(j + 1, (j + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const bf16* cK = sK + (j & 1) * S::KV_ELEMS;
    const bf16* cV = sV + (j & 1) * S::KV_ELEMS;
    // ---- S = Q Kᵀ (16 rows × 64 keys per warp) ----
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(smem_u32(sQ + (warp * 16 + (lane & 15)) * S::LD + kk * 16 + (lane >> 4) * 8), a0, a1, a2, a3);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b0, b1, b2, b3;
        const int key = np * 16 + (lane >> 4) * 8 + (lane & 7);
        const int col = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(smem_u32(cK + key * S::LD + col), b0, b1, b2, b3);
        mma16816<F16>(s[2 * np], a0, a1, a2, a3, b0, b1);
        mma16816<F16>(s[2 * np + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // mask keys beyond Lk
    const int kbase = j * S::BN;
    if (kbase + S::BN > a.Lk) {
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const int c0 = kbase + n * 8 + 2 * t4;
        if (c0 >= a.Lk) s[n][0] = s[n][2] = -FLT_MAX;
        if (c0 + 1 >= a.Lk) s[n][1] = s[n][3] = -FLT_MAX;
      }
    }
    // ---- online softmax (rows g and g+8) ----
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      mx[0] = fmaxf(mx[0], fmaxf(s[n][0], s[n][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[n][2], s[n][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      corr[r] = exp2f((mrow[r] - mx[r]) * scale_log2);
      mrow[r] = mx[r];
    }
    const float ms0 = mx[0] * scale_log2, ms1 = mx[1] * scale_log2;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      s[n][0] = exp2f(s[n][0] * scale_log2 - ms0);
      s[n][1] = exp2f(s[n][1] * scale_log2 - ms0);
      s[n][2] = exp2f(s[n][2] * scale_log2 - ms1);
      s[n][3] = exp2f(s[n][3] * scale_log2 - ms1);
      rs[0] += s[n][0] + s[n][1];
      rs[1] += s[n][2] + s[n][3];
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) lrow[r] = lrow[r] * corr[r] + rs[r];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // ---- O += P V ----
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // 16 keys per step
      const uint32_t p0 = pack16(s[2 * kk][0], s[2 * kk][1], F16);
      const uint32_t p1 = pack16(s[2 * kk][2], s[2 * kk][3], F16);
      const uint32_t p2 = pack16(s[2 * kk + 1][0], s[2 * kk + 1][1], F16);
      const uint32_t p3 = pack16(s[2 * kk + 1][2], s[2 * kk + 1][3], F16);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = dp * 16 + (lane >> 4) * 8;
        ldsm_x4_t(smem_u32(cV + key * S::LD + col), b0, b1, b2, b3);
        mma16816<F16>(o[2 * dp], p0, p1, p2, p3, b0, b1);
        mma16816<F16>(o[2 * dp + 1], p0, p1, p2, p3, b2, b3);
      }
    }
    __syncthreads();
  }
  // ---- finalize ----
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffff, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffff, lrow[r], 2);
  }
  const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
  bf16* Og = a.O + (long)row * a.o_bstride + (long)head * d;
  const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    const int c = i * 8 + 2 * t4;
    if (c < d) {
      if (r0 < a.Lq)
        *reinterpret_cast<uint32_t*>(Og + (long)r0 * a.ldo + c) = pack16(o[i][0] * inv0, o[i][1] * inv0, F16);
      if (r1 < a.Lq)
        *reinterpret_cast<uint32_t*>(Og + (long)r1 * a.ldo + c) = pack16(o[i][2] * inv1, o[i][3] * inv1, F16);
    }
  }
}

// ---- short-context attention (cross-attention to the ≤ 80 cached text tokens, R28) -------------
// All keys fit one tile, so the softmax is exact in one pass (no running max / rescale), and a block
// keeps its (row, head)'s K and V resident in shared memory while it walks QT query tiles of 64
// (Q double-buffered with cp.async): K/V are read once per block instead of once per 64 queries,
// and no MMA is spent on a second, mostly masked key tile. NW warps × 16 query rows, mma.sync.
template <int D, int LKP, int NW>  // padded head dim, padded key count (multiples of 16); warps per block
struct XAttnSmem {
  static constexpr int BM = 16 * NW, LD = D + 8;
  static constexpr int Q_ELEMS = BM * LD, KV_ELEMS = LKP * LD;
  static constexpr int BYTES = (2 * Q_ELEMS + 2 * KV_ELEMS) * 2;
};

template <int D, int LKP, int NW, bool F16>
__global__ void __launch_bounds__(32 * NW) xattn_kernel(const AttnDesc a, float scale_log2, int qt_per_block) {
  pdl_wait();
  using S = XAttnSmem<D, LKP, NW>;
  constexpr int NT = 32 * NW;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);  // [2][BM][LD]
  bf16* sK = sQ + 2 * S::Q_ELEMS;                // [LKP][LD]
  bf16* sV = sK + S::KV_ELEMS;                   // [LKP][LD]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int head = blockIdx.y, row = blockIdx.z;
  const int d = a.d;
  const int kvb = a.kv_index ? a.kv_index[row] : row;
  const bf16* Qg = a.Q + (long)row * a.q_bstride + (long)head * d;
  const bf16* Kg = a.K + (long)kvb * a.kv_bstride + (long)head * d;
  const bf16* Vg = a.V + (long)kvb * a.kv_bstride + (long)head * d;
  const int nchunk = d / 8;
  const int t_begin = blockIdx.x * qt_per_block;
  const int t_end = min(t_begin + qt_per_block, (a.Lq + S::BM - 1) / S::BM);
  if (t_begin >= t_end) return;
  // zero the pad columns [d, D) of every buffer (never written by cp.async)
  if (d < D)
    for (int i = tid; i < (2 * S::BM + 2 * LKP) * (D - d); i += NT) {
      const int r = i / (D - d), c = d + i % (D - d);
      sQ[r * S::LD + c] = __float2bfloat16(0.f);
    }
  for (int i = tid; i < LKP * nchunk; i += NT) {  // K and V once; keys ≥ Lk zero-filled
    const int r = i / nchunk, c = (i % nchunk) * 8;
    const bool ok = r < a.Lk;
    const long off = (long)(ok ? r : 0) * a.ldk + c;
    cp_async16(sK + r * S::LD + c, Kg + off, ok);
    cp_async16(sV + r * S::LD + c, Vg + off, ok);
  }
  auto load_q = [&](int t, int buf) {
    const int q0 = t * S::BM;
    bf16* dq = sQ + buf * S::Q_ELEMS;
    for (int i = tid; i < S::BM * nchunk; i += NT) {
      const int r = i / nchunk, c = (i % nchunk) * 8;
      const bool ok = q0 + r < a.Lq;
      cp_async16(dq + r * S::LD + c, Qg + (long)(ok ? q0 + r : 0) * a.ldq + c, ok);
    }
  };
  load_q(t_begin, 0);
  cp_async_commit();
  const int g = lane >> 2, t4 = lane & 3;
  bf16* Og = a.O + (long)row * a.o_bstride + (long)head * d;
  for (int t = t_begin; t < t_end; ++t) {
    const int buf = (t - t_begin) & 1;
    if (t + 1 < t_end) load_q(t + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const bf16* cQ = sQ + buf * S::Q_ELEMS;
    // ---- S = Q Kᵀ: 16 rows × LKP keys per warp ----
    float s[LKP / 8][4];
#pragma unroll
    for (int n = 0; n < LKP / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(smem_u32(cQ + (warp * 16 + (lane & 15)) * S::LD + kk * 16 + (lane >> 4) * 8), a0, a1, a2, a3);
#pragma unroll
      for (int np = 0; np < LKP / 16; ++np) {
        uint32_t b0, b1, b2, b3;
        const int key = np * 16 + (lane >> 4) * 8 + (lane & 7);
        const int col = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(smem_u32(sK + key * S::LD + col), b0, b1, b2, b3);
        mma16816<F16>(s[2 * np], a0, a1, a2, a3, b0, b1);
        mma16816<F16>(s[2 * np + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // ---- exact softmax over the (masked) keys, rows g and g + 8 ----
    float mx[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
    for (int n = 0; n < LKP / 8; ++n) {
      const int c0 = n * 8 + 2 * t4;
      if (c0 >= a.Lk) s[n][0] = s[n][2] = -FLT_MAX;
      if (c0 + 1 >= a.Lk) s[n][1] = s[n][3] = -FLT_MAX;
      mx[0] = fmaxf(mx[0], fmaxf(s[n][0], s[n][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[n][2], s[n][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
    }
    const float ms0 = mx[0] * scale_log2, ms1 = mx[1] * scale_log2;
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int n = 0; n < LKP / 8; ++n) {
      s[n][0] = exp2f(s[n][0] * scale_log2 - ms0);
      s[n][1] = exp2f(s[n][1] * scale_log2 - ms0);
      s[n][2] = exp2f(s[n][2] * scale_log2 - ms1);
      s[n][3] = exp2f(s[n][3] * scale_log2 - ms1);
      rs[0] += s[n][0] + s[n][1];
      rs[1] += s[n][2] + s[n][3];
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffff, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffff, rs[r], 2);
    }
    // ---- O = P V ----
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < LKP / 16; ++kk) {
      const uint32_t p0 = pack16(s[2 * kk][0], s[2 * kk][1], F16);
      const uint32_t p1 = pack16(s[2 * kk][2], s[2 * kk][3], F16);
      const uint32_t p2 = pack16(s[2 * kk + 1][0], s[2 * kk + 1][1], F16);
      const uint32_t p3 = pack16(s[2 * kk + 1][2], s[2 * kk + 1][3], F16);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = dp * 16 + (lane >> 4) * 8;
        ldsm_x4_t(smem_u32(sV + key * S::LD + col), b0, b1, b2, b3);
        mma16816<F16>(o[2 * dp], p0, p1, p2, p3, b0, b1);
        mma16816<F16>(o[2 * dp + 1], p0, p1, p2, p3, b2, b3);
      }
    }
    const float inv0 = 1.f / rs[0], inv1 = 1.f / rs[1];
    const int r0 = t * S::BM + warp * 16 + g, r1 = r0 + 8;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int c = i * 8 + 2 * t4;
      if (c < d) {
        if (r0 < a.Lq)
          *reinterpret_cast<uint32_t*>(Og + (long)r0 * a.ldo + c) = pack16(o[i][0] * inv0, o[i][1] * inv0, F16);
        if (r1 < a.Lq)
          *reinterpret_cast<uint32_t*>(Og + (long)r1 * a.ldo + c) = pack16(o[i][2] * inv1, o[i][3] * inv1, F16);
      }
    }
    __syncthreads();  // the buffer of tile t is refilled by the next iteration's prefetch
  }
}

template <int D, int LKP, int NW, bool F16>
static void launch_xattn(const AttnDesc& a, cudaStream_t st) {
  using S = XAttnSmem<D, LKP, NW>;
  static bool set = false;
  if (!set) {
    SD_CUDA(cudaFuncSetAttribute(xattn_kernel<D, LKP, NW, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::BYTES));
    set = true;
  }
  const int tiles = cdiv(a.Lq, S::BM);
  // enough blocks for ~4 waves of 148 SMs, each walking a contiguous run of query tiles
  const long pairs = (long)a.rows * a.heads;
  int per = (int)std::max<long>(1, (long)tiles * pairs / (148L * 16));
  per = std::min(per, 16);
  dim3 grid(cdiv(tiles, per), a.heads, a.rows);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)a.d);
  launch_k(xattn_kernel<D, LKP, NW, F16>, grid, 32 * NW, S::BYTES, st, a, scale_log2, per);
  SD_CHECK_LAUNCH();
}

template <int D, bool F16>
static void launch_attn(const AttnDesc& a, cudaStream_t st) {
  using S = AttnSmem<D>;
  static bool set = false;
  if (!set) {
    SD_CUDA(cudaFuncSetAttribute(attn_kernel<D, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::BYTES));
    set = true;
  }
  dim3 grid(cdiv(a.Lq, S::BM), a.heads, a.rows);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)a.d);
  launch_k(attn_kernel<D, F16>, grid, 128, S::BYTES, st, a, scale_log2);
  SD_CHECK_LAUNCH();
}

template <bool F16>
static void attention16(const AttnDesc& a, cudaStream_t st) {
  if (a.d % 8 || (a.ldq | a.ldk | a.ldo) % 8) throw CudaError("attention: d and strides must be multiples of 8");
  static int nw = -1;  // SD_XATTN_NW=4|8: warps per short-context block (4: kbench r01, 53 vs 75 µs at 64²)
  if (nw < 0) {
    const char* e = getenv("SD_XATTN_NW");
    nw = e && atoi(e) == 8 ? 8 : 4;
  }
  if (a.Lk <= 16 || (a.Lk <= 80 && a.d > 16)) {  // short context (the cached text tokens): one key tile
#define SD_XA(D_, L_) return nw == 4 ? launch_xattn<D_, L_, 4, F16>(a, st) : launch_xattn<D_, L_, 8, F16>(a, st)
    if (a.Lk <= 16) {
      if (a.d <= 16) SD_XA(16, 16);
      if (a.d <= 32) SD_XA(32, 16);
    } else {
      if (a.d <= 48) SD_XA(48, 80);
      if (a.d <= 64) SD_XA(64, 80);
      if (a.d <= 80) SD_XA(80, 80);
      if (a.d <= 160) SD_XA(160, 80);
    }
#undef SD_XA
  }
  if (a.d <= 16) launch_attn<16, F16>(a, st);
  else if (a.d <= 32) launch_attn<32, F16>(a, st);
  else if (a.d <= 48) launch_attn<48, F16>(a, st);
  else if (a.d <= 64) launch_attn<64, F16>(a, st);
  else if (a.d <= 80) launch_attn<80, F16>(a, st);
  else if (a.d <= 128) launch_attn<128, F16>(a, st);
  else if (a.d <= 160) launch_attn<160, F16>(a, st);
  else throw CudaError("attention: head dim > 160 uses the GEMM path");
}

void attention(const AttnDesc& a, cudaStream_t st) { attention16<false>(a, st); }
void attention(const AttnDescT<f16>& a, cudaStream_t st) {
  static_assert(sizeof(AttnDescT<f16>) == sizeof(AttnDesc), "AttnDescT layouts must match");
  AttnDesc b;
  memcpy(static_cast<void*>(&b), static_cast<const void*>(&a), sizeof(b));
  attention16<true>(b, st);
}

// ---- row softmax (VAE single-head attention, d = 512, via GEMMs) ------------------------------
__global__ void softmax_rows_kernel(const float* __restrict__ S, bf16* __restrict__ P, int cols, int is_f16) {
  pdl_wait();
  const long r = blockIdx.x;
  const float* s = S + r * cols;
  __shared__ float red[32];
  float m = -FLT_MAX;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) m = fmaxf(m, s[c]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -FLT_MAX;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) sum += __expf(s[c] - m);
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffff, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.f / red[0];
  for (int c = threadIdx.x; c < cols; c += blockDim.x) P[r * cols + c] = to16(__expf(s[c] - m) * inv, is_f16);
}

void softmax_rows(const float* S, bf16* P, int rows, int cols, cudaStream_t st) {
  launch_k(softmax_rows_kernel, rows, 256, 0, st, S, P, cols, 0);
  SD_CHECK_LAUNCH();
}
void softmax_rows(const float* S, f16* P, int rows, int cols, cudaStream_t st) {
  launch_k(softmax_rows_kernel, rows, 256, 0, st, S, reinterpret_cast<bf16*>(P), cols, 1);
  SD_CHECK_LAUNCH();
}

}  // namespace sd
