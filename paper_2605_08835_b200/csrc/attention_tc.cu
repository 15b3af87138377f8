// tcgen05 / TMEM / TMA flash attention for the UNet self-attention (reading R28):
// O = softmax(Q Kᵀ/√d) V per (batch row, head), head dims d ∈ {40, 64, 80}.
//
// One CTA = 128 queries of one (row, head); it streams the keys in blocks of 128.
//   warp 0      TMA: Q once; K (token-major, from the fused q|k buffer) and Vᵀ (channel-major,
//               produced directly by the V GEMM) tiles into a STAGES-deep ring
//   warp 1      MMA: S_j = Q·K_jᵀ (M=128, N=128, K=d) into TMEM (double-buffered), then
//               O += P_{j-1}·V_{j-1} (M=128, N=dpad, K=128) into a TMEM accumulator
//   warps 2..5  softmax: one query row per thread — tcgen05.ld of S, running max / sum in fp32,
//               P = exp2(s·log2e/√d − m) as bf16 into a swizzled smem tile (A operand of the PV
//               MMA), and O ← α·O in TMEM when the running max grows; finally O/l → bf16.
// S never leaves the SM; P never leaves shared memory. Bound: MUFU exp2 (16/clk/SM) at d ≤ 80.
#include <float.h>

#include "common.cuh"
#include "kernels_ew.h"

namespace sd {

// NB = number of S (TMEM) / P (smem) buffers. NB = 2: one CTA per SM, S_{j+1} computed while the
// softmax works on S_j. NB = 1: 256 TMEM columns and ~105 KB smem so two CTAs share an SM and
// interleave their MMA / softmax phases (the MMA of S_{j+1} still overlaps the tail of softmax_j).
template <int D, int NB>
struct TcAttn {
  static constexpr int BQ = 128, BK = 128;
  static constexpr int KQ = (D + 63) / 64;       // 64-column blocks of the head dim (Q/K tiles)
  static constexpr int K16 = (D + 15) / 16;      // MMA k-steps of Q·Kᵀ
  static constexpr int NPV = (D + 15) / 16 * 16; // N of the PV MMA (d padded to 16)
  static constexpr int Q_BYTES = KQ * BQ * 128;
  static constexpr int K_BYTES = KQ * BK * 128;
  static constexpr int V_BYTES = 2 * NPV * 128;  // two 64-key blocks of Vᵀ rows
  static constexpr int STAGE = K_BYTES + V_BYTES;
  static constexpr int STAGES = (NB == 2 && D <= 64) ? 3 : 2;
  static constexpr int P_BYTES = 2 * BQ * 128;   // one P tile: 128 rows × 128 keys bf16
  static constexpr int SMEM = 1024 + Q_BYTES + STAGES * STAGE + NB * P_BYTES + 256;
  static constexpr int TMEM_COLS = NB == 2 ? 512 : 256;
  static constexpr int O_COL = NB * 128;         // O accumulator after the S buffers
  static_assert(V_BYTES % 1024 == 0, "Vᵀ tile rows must be a multiple of 8");
  static_assert(NPV <= 128, "O must fit beside the S buffers");
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D, int NB>
__global__ void __launch_bounds__(192, 3 - NB)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tqk, const __grid_constant__ CUtensorMap tvt, bf16* __restrict__ O,
                   int ldo, int C, int P, int Lk, float scale_log2) {
  using A = TcAttn<D, NB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + A::Q_BYTES;
  uint8_t* sP = sKV + A::STAGES * A::STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + NB * A::P_BYTES);
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;
  uint64_t* kv_empty = kv_full + A::STAGES;
  uint64_t* s_full = kv_empty + A::STAGES;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* pv_done = p_full + 2;
  uint64_t* q_ready = pv_done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, head = blockIdx.y, row = blockIdx.z;
  const int q0 = qt * A::BQ;
  const int nb = (Lk + A::BK - 1) / A::BK;
  const int tok0 = row * P;  // first token of this batch row in the token-major buffers
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < A::STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 4);
      mbar_init(&p_full[s], 4);
    }
    mbar_init(pv_done, 1);
    mbar_init(q_ready, 4);
    fence_mbar_init();
    tma_prefetch(&tqk);
    tma_prefetch(&tvt);
  }
  if (warp == 1) tmem_alloc(tmem_slot, A::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S buffers at columns 0 / 128, O at 256

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_expect_tx(q_full, A::Q_BYTES);
      for (int kb = 0; kb < A::KQ; ++kb)
        tma_load_2d(sQ + kb * A::BQ * 128, &tqk, q_full, head * D + kb * 64, tok0 + q0);
      for (int j = 0; j < nb; ++j) {
        const int s = j % A::STAGES;
        mbar_wait(&kv_empty[s], ((j / A::STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], A::STAGE);
        uint8_t* st = sKV + s * A::STAGE;
        for (int kb = 0; kb < A::KQ; ++kb)
          tma_load_2d(st + kb * A::BK * 128, &tqk, &kv_full[s], C + head * D + kb * 64, tok0 + j * A::BK);
        for (int h = 0; h < 2; ++h)
          tma_load_2d(st + A::K_BYTES + h * A::NPV * 128, &tvt, &kv_full[s], tok0 + j * A::BK + h * 64, head * D);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id_s = make_idesc_bf16(128, 128);
      constexpr uint32_t id_pv = make_idesc_bf16(128, A::NPV);
      mbar_wait(q_ready, 0);  // Q landed and its padded columns were zeroed by the softmax warps
      tc_fence_after();
      const uint32_t aq = smem_u32(sQ);
      for (int j = 0; j <= nb; ++j) {
        if (j < nb) {
          const int s = j % A::STAGES, sb = j % NB;
          mbar_wait(&kv_full[s], (j / A::STAGES) & 1);
          if (j >= NB) mbar_wait(&s_empty[sb], (j / NB - 1) & 1);
          tc_fence_after();
          const uint32_t ak = smem_u32(sKV + s * A::STAGE);
#pragma unroll
          for (int k = 0; k < A::K16; ++k) {
            const uint32_t off = (k >> 2) * (A::BQ * 128) + (k & 3) * 32;
            umma_bf16(tmem + sb * 128, make_sdesc_sw128(aq + off), make_sdesc_sw128(ak + off), id_s, k > 0);
          }
          umma_commit(&s_full[sb]);
        }
        if (j >= 1) {
          const int jp = j - 1, pb = jp % NB, sp = jp % A::STAGES;
          mbar_wait(&p_full[pb], (jp / NB) & 1);
          tc_fence_after();
          const uint32_t ap = smem_u32(sP + pb * A::P_BYTES);
          const uint32_t av = smem_u32(sKV + sp * A::STAGE + A::K_BYTES);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t offp = (k >> 2) * (A::BQ * 128) + (k & 3) * 32;
            const uint32_t offv = (k >> 2) * (A::NPV * 128) + (k & 3) * 32;
            umma_bf16(tmem + A::O_COL, make_sdesc_sw128(ap + offp), make_sdesc_sw128(av + offv), id_pv, (jp | k) != 0);
          }
          umma_commit(&kv_empty[sp]);
          umma_commit(pv_done);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax warps: thread ↔ query row r ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float m = -FLT_MAX, l = 0.f;
    mbar_wait(q_full, 0);
    if (D % 16 != 0) {
      // zero Q columns [D, 16·K16) of this thread's row: they belong to the next head and the
      // padded k-step of Q·Kᵀ reads them
      uint8_t* qrow = sQ + ((D / 64) * A::BQ * 128) + r * 128;
      const int c0 = (D % 64) / 8;  // first 16-byte chunk to clear
      for (int c = c0; c < (A::NPV % 64 ? A::NPV % 64 : 64) / 8; ++c)
        *reinterpret_cast<uint4*>(qrow + ((c ^ (r & 7)) << 4)) = make_uint4(0, 0, 0, 0);
      fence_proxy_async_smem();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(q_ready);
    for (int j = 0; j < nb; ++j) {
      const int sb = j % NB;
      mbar_wait(&s_full[sb], (j / NB) & 1);
      tc_fence_after();
      // pass 1: row max over the 128 scores (TMEM is re-read in pass 2 instead of holding 128
      // registers; keys beyond Lk are masked)
      const bool ragged = (j + 1) * A::BK > Lk;
      float mx = m;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t t[32];
        tmem_ld32(tmem + lane_base + sb * 128 + c * 32, t);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (!ragged || j * A::BK + c * 32 + i < Lk) mx = fmaxf(mx, __uint_as_float(t[i]));
      }
      const float ms = mx * scale_log2;
      const float alpha = ex2((m - mx) * scale_log2);
      // pass 2: P = exp2(s·scale − m) packed to bf16
      float sum = 0.f;
      uint32_t pk[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t t[32];
        tmem_ld32(tmem + lane_base + sb * 128 + c * 32, t);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float s0 = __uint_as_float(t[2 * i]), s1 = __uint_as_float(t[2 * i + 1]);
          if (ragged) {
            if (j * A::BK + c * 32 + 2 * i >= Lk) s0 = -FLT_MAX;
            if (j * A::BK + c * 32 + 2 * i + 1 >= Lk) s1 = -FLT_MAX;
          }
          const float p0 = ex2(fmaf(s0, scale_log2, -ms));
          const float p1 = ex2(fmaf(s1, scale_log2, -ms));
          sum += p0 + p1;
          pk[c * 16 + i] = pack_bf16(p0, p1);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      l = l * alpha + sum;
      m = mx;
      if (j >= 1) {
        mbar_wait(pv_done, (j - 1) & 1);  // PV_{j-1} done: O is stable and P buffer (j&1) is free
        tc_fence_after();
        if (__any_sync(0xffffffff, alpha < 1.f)) {
#pragma unroll
          for (int c = 0; c < A::NPV / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(tmem + lane_base + A::O_COL + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(tmem + lane_base + A::O_COL + c * 16, o);
          }
          tmem_wait_st();
        }
      }
      // P row → swizzled smem (two 64-key K-blocks, 128 B per row, 16-byte chunk c at c ^ (r & 7))
      uint8_t* prow = sP + sb * A::P_BYTES + r * 128;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = kb * 32 + c * 4;
          *reinterpret_cast<uint4*>(prow + kb * (A::BQ * 128) + ((c ^ (r & 7)) << 4)) =
              make_uint4(pk[i], pk[i + 1], pk[i + 2], pk[i + 3]);
        }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
    }
    // ---------------- epilogue: O / l → bf16 ----------------
    mbar_wait(pv_done, (nb - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const int qi = q0 + r;
    bf16* orow = O + (long)(tok0 + qi) * ldo + head * D;
#pragma unroll
    for (int c = 0; c < A::NPV / 16; ++c) {
      uint32_t o[16];
      tmem_ld16(tmem + lane_base + A::O_COL + c * 16, o);
      tmem_wait_ld();
      if (qi < P) {
#pragma unroll
        for (int i = 0; i < 16; i += 8) {
          const int col = c * 16 + i;
          if (col + 8 <= D)
            *reinterpret_cast<uint4*>(orow + col) =
                make_uint4(pack_bf16(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv),
                           pack_bf16(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv),
                           pack_bf16(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv),
                           pack_bf16(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, A::TMEM_COLS);
}

// host ------------------------------------------------------------------------------------------
void make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
                  uint32_t box_out);

template <int D, int NB>
static void launch_tc(const bf16* qk, const bf16* vt, bf16* O, int rows, int heads, int C, int P, cudaStream_t st) {
  using A = TcAttn<D, NB>;
  static bool set = false;
  if (!set) {
    SD_CUDA(cudaFuncSetAttribute(attn_tc_kernel<D, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM));
    set = true;
  }
  const long T = (long)rows * P;
  CUtensorMap mqk, mvt;
  make_tmap_2d(&mqk, qk, (uint64_t)2 * C, (uint64_t)T, (uint64_t)2 * C * 2, 64, 128);
  make_tmap_2d(&mvt, vt, (uint64_t)T, (uint64_t)C, (uint64_t)T * 2, 64, A::NPV);
  dim3 grid(cdiv(P, A::BQ), heads, rows);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  attn_tc_kernel<D, NB><<<grid, 192, A::SMEM, st>>>(mqk, mvt, O, C, C, P, P, scale_log2);
  SD_CHECK_LAUNCH();
}

bool attention_tc_supported(int d, int P, int C) {
  return (d == 40 || d == 64 || d == 80) && P % 128 == 0 && C % 8 == 0;
}

// qk: [rows·P][2C] (q | k), vt: [C][rows·P] (Vᵀ), O: [rows·P][C]
void attention_tc(const bf16* qk, const bf16* vt, bf16* O, int rows, int heads, int d, int C, int P,
                  cudaStream_t st) {
  switch (d) {
    case 40: launch_tc<40, 1>(qk, vt, O, rows, heads, C, P, st); break;
    case 64: launch_tc<64, 2>(qk, vt, O, rows, heads, C, P, st); break;  // measured: NB=2 1.18× faster at d=64
    case 80: launch_tc<80, 2>(qk, vt, O, rows, heads, C, P, st); break;
    default: throw CudaError("attention_tc: unsupported head dim");
  }
}

}  // namespace sd
