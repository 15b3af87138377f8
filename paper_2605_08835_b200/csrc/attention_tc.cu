// tcgen05 / TMEM / TMA flash attention for the UNet self-attention (reading R28):
// O = softmax(Q Kᵀ/√d) V per (batch row, head), head dims d ∈ {40, 64, 80}.
//
// One CTA = 128 queries of one (row, head); it streams the keys in blocks of 128.
//   warp 0      TMA: Q once; K (token-major, from the fused q|k buffer) and Vᵀ (channel-major,
//               produced directly by the V GEMM) tiles into a STAGES-deep ring
//   warp 1      MMA: S_j = Q·K_jᵀ (M=128, N=128, K=d) into TMEM (double-buffered), then
//               O += P_{j-1}·V_{j-1} (M=128, N=dpad, K=128) into a TMEM accumulator
//   softmax     SPLIT threads per query row (d = 40: 2, each owning 64 key columns) — tcgen05.ld of
//               S, running max / sum in fp32, P = exp2(s·log2e/√d − m) as bf16 into a swizzled smem
//               tile (A operand of the PV MMA), and O ← α·O in TMEM when the running max grows
//               (lazily, threshold 2⁸); finally O/l → bf16. At d = 40 the scores are read from TMEM
//               once, the S buffer is handed back before the exps, 1/8 of the exps run on the FMA
//               pipe (ex2_poly) to relieve MUFU, and P goes back to TMEM (tcgen05.st) as the A
//               operand of the PV MMA instead of through shared memory (SD_ATTN_EMU, below).
// S never leaves the SM; P never leaves shared memory. Bound: MUFU exp2 (16/clk/SM) at d ≤ 80.
#include <float.h>

#include <type_traits>

#include "common.cuh"
#include "kernels_ew.h"

namespace sd {

// NB = number of S (TMEM) / P (smem) buffers. NB = 2: one CTA per SM, S_{j+1} computed while the
// softmax works on S_j. NB = 1: 256 TMEM columns and ~105 KB smem so two CTAs share an SM and
// interleave their MMA / softmax phases (the MMA of S_{j+1} still overlaps the tail of softmax_j).
// PT = 1: P lives in TMEM (OP 4 / 5) — no P tile in smem, whose space goes to a deeper K/V ring
template <int D, int NB, int SPLIT = 1, int EMU = 0, int PT = 0>
struct TcAttn {
  static constexpr int BQ = 128, BK = 128;
  // T64 (d = 160): two 64-column SW128 blocks + one 32-column SW64 tail per Q / K tile, so that two K/V
  // stages fit in shared memory (three full blocks would need 233.7 KB)
  static constexpr bool T64 = D == 160;
  static constexpr int KQ = T64 ? 2 : (D + 63) / 64;  // full 64-column blocks of the head dim (Q/K tiles)
  static constexpr int K16 = (D + 15) / 16;           // MMA k-steps of Q·Kᵀ
  static constexpr int NPV = (D + 15) / 16 * 16; // N of the PV MMA (d padded to 16)
  static constexpr int Q_BYTES = KQ * BQ * 128 + (T64 ? BQ * 64 : 0);
  static constexpr int K_BYTES = KQ * BK * 128 + (T64 ? BK * 64 : 0);
  static constexpr int V_BYTES = 2 * NPV * 128;  // two 64-key blocks of Vᵀ rows
  static constexpr int STAGE = K_BYTES + V_BYTES;
  static constexpr int STAGES = D > 128 ? 2 : PT ? (NB == 2 && D <= 64 ? 4 : 3) : ((NB == 2 && D <= 64) ? 3 : 2);
  static constexpr int P_BYTES = PT ? 0 : 2 * BQ * 128;  // one P tile: 128 rows × 128 keys bf16
  static constexpr int X_BYTES = 3 * 2 * 128 * 4;  // row-max / row-sum exchange of the SPLIT halves
  static constexpr int SMEM = 1024 + Q_BYTES + STAGES * STAGE + NB * P_BYTES + X_BYTES + 256;
  static constexpr int THREADS = 64 + 128 * SPLIT;
  static constexpr int TMEM_COLS = (NB == 2 || (PT && NPV > 64)) ? 512 : 256;  // S | O | P must fit
  static constexpr int O_COL = NB * 128;         // O accumulator after the S buffers
  static constexpr int P_COL =  // P (16-bit, 2 per column) in TMEM (OP ≥ 4), after O
      NB == 1 ? (NPV <= 64 ? 192 : (NPV <= 128 ? 256 : 128 + NPV)) : 384;
  static_assert(V_BYTES % 1024 == 0, "Vᵀ tile rows must be a multiple of 8");
  static_assert(NPV <= 128 || (NB == 1 && PT && P_COL + 64 <= 512), "O must fit beside the S buffers");
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
// D[tmem] (+)= A[tmem] · B[smem]ᵀ (kind::f16): A read from Tensor Memory, M rows = lanes, K packed
// two bf16 per 32-bit column
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// two 2^x on the FMA pipe with packed fp32 pairs (ex2_poly's method, FADD2 / FFMA2 for the float parts)
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
  x0 = fmaxf(x0, -120.f);
  x1 = fmaxf(x1, -120.f);
  float t0 = x0, t1 = x1;
  fadd2(t0, t1, 12582912.f, 12582912.f);  // rint by the 1.5·2²³ magic add
  float r0 = t0, r1 = t1;
  fadd2(r0, r1, -12582912.f, -12582912.f);
  float f0 = x0, f1 = x1;
  fadd2(f0, f1, -r0, -r1);
  float p0, p1;
  ffma2(p0, p1, 0.05520857f, 0.05520857f, f0, f1, 0.24226530f, 0.24226530f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.69324851f, 0.69324851f);
  ffma2(p0, p1, p0, p1, f0, f1, 1.0f, 1.0f);
  y0 = __int_as_float(__float_as_int(p0) + ((__float_as_int(t0) - 0x4B400000) << 23));
  y1 = __int_as_float(__float_as_int(p1) + ((__float_as_int(t1) - 0x4B400000) << 23));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA / ALU pipes (relieves MUFU, the bound of the softmax): x = j + f with j = rint(x)
// (1.5·2²³ magic add), f ∈ [−½, ½]; 2^f by a degree-3 polynomial fitted for relative error
// (max 1.2e-4 — far below bf16 P's 3.9e-3); 2^j added into the exponent field. x is clamped to −120
// (the result is then < 1e-36, i.e. zero next to a row sum ≥ 1).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -120.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05520857f, f, 0.24226530f), f, 0.69324851f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// OP = 1 (SPLIT = 2 only): the thread's 64 scores are read from TMEM once and kept in registers for
// both passes, and the S buffer is released to the MMA warp right after the loads, so S_{j+1} is
// computed while this block's exps run; P is packed in place over the scores (register budget)
// Where Q, K and Vᵀ come from. Self-attention: tq = tk = the fused q|k buffer (K at column C), Vᵀ
// [C][rows·P]; keys of batch row r start at token r·P. Cross-attention (K7): tq = the Q projection,
// tk = the text-K cache [slots·Lk][kv_width] and tvt = the text-Vᵀ cache [kv_width][ldkeys], both
// written once per prompt at admission; batch row r reads the Lk keys of prompt slot kv_index[r].
struct AttnTcArgs {
  bf16* O;
  int ldo, P, Lk;
  float scale_log2;
  int qcol0, kcol0, vrow0;  // column of head 0 in tq / tk; row of head 0's channels in tvt
  const int* kv_index;      // nullptr: self-attention
  int vt_slot;              // cross-attention: key columns per slot in tvt (Lk rounded up to 8: TMA needs the
                            // inner box start 16-byte aligned)
};

template <int D, int NB, int SPLIT, int EMU, int OP, bool F16>  // F16: fp16 operands (SD_PREC_FP16)
__global__ void __launch_bounds__(64 + 128 * SPLIT, 3 - NB)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tvt, const __grid_constant__ CUtensorMap tq_t,
                   const __grid_constant__ CUtensorMap tk_t, const AttnTcArgs a) {
  const int P = a.P, Lk = a.Lk, ldo = a.ldo;
  constexpr bool is_f16 = F16;
  const float scale_log2 = a.scale_log2;
  bf16* __restrict__ O = a.O;
  using A = TcAttn<D, NB, SPLIT, EMU, (OP == 4 || OP == 5) ? 1 : 0>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (SWIZZLE_128B atoms); offsetting the shared array itself keeps the pointer in the
  // shared state space, so the compiler emits STS / LDS rather than generic ST / LD
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + A::Q_BYTES;
  uint8_t* sP = sKV + A::STAGES * A::STAGE;
  float* sX = reinterpret_cast<float*>(sP + NB * A::P_BYTES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + NB * A::P_BYTES + A::X_BYTES);
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
      mbar_init(&s_empty[s], 4 * SPLIT);
      mbar_init(&p_full[s], 4 * SPLIT);
    }
    mbar_init(pv_done, 1);
    mbar_init(q_ready, 4 * SPLIT);
    fence_mbar_init();
    tma_prefetch(&tq);
    if (A::T64) {
      tma_prefetch(&tq_t);
      tma_prefetch(&tk_t);
    }
    tma_prefetch(&tk);
    tma_prefetch(&tvt);
  }
  if (warp == 1) tmem_alloc(tmem_slot, A::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S buffers at columns 0 / 128, O at 256
  pdl_wait();  // the prologue above overlapped the previous grid's tail (PDL)
  // first key row of this batch row in tk / first key column in tvt
  const int slot = a.kv_index ? __ldg(a.kv_index + row) : 0;
  const int key0 = a.kv_index ? slot * Lk : tok0;
  const int vkey0 = a.kv_index ? slot * a.vt_slot : tok0;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_expect_tx(q_full, A::Q_BYTES);
      for (int kb = 0; kb < A::KQ; ++kb)
        tma_load_2d(sQ + kb * A::BQ * 128, &tq, q_full, a.qcol0 + head * D + kb * 64, tok0 + q0);
      if (A::T64) tma_load_2d(sQ + A::KQ * A::BQ * 128, &tq_t, q_full, a.qcol0 + head * D + A::KQ * 64, tok0 + q0);
      for (int j = 0; j < nb; ++j) {
        const int s = j % A::STAGES;
        mbar_wait_sleep(&kv_empty[s], ((j / A::STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], A::STAGE);
        uint8_t* st = sKV + s * A::STAGE;
        for (int kb = 0; kb < A::KQ; ++kb)
          tma_load_2d(st + kb * A::BK * 128, &tk, &kv_full[s], a.kcol0 + head * D + kb * 64, key0 + j * A::BK);
        if (A::T64)
          tma_load_2d(st + A::KQ * A::BK * 128, &tk_t, &kv_full[s], a.kcol0 + head * D + A::KQ * 64,
                      key0 + j * A::BK);
        for (int h = 0; h < 2; ++h)
          tma_load_2d(st + A::K_BYTES + h * A::NPV * 128, &tvt, &kv_full[s], vkey0 + j * A::BK + h * 64,
                      a.vrow0 + head * D);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id_s = make_idesc16(128, 128, F16);
      constexpr uint32_t id_pv = make_idesc16(128, A::NPV, F16);
      mbar_wait(q_ready, 0);  // Q landed and its padded columns were zeroed by the softmax warps
      tc_fence_after();
      const uint32_t aq = smem_u32(sQ);
      for (int j = 0; j <= nb; ++j) {
        if (j < nb) {
          const int s = j % A::STAGES, sb = j % NB;
          mbar_wait_sleep(&kv_full[s], (j / A::STAGES) & 1);
          if (j >= NB) mbar_wait_sleep(&s_empty[sb], (j / NB - 1) & 1);
          tc_fence_after();
          const uint32_t ak = smem_u32(sKV + s * A::STAGE);
#pragma unroll
          for (int k = 0; k < A::K16; ++k) {
            if (A::T64 && k >= 4 * A::KQ) {  // the 32-column SW64 tail: 64-byte rows, k-steps 32 bytes apart
              const uint32_t off = A::KQ * (A::BQ * 128) + (k - 4 * A::KQ) * 32;
              umma_bf16(tmem + sb * 128, make_sdesc_sw64(aq + off), make_sdesc_sw64(ak + off), id_s, 1);
            } else {
              const uint32_t off = (k >> 2) * (A::BQ * 128) + (k & 3) * 32;
              umma_bf16(tmem + sb * 128, make_sdesc_sw128(aq + off), make_sdesc_sw128(ak + off), id_s, k > 0);
            }
          }
          umma_commit(&s_full[sb]);
        }
        if (j >= 1) {
          const int jp = j - 1, pb = jp % NB, sp = jp % A::STAGES;
          mbar_wait_sleep(&p_full[pb], (jp / NB) & 1);
          tc_fence_after();
          const uint32_t ap = smem_u32(sP + pb * A::P_BYTES);
          const uint32_t av = smem_u32(sKV + sp * A::STAGE + A::K_BYTES);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t offp = (k >> 2) * (A::BQ * 128) + (k & 3) * 32;
            const uint32_t offv = (k >> 2) * (A::NPV * 128) + (k & 3) * 32;
            if constexpr (OP == 4 || OP == 5)  // A = P from TMEM: 16 keys = 8 packed columns per k-step
              umma_bf16_ts(tmem + A::O_COL, tmem + A::P_COL + k * 8, make_sdesc_sw128(av + offv), id_pv,
                           (jp | k) != 0);
            else
              umma_bf16(tmem + A::O_COL, make_sdesc_sw128(ap + offp), make_sdesc_sw128(av + offv), id_pv,
                        (jp | k) != 0);
          }
          umma_commit(&kv_empty[sp]);
          umma_commit(pv_done);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax warps: SPLIT threads per query row r ----------------
    // warp w accesses TMEM lane quarter w % 4; with SPLIT = 2, warps w and w + 4 share the rows of a
    // quarter and take the key columns [64h, 64h + 64) each (h = half), exchanging the row max
    // through smem once per key block (named barrier per quarter)
    constexpr int CPT = 128 / SPLIT, NCH = CPT / 32;
    constexpr bool DBUF = !(NB == 1 && SPLIT == 1);
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float m = -FLT_MAX, l = 0.f;
    mbar_wait(q_full, 0);
    if (D % 16 != 0 && h == 0) {
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
      mbar_wait_sleep(&s_full[sb], (j / NB) & 1);
      tc_fence_after();
      const uint32_t sbase = tmem + lane_base + sb * 128 + h * CPT;
      uint32_t ta[32], tb[32];
      if constexpr (OP >= 1 && OP <= 4) {
        static_assert(SPLIT == 2, "one-pass softmax needs 64 columns per thread");  // OP ≥ 1
        tmem_ld32_nw(sbase, ta);
        tmem_ld32_nw(sbase + 32, tb);
        tmem_wait_ld_tied(ta);
        tmem_wait_ld_tied(tb);
        tc_fence_before();  // the scores are in registers: S buffer free for S_{j+1}
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        if (j == nb - 1 && (Lk & (A::BK - 1))) {
          // ragged last key block (cross-attention: 77 text tokens; the 8×8 mid block: 64 tokens):
          // keys ≥ Lk get −∞ (P = 0; their K / Vᵀ rows are finite memory beyond the valid keys)
          const int valid = Lk - j * A::BK - h * 64;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (i >= valid) ta[i] = __float_as_uint(-INFINITY);
            if (32 + i >= valid) tb[i] = __float_as_uint(-INFINITY);
          }
        }
        float mx4[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(ta[i]));
          mx4[(i + 2) & 3] = fmaxf(mx4[(i + 2) & 3], __uint_as_float(tb[i]));
        }
        float mxb = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        sX[((j & 1) * 2 + h) * 128 + r] = mxb;
        named_bar_sync(1 + q, 64);
        mxb = fmaxf(mxb, sX[((j & 1) * 2 + (h ^ 1)) * 128 + r]);
        const bool upd = (mxb - m) * scale_log2 > 8.f;
        const float mnew = upd ? mxb : m;
        const float alpha = upd ? ex2((m - mnew) * scale_log2) : 1.f;
        const float ms = mnew * scale_log2;
        float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (OP == 4) {
          // packed fp32 pairs (FFMA2 / FADD2) and one pair in PER on the FMA pipe (ex2_poly2); the other
          // pairs on MUFU. P packed in place: ta[i] ← 16-bit pair (p(ta[2i]), p(ta[2i+1]))
          constexpr int PER = EMU > 0 ? EMU : 8;
          float sp0[4] = {0.f, 0.f, 0.f, 0.f}, sp1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = 0; i < 32; ++i) {  // i < 16: ta pairs, i ≥ 16: tb pairs
            uint32_t (&src)[32] = i < 16 ? ta : tb;
            const int ii = i & 15;
            float x0, x1;
            ffma2(x0, x1, __uint_as_float(src[2 * ii]), __uint_as_float(src[2 * ii + 1]), scale_log2, scale_log2,
                  -ms, -ms);
            float p0, p1;
            if (i % PER == PER - 1) {
              ex2_poly2(x0, x1, p0, p1);
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            fadd2(sp0[i & 3], sp1[i & 3], p0, p1);
            src[ii] = pack16(p0, p1, is_f16);
          }
          sum8[0] = (sp0[0] + sp1[0]) + (sp0[1] + sp1[1]);
          sum8[1] = (sp0[2] + sp1[2]) + (sp0[3] + sp1[3]);
        } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {  // P packed in place: ta[i] ← bf16x2(p(ta[2i]), p(ta[2i+1]))
          const float x0 = fmaf(__uint_as_float(ta[2 * i]), scale_log2, -ms);
          const float x1 = fmaf(__uint_as_float(ta[2 * i + 1]), scale_log2, -ms);
          const bool emu = OP >= 2 && (i % (OP == 3 ? 4 : 8)) == 3;  // OP 2, 4 / 3: 1/8 / 1/4 on the FMA pipe
          const float p0 = emu ? ex2_poly(x0) : ex2(x0);
          const float p1 = emu ? ex2_poly(x1) : ex2(x1);
          sum8[i & 7] += p0 + p1;
          ta[i] = pack16(p0, p1, is_f16);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float x0 = fmaf(__uint_as_float(tb[2 * i]), scale_log2, -ms);
          const float x1 = fmaf(__uint_as_float(tb[2 * i + 1]), scale_log2, -ms);
          const bool emu = OP >= 2 && (i % (OP == 3 ? 4 : 8)) == 1;
          const float p0 = emu ? ex2_poly(x0) : ex2(x0);
          const float p1 = emu ? ex2_poly(x1) : ex2(x1);
          sum8[i & 7] += p0 + p1;
          tb[i] = pack16(p0, p1, is_f16);
        }
        }
        const float sum = ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
        l = l * alpha + sum;
        m = mnew;
        if (j >= 1) {
          mbar_wait_sleep(pv_done, (j - 1) & 1);
          tc_fence_after();
          if (h == 0 && __any_sync(0xffffffff, alpha < 1.f)) {
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
        if constexpr (OP == 4) {
          // P stays in TMEM (the A operand of the PV MMA): this thread's 64 keys = 32 packed columns
          uint32_t (&pa)[16] = reinterpret_cast<uint32_t(&)[16]>(ta);
          uint32_t (&pb)[16] = reinterpret_cast<uint32_t(&)[16]>(tb);
          tmem_st16(tmem + lane_base + A::P_COL + h * 32, pa);
          tmem_st16(tmem + lane_base + A::P_COL + h * 32 + 16, pb);
          tmem_wait_st();
        } else {
          uint8_t* prow = sP + sb * A::P_BYTES + h * (A::BQ * 128) + r * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) =
                make_uint4(ta[c * 4], ta[c * 4 + 1], ta[c * 4 + 2], ta[c * 4 + 3]);
            *reinterpret_cast<uint4*>(prow + (((c + 4) ^ (r & 7)) << 4)) =
                make_uint4(tb[c * 4], tb[c * 4 + 1], tb[c * 4 + 2], tb[c * 4 + 3]);
          }
          fence_proxy_async_smem();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        continue;
      }
      // pass 1: row max over this thread's scores — 4 independent max chains, the next 32-column TMEM
      // load in flight while this one is reduced (TMEM is re-read in pass 2)
      float mx4[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
      tmem_ld32_nw(sbase, ta);
      tmem_wait_ld_tied(ta);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        // DBUF: the next chunk's load is in flight while this one is processed (needs 32 more registers)
        uint32_t(&cur)[32] = (DBUF && (c & 1)) ? tb : ta;
        uint32_t(&nxt)[32] = (c & 1) ? ta : tb;
        if (DBUF && c < NCH - 1) tmem_ld32_nw(sbase + (c + 1) * 32, nxt);
        if (!DBUF && c > 0) {
          tmem_ld32_nw(sbase + c * 32, ta);
          tmem_wait_ld_tied(ta);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i)
          mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(cur[i]));
        if (DBUF && c < NCH - 1) tmem_wait_ld_tied(nxt);
      }
      float mxb = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      if (SPLIT == 2) {
        sX[((j & 1) * 2 + h) * 128 + r] = mxb;
        named_bar_sync(1 + q, 64);
        mxb = fmaxf(mxb, sX[((j & 1) * 2 + (h ^ 1)) * 128 + r]);
      }
      // lazy rescaling: the running max m only moves when the block max exceeds it by more than 8 in
      // the exp2 domain (P ≤ 2⁸ stays exact in fp32 sums and bf16 P), so O is rarely rescaled
      const bool upd = (mxb - m) * scale_log2 > 8.f;
      const float mnew = upd ? mxb : m;
      const float alpha = upd ? ex2((m - mnew) * scale_log2) : 1.f;
      const float ms = mnew * scale_log2;
      // pass 2: P = exp2(s·scale − m) packed to bf16; 8 independent partial sums
      float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t pk[NCH * 16];
      tmem_ld32_nw(sbase, ta);
      tmem_wait_ld_tied(ta);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        // DBUF: the next chunk's load is in flight while this one is processed (needs 32 more registers)
        uint32_t(&cur)[32] = (DBUF && (c & 1)) ? tb : ta;
        uint32_t(&nxt)[32] = (c & 1) ? ta : tb;
        if (DBUF && c < NCH - 1) tmem_ld32_nw(sbase + (c + 1) * 32, nxt);
        if (!DBUF && c > 0) {
          tmem_ld32_nw(sbase + c * 32, ta);
          tmem_wait_ld_tied(ta);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float s0 = __uint_as_float(cur[2 * i]), s1 = __uint_as_float(cur[2 * i + 1]);
          const float x0 = fmaf(s0, scale_log2, -ms), x1 = fmaf(s1, scale_log2, -ms);
          float p0, p1;
          if (EMU > 0 && i % EMU == EMU - 1) {  // 1 pair in EMU on the FMA pipe
            p0 = ex2_poly(x0);
            p1 = ex2_poly(x1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          sum8[i & 7] += p0 + p1;
          pk[c * 16 + i] = pack16(p0, p1, is_f16);
        }
        if (DBUF && c < NCH - 1) tmem_wait_ld_tied(nxt);
      }
      const float sum = ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      l = l * alpha + sum;  // this thread's columns; the halves are added after the last block
      m = mnew;
      if (j >= 1) {
        mbar_wait_sleep(pv_done, (j - 1) & 1);  // PV_{j-1} done: O is stable and P buffer (j&1) is free
        tc_fence_after();
        if (h == 0 && __any_sync(0xffffffff, alpha < 1.f)) {
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
      if constexpr (OP == 5) {
        // P back to TMEM (A operand of the PV MMA): this thread's CPT keys = CPT / 2 packed columns
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tmem_st16(tmem + lane_base + A::P_COL + h * (CPT / 2) + c * 16,
                    reinterpret_cast<uint32_t(&)[16]>(pk[c * 16]));
        tmem_wait_st();
      } else {
        // P row → swizzled smem (64-key K-blocks, 128 B per row, 16-byte chunk c at c ^ (r & 7))
        uint8_t* prow = sP + sb * A::P_BYTES + r * 128;
#pragma unroll
        for (int kk = 0; kk < NCH / 2; ++kk)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int i = kk * 32 + c * 4;
            const int kb = h * (NCH / 2) + kk;
            *reinterpret_cast<uint4*>(prow + kb * (A::BQ * 128) + ((c ^ (r & 7)) << 4)) =
                make_uint4(pk[i], pk[i + 1], pk[i + 2], pk[i + 3]);
          }
        fence_proxy_async_smem();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
    }
    // ---------------- epilogue: O / l → bf16 ----------------
    if (SPLIT == 2) {
      sX[(2 * 2 + h) * 128 + r] = l;  // rows of the exchange area not used by the last key blocks
      named_bar_sync(1 + q, 64);
      l = sX[(2 * 2 + 0) * 128 + r] + sX[(2 * 2 + 1) * 128 + r];
    }
    mbar_wait(pv_done, (nb - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const int qi = q0 + r;
    bf16* orow = O + (long)(tok0 + qi) * ldo + head * D;
#pragma unroll
    for (int c = 0; c < A::NPV / 16; ++c) {
      if (c % SPLIT != h) continue;
      uint32_t o[16];
      tmem_ld16(tmem + lane_base + A::O_COL + c * 16, o);
      tmem_wait_ld();
      if (qi < P) {
#pragma unroll
        for (int i = 0; i < 16; i += 8) {
          const int col = c * 16 + i;
          if (col + 8 <= D)
            *reinterpret_cast<uint4*>(orow + col) =
                make_uint4(pack16(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv, is_f16),
                           pack16(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv, is_f16),
                           pack16(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv, is_f16),
                           pack16(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv, is_f16));
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
static bool env_on(const char* name) {
  const char* e = getenv(name);
  return !(e && e[0] == '0');
}

void make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
                  uint32_t box_out, bool is_f16, bool swz64 = false);

// the three operand tensors of one launch (host side)
struct TcSrc {
  const void* q;
  long q_rows;
  int ldq;
  const void* k;
  long k_rows;
  int ldk;
  const void* vt;
  long vt_rows, ld_keys;
  int qcol0, kcol0, vrow0, Lk;
  const int* kv_index;
};

template <int D, int NB, int SPLIT, int EMU = 0, int OP = 0>
static void launch_tc(const TcSrc& sr, bf16* O, int ldo, int rows, int heads, int P, cudaStream_t st, bool f16) {
  using A = TcAttn<D, NB, SPLIT, EMU, (OP == 4 || OP == 5) ? 1 : 0>;
  static bool set = false;
  if (!set) {
    SD_CUDA(cudaFuncSetAttribute(attn_tc_kernel<D, NB, SPLIT, EMU, OP, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM));
    SD_CUDA(cudaFuncSetAttribute(attn_tc_kernel<D, NB, SPLIT, EMU, OP, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM));
    set = true;
  }
  CUtensorMap mq, mk, mvt;
  make_tmap_2d(&mq, sr.q, (uint64_t)sr.ldq, (uint64_t)sr.q_rows, (uint64_t)sr.ldq * 2, 64, 128, f16);
  if (sr.k == sr.q && sr.ldk == sr.ldq && sr.k_rows == sr.q_rows)
    mk = mq;
  else
    make_tmap_2d(&mk, sr.k, (uint64_t)sr.ldk, (uint64_t)sr.k_rows, (uint64_t)sr.ldk * 2, 64, 128, f16);
  make_tmap_2d(&mvt, sr.vt, (uint64_t)sr.ld_keys, (uint64_t)sr.vt_rows, (uint64_t)sr.ld_keys * 2, 64, A::NPV, f16);
  CUtensorMap mq_t = mq, mk_t = mk;  // d = 160: 32-column SW64 tail boxes of Q and K
  if (A::T64) {
    make_tmap_2d(&mq_t, sr.q, (uint64_t)sr.ldq, (uint64_t)sr.q_rows, (uint64_t)sr.ldq * 2, 32, 128, f16, true);
    make_tmap_2d(&mk_t, sr.k, (uint64_t)sr.ldk, (uint64_t)sr.k_rows, (uint64_t)sr.ldk * 2, 32, 128, f16, true);
  }
  dim3 grid(cdiv(P, A::BQ), heads, rows);
  AttnTcArgs a;
  a.O = O;
  a.ldo = ldo;
  a.P = P;
  a.Lk = sr.Lk;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  a.qcol0 = sr.qcol0;
  a.kcol0 = sr.kcol0;
  a.vrow0 = sr.vrow0;
  a.kv_index = sr.kv_index;
  a.vt_slot = (sr.Lk + 7) / 8 * 8;
  if (f16)
    launch_k(attn_tc_kernel<D, NB, SPLIT, EMU, OP, true>, grid, A::THREADS, A::SMEM, st, mq, mk, mvt, mq_t, mk_t, a);
  else
    launch_k(attn_tc_kernel<D, NB, SPLIT, EMU, OP, false>, grid, A::THREADS, A::SMEM, st, mq, mk, mvt, mq_t, mk_t, a);
  SD_CHECK_LAUNCH();
}

// SD_ATTN_SPLIT=1|2: softmax threads per query row at d = 40 (default 2)
static int attn_split() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_ATTN_SPLIT");
    v = e ? atoi(e) : 2;
    if (v != 1) v = 2;
  }
  return v;
}

// SD_ATTN_EMU selects the d = 40 softmax variant (kbench r01, [16, 8, 40, 4096]):
//   0  two TMEM passes, all exps on MUFU, P through smem          0.794 ms
//   4  two passes, 1/4 of the exps on the FMA pipe (ex2_poly)     slower
//   5  one TMEM pass (OP 1), S released before the exps           0.784 ms
//   6  one pass + 1/8 of the exps on the FMA pipe (OP 2)          0.769 ms
//   7  one pass + 1/4 on the FMA pipe (OP 3)                      0.804 ms
//   8  OP 2 + P kept in TMEM as the A operand of the PV MMA       0.751 ms → 0.664 ms once the freed
//      P smem became a third K/V stage (default; no P smem stores, no async-proxy fence)
static int attn_emu() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_ATTN_EMU");
    v = e ? atoi(e) : 8;
    if (v != 0 && v != 4 && (v < 5 || v > 8)) v = 8;
  }
  return v;
}
// SD_ATTN_EF=8|4|3: one softmax pair in EF computes its exponentials on the FMA pipe (d = 40, OP 4).
// Default by precision (kbench [16, 8, 40, 4096], B200): bf16 EF 8 675 µs (EF 3: 682); fp16 EF 3 690 µs
// (EF 8: 709) — the fp16 P conversion competes with the exponentials, so fp16 moves more of them off MUFU
static int attn_ef(bool f16) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_ATTN_EF");
    v = e ? atoi(e) : 0;
    if (v != 4 && v != 3 && v != 8) v = 0;
  }
  return v ? v : (f16 ? 3 : 8);
}
// SD_ATTN_NB=1|2: S / P buffers at d = 40 (default 1: two CTAs per SM)
static int attn_nb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_ATTN_NB");
    v = e ? atoi(e) : 1;
    if (v != 2) v = 1;
  }
  return v;
}

bool attention_tc_supported(int d, int P, int C) {
  static const bool d160 = env_on("SD_ATTN160_TC");  // SD_ATTN160_TC=0: d = 160 on the mma.sync kernel
  if (d == 160 && !d160) return false;
  // ragged key blocks (P % 128 != 0) are masked by the default OP-4 softmax only
  // self-attention Vᵀ key columns start at row·P: 16-byte aligned needs P % 8 == 0
  return (d == 40 || d == 64 || d == 80 || d == 160) && (P % 128 == 0 || (attn_emu() == 8 && P % 8 == 0)) &&
         C % 8 == 0;
}

// qk: [rows·P][2C] (q | k), vt: [C][rows·P] (Vᵀ), O: [rows·P][C]
static void attention_tc16(const TcSrc& sr, bf16* O, int ldo, int rows, int heads, int d, int P, cudaStream_t st,
                           bool f16) {
  if (sr.Lk % 128 && attn_emu() != 8) throw CudaError("attention_tc: ragged keys need the default (OP 4) variant");
  switch (d) {
    case 40:
      switch (attn_nb() * 100 + attn_split() * 10 + attn_emu()) {
        case 110: launch_tc<40, 1, 1, 0>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 114: launch_tc<40, 1, 1, 4>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 124: launch_tc<40, 1, 2, 4>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 210: launch_tc<40, 2, 1, 0>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 220: launch_tc<40, 2, 2, 0>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 224: launch_tc<40, 2, 2, 4>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 125: launch_tc<40, 1, 2, 0, 1>(sr, O, ldo, rows, heads, P, st, f16); break;  // SD_ATTN_EMU=5: one-pass
        case 225: launch_tc<40, 2, 2, 0, 1>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 126: launch_tc<40, 1, 2, 0, 2>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 127: launch_tc<40, 1, 2, 0, 3>(sr, O, ldo, rows, heads, P, st, f16); break;
        case 128:  // SD_ATTN_EMU=8 (default): P in TMEM; SD_ATTN_EF = pairs per FMA-pipe exp pair (8 / 4 / 3)
          if (attn_ef(f16) == 4)
            launch_tc<40, 1, 2, 4, 4>(sr, O, ldo, rows, heads, P, st, f16);
          else if (attn_ef(f16) == 3)
            launch_tc<40, 1, 2, 3, 4>(sr, O, ldo, rows, heads, P, st, f16);
          else
            launch_tc<40, 1, 2, 0, 4>(sr, O, ldo, rows, heads, P, st, f16);
          break;
        default: launch_tc<40, 1, 2, 0>(sr, O, ldo, rows, heads, P, st, f16); break;
      }
      break;
    case 64:  // SD_ATTN_EMU=8 (default): the d = 40 structure — two CTAs per SM, two softmax threads per
              // row, one TMEM pass, P in TMEM (S 128 | O 64 | P 64 columns): SDXL [16,10,64,4096] 1.27 → 1.16
              // ms vs NB = 2 / one thread per row (which was 1.18× faster than NB = 1 with P in smem)
      if (attn_emu() == 8 && getenv("SD_ATTN_EF") && attn_ef(f16) == 3)  // measured: EF 8 faster at d = 64
        launch_tc<64, 1, 2, 3, 4>(sr, O, ldo, rows, heads, P, st, f16);
      else if (attn_emu() == 8)
        launch_tc<64, 1, 2, 0, 4>(sr, O, ldo, rows, heads, P, st, f16);
      else if (attn_emu() == 5)
        launch_tc<64, 2, 1, 0, 5>(sr, O, ldo, rows, heads, P, st, f16);
      else if (attn_emu() != 4)
        launch_tc<64, 2, 1, 0>(sr, O, ldo, rows, heads, P, st, f16);
      else
        launch_tc<64, 2, 1, 4>(sr, O, ldo, rows, heads, P, st, f16);
      break;
    case 80:  // SD_ATTN_EMU=8 (default): two softmax threads per row, one TMEM pass, P in TMEM; S | O | P
              // need 272 columns, so one CTA per SM (512 allocated): [16,8,80,1024] 87.9 → 83.1 µs
      if (attn_emu() == 8 && getenv("SD_ATTN_EF") && attn_ef(f16) == 3)  // measured: EF 8 faster at d = 80
        launch_tc<80, 1, 2, 3, 4>(sr, O, ldo, rows, heads, P, st, f16);
      else if (attn_emu() == 8)
        launch_tc<80, 1, 2, 0, 4>(sr, O, ldo, rows, heads, P, st, f16);
      else if (attn_emu() == 5)
        launch_tc<80, 2, 1, 0, 5>(sr, O, ldo, rows, heads, P, st, f16);
      else if (attn_emu() != 4)
        launch_tc<80, 2, 1, 0>(sr, O, ldo, rows, heads, P, st, f16);
      else
        launch_tc<80, 2, 1, 4>(sr, O, ldo, rows, heads, P, st, f16);
      break;
    case 160:  // SD-1.5 16×16 and the 8×8 mid block: S | O (160) | P in 512 columns, one K/V stage
      launch_tc<160, 1, 2, 0, 4>(sr, O, ldo, rows, heads, P, st, f16);
      break;
    default: throw CudaError("attention_tc: unsupported head dim");
  }
}

static TcSrc self_src(const void* qk, const void* vt, int rows, int C, int P) {
  const long T = (long)rows * P;
  TcSrc sr{};
  sr.q = sr.k = qk;
  sr.q_rows = sr.k_rows = T;
  sr.ldq = sr.ldk = 2 * C;
  sr.vt = vt;
  sr.vt_rows = C;
  sr.ld_keys = T;
  sr.qcol0 = 0;
  sr.kcol0 = C;
  sr.vrow0 = 0;
  sr.Lk = P;
  sr.kv_index = nullptr;
  return sr;
}
void attention_tc(const bf16* qk, const bf16* vt, bf16* O, int rows, int heads, int d, int C, int P, cudaStream_t st) {
  attention_tc16(self_src(qk, vt, rows, C, P), O, C, rows, heads, d, P, st, false);
}
void attention_tc(const f16* qk, const f16* vt, f16* O, int rows, int heads, int d, int C, int P, cudaStream_t st) {
  attention_tc16(self_src(qk, vt, rows, C, P), reinterpret_cast<bf16*>(O), C, rows, heads, d, P, st, true);
}

// cross-attention over the cached text tokens (K7): Q [rows·P][C]; kcache [n_slots·Lk][ldk] with this
// layer's K at column kcol; vtcache [vt_rows][ld_keys] with this layer's Vᵀ at row vrow (key j of slot s
// at column s·⌈Lk⌉₈ + j); kv_index [rows] = slot per batch row (device)
template <class T>
static void xattn_tc_impl(const T* q, const T* kcache, int ldk, long n_slots, int kcol, const T* vtcache,
                          long vt_rows, long ld_keys, int vrow, const int* kv_index, int Lk, T* O, int rows, int heads,
                          int d, int C, int P, cudaStream_t st) {
  TcSrc sr{};
  sr.q = q;
  sr.q_rows = (long)rows * P;
  sr.ldq = C;
  sr.k = kcache;
  sr.k_rows = n_slots * Lk;
  sr.ldk = ldk;
  sr.vt = vtcache;
  sr.vt_rows = vt_rows;
  sr.ld_keys = ld_keys;
  sr.qcol0 = 0;
  sr.kcol0 = kcol;
  sr.vrow0 = vrow;
  sr.Lk = Lk;
  sr.kv_index = kv_index;
  attention_tc16(sr, reinterpret_cast<bf16*>(O), C, rows, heads, d, P, st, std::is_same<T, f16>::value);
}
void xattention_tc(const bf16* q, const bf16* kc, int ldk, long n_slots, int kcol, const bf16* vtc, long vt_rows,
                   long ld_keys, int vrow, const int* kv_index, int Lk, bf16* O, int rows, int heads, int d, int C, int P,
                   cudaStream_t st) {
  xattn_tc_impl(q, kc, ldk, n_slots, kcol, vtc, vt_rows, ld_keys, vrow, kv_index, Lk, O, rows, heads, d, C, P, st);
}
void xattention_tc(const f16* q, const f16* kc, int ldk, long n_slots, int kcol, const f16* vtc, long vt_rows,
                   long ld_keys, int vrow, const int* kv_index, int Lk, f16* O, int rows, int heads, int d, int C, int P,
                   cudaStream_t st) {
  xattn_tc_impl(q, kc, ldk, n_slots, kcol, vtc, vt_rows, ld_keys, vrow, kv_index, Lk, O, rows, heads, d, C, P, st);
}

}  // namespace sd
