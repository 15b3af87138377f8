// tcgen05 cross-attention over the cached text tokens (readings R28, R2): O = softmax(Q·Kᵀ/√d)·V
// with ≤ 80 keys (77 text tokens), one block of keys, so the softmax of a query tile is exact in one pass.
//
// A CTA owns one (batch row, head) and walks a run of 128-query tiles, keeping that row's K and Vᵀ (one
// TMA load each) resident in shared memory — the per-tile cost is then Q in, O out, and the exps:
//   warp 0      TMA: K and Vᵀ once; Q tiles into a 2-deep ring
//   warp 1      MMA: S_t = Q_t·Kᵀ (M 128, N 80, K = d) into TMEM S buffer t mod 2, then
//               O = P_{t-1}·V (A = P from TMEM, K = 80 keys) into the TMEM O accumulator
//   warps 2-9   softmax, two threads per query row (40 keys each; keys ≥ Lk masked to −∞); P (16-bit) is
//               written back IN PLACE over the S columns just read — the A operand of the PV MMA — then
//               the epilogue of the previous tile: O/l → 16-bit rows of O
// TMEM: S/P 2 × 80 | O (48 / 64 / 80 columns) ≤ 256 → two CTAs per SM (the per-tile chain S → softmax →
// PV → epilogue of one CTA overlaps the other's). P_t overwrites S_t: the S MMA of tile t + 2 (same
// buffer) is issued after the PV MMA of tile t (it waits for P_{t+1}, written after P_t), and tcgen05
// MMAs of one issuing thread execute in order.
#include <float.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "kernels_ew.h"

namespace sd {

namespace {

constexpr int XK = 80;  // keys per tile (≥ Lk): N of the S MMA, K of the PV MMA

template <int D>
struct XA {
  static constexpr int KQ = (D + 63) / 64;        // 64-column blocks of the head dim
  static constexpr int K16 = (D + 15) / 16;       // k-steps of Q·Kᵀ
  static constexpr int NPV = (D + 15) / 16 * 16;  // N of the PV MMA
  static constexpr int Q_BYTES = KQ * 128 * 128;
  static constexpr int K_BYTES = KQ * XK * 128;
  static constexpr int V_BYTES = 2 * NPV * 128;   // Vᵀ rows: keys 0..63 | 64..79 (SW128 blocks of 64 keys)
  static constexpr int X_BYTES = 2 * 2 * 128 * 4; // row max / row sum exchange of the two halves
  static constexpr int SMEM = 1024 + 2 * Q_BYTES + K_BYTES + V_BYTES + X_BYTES + 256;
  static constexpr int S_STRIDE = XK, O_COL = 2 * S_STRIDE;
  static_assert(O_COL + NPV <= 256, "S/P | O must fit 256 TMEM columns");
  static_assert(V_BYTES % 1024 == 0 && K_BYTES % 1024 == 0, "tiles must be whole 8-row swizzle groups");
};

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void st4(uint32_t taddr, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct XArgs {
  bf16* O;
  int ldo, P, Lk, vt_slot, tiles_per_cta;
  float scale_log2;
  int qcol0, kcol0, vrow0;
  const int* kv_index;
};

}  // namespace

template <int D, bool F16>
__global__ void __launch_bounds__(320, 2)
    xattn_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tvt, const XArgs a) {
  using A = XA<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                        // [2][Q_BYTES]
  uint8_t* sK = sQ + 2 * A::Q_BYTES;
  uint8_t* sV = sK + A::K_BYTES;
  float* sX = reinterpret_cast<float*>(sV + A::V_BYTES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sX) + A::X_BYTES);
  uint64_t* kv_full = bar;          // K and Vᵀ landed
  uint64_t* kv_ready = bar + 1;     // K's padded columns zeroed (softmax warps)
  uint64_t* q_full = bar + 2;       // [2]
  uint64_t* q_empty = bar + 4;      // [2] (MMA commit)
  uint64_t* s_full = bar + 6;       // [2] (MMA commit)
  uint64_t* p_full = bar + 8;       // [2] (8 softmax warps)
  uint64_t* o_full = bar + 10;      // PV done (MMA commit)
  uint64_t* o_empty = bar + 11;     // O drained (8 softmax warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y, row = blockIdx.z;
  const int ntiles = (a.P + 127) / 128;
  const int t0 = blockIdx.x * a.tiles_per_cta;
  const int T = min(a.tiles_per_cta, ntiles - t0);  // query tiles of this CTA (≥ 1)
  const int tok0 = row * a.P;
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_ready, 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 8);
    fence_mbar_init();
    tma_prefetch(&tq);
    tma_prefetch(&tk);
    tma_prefetch(&tvt);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (T <= 0) {
    // nothing to do (cannot happen with the host's grid); keep the dealloc path uniform
  } else if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const int slot = __ldg(a.kv_index + row);
      mbar_expect_tx(kv_full, A::K_BYTES + A::V_BYTES);
      for (int kb = 0; kb < A::KQ; ++kb)
        tma_load_2d(sK + kb * XK * 128, &tk, kv_full, a.kcol0 + head * D + kb * 64, slot * a.Lk);
      for (int h = 0; h < 2; ++h)
        tma_load_2d(sV + h * A::NPV * 128, &tvt, kv_full, slot * a.vt_slot + h * 64, a.vrow0 + head * D);
      for (int t = 0; t < T; ++t) {
        const int b = t & 1;
        if (t >= 2) mbar_wait_sleep(&q_empty[b], ((t >> 1) - 1) & 1);
        mbar_expect_tx(&q_full[b], A::Q_BYTES);
        for (int kb = 0; kb < A::KQ; ++kb)
          tma_load_2d(sQ + b * A::Q_BYTES + kb * 128 * 128, &tq, &q_full[b], a.qcol0 + head * D + kb * 64,
                      tok0 + (t0 + t) * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id_s = make_idesc16(128, XK, F16);
      constexpr uint32_t id_pv = make_idesc16(128, A::NPV, F16);
      mbar_wait(kv_ready, 0);
      tc_fence_after();
      const uint32_t ak = smem_u32(sK), av = smem_u32(sV);
      for (int t = 0; t <= T; ++t) {
        if (t < T) {
          // S_t into buffer t mod 2: P_{t−2} there was consumed by the PV MMA issued in iteration t − 1,
          // which executes before this one
          const int b = t & 1;
          mbar_wait_sleep(&q_full[b], (t >> 1) & 1);
          tc_fence_after();
          const uint32_t aq = smem_u32(sQ + b * A::Q_BYTES);
#pragma unroll
          for (int k = 0; k < A::K16; ++k) {
            const uint32_t offq = (k >> 2) * (128 * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (XK * 128) + (k & 3) * 32;
            umma_bf16(tmem + b * A::S_STRIDE, make_sdesc_sw128(aq + offq), make_sdesc_sw128(ak + offk), id_s,
                      k > 0);
          }
          umma_commit(&s_full[b]);
          umma_commit(&q_empty[b]);
        }
        if (t >= 1) {
          const int tp = t - 1, pb = tp & 1;
          mbar_wait_sleep(&p_full[pb], (tp >> 1) & 1);
          if (tp >= 1) mbar_wait_sleep(o_empty, (tp - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < XK / 16; ++k) {  // 80 keys = 5 k-steps of 16; A = P (8 packed columns per k-step)
            const uint32_t offv = (k >> 2) * (A::NPV * 128) + (k & 3) * 32;
            mma_ts(tmem + A::O_COL, tmem + pb * A::S_STRIDE + k * 8, make_sdesc_sw128(av + offv), id_pv, k != 0);
          }
          umma_commit(o_full);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax + epilogue: two threads per query row, 40 keys each ----------------
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    if (h == 0) {
      // zero K's columns [D, 16·K16) (the next head's channels) so that Q's junk there multiplies zeros
      mbar_wait(kv_full, 0);
      if (D % 16) {
        uint8_t* krow = sK + (D / 64) * XK * 128 + r * 128;
        if (r < XK)
          for (int c = (D % 64) / 8; c < (A::NPV % 64 ? A::NPV % 64 : 64) / 8; ++c)
            *reinterpret_cast<uint4*>(krow + ((c ^ (r & 7)) << 4)) = make_uint4(0, 0, 0, 0);
        fence_proxy_async_smem();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(kv_ready);
    }
    float l_prev = 1.f;
    const int valid = a.Lk - h * 40;  // keys of this thread's 40 columns that exist (warp-uniform)
    for (int t = 0; t <= T; ++t) {
      float l_cur = 1.f;
      uint32_t pk[20];
      const int b = t & 1;
      if (t < T) {
        mbar_wait_sleep(&s_full[b], (t >> 1) & 1);
        tc_fence_after();
        uint32_t s[40];
        uint32_t(&s0)[32] = reinterpret_cast<uint32_t(&)[32]>(s[0]);
        uint32_t(&s1)[8] = reinterpret_cast<uint32_t(&)[8]>(s[32]);
        const uint32_t sa = tmem + lane_base + b * A::S_STRIDE + h * 40;
        tmem_ld32_nw(sa, s0);
        ld8(sa + 32, s1);
        tmem_wait_ld_tied(s0);
        wait_ld();
        float mx = -FLT_MAX;
#pragma unroll
        for (int i = 0; i < 40; ++i) {
          if (i >= valid) s[i] = __float_as_uint(-INFINITY);
          mx = fmaxf(mx, __uint_as_float(s[i]));
        }
        sX[(b * 2 + h) * 128 + r] = mx;
        named_bar_sync(1 + q, 64);
        mx = fmaxf(mx, sX[(b * 2 + (h ^ 1)) * 128 + r]);
        const float ms = mx * a.scale_log2;
        float sum = 0.f;
        // exponentials only for the 8-key chunks that hold valid keys (valid is warp-uniform)
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          if (c * 8 < valid) {
#pragma unroll
            for (int i = c * 4; i < c * 4 + 4; ++i) {
              const float p0 = ex2f(fmaf(__uint_as_float(s[2 * i]), a.scale_log2, -ms));
              const float p1 = ex2f(fmaf(__uint_as_float(s[2 * i + 1]), a.scale_log2, -ms));
              sum += p0 + p1;
              pk[i] = pack16(p0, p1, F16);
            }
          } else {
#pragma unroll
            for (int i = c * 4; i < c * 4 + 4; ++i) pk[i] = 0u;
          }
        }
        l_cur = sum;
      }
      if (t >= 1) {
        // epilogue of tile t − 1: O / l → 16-bit rows of O (before P_t is published, so the PV MMA of
        // tile t cannot overwrite O while it is read)
        const int tp = t - 1;
        mbar_wait_sleep(o_full, tp & 1);
        tc_fence_after();
        const float inv = 1.f / l_prev;
        const int qi = (t0 + tp) * 128 + r;
        bf16* orow = a.O + (long)(tok0 + qi) * a.ldo + head * D;
#pragma unroll
        for (int c = 0; c < A::NPV / 16; ++c) {
          if (c % 2 != h) continue;
          uint32_t o[16];
          ld16(tmem + lane_base + A::O_COL + c * 16, o);
          wait_ld();
          if (qi < a.P) {
#pragma unroll
            for (int i = 0; i < 16; i += 8) {
              const int col = c * 16 + i;
              if (col + 8 <= D)
                *reinterpret_cast<uint4*>(orow + col) =
                    make_uint4(pack16(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv, F16),
                               pack16(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv, F16),
                               pack16(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv, F16),
                               pack16(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv, F16));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty);
      }
      if (t < T) {
        // P_t in place over this thread's S columns: packed keys [40h, 40h + 40) → columns [20h, 20h + 20)
        uint32_t(&pa)[16] = reinterpret_cast<uint32_t(&)[16]>(pk[0]);
        uint32_t(&pc)[4] = reinterpret_cast<uint32_t(&)[4]>(pk[16]);
        const uint32_t pa_addr = tmem + lane_base + b * A::S_STRIDE + h * 20;
        // the partner half may still be reading its S columns [40, 80) — they overlap P's [20, 40) only for
        // h = 1 writing over keys 20..39 of h = 0, which h = 0 read before the max exchange above
        st16(pa_addr, pa);
        st4(pa_addr + 16, pc);
        wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        // row sum of both halves (the exchange slots of buffer b are free again: the partner read the max)
        named_bar_sync(1 + q, 64);
        sX[(b * 2 + h) * 128 + r] = l_cur;
        named_bar_sync(1 + q, 64);
        l_cur += sX[(b * 2 + (h ^ 1)) * 128 + r];
      }
      l_prev = l_cur;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

void make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
                  uint32_t box_out, bool is_f16, bool swz64 = false);

template <int D, bool F16>
static void launch_x(const void* q, const void* kc, int ldk, long n_slots, int kcol, const void* vtc, long vt_rows,
                     long ld_keys, int vrow, const int* kv_index, int Lk, void* O, int rows, int heads, int C, int P,
                     cudaStream_t st) {
  using A = XA<D>;
  static bool set = false;
  if (!set) {
    SD_CUDA(cudaFuncSetAttribute(xattn_tc_kernel<D, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM));
    set = true;
  }
  CUtensorMap mq, mk, mvt;
  make_tmap_2d(&mq, q, (uint64_t)C, (uint64_t)rows * P, (uint64_t)C * 2, 64, 128, F16);
  make_tmap_2d(&mk, kc, (uint64_t)ldk, (uint64_t)n_slots * Lk, (uint64_t)ldk * 2, 64, XK, F16);
  make_tmap_2d(&mvt, vtc, (uint64_t)ld_keys, (uint64_t)vt_rows, (uint64_t)ld_keys * 2, 64, A::NPV, F16);
  const int ntiles = (P + 127) / 128;
  // enough CTAs for ~2 resident per SM over the (row, head) pairs; each walks a contiguous run of
  // query tiles
  const long pairs = (long)rows * heads;
  int per = (int)std::max<long>(1, (long)ntiles * pairs / (2L * stream_sms(st)));
  per = std::min(per, ntiles);
  XArgs a;
  a.O = static_cast<bf16*>(O);
  a.ldo = C;
  a.P = P;
  a.Lk = Lk;
  a.vt_slot = (Lk + 7) / 8 * 8;
  a.tiles_per_cta = per;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  a.qcol0 = 0;
  a.kcol0 = kcol;
  a.vrow0 = vrow;
  a.kv_index = kv_index;
  launch_k(xattn_tc_kernel<D, F16>, dim3((ntiles + per - 1) / per, heads, rows), 320, (size_t)A::SMEM, st, mq, mk, mvt,
           a);
  SD_CHECK_LAUNCH();
}

bool xattention_tc2_supported(int d, int Lk) { return (d == 40 || d == 64 || d == 80) && Lk <= XK; }

template <bool F16>
static void xattn2(const void* q, const void* kc, int ldk, long n_slots, int kcol, const void* vtc, long vt_rows,
                   long ld_keys, int vrow, const int* kv_index, int Lk, void* O, int rows, int heads, int d, int C,
                   int P, cudaStream_t st) {
  switch (d) {
    case 40: launch_x<40, F16>(q, kc, ldk, n_slots, kcol, vtc, vt_rows, ld_keys, vrow, kv_index, Lk, O, rows, heads, C, P, st); break;
    case 64: launch_x<64, F16>(q, kc, ldk, n_slots, kcol, vtc, vt_rows, ld_keys, vrow, kv_index, Lk, O, rows, heads, C, P, st); break;
    case 80: launch_x<80, F16>(q, kc, ldk, n_slots, kcol, vtc, vt_rows, ld_keys, vrow, kv_index, Lk, O, rows, heads, C, P, st); break;
    default: throw CudaError("xattention_tc2: head dim must be 40, 64 or 80");
  }
}

void xattention_tc2(const bf16* q, const bf16* kc, int ldk, long n_slots, int kcol, const bf16* vtc, long vt_rows,
                    long ld_keys, int vrow, const int* kv_index, int Lk, bf16* O, int rows, int heads, int d, int C,
                    int P, cudaStream_t st) {
  xattn2<false>(q, kc, ldk, n_slots, kcol, vtc, vt_rows, ld_keys, vrow, kv_index, Lk, O, rows, heads, d, C, P, st);
}
void xattention_tc2(const f16* q, const f16* kc, int ldk, long n_slots, int kcol, const f16* vtc, long vt_rows,
                    long ld_keys, int vrow, const int* kv_index, int Lk, f16* O, int rows, int heads, int d, int C,
                    int P, cudaStream_t st) {
  xattn2<true>(q, kc, ldk, n_slots, kcol, vtc, vt_rows, ld_keys, vrow, kv_index, Lk, O, rows, heads, d, C, P, st);
}

}  // namespace sd
