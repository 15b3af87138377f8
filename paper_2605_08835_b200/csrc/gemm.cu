// tcgen05 / TMEM / TMA GEMM and implicit-GEMM 3x3 convolution for sm_100a.
//
// One persistent, warp-specialised kernel template gemm_kernel<BN, CG, MODE> (MODE = dense / conv3):
//   warp 0      TMA producer   (one elected lane): A and B tiles into a STAGES-deep smem ring
//   warp 1      MMA issuer     (one elected lane of the leader CTA): tcgen05.mma into a
//                              double-buffered TMEM accumulator; also owns TMEM alloc/dealloc
//   warps 2..   epilogue       tcgen05.ld → bias / temb / act / residual → bf16|fp32 stores (8 warps for
//                              conv3, 16 for dense: 2 or 4 per TMEM lane quarter)
// CG = 1: one CTA computes a 128×BN tile.
// CG = 2: a CTA pair (cluster of 2, cta_group::2) computes a 256×BN tile: each CTA loads its 128
//         rows of A and half of B, the leader issues 256×BN×16 MMAs reading both CTAs' smem, and
//         each CTA drains its 128 accumulator rows from its own TMEM. Per-SM operand traffic per
//         FLOP drops by (1/BN + 1/128) → (1/BN + 1/256) — the lever against the L2 bandwidth wall.
// smem operands are K-major with the 128-byte swizzle written by TMA and described to the tensor
// core by SWIZZLE_128B UMMA descriptors (8-row groups 1024 B apart).
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace sd {

struct GemmArgs {
  int mode;
  int M, N;
  int B, H, W, wt, ht, bt, tiles_x, tiles_y;
  int stride;         // conv3: input pixel = stride·output pixel + tap offset
  int kb_src[2];      // K blocks (of 64 channels) per tap for each source
  int nsrc;
  int num_kb;         // K blocks per tile
  int m_tiles, n_tiles, m_tile_begin;   // m_tiles counts tiles of 128*CG rows
  void* out;
  int ldo, col_off, out_f32;
  const float* bias;
  int bias_per_row;
  float alpha;
  const float* temb;
  int ld_temb, rows_per_img;
  const bf16* res;
  int ldr;
  int act;
  int tma_store;      // bf16 output through the per-warp smem slab + TMA store
  int res_tma;        // dense: the residual sub-tile arrives by TMA in the staging slab (coalesced)
  int gelu_tanh;      // GEGLU: tanh form of GELU on MUFU tanh.approx (default; SD_GELU_TANH=0 = erf form)
  int f16;            // 16-bit operands / outputs are fp16 (SD_PREC_FP16) instead of bf16
  int dbg;            // experiment switch (SD_EPI_DBG): 1 = no store, 2 = no bias, 3 = no TMEM load
  int splits, kps;    // split-K: K blocks [s·kps, (s+1)·kps) of split s
  float* part;        // split-K fp32 partials [splits][M][N] (raw accumulators)
  // GroupNorm statistics of the stored output (the consumer's GN skips its statistics pass): per
  // 32-pixel output quarter ("slot", wholly inside one image) and channel, (Σy, Σy²) over the quarter's
  // 32 stored 16-bit values → gn_part[(img · gn_slots + slot) · N + n] (float2). Slot of a conv quarter
  // box sw × sh at (x, y): (y / sh) · (W / sw) + x / sw; of a dense quarter: (row mod gn_P) / 32.
  float2* gn_part;
  int gn_P, gn_slots, gn_sw, gn_sh;
  // NH = 2 (BN = 320) tail balancing: work units u < full_units are whole tiles; the last tiles (one
  // partial wave) are split into their two 160-column N-halves, units full_units + 2i + h → tile
  // full_units + i, half h. The same N = 160 MMAs over the same K blocks either way: bitwise identical.
  int full_units, total_units;
  const float2* ln_stat;  // folded LayerNorm (GemmDescT::ln_stat)
  const float* ln_wbar;
  int ln_cols;
};

// folded LayerNorm: o ← rstd·(o − μ·w̄) for the 32 columns [col, col + 32) of this lane's row (before the bias)
__device__ __forceinline__ void ln_correct32(const GemmArgs& g, float* o, long prow, bool valid, int col) {
  if (!g.ln_cols) {
    const float2 st = valid ? __ldg(g.ln_stat + prow) : make_float2(0.f, 0.f);
    if (col + 32 <= g.N) {
      const float4* w4 = reinterpret_cast<const float4*>(g.ln_wbar + col);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 w = __ldg(w4 + i);
        o[4 * i] = st.y * fmaf(-st.x, w.x, o[4 * i]);
        o[4 * i + 1] = st.y * fmaf(-st.x, w.y, o[4 * i + 1]);
        o[4 * i + 2] = st.y * fmaf(-st.x, w.z, o[4 * i + 2]);
        o[4 * i + 3] = st.y * fmaf(-st.x, w.w, o[4 * i + 3]);
      }
    } else {
      for (int i = 0; i < 32 && col + i < g.N; ++i) o[i] = st.y * fmaf(-st.x, __ldg(g.ln_wbar + col + i), o[i]);
    }
  } else {
    const float wb = valid ? __ldg(g.ln_wbar + prow) : 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float2 st = col + i < g.N ? __ldg(g.ln_stat + col + i) : make_float2(0.f, 0.f);
      o[i] = st.y * fmaf(-st.x, wb, o[i]);
    }
  }
}

// work unit u → tile index and N-half selector (−1 = whole tile; 0 / 1 = that 160-column half)
__device__ __forceinline__ int decode_unit(const GemmArgs& g, int u, int& hsel) {
  if (u < g.full_units) {
    hsel = -1;
    return u;
  }
  hsel = (u - g.full_units) & 1;
  return g.full_units + ((u - g.full_units) >> 1);
}

// tile t → (M tile, N tile, K-block range); tiles of split s follow those of split s-1
__device__ __forceinline__ void decode_tile(const GemmArgs& g, int t, int& mt, int& nt, int& s, int& kb0, int& kb1) {
  const int per = g.m_tiles * g.n_tiles;
  s = t / per;
  const int r = t - s * per;
  mt = g.m_tile_begin + r / g.n_tiles;
  nt = r % g.n_tiles;
  kb0 = s * g.kps;
  kb1 = min(g.num_kb, kb0 + g.kps);
}

template <int BN, int CG, int EPW = 8>
struct Cfg {
  static constexpr int BM = 128, BK = 64;
  // BN = 320 (conv3, CTA pairs): two N = 160 MMAs per k-step share the A operand — A is read from smem
  // once per 320 output columns instead of once per 160 (the N = 160 tiles were operand-bandwidth bound:
  // tensor pipe ~51 %, with the MMA warp never waiting on data or the epilogue)
  static constexpr int NH = BN > 256 ? 2 : 1;                    // MMA N-halves per k-step
  static constexpr int MMA_N = BN / NH;
  static constexpr int A_BYTES = BM * BK * 2;                    // 16 KB (this CTA's rows)
  static constexpr int B_ROWS = BN / CG;                         // B rows loaded by this CTA
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // EPW epilogue warps (8, or 16 for the short-K dense GEMMs whose epilogue is the critical path), each
  // with 2 × 2 KB staging slabs; the operand ring gets the rest of 224 KB
  static constexpr int STAGING = EPW * 2 * 2048;
  static constexpr int RING = 224 * 1024 - STAGING;
  static constexpr int STAGES = RING / STAGE > 8 ? 8 : RING / STAGE;
  static constexpr int TMEM_STRIDE = BN <= 64 ? 64 : (BN <= 128 ? 128 : (BN <= 256 ? 256 : BN));
  static constexpr int NACC = 2 * TMEM_STRIDE <= 512 ? 2 : 1;    // double-buffered accumulator if it fits
  static constexpr int TMEM_COLS = NACC == 2 ? 2 * TMEM_STRIDE : 512;
  static constexpr int SMEM = 1024 + STAGES * STAGE + STAGING + 1024;
  static_assert(B_BYTES % 1024 == 0, "B tile must be a whole number of 8-row swizzle groups");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA rank 0 of the cluster
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}

template <int CG>
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, uint64_t* bar, uint32_t bar_l, int c0, int c1) {
  if (CG == 1) {
    tma_load_2d(dst, m, bar, c0, c1);
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_l), "r"(c0), "r"(c1)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, uint32_t bar_l, int c0, int c1,
                                     int c2) {
  if (CG == 1) {
    tma_load_3d(dst, m, bar, c0, c1, c2);
  } else {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_l), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, uint32_t bar_l, int c0, int c1,
                                     int c2, int c3) {
  if (CG == 1) {
    tma_load_4d(dst, m, bar, c0, c1, c2, c3);
  } else {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_l), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (CG == 1) {
    umma_bf16(d, a, b, idesc, acc);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}
// commit → arrive on `bar` (CG = 2: on the barrier at the same offset in both CTAs of the pair)
template <int CG>
__device__ __forceinline__ void commit(uint64_t* bar) {
  if (CG == 1) {
    umma_commit(bar);
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* dst, uint32_t ncols) {
  if (CG == 1) {
    tmem_alloc(dst, ncols);
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t ncols) {
  if (CG == 1)
    tmem_dealloc(taddr, ncols);
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// ---- epilogue --------------------------------------------------------------------------------
// Each epilogue warp owns 32 accumulator rows (its TMEM lane quarter). Per 32-column chunk:
// tcgen05.ld → fp32 math (α, bias, temb, act, residual) → bf16 → a 2 KB per-warp staging slab in
// smem (64-byte rows, 64B swizzle) → one TMA store of the 32×32 sub-tile (coalesced, clipped to the
// tensor bounds by the hardware). fp32 outputs (ε, temb projections) use direct stores.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// (Σy, Σy²) per column of a staged 32×32 16-bit sub-tile (64-byte rows, 64B swizzle as written by
// stage_store): lane (h, w) reads the column pair w (channels 2w, 2w+1) of rows 2k + h, k = 0..15 — the
// two rows of one LDS are the two halves of one 128-byte line, so every load is bank-conflict free — then
// one xor-16 exchange; lanes 0..15 store (S_2w, Q_2w, S_2w+1, Q_2w+1). Fixed order: deterministic.
template <bool F16>
__device__ __forceinline__ void gn_colstats(const uint8_t* buf, int lane, float2* dst) {
  const int h = lane >> 4, w = lane & 15;
  float s0 = 0.f, s1 = 0.f, q0 = 0.f, q1 = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int r = 2 * k + h;
    const uint32_t u = *reinterpret_cast<const uint32_t*>(buf + r * 64 + (((w >> 2) ^ (k & 3)) << 4) + (w & 3) * 4);
    float a, b;
    if (F16) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u));
      a = f.x, b = f.y;
    } else {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
      a = f.x, b = f.y;
    }
    s0 += a;
    s1 += b;
    q0 = fmaf(a, a, q0);
    q1 = fmaf(b, b, q1);
  }
  s0 += __shfl_xor_sync(0xffffffff, s0, 16);
  s1 += __shfl_xor_sync(0xffffffff, s1, 16);
  q0 += __shfl_xor_sync(0xffffffff, q0, 16);
  q1 += __shfl_xor_sync(0xffffffff, q1, 16);
  if (lane < 16) reinterpret_cast<float4*>(dst)[w] = make_float4(s0, q0, s1, q1);
}

struct EpiCtx {
  uint8_t* stage;   // this warp's 2 × 2 KB staging slabs
  int slot;         // alternating slab
  int sx, sy, sb;   // this warp's slab origin (conv: pixel coords; dense: row in sx)
  uint64_t* rbar;   // this warp's 2 residual-arrival barriers (one per slab)
  uint32_t rph;     // their phase bits
};

// write 32 fp32 values (this lane's row, columns [col, col+32)) to the staging slab and TMA-store it
template <int MODE, bool F16>
__device__ __forceinline__ void stage_store(const GemmArgs& g, const CUtensorMap* om, EpiCtx& ec, const float* o,
                                            int col, int lane, bool slab_ready = false, float2* gn_dst = nullptr) {
  uint8_t* buf = ec.stage + ec.slot * 2048;
  if (!slab_ready) {
    if (lane == 0) bulk_wait_read<1>();    // the store issued two chunks ago has finished reading
    __syncwarp();
  }
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 v = make_uint4(pack16(o[8 * c], o[8 * c + 1], F16), pack16(o[8 * c + 2], o[8 * c + 3], F16),
                               pack16(o[8 * c + 4], o[8 * c + 5], F16), pack16(o[8 * c + 6], o[8 * c + 7], F16));
    *reinterpret_cast<uint4*>(buf + lane * 64 + ((c ^ sw) << 4)) = v;
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (MODE == GEMM_DENSE)
      tma_store_2d(om, buf, col, ec.sx);
    else
      tma_store_4d(om, buf, col, ec.sx, ec.sy, ec.sb);
    bulk_commit();
  }
  if (gn_dst) gn_colstats<F16>(buf, lane, gn_dst);  // the slab is only read: concurrent with the TMA store
  ec.slot ^= 1;
}

// o[0..32) += p[0..32) with 16-byte read-only loads (p 16-byte aligned: bias / temb rows are)
__device__ __forceinline__ void add32(float* o, const float* p) {
  const float4* p4 = reinterpret_cast<const float4*>(p);
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __ldg(p4 + i);  // all loads in flight before the adds
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    fadd2(o[4 * i], o[4 * i + 1], v[i].x, v[i].y);
    fadd2(o[4 * i + 2], o[4 * i + 3], v[i].z, v[i].w);
  }
}

// residual of 32 columns of one row (16-byte read-only loads)
__device__ __forceinline__ void res_load32(uint4 (&r)[4], const bf16* rp) {
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = __ldg(reinterpret_cast<const uint4*>(rp) + i);
}

// `tfull` / `tphase`: the accumulator-ready barrier of this tile
// NW epilogue warps share each TMEM lane quarter; warp `half` (0 … NW−1) takes the 32-column chunks
// c ≡ half (mod NW)
template <int BN, int MODE, bool F16, int NW>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& g, const CUtensorMap* om, const CUtensorMap* res_map,
                                              EpiCtx& ec, uint32_t tbase,
                                              int mbox, int n0, int q, int lane, int half, int split, uint64_t* tfull,
                                              uint32_t tphase, int c_lo = 0, int c_hi = BN / 32) {
  // chunks [c_lo, c_hi) of the tile; chunk c's accumulator columns start at tbase + (c − c_lo)·32
  const int r = q * 32 + lane;
  long prow;
  int img;
  bool valid;
  if (MODE == GEMM_DENSE) {
    prow = (long)mbox * 128 + r;
    valid = prow < g.M;
    img = (int)(prow / g.rows_per_img);
    ec.sx = mbox * 128 + q * 32;
  } else {
    const int tx = mbox % g.tiles_x;
    const int ty = (mbox / g.tiles_x) % g.tiles_y;
    const int tb = mbox / (g.tiles_x * g.tiles_y);
    const int xx = tx * g.wt + r % g.wt;
    const int yy = ty * g.ht + (r / g.wt) % g.ht;
    const int bb = tb * g.bt + r / (g.wt * g.ht);
    valid = xx < g.W && yy < g.H && bb < g.B;
    prow = ((long)bb * g.H + yy) * g.W + xx;
    img = bb;
    const int r0 = q * 32;
    ec.sx = tx * g.wt + r0 % g.wt;
    ec.sy = ty * g.ht + (r0 / g.wt) % g.ht;
    ec.sb = tb * g.bt + r0 / (g.wt * g.ht);
  }
  // GN statistics slot of this warp's 32-row quarter (warp-uniform; the host checked that a quarter
  // never straddles two images and that whole quarters are in or out of range)
  int gq_img = 0, gq_slot = 0;
  bool gq_valid = false;
  if (g.gn_part) {
    if (MODE == GEMM_DENSE) {
      const long r0 = (long)mbox * 128 + q * 32;
      gq_valid = r0 < g.M;
      gq_img = (int)(r0 / g.gn_P);
      gq_slot = (int)(r0 - (long)gq_img * g.gn_P) >> 5;
    } else {
      gq_valid = ec.sb < g.B;
      gq_img = ec.sb;
      gq_slot = (ec.sy / g.gn_sh) * (g.W / g.gn_sw) + ec.sx / g.gn_sw;
    }
  }
  mbar_wait(tfull, tphase);
  tc_fence_after();
  if (g.act == ACT_GEGLU) {
    // columns [128j, 128j+64) = value, [128j+64, 128j+128) = gate; output width BN/2
#pragma unroll 1
    for (int ci = half; ci < 2 * (BN / 128); ci += NW) {  // (128-column group j, 32-column half h) items
      const int j = ci >> 1, h = ci & 1;
      {
        uint32_t rv[32], rg[32];
        const int cv = j * 128 + h * 32, cgc = cv + 64;
        tmem_ld32(tbase + cv, rv);
        tmem_ld32(tbase + cgc, rg);
        const int ocol = (n0 >> 1) + j * 64 + h * 32;
        if (ocol >= (g.N >> 1)) continue;  // warp-uniform
        float o[32];
        float vv[32], gg[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          vv[i] = __uint_as_float(rv[i]) * g.alpha;
          gg[i] = __uint_as_float(rg[i]) * g.alpha;
        }
        if (g.ln_stat) {
          ln_correct32(g, vv, prow, valid, n0 + cv);
          ln_correct32(g, gg, prow, valid, n0 + cgc);
        }
        if (g.bias) {
          add32(vv, g.bias + n0 + cv);
          add32(gg, g.bias + n0 + cgc);
        }
        if (g.gelu_tanh) {
          // GELU(x) ≈ ½x(1 + tanh(√(2/π)(x + 0.044715x³))): |Δ| ≤ 4.7e-4 from the erf form, plus the
          // tanh.approx error (≤ ½|x|·2^-10.9 absolute; not below an ulp for negative x, DESIGN R33); 6 instructions instead
          // of the 15 of the erf polynomial (the FF1 epilogue was issue-bound: 64 % issue, 36 % tensor
          // pipe) → FF1 at 64×64: 135 → 109 µs
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = gg[i];
            const float u = x * fmaf(0.0356774081f * x, x, 0.7978845608f);  // √(2/π)·(x + 0.044715·x³)
            float t;
            asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
            const float hx = 0.5f * x;
            o[i] = vv[i] * fmaf(hx, t, hx);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = vv[i] * gelu_f(gg[i]);
        }
        if (g.res && valid) {
          const bf16* rp = g.res + prow * g.ldr + ocol;
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] += cvt16(rp[i], F16);
        }
        stage_store<MODE, F16>(g, om, ec, o, ocol, lane);
      }
    }
    return;
  }
#pragma unroll 1
  for (int c = c_lo + (half - c_lo % NW + NW) % NW; c < c_hi; c += NW) {  // NW warps per lane quarter: c ≡ half
    uint32_t rv[32];
    const bool rt = g.res_tma && n0 + c * 32 < g.N;  // warp-uniform
    if (rt) {
      // the slab is free once the store issued from it two chunks ago has read it; the 32×32 residual
      // sub-tile then lands in it (same 64B swizzle as the output box) while the accumulator is read
      if (lane == 0) {
        bulk_wait_read<1>();
        mbar_expect_tx(&ec.rbar[ec.slot], 2048);
        tma_load_2d(ec.stage + ec.slot * 2048, res_map, &ec.rbar[ec.slot], n0 + c * 32, ec.sx);
      }
      __syncwarp();
    }
    const int col = n0 + c * 32;
    // the chunk's bias (one 128-byte row, the same for every lane: L1 broadcast) is requested before the
    // accumulator read, so its latency overlaps the TMEM load instead of following it (measured on
    // [65536, 320, 320]: skipping the bias entirely saved 13 % of the kernel — the serial LDG chain)
    const bool pre_b = g.bias && !g.bias_per_row && g.dbg != 2 && col + 32 <= g.N && g.splits == 1;
    float4 bv[8];
    if (pre_b) {
      const float4* b4 = reinterpret_cast<const float4*>(g.bias + col);
#pragma unroll
      for (int i = 0; i < 8; ++i) bv[i] = __ldg(b4 + i);
    }
    if (g.dbg != 3) {
      tmem_ld32(tbase + (c - c_lo) * 32, rv);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) rv[i] = 0;
    }
    if (col >= g.N) continue;  // warp-uniform
    if (g.splits > 1) {
      // split-K: raw fp32 partial sums; bias / temb / act / residual are applied by splitk_reduce
      if (valid) {
        float* pp = g.part + ((long)split * g.M + prow) * g.N + col;
        if (col + 32 <= g.N) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(pp)[i] =
                make_float4(__uint_as_float(rv[4 * i]), __uint_as_float(rv[4 * i + 1]),
                            __uint_as_float(rv[4 * i + 2]), __uint_as_float(rv[4 * i + 3]));
        } else {
          for (int i = 0; i < 32 && col + i < g.N; ++i) pp[i] = __uint_as_float(rv[i]);
        }
      }
      continue;
    }
    float o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(rv[i]);
    if (g.alpha != 1.f) {  // warp-uniform; most GEMMs have α = 1
#pragma unroll
      for (int i = 0; i < 32; i += 2) fmul2(o[i], o[i + 1], g.alpha, g.alpha);
    }
    const bool full32 = col + 32 <= g.N;
    if (g.ln_stat) ln_correct32(g, o, prow, valid, col);
    if (pre_b) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        fadd2(o[4 * i], o[4 * i + 1], bv[i].x, bv[i].y);
        fadd2(o[4 * i + 2], o[4 * i + 3], bv[i].z, bv[i].w);
      }
    } else if (g.bias && g.dbg != 2) {
      if (g.bias_per_row) {
        const float bv = valid ? g.bias[prow] : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] += bv;
      } else if (full32) {
        add32(o, g.bias + col);
      } else {
        for (int i = 0; i < 32 && col + i < g.N; ++i) o[i] += __ldg(g.bias + col + i);
      }
    }
    if (g.temb && valid) {
      const float* tp = g.temb + (long)img * g.ld_temb + col;
      if (full32) {
        add32(o, tp);
      } else {
        for (int i = 0; i < 32 && col + i < g.N; ++i) o[i] += __ldg(tp + i);
      }
    }
    if (g.act == ACT_SILU) {
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = silu_f(o[i]);
    }
    if (rt) {
      mbar_wait(&ec.rbar[ec.slot], (ec.rph >> ec.slot) & 1);
      ec.rph ^= 1u << ec.slot;
      const uint8_t* buf = ec.stage + ec.slot * 2048;
      const int sw = (lane >> 1) & 3;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 u = *reinterpret_cast<const uint4*>(buf + lane * 64 + ((i ^ sw) << 4));
        const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
        for (int k = 0; k < 8; k += 2)
          fadd2(o[8 * i + k], o[8 * i + k + 1], cvt16(e[k], F16), cvt16(e[k + 1], F16));
      }
    } else if (g.res && valid) {
      const bf16* rp = g.res + prow * g.ldr + col;
      if (full32) {
        uint4 u4[4];
        res_load32(u4, rp);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bf16* e = reinterpret_cast<const bf16*>(&u4[i]);
#pragma unroll
          for (int k = 0; k < 8; ++k) o[8 * i + k] += cvt16(e[k], F16);
        }
      } else {
        for (int i = 0; i < 32 && col + i < g.N; ++i) o[i] += cvt16(rp[i], F16);
      }
    }
    if (g.dbg == 1) {
      if (o[0] == 12345.f) g.res ? (void)0 : __trap();
    } else if (g.tma_store) {
      float2* gd = nullptr;
      if (g.gn_part && gq_valid) gd = g.gn_part + ((long)gq_img * g.gn_slots + gq_slot) * g.N + col;
      stage_store<MODE, F16>(g, om, ec, o, col, lane, rt, gd);
    } else if (valid) {
      if (g.out_f32) {
        float* op = reinterpret_cast<float*>(g.out) + prow * g.ldo + g.col_off + col;
        if (full32 && ((g.ldo | g.col_off) & 3) == 0) {
          float4* o4 = reinterpret_cast<float4*>(op);
#pragma unroll
          for (int i = 0; i < 8; ++i) o4[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        } else {
          for (int i = 0; i < 32 && col + i < g.N; ++i) op[i] = o[i];
        }
      } else {
        bf16* op = reinterpret_cast<bf16*>(g.out) + prow * g.ldo + g.col_off + col;
        if (full32 && ((g.ldo | g.col_off) & 7) == 0) {
          uint4* o4 = reinterpret_cast<uint4*>(op);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            o4[i] = make_uint4(pack16(o[8 * i], o[8 * i + 1], F16), pack16(o[8 * i + 2], o[8 * i + 3], F16),
                               pack16(o[8 * i + 4], o[8 * i + 5], F16), pack16(o[8 * i + 6], o[8 * i + 7], F16));
        } else {
          for (int i = 0; i < 32 && col + i < g.N; ++i) op[i] = to16(o[i], F16);
        }
      }
    }
  }
}

template <int BN, int CG, int MODE, bool F16, int EPW>
__global__ void __launch_bounds__(64 + 32 * EPW, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                const __grid_constant__ CUtensorMap tb0, const __grid_constant__ CUtensorMap tb1,
                const __grid_constant__ CUtensorMap tout, const __grid_constant__ CUtensorMap tres,
                const GemmArgs g) {
  using C = Cfg<BN, CG, EPW>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (SWIZZLE_128B atoms); offsetting the shared array itself keeps the pointer in the
  // shared state space, so the compiler emits STS / LDS rather than generic ST / LD
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sStage = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + C::STAGING);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 3;  // 2 accumulators, or 3 rotating 160-column halves (NH = 2)
  uint64_t* rbar = tempty + 3;  // [EPW epilogue warps][2 slabs]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2 * EPW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPW * CG);
    }
    for (int s = 0; s < 2 * EPW; ++s) mbar_init(&rbar[s], 1);
    fence_mbar_init();
    tma_prefetch(&ta0);
    tma_prefetch(&tb0);
    if (g.nsrc > 1) {
      tma_prefetch(&ta1);
      tma_prefetch(&tb1);
    }
    if (g.res_tma) tma_prefetch(&tres);
  }
  if (warp == 1) tmem_alloc_cg<CG>(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // barrier init, TMEM alloc and descriptor prefetch above overlapped the previous grid (PDL)

  const int total = g.total_units;
  const int worker = blockIdx.x / CG, nworkers = gridDim.x / CG;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (both CTAs of a pair load their halves) =================
      int stage = 0;
      uint32_t phase = 0;
      for (int u = worker; u < total; u += nworkers) {
        int hsel;
        const int t = decode_unit(g, u, hsel);
        int mt, nt, sp, kb0, kb1;
        decode_tile(g, t, mt, nt, sp, kb0, kb1);
        const int mbox = mt * CG + (int)rank;  // this CTA's 128-row box
        const int n0 = nt * BN + (int)rank * C::B_ROWS;
        int m0 = 0, x0 = 0, y0 = 0, b0 = 0;
        if (MODE == GEMM_DENSE) {
          m0 = mbox * C::BM;
        } else {
          const int tx = mbox % g.tiles_x;
          const int ty = (mbox / g.tiles_x) % g.tiles_y;
          const int tb = mbox / (g.tiles_x * g.tiles_y);
          x0 = tx * g.wt;
          y0 = ty * g.ht;
          b0 = tb * g.bt;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint32_t bar_l = 0;
          // experiment switches (SD_EPI_DBG; results are garbage): 5 = B loaded only for a tile's first K
          // block, 6 = A only for the first — how much of the time the operand feed of each costs
          const bool skipB = g.dbg == 5 && kb != kb0, skipA = g.dbg == 6 && kb != kb0;
          const int bytes = C::STAGE - (skipB ? C::B_BYTES : 0) - (skipA ? C::A_BYTES : 0) -
                            (hsel >= 0 && !skipB ? C::B_BYTES / 2 : 0);  // a half unit loads one N-half of B
          if (CG == 1) {
            mbar_expect_tx(&full[stage], bytes);
          } else {
            bar_l = leader_addr(&full[stage]);
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * bytes);
          }
          void* dA = sA + stage * C::A_BYTES;
          void* dB = sB + stage * C::B_BYTES;
          if (MODE == GEMM_DENSE) {
            // two sources (a channel concat never materialised): K blocks [0, kb_src0) from source 0
            const bool s1 = g.nsrc > 1 && kb >= g.kb_src[0];
            const int kk = s1 ? kb - g.kb_src[0] : kb;
            if (!skipA) tma2<CG>(dA, s1 ? &ta1 : &ta0, &full[stage], bar_l, kk * C::BK, m0);
            if (!skipB) tma2<CG>(dB, s1 ? &tb1 : &tb0, &full[stage], bar_l, kk * C::BK, n0);
          } else {
            int r = kb, src = 0;
            if (r >= 9 * g.kb_src[0]) {
              r -= 9 * g.kb_src[0];
              src = 1;
            }
            const int tap = r / g.kb_src[src], cb = r % g.kb_src[src];
            const int dy = tap / 3 - 1, dx = tap % 3 - 1;
            const CUtensorMap* ma = src ? &ta1 : &ta0;
            const CUtensorMap* mb = src ? &tb1 : &tb0;
            if (!skipA) tma4<CG>(dA, ma, &full[stage], bar_l, cb * C::BK, g.stride * x0 + dx, g.stride * y0 + dy, b0);
            if (skipB) {
            } else if (C::NH == 1) {
              tma3<CG>(dB, mb, &full[stage], bar_l, cb * C::BK, tap, n0);
            } else {  // this CTA's slice of each N-half: rows nt·BN + h·MMA_N + rank·MMA_N/CG
#pragma unroll
              for (int h = 0; h < C::NH; ++h)
                if (hsel < 0 || h == hsel)
                  tma3<CG>(static_cast<uint8_t*>(dB) + h * (C::B_ROWS / C::NH) * 128, mb, &full[stage], bar_l,
                         cb * C::BK, tap, nt * BN + h * C::MMA_N + (int)rank * (C::MMA_N / CG));
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ================= MMA issuer (leader CTA) =================
      const uint32_t idesc = make_idesc16(128 * CG, C::MMA_N, F16);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, jh = 0;
      for (int u = worker; u < total; u += nworkers, ++it) {
        int hsel;
        const int t = decode_unit(g, u, hsel);
        const int acc = C::NACC == 2 ? (it & 1) : 0;
        const uint32_t acc_phase = C::NACC == 2 ? ((it >> 1) & 1) : (it & 1);
        // NH = 2 (BN = 320): each 160-column half computed takes the next global half index j (jh, jh + 1,
        // …), in rotating buffers j mod 3 of 160 TMEM columns (480 of 512): the next tile's MMAs start as
        // soon as this tile's first half is drained, instead of after its whole epilogue. A half unit
        // (tail balancing) computes only its half h = hsel.
        uint32_t dh[2] = {0u, 0u};
        int jb[2] = {0, 0};
        if constexpr (C::NH == 2) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (hsel >= 0 && h != hsel) continue;
            const int j = jh++, b = j % 3;
            mbar_wait(&tempty[b], ((j / 3) & 1) ^ 1);
            dh[h] = tmem_base + b * C::MMA_N;
            jb[h] = b;
          }
        } else {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          dh[0] = tmem_base + acc * C::TMEM_STRIDE;
          dh[1] = dh[0] + C::MMA_N;
        }
        tc_fence_after();
        int mt, nt, sp, kb0, kb1;
        decode_tile(g, t, mt, nt, sp, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k)
#pragma unroll
            for (int h = 0; h < C::NH; ++h)  // N-half h: B rows [h·B_ROWS/NH, …) of every CTA, TMEM cols h·MMA_N
              if (hsel < 0 || h == hsel)
                mma<CG>(dh[h], make_sdesc_sw128(a0 + k * 32),
                        make_sdesc_sw128(b0 + h * (C::B_ROWS / C::NH) * 128 + k * 32), idesc,
                        (kb != kb0 || k != 0) ? 1u : 0u);
          commit<CG>(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (C::NH == 2) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (hsel < 0 || h == hsel) commit<CG>(&tfull[jb[h]]);
        } else {
          commit<CG>(&tfull[acc]);
        }
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue (warps 2..9 → TMEM lane quarters 2,3,0,1,2,3,0,1; two warps per quarter split
    // the 32-column chunks, so the epilogue keeps up with short-K tiles) =====
    const int q = warp & 3;
    EpiCtx ec{sStage + (warp - 2) * 4096, 0, 0, 0, 0, rbar + (warp - 2) * 2, 0u};
    int it = 0, jh = 0;
    for (int u = worker; u < total; u += nworkers, ++it) {
      int hsel;
      const int t = decode_unit(g, u, hsel);
      const int acc = C::NACC == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = C::NACC == 2 ? ((it >> 1) & 1) : (it & 1);
      int mt, nt, sp, kb0, kb1;
      decode_tile(g, t, mt, nt, sp, kb0, kb1);
      auto release = [&](int b) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 1) {
            mbar_arrive(&tempty[b]);
          } else {
            const uint32_t a = leader_addr(&tempty[b]);
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
          }
        }
      };
      const uint32_t lq = (uint32_t)(q * 32) << 16;
      if constexpr (C::NH == 2) {
        // the tile's two 160-column halves from their rotating buffers, first half first (its release lets
        // the next tile's MMAs start)
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (hsel >= 0 && h != hsel) continue;  // a half unit drains only its half
          const int j = jh++, b = j % 3;
          epilogue_tile<BN, MODE, F16, EPW / 4>(g, &tout, &tres, ec, tmem_base + lq + b * C::MMA_N, mt * CG + (int)rank,
                                                nt * BN, q, lane, (warp - 2) >> 2, sp, &tfull[b], (j / 3) & 1,
                                                h * (BN / 64), (h + 1) * (BN / 64));
          release(b);
        }
      } else {
        const uint32_t tbase = tmem_base + lq + acc * C::TMEM_STRIDE;
        epilogue_tile<BN, MODE, F16, EPW / 4>(g, &tout, &tres, ec, tbase, mt * CG + (int)rank, nt * BN, q, lane,
                                              (warp - 2) >> 2, sp, &tfull[acc], acc_phase);
        release(acc);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_cg<CG>(tmem_base, C::TMEM_COLS);
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e == cudaSuccess && q == cudaDriverEntryPointSuccess) fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 16-bit element type of the maps built by this thread's current gemm() call (bf16, or fp16)
static thread_local CUtensorMapDataType t_map_dtype = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;

static void make_map(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                     const uint32_t* elem_strides = nullptr) {
  cuuint64_t gd[5], gs[5];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    es[i] = elem_strides ? elem_strides[i] : 1;
    if (i + 1 < rank) gs[i] = strides_bytes[i];
  }
  CUresult r = encode_fn()(m, t_map_dtype, rank, const_cast<void*>(ptr), gd, gs, bx, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

void make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
                  uint32_t box_out, bool is_f16, bool swz64) {
  uint64_t d[2] = {inner, outer}, s[1] = {row_bytes};
  uint32_t b[2] = {box_in, box_out};
  t_map_dtype = is_f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  make_map(m, ptr, 2, d, s, b, swz64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
  t_map_dtype = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    SD_CUDA(cudaGetDevice(&dev));
    SD_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

static int pow2_div(int v, int cap) {
  int p = 1;
  while (p * 2 <= cap && v % (p * 2) == 0) p *= 2;
  return p;
}

void conv3_tile_geometry(int B, int H, int W, int* wt, int* ht, int* bt) {
  *wt = pow2_div(W, 128);
  *ht = pow2_div(H, 128 / *wt);
  *bt = 128 / (*wt * *ht);
  (void)B;
}


// split-K reduction: out = epilogue(Σ_s part[s]) in fixed split order (deterministic)
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int S, long M, int N, const float* __restrict__ bias,
                                     const float* __restrict__ temb, int ld_temb, int rows_per_img,
                                     const bf16* __restrict__ res, int ldr, int act, float alpha, bf16* __restrict__ out,
                                     int ldo, int col_off, int is_f16) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;  // one group of 4 columns
  const int nq = N / 4;
  if (i >= M * nq) return;
  const long m = i / nq;
  const int n = (int)(i % nq) * 4;
  // every split's 16-byte load issued before the first add (S ≤ 8), summed in split order
  float4 v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s < S) v[s] = reinterpret_cast<const float4*>(part + ((long)s * M + m) * N + n)[0];
  float4 acc = v[0];
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s < S) {
      acc.x += v[s].x;
      acc.y += v[s].y;
      acc.z += v[s].z;
      acc.w += v[s].w;
    }
  float o[4] = {acc.x * alpha, acc.y * alpha, acc.z * alpha, acc.w * alpha};
  for (int k = 0; k < 4; ++k) {
    if (bias) o[k] += bias[n + k];
    if (temb) o[k] += temb[(m / rows_per_img) * ld_temb + n + k];
    if (act == ACT_SILU) o[k] = silu_f(o[k]);
    if (res) o[k] += cvt16(res[m * ldr + n + k], is_f16);
  }
  uint2 pk = make_uint2(pack16(o[0], o[1], is_f16), pack16(o[2], o[3], is_f16));
  *reinterpret_cast<uint2*>(out + m * ldo + col_off + n) = pk;
}

template <int BN, int CG, int MODE, int EPW>
static void launch(const CUtensorMap* m, const GemmArgs& a, cudaStream_t st) {
  using C = Cfg<BN, CG, EPW>;
  static bool attr_set = false;
  if (!attr_set) {
    SD_CUDA(cudaFuncSetAttribute(gemm_kernel<BN, CG, MODE, false, EPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM));
    SD_CUDA(cudaFuncSetAttribute(gemm_kernel<BN, CG, MODE, true, EPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM));
    attr_set = true;
  }
  const int tiles = a.m_tiles * a.n_tiles * a.splits;
  int workers = stream_sms(st) / CG;
  if (tiles < workers) workers = tiles;
  if (workers <= 0) return;
  // NH = 2 tail balancing: a last partial wave of ≤ workers/2 tiles runs as 2× as many half-tile units
  // (SD_TAIL_HALVES=0 disables); results are bitwise the same
  GemmArgs b = a;
  b.full_units = tiles;
  b.total_units = tiles;
  {
    static int th = -1;
    if (th < 0) {
      const char* e = getenv("SD_TAIL_HALVES");
      th = !(e && e[0] == '0');
    }
    const int tail = tiles % workers;
    if (C::NH == 2 && th && a.splits == 1 && tiles > workers && tail > 0 && 2 * tail <= workers) {
      b.full_units = tiles - tail;
      b.total_units = b.full_units + 2 * tail;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(workers * CG);
  cfg.blockDim = dim3(64 + 32 * EPW);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 2 : 1;
  if (a.f16)
    SD_CUDA(cudaLaunchKernelEx(&cfg, gemm_kernel<BN, CG, MODE, true, EPW>, m[0], m[1], m[2], m[3], m[4], m[5], b));
  else
    SD_CUDA(cudaLaunchKernelEx(&cfg, gemm_kernel<BN, CG, MODE, false, EPW>, m[0], m[1], m[2], m[3], m[4], m[5], b));
  SD_CHECK_LAUNCH();
}

// conv3 and dense launches are separate instantiations (distinct kernel names in launch lists)
template <int MODE, int EPW>
static void dispatch_w(int bn, int cg, const CUtensorMap* maps, const GemmArgs& a, cudaStream_t st) {
  switch (bn * 4 + cg) {
    case 64 * 4 + 1: launch<64, 1, MODE, EPW>(maps, a, st); break;
    case 128 * 4 + 1: launch<128, 1, MODE, EPW>(maps, a, st); break;
    case 160 * 4 + 1: launch<160, 1, MODE, EPW>(maps, a, st); break;
    case 256 * 4 + 1: launch<256, 1, MODE, EPW>(maps, a, st); break;
    case 128 * 4 + 2: launch<128, 2, MODE, EPW>(maps, a, st); break;
    case 160 * 4 + 2: launch<160, 2, MODE, EPW>(maps, a, st); break;
    case 256 * 4 + 2: launch<256, 2, MODE, EPW>(maps, a, st); break;
    case 320 * 4 + 2: launch<320, 2, MODE, EPW>(maps, a, st); break;
    default: throw CudaError("unsupported BN/CG");
  }
}
// epilogue warps: 12 (3 per TMEM lane quarter) for dense launches with K ≤ 320 (5 K blocks) that are not
// GEGLU, else 8. With such short K the epilogue's serial chunk chain per warp (TMEM load → math →
// staging → TMA store) is the critical path — [65536, 320, 320]: 25.0 µs with stores, 19.0 µs without,
// and removing either operand's loads changed nothing — and 3 warps per quarter cut the longest chain
// of a BN = 160 tile from 3 chunks to 2: 25.3 → 22.9 µs, [65536, 960, 320] 64.0 → 60.0 µs, with the
// residual 32.2 → 30.3 µs. Longer K and GEGLU lose 2-4 % (fewer ring stages in the smaller smem share,
// 128 registers). 16 warps would cap registers at 96 (18 warps, 5 per SMSP: 200-byte spills).
// SD_EPI_WARPS=8 turns the 12-warp form off.
static int epi_warps(int mode, const GemmArgs& a) {
  static int e = -1;
  if (e < 0) {
    const char* s = getenv("SD_EPI_WARPS");
    e = s ? atoi(s) : 12;
  }
  return mode == GEMM_DENSE && e == 12 && a.num_kb <= 5 && a.act != ACT_GEGLU ? 12 : 8;
}
template <int MODE>
static void dispatch(int bn, int cg, const CUtensorMap* maps, const GemmArgs& a, cudaStream_t st) {
  if constexpr (MODE == GEMM_DENSE) {
    if (epi_warps(MODE, a) == 12) {
      dispatch_w<MODE, 12>(bn, cg, maps, a, st);
      return;
    }
  }
  dispatch_w<MODE, 8>(bn, cg, maps, a, st);
}

static int pick_bn(int N, int act) {
  if (act == ACT_GEGLU) {
    static int e = -1;  // SD_GEGLU_BN=128 (experiments; measured 1.4× slower at 64×64)
    if (e < 0) {
      const char* s = getenv("SD_GEGLU_BN");
      e = s ? atoi(s) : 0;
    }
    return (e == 128 || N % 256) ? 128 : 256;
  }
  if (N <= 64) return 64;
  if (N % 256 == 0) return 256;
  if (N % 160 == 0) return 160;
  if (N <= 128 || N % 128 == 0) return 128;
  return 256;
}

int g_cg_override = -1;
int g_pdl = [] {  // SD_PDL=0: plain stream-ordered launches
  const char* e = getenv("SD_PDL");
  return e && e[0] == '0' ? 0 : 1;
}();  // 0 = heuristic, 1 / 2 = force (tests, SD_GEMM_CG)

static int conv_num_kb(const GemmDesc& d) {
  int kb = 0;
  for (int s = 0; s < d.nsrc; ++s) kb += 9 * cdiv(d.cs[s], 64);
  return kb;
}

int gemm_splits(const GemmDesc& d) {
  static int env = -2;
  if (env == -2) {
    const char* s = getenv("SD_SPLITK");
    env = s ? atoi(s) : -1;
  }
  if (d.splits == 1 || d.ln_stat) return 1;
  if (d.act == ACT_GEGLU || d.out_f32 || d.bias_per_row || d.N % 4 || d.ldo % 4 || d.col_off % 4) return 1;
  if (d.mode == GEMM_DENSE) {
    // dense: only an explicit split count (the caller picks it from the layer, never from the batch, so
    // results stay batch-invariant); K blocks of 64 split evenly, ≥ 4 per split
    if (d.splits <= 1) return 1;
    const int kbd = cdiv(d.K, 64);
    const int sd = std::max(1, std::min(d.splits, std::min(8, kbd / 4)));
    return cdiv(kbd, cdiv(kbd, sd));
  }
  const int kb = conv_num_kb(d);
  int s = d.splits;
  if (s == 0) {
    // the 8×8 level of SD-1.5 (1280 / 2560 channels): 40 output tiles at 8 requests × CFG leave
    // most of the 148 SMs idle over 180–360 K blocks; 3 splits make one full wave
    // the 16×16 level too: 80 pair tiles are 1.08 waves of 74 pairs at 16 rows; 3 splits measured
    // [16, 16, 16, 1280, 1280] 116.7 → 105.1 µs (2 splits: 109.7). SD_SPLIT16=1 turns it off.
    static int s16 = -2;
    if (s16 == -2) {
      const char* e = getenv("SD_SPLIT16");
      s16 = e ? atoi(e) : 3;
    }
    if ((long)d.H * d.W == 256 && kb >= 90 && s16 > 1) {
      s = s16;
    } else {
      if ((long)d.H * d.W > 64 || kb < 90) return 1;
      s = env >= 0 ? env : 3;
    }
  }
  s = std::max(1, std::min(s, std::min(8, kb)));
  const int kps = cdiv(kb, s);
  return cdiv(kb, kps);
}

size_t gemm_split_ws_bytes(const GemmDesc& d) {
  const int s = gemm_splits(d);
  if (s <= 1) return 0;
  const long M = d.mode == GEMM_DENSE ? (long)d.M : (long)d.B * d.H * d.W;
  return (size_t)s * M * d.N * sizeof(float);
}

bool gemm_gn_ok(const GemmDesc& d) {
  if (d.out_f32 || d.act == ACT_GEGLU || d.col_off || d.ldo != d.N || d.N % 32 || d.bias_per_row) return false;
  if (gemm_splits(d) > 1) return false;
  if (d.mode == GEMM_DENSE) return d.gn_P > 0 && d.gn_P % 32 == 0 && d.M % d.gn_P == 0;
  int wt, ht, bt;
  conv3_tile_geometry(d.B, d.H, d.W, &wt, &ht, &bt);
  return wt * ht >= 32 && d.W % wt == 0 && d.H % ht == 0;
}

void gemm(const GemmDesc& d, cudaStream_t st) {
  if (d.gn_part && !gemm_gn_ok(d)) throw CudaError("gemm: GroupNorm statistics requested for an ineligible launch");
  if (g_cg_override < 0) {
    const char* s = getenv("SD_GEMM_CG");
    g_cg_override = s ? atoi(s) : 0;
  }
  GemmArgs a{};
  CUtensorMap maps[6];
  memset(maps, 0, sizeof(maps));
  a.mode = d.mode;
  a.f16 = d.f16;
  t_map_dtype = d.f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  a.N = d.N;
  static int bn_env = -1;  // SD_GEMM_BN: force the N tile of dense GEMMs (experiments)
  if (bn_env < 0) {
    const char* e = getenv("SD_GEMM_BN");
    bn_env = e ? atoi(e) : 0;
  }
  int bn = d.bn ? d.bn : (bn_env && d.mode == GEMM_DENSE && d.act != ACT_GEGLU ? bn_env : pick_bn(d.N, d.act));
  if (d.act == ACT_GEGLU && bn % 128) throw CudaError("GEGLU needs BN multiple of 128");
  a.n_tiles = cdiv(d.N, bn);
  int m_boxes = 0;
  if (d.mode == GEMM_DENSE) {
    if (d.K % 8 || d.lda % 8 || d.ldb % 8) throw CudaError("dense GEMM: K/lda/ldb must be multiples of 8");
    a.M = d.M;
    m_boxes = cdiv(d.M, 128);
    a.nsrc = d.nsrc;
    if (d.nsrc == 2) {  // A = [xs[0] | xs[1]] (cs[0] + cs[1] = K columns), B = [Bw[0] | Bw[1]] (row stride ldb)
      if (d.cs[0] % 8 || d.cs[1] % 8 || d.cs[0] + d.cs[1] != d.K) throw CudaError("dense GEMM: bad source split");
      a.kb_src[0] = cdiv(d.cs[0], 64);
      a.kb_src[1] = cdiv(d.cs[1], 64);
      a.num_kb = a.kb_src[0] + a.kb_src[1];
    } else {
      a.num_kb = cdiv(d.K, 64);
    }
  } else {
    if (d.stride != 1 && (d.stride != 2 || d.nsrc != 1)) throw CudaError("conv3: stride 1, or 2 with one source");
    a.B = d.B;
    a.H = d.H;
    a.W = d.W;
    a.stride = d.stride;
    a.M = d.B * d.H * d.W;
    conv3_tile_geometry(d.B, d.H, d.W, &a.wt, &a.ht, &a.bt);
    a.tiles_x = cdiv(d.W, a.wt);
    a.tiles_y = cdiv(d.H, a.ht);
    m_boxes = a.tiles_x * a.tiles_y * cdiv(d.B, a.bt);
    a.nsrc = d.nsrc;
    a.num_kb = 0;
    for (int s = 0; s < d.nsrc; ++s) {
      if (d.cs[s] % 8) throw CudaError("conv3: channels must be a multiple of 8");
      a.kb_src[s] = cdiv(d.cs[s], 64);
      a.num_kb += 9 * a.kb_src[s];
    }
  }
  a.ln_stat = d.ln_stat;
  a.ln_wbar = d.ln_wbar;
  a.ln_cols = d.ln_cols;
  if (d.ln_stat && (d.mode != GEMM_DENSE || !d.ln_wbar || d.act == ACT_SILU))
    throw CudaError("gemm: folded LayerNorm needs a dense launch with w-bar (no SiLU)");
  a.gn_part = d.gn_part;
  if (d.gn_part) {
    const int P = d.mode == GEMM_DENSE ? d.gn_P : d.H * d.W;
    a.gn_P = P;
    a.gn_slots = P / 32;
    a.gn_sw = d.mode == GEMM_DENSE ? 32 : (a.wt < 32 ? a.wt : 32);
    a.gn_sh = 32 / a.gn_sw;
  }
  a.splits = 1;
  a.kps = a.num_kb;
  a.part = nullptr;
  {
    const int s = gemm_splits(d);
    if (s > 1 && d.m_tile_count < 0 && d.split_ws && d.split_ws_bytes >= gemm_split_ws_bytes(d)) {
      a.kps = cdiv(a.num_kb, s);
      a.splits = s;
      a.part = d.split_ws;
    }
  }
  int box_begin = d.m_tile_begin, box_count = d.m_tile_count >= 0 ? d.m_tile_count : m_boxes;
  // pair tiles (256 rows, half of B per CTA) when the weights dominate the operand traffic
  // (M ≤ 16·N; measured on B200: 16×16 / 8×8 / 32×32×1280 convs gain up to 1.4×, 64×64 ones lose)
  // pairs when the weights dominate the operand traffic (M ≤ 16·N: the 16×16 / 8×8 UNet levels gain
  // up to 1.4×; short-K dense GEMMs at M = 65536 lose). conv3 layers of 64×64 … 256×256 pixels also
  // take pairs (kbench r01: +3-5 %; at 32×32 and 512×512 they lose 1-11 %); SD_CONV_CG_OLD=1 = M-rule only.
  static int conv_old = -1;
  if (conv_old < 0) {
    const char* s = getenv("SD_CONV_CG_OLD");
    conv_old = s && s[0] == '1';
  }
  const bool pair_ok = box_begin % 2 == 0 && bn >= 128;
  const long hw = (long)d.H * d.W;
  const bool conv_pair = d.mode == GEMM_CONV3 && !conv_old && hw >= 4096 && hw <= 65536;
  int cg = (pair_ok && (((long)box_count * 128 <= 16L * d.N) || conv_pair)) ? 2 : 1;
  if (g_cg_override == 1 || g_cg_override == 2) cg = g_cg_override;
  if (cg == 2 && (box_begin % 2 || bn < 128)) cg = 1;
  // paired conv tiles with N a multiple of 320 (the 64×64 / 32×32 levels): BN = 320 = two N = 160 MMAs
  // sharing A (SD_CONV_BN320=0: BN = 160)
  static int bn320 = -1;
  if (bn320 < 0) {
    const char* e = getenv("SD_CONV_BN320");
    bn320 = !(e && e[0] == '0');
  }
  if (bn320 && d.mode == GEMM_CONV3 && cg == 2 && bn == 160 && d.N % 320 == 0 && !d.bn) {
    bn = 320;
    a.n_tiles = cdiv(d.N, bn);
  }
  const uint32_t brows = (uint32_t)(bn / cg / (bn > 256 ? 2 : 1));
  if (d.mode == GEMM_DENSE && d.nsrc == 2) {
    for (int s = 0; s < 2; ++s) {  // source s: its own activation tensor [M][cs] and weight columns
      uint64_t dA[2] = {(uint64_t)d.cs[s], (uint64_t)d.M}, sA[1] = {(uint64_t)d.cs[s] * 2};
      uint32_t bA[2] = {64, 128};
      make_map(&maps[s], d.xs[s], 2, dA, sA, bA);
      uint64_t dB[2] = {(uint64_t)d.cs[s], (uint64_t)d.N}, sB[1] = {(uint64_t)d.ldb * 2};
      uint32_t bB[2] = {64, brows};
      make_map(&maps[2 + s], d.Bw[s], 2, dB, sB, bB);
    }
  } else if (d.mode == GEMM_DENSE) {
    uint64_t dA[2] = {(uint64_t)d.K, (uint64_t)d.M}, sA[1] = {(uint64_t)d.lda * 2};
    uint32_t bA[2] = {64, 128};
    make_map(&maps[0], d.A, 2, dA, sA, bA);
    uint64_t dB[2] = {(uint64_t)d.K, (uint64_t)d.N}, sB[1] = {(uint64_t)d.ldb * 2};
    uint32_t bB[2] = {64, brows};
    make_map(&maps[2], d.Bw[0], 2, dB, sB, bB);
    maps[1] = maps[0];
    maps[3] = maps[2];
  } else {
    const int sd = d.stride;  // stride 2: the box spans 2·wt × 2·ht input pixels, every second one loaded
    const uint64_t Wi = (uint64_t)d.W * sd, Hi = (uint64_t)d.H * sd;
    for (int s = 0; s < d.nsrc; ++s) {
      uint64_t dA[4] = {(uint64_t)d.cs[s], Wi, Hi, (uint64_t)d.B};
      uint64_t sA[3] = {(uint64_t)d.cs[s] * 2, (uint64_t)d.cs[s] * 2 * Wi, (uint64_t)d.cs[s] * 2 * Wi * Hi};
      uint32_t bA[4] = {64, (uint32_t)(a.wt * sd), (uint32_t)(a.ht * sd), (uint32_t)a.bt};
      uint32_t eA[4] = {1, (uint32_t)sd, (uint32_t)sd, 1};
      make_map(&maps[s], d.xs[s], 4, dA, sA, bA, CU_TENSOR_MAP_SWIZZLE_128B, eA);
      uint64_t dB[3] = {(uint64_t)d.cs[s], 9, (uint64_t)d.N};
      uint64_t sB[2] = {(uint64_t)d.cs[s] * 2, (uint64_t)d.cs[s] * 2 * 9};
      uint32_t bB[3] = {64, 1, brows};
      make_map(&maps[2 + s], d.Bw[s], 3, dB, sB, bB);
    }
    if (d.nsrc == 1) {
      maps[1] = maps[0];
      maps[3] = maps[2];
    }
  }
  a.m_tile_begin = box_begin / cg;
  a.m_tiles = cdiv(box_count, cg);
  a.out = d.out;
  a.ldo = d.ldo;
  a.col_off = d.col_off;
  a.out_f32 = d.out_f32;
  a.bias = d.bias;
  a.bias_per_row = d.bias_per_row;
  a.alpha = d.alpha;
  a.temb = d.temb;
  a.ld_temb = d.ld_temb;
  a.rows_per_img = d.rows_per_img > 0 ? d.rows_per_img : 1;
  a.res = d.res;
  a.ldr = d.ldr;
  a.act = d.act;
  {
    static int gt = -1;
    if (gt < 0) {
      const char* e = getenv("SD_GELU_TANH");
      gt = e ? atoi(e) : 1;
    }
    a.gelu_tanh = gt;
  }
  // bf16 outputs go through the TMA store path (box = one warp's 32 rows × 32 columns)
  const int n_out = d.act == ACT_GEGLU ? d.N / 2 : d.N;
  a.tma_store = (!d.out_f32 && d.ldo % 8 == 0 && d.col_off % 8 == 0 && n_out % 8 == 0 && a.splits == 1) ? 1 : 0;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* s = getenv("SD_EPI_DBG");
      dbg = s ? atoi(s) : 0;
    }
    a.dbg = dbg;
    if (dbg == 4) a.tma_store = 0;  // direct stores
  }
  if (d.gn_part && !a.tma_store) throw CudaError("gemm: GroupNorm statistics need the TMA-store epilogue");
  if (a.tma_store) {
    const bf16* ob = reinterpret_cast<const bf16*>(d.out) + d.col_off;
    if (d.mode == GEMM_DENSE) {
      uint64_t dO[2] = {(uint64_t)n_out, (uint64_t)d.M}, sO[1] = {(uint64_t)d.ldo * 2};
      uint32_t bO[2] = {32, 32};
      make_map(&maps[4], ob, 2, dO, sO, bO, CU_TENSOR_MAP_SWIZZLE_64B);
    } else {
      const int sw = a.wt < 32 ? a.wt : 32;
      const int sh = a.ht < 32 / sw ? a.ht : 32 / sw;
      const int sb = 32 / (sw * sh);
      uint64_t dO[4] = {(uint64_t)n_out, (uint64_t)d.W, (uint64_t)d.H, (uint64_t)d.B};
      uint64_t sO[3] = {(uint64_t)d.ldo * 2, (uint64_t)d.ldo * 2 * d.W, (uint64_t)d.ldo * 2 * d.W * d.H};
      uint32_t bO[4] = {32, (uint32_t)sw, (uint32_t)sh, (uint32_t)sb};
      make_map(&maps[4], ob, 4, dO, sO, bO, CU_TENSOR_MAP_SWIZZLE_64B);
    }
  } else {
    if (d.act == ACT_GEGLU) throw CudaError("GEGLU epilogue needs a bf16, 16-byte aligned output");
    maps[4] = maps[0];
  }
  // dense residual through TMA (the per-lane row loads cost one L1 wavefront per row: 32 per warp
  // instruction); SD_RES_TMA=0 keeps the direct loads (A/B)
  static int res_tma_env = -1;
  if (res_tma_env < 0) {
    const char* e = getenv("SD_RES_TMA");
    res_tma_env = e ? atoi(e) : 1;
  }
  maps[5] = maps[0];
  if (res_tma_env && a.tma_store && d.res && d.mode == GEMM_DENSE && d.act != ACT_GEGLU && d.ldr % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(d.res) & 15) == 0 && a.dbg == 0) {
    uint64_t dR[2] = {(uint64_t)d.N, (uint64_t)d.M}, sR[1] = {(uint64_t)d.ldr * 2};
    uint32_t bR[2] = {32, 32};
    make_map(&maps[5], d.res, 2, dR, sR, bR, CU_TENSOR_MAP_SWIZZLE_64B);
    a.res_tma = 1;
  }
  t_map_dtype = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (d.mode == GEMM_DENSE)
    dispatch<GEMM_DENSE>(bn, cg, maps, a, st);
  else
    dispatch<GEMM_CONV3>(bn, cg, maps, a, st);
  if (a.splits > 1) {
    const long n4 = (long)a.M * (d.N / 4);
    launch_k(splitk_reduce_kernel, (unsigned)cdiv(n4, 256), 256, 0, st, 
        a.part, a.splits, a.M, d.N, d.bias, d.temb, d.ld_temb,
        d.mode == GEMM_DENSE ? (d.rows_per_img > 0 ? d.rows_per_img : 1) : d.H * d.W, d.res, d.ldr, d.act, d.alpha,
        reinterpret_cast<bf16*>(d.out), d.ldo, d.col_off, d.f16);
    SD_CHECK_LAUNCH();
  }
}

// SD_PREC_FP16: the same kernels; the descriptor differs only in its pointer types
static GemmDesc as16(const GemmDescT<f16>& d) {
  static_assert(sizeof(GemmDescT<f16>) == sizeof(GemmDesc), "GemmDescT layouts must match");
  GemmDesc b;
  memcpy(static_cast<void*>(&b), static_cast<const void*>(&d), sizeof(b));
  b.f16 = 1;
  return b;
}
void gemm(const GemmDescT<f16>& d, cudaStream_t st) { gemm(as16(d), st); }
int gemm_splits(const GemmDescT<f16>& d) { return gemm_splits(as16(d)); }
bool gemm_gn_ok(const GemmDescT<f16>& d) { return gemm_gn_ok(as16(d)); }
size_t gemm_split_ws_bytes(const GemmDescT<f16>& d) { return gemm_split_ws_bytes(as16(d)); }

}  // namespace sd
