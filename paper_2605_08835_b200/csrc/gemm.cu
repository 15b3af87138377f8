// tcgen05 / TMEM / TMA GEMM and implicit-GEMM 3x3 convolution for sm_100a.
//
// One persistent, warp-specialised kernel:
//   warp 0      TMA producer   (one elected lane): A and B tiles into a STAGES-deep smem ring
//   warp 1      MMA issuer     (one elected lane): tcgen05.mma 128×BN×16 into a double-buffered
//                              TMEM accumulator; also owns TMEM alloc/dealloc
//   warps 2..5  epilogue       tcgen05.ld → bias / temb / act / residual → bf16|fp32 stores
// smem operands are K-major with the 128-byte swizzle written by TMA and described to the
// tensor core by SWIZZLE_128B UMMA descriptors (8-row groups 1024 B apart).
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace sd {

struct GemmArgs {
  int mode;
  int M, N;
  int B, H, W, wt, ht, bt, tiles_x, tiles_y;
  int kb_src[2];      // K blocks (of 64 channels) per tap for each source
  int nsrc;
  int num_kb;         // K blocks per tile
  int m_tiles, n_tiles, m_tile_begin;
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
};

template <int BN>
struct Cfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;                    // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGES = BN >= 256 ? 4 : (BN >= 160 ? 5 : 6);
  static constexpr int TMEM_STRIDE = BN <= 64 ? 64 : (BN <= 128 ? 128 : 256);
  static constexpr int TMEM_COLS = 2 * TMEM_STRIDE;
  static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + 256;
};

template <int BN>
__global__ void __launch_bounds__(192, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                const __grid_constant__ CUtensorMap tb0, const __grid_constant__ CUtensorMap tb1, const GemmArgs g) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_mbar_init();
    tma_prefetch(&ta0);
    tma_prefetch(&tb0);
    if (g.nsrc > 1) {
      tma_prefetch(&ta1);
      tma_prefetch(&tb1);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total = g.m_tiles * g.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer =================
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int mt = g.m_tile_begin + t / g.n_tiles, nt = t % g.n_tiles;
        const int n0 = nt * BN;
        int m0 = 0, x0 = 0, y0 = 0, b0 = 0;
        if (g.mode == GEMM_DENSE) {
          m0 = mt * C::BM;
        } else {
          const int tx = mt % g.tiles_x;
          const int ty = (mt / g.tiles_x) % g.tiles_y;
          const int tb = mt / (g.tiles_x * g.tiles_y);
          x0 = tx * g.wt;
          y0 = ty * g.ht;
          b0 = tb * g.bt;
        }
        for (int kb = 0; kb < g.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
          void* dA = sA + stage * C::A_BYTES;
          void* dB = sB + stage * C::B_BYTES;
          if (g.mode == GEMM_DENSE) {
            tma_load_2d(dA, &ta0, &full[stage], kb * C::BK, m0);
            tma_load_2d(dB, &tb0, &full[stage], kb * C::BK, n0);
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
            tma_load_4d(dA, ma, &full[stage], cb * C::BK, x0 + dx, y0 + dy, b0);
            tma_load_3d(dB, mb, &full[stage], cb * C::BK, tap, n0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer =================
      constexpr uint32_t idesc = make_idesc_bf16(128, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * C::TMEM_STRIDE;
        for (int kb = 0; kb < g.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            umma_bf16(d, make_sdesc_sw128(a0 + k * 32), make_sdesc_sw128(b0 + k * 32), idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue (warps 2..5 → TMEM lane quarters 2,3,0,1) =================
    const int q = warp & 3;
    const int r = q * 32 + lane;          // accumulator row = TMEM lane
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int mt = g.m_tile_begin + t / g.n_tiles, nt = t % g.n_tiles;
      const int n0 = nt * BN;
      long prow;       // output row index (pixel or m)
      int img;
      bool valid;
      if (g.mode == GEMM_DENSE) {
        prow = (long)mt * 128 + r;
        valid = prow < g.M;
        img = (int)(prow / g.rows_per_img);
      } else {
        const int tx = mt % g.tiles_x;
        const int ty = (mt / g.tiles_x) % g.tiles_y;
        const int tb = mt / (g.tiles_x * g.tiles_y);
        const int xx = tx * g.wt + r % g.wt;
        const int yy = ty * g.ht + (r / g.wt) % g.ht;
        const int bb = tb * g.bt + r / (g.wt * g.ht);
        valid = xx < g.W && yy < g.H && bb < g.B;
        prow = ((long)bb * g.H + yy) * g.W + xx;
        img = bb;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * C::TMEM_STRIDE;
      if (g.act == ACT_GEGLU) {
        // columns [128j, 128j+64) = value, [128j+64, 128j+128) = gate; output width BN/2
#pragma unroll 1
        for (int j = 0; j < BN / 128; ++j) {
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            uint32_t rv[32], rg[32];
            const int cv = j * 128 + h * 32, cg = cv + 64;
            tmem_ld32(tbase + cv, rv);
            tmem_ld32(tbase + cg, rg);
            const int ocol = (n0 >> 1) + j * 64 + h * 32;   // output column base
            if (valid && ocol < (g.N >> 1)) {
              float o[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float v = __uint_as_float(rv[i]) * g.alpha;
                float gt = __uint_as_float(rg[i]) * g.alpha;
                if (g.bias) {
                  v += g.bias[n0 + cv + i];
                  gt += g.bias[n0 + cg + i];
                }
                o[i] = v * gelu_f(gt);
              }
              bf16* op = reinterpret_cast<bf16*>(g.out) + prow * g.ldo + g.col_off + ocol;
              if (g.res) {
                const bf16* rp = g.res + prow * g.ldr + ocol;
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] += __bfloat162float(rp[i]);
              }
              uint4* o4 = reinterpret_cast<uint4*>(op);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                o4[i] = make_uint4(pack_bf16(o[8 * i], o[8 * i + 1]), pack_bf16(o[8 * i + 2], o[8 * i + 3]),
                                   pack_bf16(o[8 * i + 4], o[8 * i + 5]), pack_bf16(o[8 * i + 6], o[8 * i + 7]));
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t rv[32];
          tmem_ld32(tbase + c * 32, rv);
          const int col = n0 + c * 32;
          if (valid && col < g.N) {
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(rv[i]) * g.alpha;
            if (g.bias) {
              if (g.bias_per_row) {
                const float bv = g.bias[prow];
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] += bv;
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] += (col + i < g.N) ? g.bias[col + i] : 0.f;
              }
            }
            if (g.temb) {
              const float* tp = g.temb + (long)img * g.ld_temb + col;
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] += (col + i < g.N) ? tp[i] : 0.f;
            }
            if (g.act == ACT_SILU) {
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = silu_f(o[i]);
            }
            const bool full32 = col + 32 <= g.N;
            if (g.res) {
              const bf16* rp = g.res + prow * g.ldr + col;
              if (full32) {
                const uint4* r4 = reinterpret_cast<const uint4*>(rp);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  uint4 u = r4[i];
                  const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
                  for (int k = 0; k < 8; ++k) o[8 * i + k] += __bfloat162float(e[k]);
                }
              } else {
                for (int i = 0; i < 32 && col + i < g.N; ++i) o[i] += __bfloat162float(rp[i]);
              }
            }
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
                  o4[i] = make_uint4(pack_bf16(o[8 * i], o[8 * i + 1]), pack_bf16(o[8 * i + 2], o[8 * i + 3]),
                                     pack_bf16(o[8 * i + 4], o[8 * i + 5]), pack_bf16(o[8 * i + 6], o[8 * i + 7]));
              } else {
                for (int i = 0; i < 32 && col + i < g.N; ++i) op[i] = __float2bfloat16(o[i]);
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, C::TMEM_COLS);
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

static void make_map(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box) {
  cuuint64_t gd[5], gs[5];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) gs[i] = strides_bytes[i];
  }
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), gd, gs, bx, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
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

template <int BN>
static void launch(const CUtensorMap* m, const GemmArgs& a, cudaStream_t st) {
  using C = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    SD_CUDA(cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const int total = a.m_tiles * a.n_tiles;
  const int grid = total < num_sms() ? total : num_sms();
  if (grid <= 0) return;
  gemm_kernel<BN><<<grid, 192, C::SMEM, st>>>(m[0], m[1], m[2], m[3], a);
  SD_CHECK_LAUNCH();
}

static int pick_bn(int N, int act) {
  if (act == ACT_GEGLU) return N % 256 == 0 ? 256 : 128;
  if (N <= 64) return 64;
  if (N % 256 == 0) return 256;
  if (N % 160 == 0) return 160;
  if (N <= 128 || N % 128 == 0) return 128;
  return 256;
}

void gemm(const GemmDesc& d, cudaStream_t st) {
  GemmArgs a{};
  CUtensorMap maps[4];
  memset(maps, 0, sizeof(maps));
  a.mode = d.mode;
  a.N = d.N;
  int bn = d.bn ? d.bn : pick_bn(d.N, d.act);
  if (d.act == ACT_GEGLU && bn % 128) throw CudaError("GEGLU needs BN multiple of 128");
  a.n_tiles = cdiv(d.N, bn);
  if (d.mode == GEMM_DENSE) {
    if (d.K % 8 || d.lda % 8 || d.ldb % 8) throw CudaError("dense GEMM: K/lda/ldb must be multiples of 8");
    a.M = d.M;
    a.m_tiles = cdiv(d.M, 128);
    a.num_kb = cdiv(d.K, 64);
    a.nsrc = 1;
    uint64_t dA[2] = {(uint64_t)d.K, (uint64_t)d.M}, sA[1] = {(uint64_t)d.lda * 2};
    uint32_t bA[2] = {64, 128};
    make_map(&maps[0], d.A, 2, dA, sA, bA);
    uint64_t dB[2] = {(uint64_t)d.K, (uint64_t)d.N}, sB[1] = {(uint64_t)d.ldb * 2};
    uint32_t bB[2] = {64, (uint32_t)bn};
    make_map(&maps[2], d.Bw[0], 2, dB, sB, bB);
    maps[1] = maps[0];
    maps[3] = maps[2];
  } else {
    a.B = d.B;
    a.H = d.H;
    a.W = d.W;
    a.M = d.B * d.H * d.W;
    conv3_tile_geometry(d.B, d.H, d.W, &a.wt, &a.ht, &a.bt);
    a.tiles_x = cdiv(d.W, a.wt);
    a.tiles_y = cdiv(d.H, a.ht);
    a.m_tiles = a.tiles_x * a.tiles_y * cdiv(d.B, a.bt);
    a.nsrc = d.nsrc;
    a.num_kb = 0;
    for (int s = 0; s < d.nsrc; ++s) {
      if (d.cs[s] % 8) throw CudaError("conv3: channels must be a multiple of 8");
      a.kb_src[s] = cdiv(d.cs[s], 64);
      a.num_kb += 9 * a.kb_src[s];
      uint64_t dA[4] = {(uint64_t)d.cs[s], (uint64_t)d.W, (uint64_t)d.H, (uint64_t)d.B};
      uint64_t sA[3] = {(uint64_t)d.cs[s] * 2, (uint64_t)d.cs[s] * 2 * d.W, (uint64_t)d.cs[s] * 2 * d.W * d.H};
      uint32_t bA[4] = {64, (uint32_t)a.wt, (uint32_t)a.ht, (uint32_t)a.bt};
      make_map(&maps[s], d.xs[s], 4, dA, sA, bA);
      uint64_t dB[3] = {(uint64_t)d.cs[s], 9, (uint64_t)d.N};
      uint64_t sB[2] = {(uint64_t)d.cs[s] * 2, (uint64_t)d.cs[s] * 2 * 9};
      uint32_t bB[3] = {64, 1, (uint32_t)bn};
      make_map(&maps[2 + s], d.Bw[s], 3, dB, sB, bB);
    }
    if (d.nsrc == 1) {
      maps[1] = maps[0];
      maps[3] = maps[2];
    }
  }
  a.m_tile_begin = d.m_tile_begin;
  if (d.m_tile_count >= 0) a.m_tiles = d.m_tile_count;
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
  switch (bn) {
    case 64: launch<64>(maps, a, st); break;
    case 128: launch<128>(maps, a, st); break;
    case 160: launch<160>(maps, a, st); break;
    case 256: launch<256>(maps, a, st); break;
    default: throw CudaError("unsupported BN");
  }
}

}  // namespace sd
