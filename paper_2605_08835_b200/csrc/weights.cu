// On-device weight initialisation with the counter-based generator specified in synth/__init__.py
// (R20 re-specified so both sides can implement it): u = (mix64(seed + (i+1)·φ) >> 40)·2⁻²⁴,
// t = (u − ½)·2, w = fl32(t·bound); γ = 1 + fl32(t·0.1f); β = fl32(t·0.1f). Written directly into
// the kernel-side layout (conv [O][9][I], GEGLU row interleave) and rounded to bf16 (RNE).
#include "common.cuh"
#include "kernels_ew.h"

namespace sd {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float gen(const WeightInit& w, long i) {
  const uint64_t bits = mix64(w.tseed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull);
  const float u = __fmul_rn((float)(bits >> 40), 5.9604644775390625e-08f);  // 2^-24
  const float t = __fmul_rn(__fsub_rn(u, 0.5f), 2.0f);
  if (w.kind == WK_UNIFORM) return __fmul_rn(t, w.bound);
  const float v = __fmul_rn(t, 0.1f);
  return w.kind == WK_GAMMA ? __fadd_rn(1.0f, v) : v;
}

__global__ void init_weight_kernel(const WeightInit w) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  const float v = w.src ? w.src[i] : gen(w, i);
  void* dst = w.dst0;
  long off = i;
  if (w.layout == WL_CONV3) {
    const int tap = (int)(i % 9);
    const long oc = i / 9;
    const int c = (int)(oc % w.I);
    const int o = (int)(oc / w.I);
    if (c < w.I1) {
      off = ((long)o * 9 + tap) * w.Ipad + c;
    } else {
      dst = w.dst1;
      off = ((long)o * 9 + tap) * (w.I - w.I1) + (c - w.I1);
    }
  } else if (w.layout == WL_GEGLU) {
    const int cols = (int)(w.n / (2 * w.F));
    const long row = i / cols;
    const int c = (int)(i % cols);
    const bool gate = row >= w.F;
    const int j = (int)(gate ? row - w.F : row);
    const long drow = (long)(j / 64) * 128 + (gate ? 64 : 0) + (j % 64);
    off = drow * cols + c;
  } else if (w.layout == WL_ROWS) {
    off = (i / w.I) * w.Ipad + (i % w.I);
  }
  if (w.out_bf16 == 2)  // SD_PREC_FP16: the generated bf16 value (R20), held in fp16; loaded values round once
    reinterpret_cast<f16*>(dst)[off] = __float2half_rn(w.src ? v : __bfloat162float(__float2bfloat16_rn(v)));
  else if (w.out_bf16)
    reinterpret_cast<bf16*>(dst)[off] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float*>(dst)[off] = v;
}

void init_weight(const WeightInit& w, cudaStream_t st) {
  if (w.n <= 0) return;
  launch_k(init_weight_kernel, cdiv(w.n, 256), 256, 0, st, w);
  SD_CHECK_LAUNCH();
}

}  // namespace sd
