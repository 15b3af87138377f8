// Memory-bound helper kernels: ragged CFG gather (K11), CFG combine + DDIM/Euler update (K12),
// timestep sinusoid (K10 front), nearest upsample, stride-2 im2col, channel concat, layout moves.
// All vectorised where the layout allows; all launch-bound at the sizes of one UNet step.
#include "common.cuh"
#include "kernels_ew.h"

namespace sd {

// K11: UNet input rows. Row ρ belongs to request r = row_req[ρ]; writes T(c_in_r · x_r) NHWC
// with channels [4, cpad) zero.  (R26 row order is encoded in row_req.)
// T = bf16 on the product path, float in the fp32 parity mode (R19); likewise below.
// one thread per (pixel, 8-channel vector): vector 0 carries the 4 latent channels, the rest of the
// cpad-channel row is zero; 16/32-byte stores
template <class T>
__global__ void gather_rows_kernel(RowMap m, int rows, int hw, int nv, T* __restrict__ out) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;  // (pixel of a row, vector)
  if (i >= (long)rows * hw * nv) return;
  const long px = i / nv;
  const int v = (int)(i - px * nv);
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (v == 0) {
    const int rho = (int)(px / hw), p = (int)(px % hw);
    const int r = m.row_req[rho];
    const float* x = m.latents[r];
    const float c = m.c_in[r];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = c * x[(long)k * hw + p];
  }
  store8(out + i * 8, o);
}

template <class T>
void gather_rows(const RowMap& m, int rows, int hw, int cpad, T* out, cudaStream_t st) {
  if (cpad % 8) throw CudaError("gather_rows: cpad must be a multiple of 8");
  const long n = (long)rows * hw * (cpad / 8);
  launch_k(gather_rows_kernel<T>, cdiv(n, 256), 256, 0, st, m, rows, hw, cpad / 8, out);
  SD_CHECK_LAUNCH();
}

// K12: per request r, ε̃ = has_uncond ? ε_u + g(ε_c − ε_u) : ε_c (R2, R3), then x ← a·x + b·ε̃
// (DDIM η=0 written as a·x + b·ε̃ with a = √(ᾱ_prev/ᾱ_t), b = √(1−ᾱ_prev) − √(ᾱ_prev(1−ᾱ_t)/ᾱ_t);
// Euler: a = 1, b = σ_{i+1} − σ_i). ε rows are NHWC fp32 [rows][hw][ld_eps] (first 4 channels);
// the cond row of request r is row r (R26).
__global__ void combine_update_kernel(RowMap m, int n_req, int hw, const float* __restrict__ eps, int ld,
                                      float* const* lat) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)n_req * hw) return;
  const int r = (int)(i / hw), p = (int)(i % hw);
  const int u = m.unc_row[r];
  const float g = m.guidance[r], a = m.coef_a[r], b = m.coef_b[r];
  const float* ec = eps + ((long)r * hw + p) * ld;
  const float* eu = u >= 0 ? eps + ((long)u * hw + p) * ld : nullptr;
  float* x = lat[r];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float e = ec[c];
    if (eu) e = eu[c] + g * (e - eu[c]);
    const long xi = (long)c * hw + p;
    x[xi] = a * x[xi] + b * e;
  }
}

void combine_update(const RowMap& m, int n_req, int hw, const float* eps, int ld_eps, float* const* lat,
                    cudaStream_t st) {
  const long n = (long)n_req * hw;
  launch_k(combine_update_kernel, cdiv(n, 256), 256, 0, st, m, n_req, hw, eps, ld_eps, lat);
  SD_CHECK_LAUNCH();
}

// K10 front: [cos(t·f_k) ‖ sin(t·f_k)], f_k = exp(−ln(10⁴)·k/half) (flip_sin_to_cos, R27).
template <class T>
__global__ void sinusoid_kernel(const float* __restrict__ t, int rows, int dim, T* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int half = dim / 2;
  if (i >= rows * half) return;
  const int r = i / half, k = i % half;
  const float f = expf(-9.210340371976184f * (float)k / (float)half);
  const float arg = t[r] * f;
  act_st(out + (long)r * dim + k, cosf(arg));
  act_st(out + (long)r * dim + half + k, sinf(arg));
}

template <class T>
void timestep_sinusoid(const float* t_row, int rows, int dim, T* out, cudaStream_t st) {
  launch_k(sinusoid_kernel<T>, cdiv(rows * dim / 2, 256), 256, 0, st, t_row, rows, dim, out);
  SD_CHECK_LAUNCH();
}

// nearest 2× upsample, NHWC, 16-byte vectors
__global__ void upsample2x_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int B, int H, int W, int V) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long n = (long)B * 2 * H * 2 * W * V;
  if (i >= n) return;
  const int v = (int)(i % V);
  long p = i / V;
  const int xo = (int)(p % (2 * W));
  p /= 2 * W;
  const int yo = (int)(p % (2 * H));
  const int b = (int)(p / (2 * H));
  y[i] = x[(((long)b * H + yo / 2) * W + xo / 2) * V + v];
}

template <class T>
void upsample2x(const T* x, T* y, int B, int H, int W, int C, cudaStream_t st) {
  const int V = C * (int)sizeof(T) / 16;
  const long n = (long)B * 4 * H * W * V;
  launch_k(upsample2x_kernel, cdiv(n, 256), 256, 0, st, reinterpret_cast<const uint4*>(x), reinterpret_cast<uint4*>(y), B,
                                                  H, W, V);
  SD_CHECK_LAUNCH();
}

// im2col for 3×3 / stride 2 / pad 1: y[(b,yo,xo)][tap·C + c] (tap-major, matches weights [N][9][C])
__global__ void im2col_s2_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int B, int H, int W, int V) {
  pdl_wait();
  const int Ho = (H + 1) / 2, Wo = (W + 1) / 2;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long n = (long)B * Ho * Wo * 9 * V;
  if (i >= n) return;
  const int v = (int)(i % V);
  long r = i / V;
  const int tap = (int)(r % 9);
  r /= 9;
  const int xo = (int)(r % Wo);
  r /= Wo;
  const int yo = (int)(r % Ho);
  const int b = (int)(r / Ho);
  const int yi = 2 * yo + tap / 3 - 1, xi = 2 * xo + tap % 3 - 1;
  uint4 val = make_uint4(0, 0, 0, 0);
  if (yi >= 0 && yi < H && xi >= 0 && xi < W) val = x[(((long)b * H + yi) * W + xi) * V + v];
  y[i] = val;
}

template <class T>
void im2col_s2(const T* x, T* y, int B, int H, int W, int C, cudaStream_t st) {
  const int V = C * (int)sizeof(T) / 16;
  const long n = (long)B * ((H + 1) / 2) * ((W + 1) / 2) * 9 * V;
  launch_k(im2col_s2_kernel, cdiv(n, 256), 256, 0, st, reinterpret_cast<const uint4*>(x), reinterpret_cast<uint4*>(y), B,
                                                 H, W, V);
  SD_CHECK_LAUNCH();
}

__global__ void concat_kernel(const uint4* __restrict__ a, int va, const uint4* __restrict__ b, int vb,
                              uint4* __restrict__ y, long P) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int V = va + vb;
  if (i >= P * V) return;
  const long p = i / V;
  const int v = (int)(i % V);
  y[i] = v < va ? a[p * va + v] : b[p * vb + (v - va)];
}

template <class T>
void concat_channels(const T* a, int ca, const T* b, int cb, T* y, long P, cudaStream_t st) {
  const int per = 16 / (int)sizeof(T);  // elements per 16-byte vector
  const long n = P * (ca + cb) / per;
  launch_k(concat_kernel, cdiv(n, 256), 256, 0, st, reinterpret_cast<const uint4*>(a), ca / per,
                                              reinterpret_cast<const uint4*>(b), cb / per, reinterpret_cast<uint4*>(y),
                                              P);
  SD_CHECK_LAUNCH();
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, bf16* __restrict__ y, long n) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __float2bfloat16(x[i]);
}

void f32_to_bf16(const float* x, bf16* y, long n, cudaStream_t st) {
  launch_k(f32_to_bf16_kernel, cdiv(n, 256), 256, 0, st, x, y, n);
  SD_CHECK_LAUNCH();
}

__global__ void f32_to_f16_kernel(const float* __restrict__ x, f16* __restrict__ y, long n) {
  pdl_wait();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __float2half_rn(x[i]);
}

void f32_to_act(const float* x, f16* y, long n, cudaStream_t st) {
  launch_k(f32_to_f16_kernel, cdiv(n, 256), 256, 0, st, x, y, n);
  SD_CHECK_LAUNCH();
}

void f32_to_act(const float* x, float* y, long n, cudaStream_t st) {
  SD_CUDA(cudaMemcpyAsync(y, x, (size_t)n * sizeof(float), cudaMemcpyDeviceToDevice, st));
}

// dst[r][0..n) = src[idx[r]][0..n) (fp32): the SDXL added embedding of each row's prompt slot
__global__ void gather_rows_f32_kernel(const float* __restrict__ src, const int* __restrict__ idx, int n,
                                       float* __restrict__ dst) {
  pdl_wait();
  const int r = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[(long)r * n + i] = src[(long)idx[r] * n + i];
}

void gather_rows_f32(const float* src, const int* idx, int rows, int n, float* dst, cudaStream_t st) {
  launch_k(gather_rows_f32_kernel, dim3(cdiv(n, 256), rows), 256, 0, st, src, idx, n, dst);
  SD_CHECK_LAUNCH();
}

template <class T>
__global__ void latent_to_nhwc_kernel(const float* __restrict__ z, int hw, float scale, int cpad, T* __restrict__ out) {
  pdl_wait();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= hw) return;
  T* o = out + (long)p * cpad;
  for (int c = 0; c < cpad; ++c) act_st(o + c, c < 4 ? z[(long)c * hw + p] * scale : 0.f);
}

template <class T>
void latent_to_nhwc(const float* z, int hw, float scale, int cpad, T* out, cudaStream_t st) {
  launch_k(latent_to_nhwc_kernel<T>, cdiv(hw, 256), 256, 0, st, z, hw, scale, cpad, out);
  SD_CHECK_LAUNCH();
}

__global__ void nhwc_to_nchw3_kernel(const float* __restrict__ x, int ld, long P, float* __restrict__ y) {
  pdl_wait();
  const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
#pragma unroll
  for (int c = 0; c < 3; ++c) y[c * P + p] = x[p * ld + c];
}

void nhwc_to_nchw3(const float* x, int ld, long P, float* y, cudaStream_t st) {
  launch_k(nhwc_to_nchw3_kernel, cdiv(P, 256), 256, 0, st, x, ld, P, y);
  SD_CHECK_LAUNCH();
}

#define SD_EW_INST(T)                                                                              \
  template void gather_rows<T>(const RowMap&, int, int, int, T*, cudaStream_t);                    \
  template void timestep_sinusoid<T>(const float*, int, int, T*, cudaStream_t);                   \
  template void upsample2x<T>(const T*, T*, int, int, int, int, cudaStream_t);                    \
  template void im2col_s2<T>(const T*, T*, int, int, int, int, cudaStream_t);                     \
  template void concat_channels<T>(const T*, int, const T*, int, T*, long, cudaStream_t);         \
  template void latent_to_nhwc<T>(const float*, int, float, int, T*, cudaStream_t);
SD_EW_INST(bf16)
SD_EW_INST(f16)
SD_EW_INST(float)

}  // namespace sd
