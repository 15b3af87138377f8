// Engine: model definitions (diffusers SD-1.5 / tiny shapes, R1, App. C), on-device weight init,
// text K/V cache, and the step-level batched UNet iteration behind sd_step_batch (SURVEY §8(a)
// rows a4-a9). Every op is one of our sm_100a kernels; there is no library or CPU fallback.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <stdlib.h>
#include <type_traits>
#include <unordered_map>

#include <nvtx3/nvToolsExt.h>
#include "engine.h"

namespace sd {

// ---------------------------------------------------------------------------------------------
// configs (must match oracle/configs.py by construction; checked end to end by the parity tests)
// ---------------------------------------------------------------------------------------------
UNetCfg unet_cfg(int model) {
  UNetCfg c;
  if (model == SD_MODEL_TINY) {
    c.block_out = {32, 64};
    c.attn = {1, 1};
    c.layers = 1;
    c.groups = 8;
    c.heads = 2;
    c.ctx_dim = 32;
    c.ctx_len = 8;
  } else if (model == SD_MODEL_SD15) {
    c.block_out = {320, 640, 1280, 1280};
    c.attn = {1, 1, 1, 0};
    c.layers = 2;
    c.groups = 32;
    c.heads = 8;
    c.ctx_dim = 768;
    c.ctx_len = 77;
  } else if (model == SD_MODEL_SDXL) {
    c.block_out = {320, 640, 1280};
    c.attn = {0, 1, 1};
    c.depth = {0, 2, 10};
    c.mid_depth = 10;
    c.layers = 2;
    c.groups = 32;
    c.heads = 0;
    c.head_dim = 64;
    c.ctx_dim = 2048;
    c.ctx_len = 77;
    c.add_time_dim = 256;
    c.pooled_dim = 1280;
  } else {  // SD_MODEL_TINY_XL
    c.block_out = {32, 64};
    c.attn = {0, 1};
    c.depth = {0, 2};
    c.mid_depth = 2;
    c.layers = 1;
    c.groups = 8;
    c.heads = 0;
    c.head_dim = 16;
    c.ctx_dim = 48;
    c.ctx_len = 8;
    c.add_time_dim = 8;
    c.pooled_dim = 40;
  }
  return c;
}

VAECfg vae_cfg(int model) {
  VAECfg c;
  if (model == SD_MODEL_TINY || model == SD_MODEL_TINY_XL) {
    c.block_out = {32, 64};
    c.layers = 1;
    c.groups = 8;
  } else {
    c.block_out = {128, 256, 512, 512};
    c.layers = 2;
    c.groups = 32;
  }
  c.sf = model == SD_MODEL_SDXL ? 0.13025f : 0.18215f;
  return c;
}

void Arena::init(size_t bytes) {
  SD_CUDA(cudaMalloc(&base, bytes));
  cap = bytes;
  used = 0;
}
void Arena::release() {
  if (base) cudaFree(base);
  base = nullptr;
  cap = used = 0;
}
void* Arena::alloc(size_t bytes) {
  size_t off = (used + 255) & ~size_t(255);
  if (off + bytes > cap) throw std::bad_alloc();
  used = off + bytes;
  return base + off;
}

// ---------------------------------------------------------------------------------------------
// generator seeds (synth/__init__.py): tensor_seed = mix64(fnv1a64(name) ^ mix64(global_seed))
// ---------------------------------------------------------------------------------------------
static uint64_t mix64h(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t fnv1a64(const std::string& s) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (unsigned char ch : s) {
    h ^= ch;
    h *= 0x100000001B3ull;
  }
  return h;
}

struct Builder {
  Engine* e;
  cudaStream_t st;
  long n_params = 0;
  template <class T>
  T* alloc(long n) {
    T* p = e->warena.get<T>((size_t)n);
    return p;
  }
  // weight matrices in the engine precision (bf16, or fp32 in the parity mode)
  wptr walloc(long n) { return e->warena.alloc((size_t)n * e->esize); }
  wptr woff(wptr base, long elems) const { return static_cast<char*>(base) + elems * (long)e->esize; }
  bool wbf() const { return !e->f32; }
  // canonical tensor `name` of n elements → generated into dst (layout given)
  void gen(const std::string& name, long n, int kind, long fan_in, int layout, void* d0, void* d1, bool bf,
           int O = 0, int I = 0, int I1 = 0, int Ipad = 0, int F = 0) {
    WeightInit w{};
    w.tseed = mix64h(fnv1a64(name) ^ mix64h(e->cfg.weight_seed));
    w.kind = kind;
    w.bound = (float)(1.0 / sqrt((double)fan_in));
    w.layout = layout;
    w.n = n;
    w.O = O;
    w.I = I;
    w.I1 = I1;
    w.Ipad = Ipad;
    w.F = F;
    w.dst0 = d0;
    w.dst1 = d1;
    w.out_bf16 = bf ? (e->f16 ? 2 : 1) : 0;
    w.src = nullptr;
    init_weight(w, st);
    e->wreg[name] = w;
    n_params += n;
  }
  float* bias(const std::string& name, int n, long fan_in, float* dst = nullptr) {
    if (!dst) dst = alloc<float>(n);
    gen(name, n, WK_UNIFORM, fan_in, WL_PLAIN, dst, nullptr, false);
    return dst;
  }
  void norm(const std::string& p, int c, float** g, float** b) {
    *g = alloc<float>(c);
    *b = alloc<float>(c);
    gen(p + ".weight", c, WK_GAMMA, 1, WL_PLAIN, *g, nullptr, false);
    gen(p + ".bias", c, WK_BETA, 1, WL_PLAIN, *b, nullptr, false);
  }
  // conv3x3 [O][I][3][3] → [O][9][Ipad] bf16
  wptr conv3(const std::string& p, int O, int I, int Ipad, float** b) {
    wptr w = walloc((long)O * 9 * Ipad);
    if (Ipad != I) SD_CUDA(cudaMemsetAsync(w, 0, (size_t)O * 9 * Ipad * e->esize, st));
    gen(p + ".weight", (long)O * I * 9, WK_UNIFORM, (long)I * 9, WL_CONV3, w, nullptr, wbf(), O, I, I, Ipad);
    if (b) *b = bias(p + ".bias", O, (long)I * 9);
    return w;
  }
  // linear / 1x1 conv [O][I] (optionally into dst rows)
  wptr lin(const std::string& p, int O, int I, float** b, wptr dst = nullptr, float* bdst = nullptr) {
    wptr w = dst ? dst : walloc((long)O * I);
    gen(p + ".weight", (long)O * I, WK_UNIFORM, I, WL_PLAIN, w, nullptr, wbf());
    if (b) *b = bias(p + ".bias", O, I, bdst);
    return w;
  }
};

static void build_res(Builder& B, const std::string& p, int cin, int cout, int* temb_cursor, ResW* r, bool temb) {
  r->cin = cin;
  r->cout = cout;
  B.norm(p + ".norm1", cin, &r->n1g, &r->n1b);
  r->w1 = B.conv3(p + ".conv1", cout, cin, cin, &r->b1);
  if (temb) {
    const int T = B.e->uc.temb_dim();
    r->temb_off = *temb_cursor;
    B.lin(p + ".time_emb_proj", cout, T, nullptr, B.woff(B.e->U.temb_all_w, (long)r->temb_off * T), nullptr);
    B.bias(p + ".time_emb_proj.bias", cout, T, B.e->U.temb_all_b + r->temb_off);
    *temb_cursor += cout;
  }
  B.norm(p + ".norm2", cout, &r->n2g, &r->n2b);
  r->w2 = B.conv3(p + ".conv2", cout, cout, cout, &r->b2);
  if (cin != cout) r->wsc = B.lin(p + ".conv_shortcut", cout, cin, &r->bsc);
}

static void build_tf(Builder& B, const std::string& p, int C, int depth, int* kv_cursor, TfW* t) {
  Engine* e = B.e;
  const int D = e->uc.ctx_dim;
  t->C = C;
  B.norm(p + ".norm", C, &t->gng, &t->gnb);
  t->wpin = B.lin(p + ".proj_in", C, C, &t->bpin);  // 1×1 conv or Linear: the same [C][C] values
  for (int d = 0; d < depth; ++d) {
    BlkW k{};
    const std::string b = p + ".transformer_blocks." + std::to_string(d);
    B.norm(b + ".norm1", C, &k.l1g, &k.l1b);
    k.wqkv = B.walloc(3L * C * C);
    B.lin(b + ".attn1.to_q", C, C, nullptr, k.wqkv);
    B.lin(b + ".attn1.to_k", C, C, nullptr, B.woff(k.wqkv, (long)C * C));
    B.lin(b + ".attn1.to_v", C, C, nullptr, B.woff(k.wqkv, 2L * C * C));
    k.wo = B.lin(b + ".attn1.to_out.0", C, C, &k.bo);
    B.norm(b + ".norm2", C, &k.l2g, &k.l2b);
    k.wq2 = B.lin(b + ".attn2.to_q", C, C, nullptr);
    k.koff = *kv_cursor;
    B.lin(b + ".attn2.to_k", C, D, nullptr, B.woff(e->U.kv_all_w, (long)k.koff * D));
    k.voff = *kv_cursor + C;
    B.lin(b + ".attn2.to_v", C, D, nullptr, B.woff(e->U.kv_all_w, (long)k.voff * D));
    *kv_cursor += 2 * C;
    k.wo2 = B.lin(b + ".attn2.to_out.0", C, C, &k.bo2);
    B.norm(b + ".norm3", C, &k.l3g, &k.l3b);
    // GEGLU proj [8C][C] with rows interleaved per 64 (value | gate) for the fused epilogue
    k.wff1 = B.walloc(8L * C * C);
    B.gen(b + ".ff.net.0.proj.weight", 8L * C * C, WK_UNIFORM, C, WL_GEGLU, k.wff1, nullptr, B.wbf(), 0, 0, 0, 0, 4 * C);
    k.bff1 = B.alloc<float>(8L * C);
    B.gen(b + ".ff.net.0.proj.bias", 8L * C, WK_UNIFORM, C, WL_GEGLU, k.bff1, nullptr, false, 0, 0, 0, 0, 4 * C);
    k.wff2 = B.lin(b + ".ff.net.2", C, 4 * C, &k.bff2);
    t->blk.push_back(k);
  }
  t->wpout = B.lin(p + ".proj_out", C, C, &t->bpout);
}

static void build_unet(Engine* e, cudaStream_t st) {
  Builder B{e, st};
  const UNetCfg& c = e->uc;
  const int L = (int)c.block_out.size();
  const int T = c.temb_dim();
  // sizes of the fused temb-projection and text-K/V weights
  int temb_total = 0, kv_total = 0;
  {
    int out = c.block_out[0];
    for (int i = 0; i < L; ++i) {
      out = c.block_out[i];
      temb_total += c.layers * out;
      kv_total += c.layers * c.depth_at(i) * 2 * out;
    }
    temb_total += 2 * c.block_out[L - 1];
    kv_total += c.mid_depth * 2 * c.block_out[L - 1];
    for (int i = 0; i < L; ++i) {
      const int o = c.block_out[L - 1 - i];
      temb_total += (c.layers + 1) * o;
      kv_total += (c.layers + 1) * c.depth_at(L - 1 - i) * 2 * o;
    }
  }
  UNetW& U = e->U;
  U.temb_all_n = temb_total;
  U.temb_all_w = B.walloc((long)temb_total * T);
  U.temb_all_b = B.alloc<float>(temb_total);
  U.kv_width = kv_total;
  U.kv_all_w = B.walloc((long)kv_total * c.ctx_dim);
  int tcur = 0, kcur = 0;

  // conv_in: input padded to 64 channels (zeros) so every TMA box is 128-byte aligned
  U.conv_in_w = B.conv3("conv_in", c.block_out[0], c.in_ch, 64, &U.conv_in_b);
  U.lin1_w = B.lin("time_embedding.linear_1", T, c.block_out[0], &U.lin1_b);
  U.lin2_w = B.lin("time_embedding.linear_2", T, T, &U.lin2_b);
  if (c.add_time_dim) {
    U.add1_w = B.lin("add_embedding.linear_1", T, c.add_in(), &U.add1_b);
    U.add2_w = B.lin("add_embedding.linear_2", T, T, &U.add2_b);
  }
  int out = c.block_out[0];
  for (int i = 0; i < L; ++i) {
    const int in = out;
    out = c.block_out[i];
    DownW d;
    d.ch = out;
    d.down = i != L - 1;
    for (int j = 0; j < c.layers; ++j) {
      ResW r;
      build_res(B, "down_blocks." + std::to_string(i) + ".resnets." + std::to_string(j), j == 0 ? in : out, out, &tcur,
                &r, true);
      d.res.push_back(r);
      if (c.attn[i]) {
        TfW t;
        build_tf(B, "down_blocks." + std::to_string(i) + ".attentions." + std::to_string(j), out, c.depth_at(i), &kcur,
                 &t);
        d.tf.push_back(t);
      }
    }
    if (d.down) d.wdown = B.conv3("down_blocks." + std::to_string(i) + ".downsamplers.0.conv", out, out, out, &d.bdown);
    U.down.push_back(d);
  }
  const int cm = c.block_out[L - 1];
  build_res(B, "mid_block.resnets.0", cm, cm, &tcur, &U.mid0, true);
  build_tf(B, "mid_block.attentions.0", cm, c.mid_depth, &kcur, &U.midtf);
  build_res(B, "mid_block.resnets.1", cm, cm, &tcur, &U.mid1, true);
  out = c.block_out[L - 1];
  for (int i = 0; i < L; ++i) {
    const int prev = out;
    out = c.block_out[L - 1 - i];
    const int in = c.block_out[std::max(L - 2 - i, 0)];
    UpW u;
    u.ch = out;
    u.up = i != L - 1;
    const int nl = c.layers + 1;
    for (int j = 0; j < nl; ++j) {
      const int skip = j == nl - 1 ? in : out;
      const int rin = j == 0 ? prev : out;
      ResW r;
      build_res(B, "up_blocks." + std::to_string(i) + ".resnets." + std::to_string(j), rin + skip, out, &tcur, &r,
                true);
      u.res.push_back(r);
      if (c.attn[L - 1 - i]) {
        TfW t;
        build_tf(B, "up_blocks." + std::to_string(i) + ".attentions." + std::to_string(j), out, c.depth_at(L - 1 - i),
                 &kcur, &t);
        u.tf.push_back(t);
      }
    }
    if (u.up) u.wup = B.conv3("up_blocks." + std::to_string(i) + ".upsamplers.0.conv", out, out, out, &u.bup);
    U.up.push_back(u);
  }
  B.norm("conv_norm_out", c.block_out[0], &U.nout_g, &U.nout_b);
  U.conv_out_w = B.conv3("conv_out", 4, c.block_out[0], c.block_out[0], &U.conv_out_b);
  if (tcur != temb_total || kcur != kv_total) throw CudaError("internal: temb/kv width mismatch");
}

static void build_vae(Engine* e, cudaStream_t st) {
  Builder B{e, st};
  const VAECfg& c = e->vc;
  VAEW& V = e->V;
  const int cm = c.block_out.back();
  V.pq_w = B.lin("post_quant_conv", 4, 4, &V.pq_b);
  // pq is applied by a tiny dense GEMM on 64-channel-padded input: store [4][64]
  {
    const size_t es = e->esize;
    wptr w64 = B.walloc(16 * 64);  // N padded to 16 rows
    SD_CUDA(cudaMemsetAsync(w64, 0, 16 * 64 * es, st));
    SD_CUDA(cudaMemcpy2DAsync(w64, 64 * es, V.pq_w, 4 * es, 4 * es, 4, cudaMemcpyDeviceToDevice, st));
    V.pq_w = w64;
    WeightInit& r = e->wreg["post_quant_conv.weight"];
    r.layout = WL_ROWS;
    r.dst0 = w64;
    r.I = 4;
    r.Ipad = 64;
  }
  V.cin_w = B.conv3("decoder.conv_in", cm, 4, 64, &V.cin_b);
  int dummy = 0;
  build_res(B, "decoder.mid_block.resnets.0", cm, cm, &dummy, &V.mid0, false);
  const std::string a = "decoder.mid_block.attentions.0";
  B.norm(a + ".group_norm", cm, &V.ag, &V.ab);
  V.wq = B.lin(a + ".to_q", cm, cm, &V.bq);
  V.wk = B.lin(a + ".to_k", cm, cm, &V.bk);
  V.wv = B.lin(a + ".to_v", cm, cm, &V.bv);
  V.wo = B.lin(a + ".to_out.0", cm, cm, &V.bo);
  build_res(B, "decoder.mid_block.resnets.1", cm, cm, &dummy, &V.mid1, false);
  const int L = (int)c.block_out.size();
  int out = c.block_out[L - 1];
  for (int i = 0; i < L; ++i) {
    const int prev = out;
    out = c.block_out[L - 1 - i];
    UpW u;
    u.ch = out;
    u.up = i != L - 1;
    for (int j = 0; j < c.layers + 1; ++j) {
      ResW r;
      build_res(B, "decoder.up_blocks." + std::to_string(i) + ".resnets." + std::to_string(j), j == 0 ? prev : out,
                out, &dummy, &r, false);
      u.res.push_back(r);
    }
    if (u.up)
      u.wup = B.conv3("decoder.up_blocks." + std::to_string(i) + ".upsamplers.0.conv", out, out, out, &u.bup);
    V.up.push_back(u);
  }
  B.norm("decoder.conv_norm_out", c.block_out[0], &V.nout_g, &V.nout_b);
  V.cout_w = B.conv3("decoder.conv_out", 3, c.block_out[0], c.block_out[0], &V.cout_b);
}

Engine::~Engine() {
  for (auto* d : free_decodes) destroy_decode(this, d);
  warena.release();
  ws.release();
  if (kv_cache) cudaFree(kv_cache);
  if (vt_cache) cudaFree(vt_cache);
  if (aug_cache) cudaFree(aug_cache);
  if (reg_scratch) cudaFree(reg_scratch);
  if (gn_ws) cudaFree(gn_ws);
  if (fold_mem) cudaFree(fold_mem);
  if (tile_scratch) cudaFree(tile_scratch);
  if (tile_ev) cudaEventDestroy(tile_ev);
  if (time_ids) cudaFree(time_ids);
  if (reg_ev) cudaEventDestroy(reg_ev);
  if (meta_dev) cudaFree(meta_dev);
  for (auto& kv : graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (int i = 0; i < 2; ++i) {
    if (meta_pinned[i]) cudaFreeHost(meta_pinned[i]);
    if (meta_ev[i]) cudaEventDestroy(meta_ev[i]);
  }
  if (cap_stream) cudaStreamDestroy(cap_stream);
}

static size_t reg_emb_bytes(const Engine* e) {
  return (((size_t)e->uc.ctx_len * e->uc.ctx_dim * e->esize) + 255) & ~size_t(255);
}

static size_t unet_ws_bytes(const Engine* e) {
  // generous bound: every intermediate of one forward at max rows / max resolution
  const long P = (long)e->cfg.max_latent_hw * e->cfg.max_latent_hw;
  const long R = e->max_rows;
  const int c0 = e->uc.block_out[0];
  // ≈ 60 tensors of R·P·c0 at the top level dominate (level k has P/4^k pixels, ≤ 4·c0 channels)
  const double top = (double)R * P * c0 * e->esize;
  // + split-K partials of one ≤ 64-pixel conv (≤ 8 splits × R·64 rows × 2·c_max fp32)
  const double split = 8.0 * R * 64 * 2 * e->uc.block_out.back() * 4;
  return (size_t)(top * 140 + split) + ((size_t)512 << 20);
}

// sd_engine_set_weight: canonical fp32 values (PyTorch layout of the named diffusers parameter) →
// the kernel-side layout, through the generator kernel's own layout transform (weights.cu)
void set_weight(Engine* e, const std::string& name, const float* host, size_t bytes) {
  auto it = e->wreg.find(name);
  if (it == e->wreg.end()) throw std::invalid_argument("sd_engine_set_weight: unknown parameter '" + name + "'");
  WeightInit w = it->second;
  if (bytes != (size_t)w.n * sizeof(float))
    throw std::invalid_argument("sd_engine_set_weight: '" + name + "' has " + std::to_string(w.n) +
                                " fp32 elements, got " + std::to_string(bytes) + " bytes");
  SD_CUDA(cudaSetDevice(e->device));
  float* d = nullptr;
  SD_CUDA(cudaMalloc(&d, bytes));
  cudaStream_t st;
  SD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  SD_CUDA(cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, st));
  w.src = d;
  init_weight(w, st);
  e->fold_dirty = true;  // folded LayerNorm weights are recomputed before the next step
  SD_CUDA(cudaStreamSynchronize(st));
  SD_CUDA(cudaStreamDestroy(st));
  SD_CUDA(cudaFree(d));
}

void build_engine(Engine* e) {
  SD_CUDA(cudaSetDevice(e->device));
  e->uc = unet_cfg(e->cfg.model);
  e->vc = vae_cfg(e->cfg.model);
  e->max_rows = 2 * e->cfg.b_max;
  e->f32 = e->cfg.precision == SD_PREC_FP32;
  e->f16 = e->cfg.precision == SD_PREC_FP16;
  e->esize = e->f32 ? 4 : 2;
  const size_t wbytes = (e->cfg.model == SD_MODEL_SD15   ? ((size_t)2200 << 20)
                         : e->cfg.model == SD_MODEL_SDXL ? ((size_t)5600 << 20)
                                                         : ((size_t)64 << 20)) *
                        (e->f32 ? 2 : 1);
  e->warena.init(wbytes);
  cudaStream_t st;
  SD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  build_unet(e, st);
  build_vae(e, st);
  SD_CUDA(cudaStreamSynchronize(st));
  SD_CUDA(cudaStreamDestroy(st));
  e->ws.init(unet_ws_bytes(e));
  {
    // off by default: measured slower on the bench step (LayerNorm 42.0 → 23.6 ms but dense GEMMs
    // 262.7 → 298.9 ms per bench step — the short-K consumer GEMMs are epilogue-bound, and the per-element
    // correction with its w̄ / per-column (μ, rstd) loads lands on that critical path); SD_LN_FOLD=1 enables
    const char* lf = getenv("SD_LN_FOLD");
    e->ln_fold = !e->f32 && (lf && lf[0] == '1');
  }
  if (e->ln_fold) {
    // folded copies of every transformer block's LN-consumer weights (3C + C + 8C rows of C) + 2 vectors each
    std::vector<TfW*> tfs;
    for (auto& d : e->U.down)
      for (auto& t : d.tf) tfs.push_back(&t);
    tfs.push_back(&e->U.midtf);
    for (auto& u : e->U.up)
      for (auto& t : u.tf) tfs.push_back(&t);
    size_t bytes = 0;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    for (TfW* t : tfs)
      for (size_t j = 0; j < t->blk.size(); ++j)
        bytes += al(12L * t->C * t->C * e->esize) + 2 * al(12L * t->C * sizeof(float)) + 1024;
    if (bytes) {
      SD_CUDA(cudaMalloc(&e->fold_mem, bytes));
      char* p = static_cast<char*>(e->fold_mem);
      auto take = [&](size_t b) {
        char* r = p;
        p += al(b);
        return r;
      };
      for (TfW* t : tfs)
        for (BlkW& k : t->blk) {
          const long C = t->C;
          k.wqkv_f = take(3 * C * C * e->esize);
          k.wq2_f = take(C * C * e->esize);
          k.wff1_f = take(8 * C * C * e->esize);
          float* v = reinterpret_cast<float*>(take(12 * C * sizeof(float)));
          k.wb_qkv = v, k.wb_q2 = v + 3 * C, k.wb_ff1 = v + 4 * C;
          v = reinterpret_cast<float*>(take(12 * C * sizeof(float)));
          k.bf_qkv = v, k.bf_q2 = v + 3 * C, k.bf_ff1 = v + 4 * C;
        }
    }
    e->fold_dirty = true;
  }
  {
    const size_t gb = gn_workspace_bytes(e->max_rows, e->cfg.max_latent_hw * e->cfg.max_latent_hw * 4, 64, 4096);
    SD_CUDA(cudaMalloc(&e->gn_ws, gb));
    SD_CUDA(cudaMemset(e->gn_ws, 0, gb));
  }
  // text K/V cache slots (slot 0 = unconditional)
  e->max_slots = 4 * e->cfg.b_max + 8;
  e->slot_elems = (long)e->uc.ctx_len * e->U.kv_width;
  SD_CUDA(cudaMalloc(&e->kv_cache, (size_t)e->max_slots * e->slot_elems * e->esize));
  SD_CUDA(cudaMemset(e->kv_cache, 0, (size_t)e->max_slots * e->slot_elems * e->esize));
  if (!e->f32) {  // finite everywhere: the cross-attention reads (and masks) keys beyond a slot's 77
    e->vt_ld = (long)e->max_slots * ((e->uc.ctx_len + 7) / 8 * 8);  // slot stride ⌈77⌉₈ = 80 keys
    SD_CUDA(cudaMalloc(&e->vt_cache, (size_t)e->U.kv_width * e->vt_ld * e->esize));
    SD_CUDA(cudaMemset(e->vt_cache, 0, (size_t)e->U.kv_width * e->vt_ld * e->esize));
  }
  if (e->uc.add_time_dim) {
    SD_CUDA(cudaMalloc(&e->aug_cache, (size_t)e->max_slots * e->uc.temb_dim() * sizeof(float)));
    SD_CUDA(cudaMemset(e->aug_cache, 0, (size_t)e->max_slots * e->uc.temb_dim() * sizeof(float)));
  }
  {
    const UNetCfg& c = e->uc;
    const size_t extra = c.add_time_dim ? ((size_t)((c.add_in() + 127) & ~127) + c.temb_dim()) * e->esize : 0;
    SD_CUDA(cudaMalloc(&e->reg_scratch, reg_emb_bytes(e) + extra + 256));
    SD_CUDA(cudaEventCreateWithFlags(&e->reg_ev, cudaEventDisableTiming));
    static const float ids[6] = {1024.f, 1024.f, 0.f, 0.f, 1024.f, 1024.f};  // R27 (orig, crop, target)
    SD_CUDA(cudaMalloc(&e->time_ids, sizeof(ids)));
    SD_CUDA(cudaMemcpy(e->time_ids, ids, sizeof(ids), cudaMemcpyHostToDevice));
  }
  e->slot_used.assign(e->max_slots, 0);
  e->slot_used[0] = 1;
  e->meta_bytes = 64 << 10;
  SD_CUDA(cudaMalloc(&e->meta_dev, e->meta_bytes));
  e->meta_host.resize(e->meta_bytes);
  for (int i = 0; i < 2; ++i) {
    SD_CUDA(cudaMallocHost(&e->meta_pinned[i], e->meta_bytes));
    SD_CUDA(cudaEventCreateWithFlags(&e->meta_ev[i], cudaEventDisableTiming));
  }
  SD_CUDA(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
  const char* ng = getenv("SD_NO_GRAPH");
  e->use_graphs = !(ng && ng[0] == '1');
  const char* at = getenv("SD_ATTN_TC");
  e->use_attn_tc = !(at && at[0] == '0') && !e->f32;
  // SD_XATTN_TC=1: cross-attention at d ≤ 80 on the general tcgen05 flash kernel (one CTA per 128-query
  // tile; with 77 keys its per-CTA setup dominates: 64² 71 µs) instead of the persistent one below
  const char* xt = getenv("SD_XATTN_TC");
  e->use_xattn_tc = e->use_attn_tc && (xt && xt[0] == '1');
  // the persistent tcgen05 cross-attention (xattention_tc.cu: K / Vᵀ resident across a run of query
  // tiles, P in place of S in TMEM, two CTAs per SM) for d = 40 / 64 / 80; SD_XATTN_TC2=0 falls back to
  // the mma.sync kernel of attention.cu
  const char* x2 = getenv("SD_XATTN_TC2");
  e->use_xattn_tc2 = e->use_attn_tc && !(x2 && x2[0] == '0');
}

// ---------------------------------------------------------------------------------------------
// text K/V cache (computed once per prompt at admission; K/V do not depend on x or t)
// ---------------------------------------------------------------------------------------------
// SDXL "text_time" added embedding of one prompt (R27): [sinusoid_256(id_k) for the 6 time ids ‖
// pooled] → Linear → SiLU → Linear, cached per slot in fp32 and added to linear_2's output per row
template <class AT>
static void added_embedding(Engine* e, const float* pooled, int slot, cudaStream_t st) {
  const UNetCfg& c = e->uc;
  const int T = c.temb_dim(), K = c.add_in(), td = c.add_time_dim;
  // scratch rows after the embedding copy (ctx_kv): [K] then [T], activation precision
  AT* row = reinterpret_cast<AT*>(e->reg_scratch + reg_emb_bytes(e));
  AT* hid = row + ((K + 127) & ~127);
  timestep_sinusoid(e->time_ids, 6, td, row, st);  // [6][td] = one row of 6·td (R27 time ids)
  f32_to_act(pooled, row + 6 * td, c.pooled_dim, st);
  GemmDescT<AT> d;
  d.A = row;
  d.M = 1;
  d.K = K;
  d.lda = K;
  d.Bw[0] = wt<AT>(e->U.add1_w);
  d.N = T;
  d.ldb = K;
  d.out = hid;
  d.ldo = T;
  d.bias = e->U.add1_b;
  d.act = ACT_SILU;
  gemm(d, st);
  GemmDescT<AT> d2;
  d2.A = hid;
  d2.M = 1;
  d2.K = T;
  d2.lda = T;
  d2.Bw[0] = wt<AT>(e->U.add2_w);
  d2.N = T;
  d2.ldb = T;
  d2.out = e->aug_cache + (long)slot * T;
  d2.ldo = T;
  d2.out_f32 = 1;
  d2.bias = e->U.add2_b;
  gemm(d2, st);
}

template <class AT>
static void ctx_kv(Engine* e, const float* emb, int len, int dim, const float* pooled, int slot, cudaStream_t st) {
  std::lock_guard<std::mutex> g(e->reg_mu);
  if (e->reg_ev_valid) SD_CUDA(cudaStreamWaitEvent(st, e->reg_ev, 0));  // the previous user is done
  AT* tmp = reinterpret_cast<AT*>(e->reg_scratch);
  f32_to_act(emb, tmp, (long)len * dim, st);
  GemmDescT<AT> d;
  d.A = tmp;
  d.M = len;
  d.K = dim;
  d.lda = dim;
  d.Bw[0] = wt<AT>(e->U.kv_all_w);
  d.N = e->U.kv_width;
  d.ldb = dim;
  d.out = static_cast<AT*>(e->kv_cache) + (long)slot * e->slot_elems;
  d.ldo = e->U.kv_width;
  gemm(d, st);
  if (e->vt_cache) {
    // the same projections transposed, [kv_width][len] at key column slot·⌈len⌉₈ of the Vᵀ cache (the B
    // operand of the cross-attention PV MMA is K-major over keys)
    GemmDescT<AT> v;
    v.A = wt<AT>(e->U.kv_all_w);
    v.M = e->U.kv_width;
    v.K = dim;
    v.lda = dim;
    v.Bw[0] = tmp;
    v.N = len;
    v.ldb = dim;
    v.out = static_cast<AT*>(e->vt_cache);
    v.ldo = (int)e->vt_ld;
    v.col_off = slot * ((len + 7) / 8 * 8);
    gemm(v, st);
  }
  if (e->uc.add_time_dim) added_embedding<AT>(e, pooled, slot, st);
  SD_CUDA(cudaEventRecord(e->reg_ev, st));
  e->reg_ev_valid = true;
}

int ctx_register(Engine* e, const float* emb, int len, int dim, const float* pooled, int pooled_dim, int slot,
                 cudaStream_t st) {
  if (len != e->uc.ctx_len || dim != e->uc.ctx_dim) throw std::invalid_argument("ctx shape mismatch");
  if (e->uc.add_time_dim && (!pooled || pooled_dim != e->uc.pooled_dim))
    throw std::invalid_argument("this model needs the pooled text embedding (SDXL added conditioning)");
  if (slot < 0) {
    std::lock_guard<std::mutex> g(e->mu);
    for (int s = 1; s < e->max_slots; ++s)
      if (!e->slot_used[s]) {
        slot = s;
        break;
      }
    if (slot < 0) throw std::runtime_error("no free ctx slot");
    e->slot_used[slot] = 1;
  }
  if (e->f32)
    ctx_kv<float>(e, emb, len, dim, pooled, slot, st);
  else if (e->f16)
    ctx_kv<f16>(e, emb, len, dim, pooled, slot, st);
  else
    ctx_kv<bf16>(e, emb, len, dim, pooled, slot, st);
  return slot;
}

// ---------------------------------------------------------------------------------------------
// UNet forward over `rows` rows at h×w (activations NHWC bf16)
// ---------------------------------------------------------------------------------------------
template <class AT>
struct Fwd {
  Engine* e;
  cudaStream_t st;
  int R;
  const float* temb_all;  // [R][temb_all_n] fp32
  const int* kv_index;    // [R] ctx slot per row
  void* gn_ws;

  AT* buf(long elems) { return e->ws.get<AT>((size_t)elems); }

  // GroupNorm statistics emitted by the producing conv / GEMM epilogue (GemmDescT::gn_part), keyed by
  // the output tensor. Every GroupNorm input of the UNet is written by conv() / linear() / gemm_out(),
  // and each of those updates its output's entry (set, or erased when the launch cannot emit them),
  // so a lookup never sees statistics of an older tensor at a reused address. Whether a launch emits
  // them depends only on the layer (gemm_gn_ok), never on the batch: batch invariance holds (I5).
  std::unordered_map<const void*, const float2*> gnp;
  bool gn_epi = false;  // SD_GN_EPI (default on for 16-bit activations)
  // statistics buffer for an output of `pixels` rows × C channels; allocate it next to the output so it
  // lives exactly as long
  float2* gn_buf(long pixels, int C) {
    if (!gn_epi) return nullptr;
    return e->ws.get<float2>((size_t)((pixels + 31) / 32) * C);
  }
  template <class D>
  void gn_note(D& d, const void* out, float2* gp) {
    if (gp && gemm_gn_ok(d)) {
      d.gn_part = gp;
      gnp[out] = gp;
    } else {
      gnp.erase(out);
    }
  }
  const float2* gn_of(const void* x) const {
    auto it = gnp.find(x);
    return it == gnp.end() ? nullptr : it->second;
  }

  void gn(const AT* x, AT* y, int P, int C, const float* g, const float* b, float eps, bool silu) {
    const float2* gp = gn_of(x);
    const int pi = e->prof.begin(PC_GN, st, (gp ? 2.0 : 3.0) * R * P * C * 2);
    if (gp)
      group_norm_parts(x, C, gp, (const AT*)nullptr, 0, (const float2*)nullptr, y, R, P, e->uc.groups, g, b, eps, silu,
                       gn_ws, st);
    else
      group_norm(x, y, R, P, C, e->uc.groups, g, b, eps, silu, gn_ws, st);
    e->prof.end(pi, st);
  }
  // folded LayerNorm: per-token (μ, rstd) only (8 bytes per token); the consumer GEMMs normalise
  const float2* ln_st(const AT* x, long T, int C) {
    float2* st_ = e->ws.get<float2>((size_t)T);
    const int pi = e->prof.begin(PC_LN, st, 1.0 * T * C * 2);
    if constexpr (!std::is_same<AT, float>::value) ln_stats(x, (int)T, C, e->uc.eps_ln, st_, st);
    e->prof.end(pi, st);
    return st_;
  }
  void ln(const AT* x, AT* y, long T, int C, const float* g, const float* b) {
    const int pi = e->prof.begin(PC_LN, st, 2.0 * T * C * 2);
    layer_norm(x, y, (int)T, C, g, b, e->uc.eps_ln, st);
    e->prof.end(pi, st);
  }
  void attn(const AttnDescT<AT>& a) {
    const int pi = e->prof.begin(PC_ATTN, st, 4.0 * a.rows * a.heads * (double)a.Lq * a.Lk * a.d);
    attention(a, st);
    e->prof.end(pi, st);
  }
  void linear(const AT* A, long M, int K, const AT* W, int N, const float* bias, void* out, int ldo,
              const AT* res = nullptr, int act = ACT_NONE, int out_f32 = 0, int cls = PC_GEMM, float2* gp = nullptr,
              int gn_P = 0, const float2* ln_st = nullptr, const float* ln_wb = nullptr, int ln_cols = 0) {
    GemmDescT<AT> d;
    d.A = A;
    d.M = (int)M;
    d.K = K;
    d.lda = K;
    d.Bw[0] = W;
    d.N = N;
    d.ldb = K;
    d.out = out;
    d.ldo = ldo;
    d.bias = bias;
    d.res = res;
    d.ldr = ldo;
    d.act = act;
    d.out_f32 = out_f32;
    d.gn_P = gn_P;
    d.ln_stat = ln_st;  // folded LayerNorm (the weights / bias passed in are W′ / b′)
    d.ln_wbar = ln_wb;
    d.ln_cols = ln_cols;
    d.bias_per_row = ln_cols;  // the Vᵀ projection: b′ per output row
    // split-K for the transformer projections of the ≤ 64-pixel levels (8×8: [1024, 1280, 1280] at 16
    // rows is 40 output tiles on 148 SMs): a function of the layer (pixels per image, K), not of the
    // batch — fp32 partials summed in split order, batch-invariant. Off by default (SD_DENSE_SPLIT=3
    // enables 3 splits): measured neutral-to-negative — the split GEMM keeps most of its fixed cost
    // (ncu: 17.8 µs per third of K vs 25.7 µs whole) and the reduce adds 7-8 µs
    const size_t mk = e->ws.mark();
    if (!std::is_same<AT, float>::value && split_P > 0 && split_P <= 64 && K >= 1280 && act != ACT_GEGLU &&
        !out_f32 && dense_split() > 1) {
      d.splits = dense_split();
      d.split_ws_bytes = gemm_split_ws_bytes(d);
      if (d.split_ws_bytes) d.split_ws = e->ws.get<float>(d.split_ws_bytes / sizeof(float));
    }
    gn_note(d, out, gp);
    const int pi = e->prof.begin(cls, st, 2.0 * M * N * K);
    gemm(d, st);
    e->prof.end(pi, st);
    e->ws.reset(mk);
  }
  int split_P = 0;  // pixels per image of the transformer being run (split-K rule of linear())
  static int dense_split() {
    static int v = -1;
    if (v < 0) {
      const char* s = getenv("SD_DENSE_SPLIT");
      v = s ? atoi(s) : 1;
    }
    return v;
  }
  // 3×3 conv, pad 1; H × W is the OUTPUT size (the input is stride·H × stride·W)
  void conv(const AT* x, int H, int W, int C, const AT* w, int N, const float* bias, void* out,
            const float* temb = nullptr, const AT* res = nullptr, int out_f32 = 0, int ldo = 0, int c_real = 0,
            int stride = 1, float2* gp = nullptr) {
    GemmDescT<AT> d;
    d.mode = GEMM_CONV3;
    d.stride = stride;
    d.xs[0] = x;
    d.cs[0] = C;
    d.B = R;
    d.H = H;
    d.W = W;
    d.Bw[0] = w;
    d.N = N;
    d.out = out;
    d.ldo = ldo ? ldo : N;
    d.bias = bias;
    d.temb = temb;
    d.ld_temb = e->U.temb_all_n;
    d.res = res;
    d.ldr = N;
    d.out_f32 = out_f32;
    const size_t mk = e->ws.mark();
    d.split_ws_bytes = gemm_split_ws_bytes(d);
    if (d.split_ws_bytes) d.split_ws = e->ws.get<float>(d.split_ws_bytes / sizeof(float));
    gn_note(d, out, gp);
    const int pi = e->prof.begin(PC_CONV, st, 2.0 * R * H * W * N * 9.0 * (c_real ? c_real : C));
    gemm(d, st);
    e->prof.end(pi, st);
    e->ws.reset(mk);
  }

  // x1 != nullptr: the block's input is the channel concat [x (C0 = r.cin − C1) | x1 (C1)] (up blocks),
  // read by the two-source GroupNorm and shortcut GEMM instead of being materialised
  AT* resblock(const ResW& r, const AT* x, int H, int W, const AT* x1 = nullptr, int C1 = 0) {
    const int P = H * W;
    const size_t mk = e->ws.mark();
    AT* out = buf((long)R * P * r.cout);  // allocated below the scratch mark
    float2* out_gp = gn_buf((long)R * P, r.cout);
    const size_t mk2 = e->ws.mark();
    (void)mk;
    AT* a = buf((long)R * P * r.cin);
    if (x1) {
      if (!r.wsc) throw std::logic_error("two-source resblock needs the 1x1 shortcut");
      const float2 *g0 = gn_of(x), *g1 = gn_of(x1);
      const int pi = e->prof.begin(PC_GN, st, (g0 && g1 ? 2.0 : 3.0) * R * P * r.cin * 2);
      if (g0 && g1)
        group_norm_parts(x, r.cin - C1, g0, x1, C1, g1, a, R, P, e->uc.groups, r.n1g, r.n1b, e->uc.eps_res, true,
                         gn_ws, st);
      else
        group_norm2(x, r.cin - C1, x1, C1, a, R, P, e->uc.groups, r.n1g, r.n1b, e->uc.eps_res, true, gn_ws, st);
      e->prof.end(pi, st);
    } else {
      gn(x, a, P, r.cin, r.n1g, r.n1b, e->uc.eps_res, true);
    }
    AT* h1 = buf((long)R * P * r.cout);
    conv(a, H, W, r.cin, wt<AT>(r.w1), r.cout, r.b1, h1, temb_all + r.temb_off, nullptr, 0, 0, 0, 1,
         gn_buf((long)R * P, r.cout));
    AT* a2 = buf((long)R * P * r.cout);
    gn(h1, a2, P, r.cout, r.n2g, r.n2b, e->uc.eps_res, true);
    const AT* sc = x;
    if (r.wsc && x1) {
      AT* s = buf((long)R * P * r.cout);
      GemmDescT<AT> d;  // shortcut over the concat: K = [x | x1], weight columns split the same way
      d.nsrc = 2;
      d.xs[0] = x;
      d.cs[0] = r.cin - C1;
      d.xs[1] = x1;
      d.cs[1] = C1;
      d.M = (int)((long)R * P);
      d.K = r.cin;
      d.lda = r.cin;
      d.Bw[0] = wt<AT>(r.wsc);
      d.Bw[1] = wt<AT>(r.wsc) + (r.cin - C1);
      d.N = r.cout;
      d.ldb = r.cin;
      d.out = s;
      d.ldo = r.cout;
      d.bias = r.bsc;
      gn_note(d, s, nullptr);
      const int pi = e->prof.begin(PC_CONV1, st, 2.0 * R * P * r.cout * r.cin);
      gemm(d, st);
      e->prof.end(pi, st);
      sc = s;
    } else if (r.wsc) {
      AT* s = buf((long)R * P * r.cout);
      linear(x, (long)R * P, r.cin, wt<AT>(r.wsc), r.cout, r.bsc, s, r.cout, nullptr, ACT_NONE, 0, PC_CONV1);
      sc = s;
    }
    conv(a2, H, W, r.cout, wt<AT>(r.w2), r.cout, r.b2, out, nullptr, sc, 0, 0, 0, 1, out_gp);
    e->ws.reset(mk2);
    return out;
  }

  AT* transformer(const TfW& t, const AT* x, int H, int W) {
    const int C = t.C, P = H * W;
    const long T = (long)R * P;
    const int heads = e->uc.heads_at(C), dh = C / heads;
    split_P = P;
    AT* out = buf(T * C);
    float2* out_gp = gn_buf(T, C);
    const size_t mk = e->ws.mark();
    AT* a = buf(T * C);
    gn(x, a, P, C, t.gng, t.gnb, e->uc.eps_tf, false);
    AT* h = buf(T * C);
    linear(a, T, C, wt<AT>(t.wpin), C, t.bpin, h, C, nullptr, ACT_NONE, 0, PC_CONV1);
    AT* hb = buf(T * C);  // ping-pong hidden state across blocks
    for (const BlkW& k : t.blk) {
      const size_t mb = e->ws.mark();
      AT* n = buf(T * C);
      const bool fold = e->ln_fold;  // LayerNorm folded into the q|k|v, q2 and FF1 GEMMs (no normalised copy)
      const float2* s1 = nullptr;
      if (fold)
        s1 = ln_st(h, T, C);
      else
        ln(h, n, T, C, k.l1g, k.l1b);
      AT* o = buf(T * C);
      bool tc = false;
      if constexpr (!std::is_same<AT, float>::value) tc = e->use_attn_tc && attention_tc_supported(dh, P, C);
      if (tc) {
        // tcgen05 flash attention: q|k token-major from one GEMM, Vᵀ channel-major from another
        AT* qk = buf(T * 2 * C);
        AT* vt = buf(T * C);
        if (fold) {
          linear(h, T, C, wt<AT>(k.wqkv_f), 2 * C, k.bf_qkv, qk, 2 * C, nullptr, ACT_NONE, 0, PC_GEMM, nullptr, 0, s1,
                 k.wb_qkv, 0);
          linear(wt<AT>(k.wqkv_f) + 2L * C * C, C, C, h, (int)T, k.bf_qkv + 2 * C, vt, (int)T, nullptr, ACT_NONE, 0,
                 PC_GEMM, nullptr, 0, s1, k.wb_qkv + 2 * C, 1);
        } else {
          linear(n, T, C, wt<AT>(k.wqkv), 2 * C, nullptr, qk, 2 * C);
          linear(wt<AT>(k.wqkv) + 2L * C * C, C, C, n, (int)T, nullptr, vt, (int)T);
        }
        const int pi = e->prof.begin(PC_ATTN, st, 4.0 * R * heads * (double)P * P * dh);
        if constexpr (!std::is_same<AT, float>::value) attention_tc(qk, vt, o, R, heads, dh, C, P, st);
        e->prof.end(pi, st);
      } else {
        AT* qkv = buf(T * 3 * C);
        if (fold)
          linear(h, T, C, wt<AT>(k.wqkv_f), 3 * C, k.bf_qkv, qkv, 3 * C, nullptr, ACT_NONE, 0, PC_GEMM, nullptr, 0, s1,
                 k.wb_qkv, 0);
        else
          linear(n, T, C, wt<AT>(k.wqkv), 3 * C, nullptr, qkv, 3 * C);
        AttnDescT<AT> ad{};
        ad.Q = qkv;
        ad.ldq = 3 * C;
        ad.q_bstride = (long)P * 3 * C;
        ad.K = qkv + C;
        ad.V = qkv + 2 * C;
        ad.ldk = 3 * C;
        ad.kv_bstride = (long)P * 3 * C;
        ad.kv_index = nullptr;
        ad.O = o;
        ad.ldo = C;
        ad.o_bstride = (long)P * C;
        ad.rows = R;
        ad.heads = heads;
        ad.d = dh;
        ad.Lq = P;
        ad.Lk = P;
        attn(ad);
      }
      AT* h2 = buf(T * C);
      linear(o, T, C, wt<AT>(k.wo), C, k.bo, h2, C, h);
      AT* q2 = buf(T * C);
      if (fold) {
        const float2* s2 = ln_st(h2, T, C);
        linear(h2, T, C, wt<AT>(k.wq2_f), C, k.bf_q2, q2, C, nullptr, ACT_NONE, 0, PC_GEMM, nullptr, 0, s2, k.wb_q2, 0);
      } else {
        ln(h2, n, T, C, k.l2g, k.l2b);
        linear(n, T, C, wt<AT>(k.wq2), C, nullptr, q2, C);
      }
      bool xtc = false, xtc2 = false;
      if constexpr (!std::is_same<AT, float>::value) {
        xtc2 = e->use_xattn_tc2 && e->vt_cache && xattention_tc2_supported(dh, e->uc.ctx_len);
        // d = 160 (the 16×16 level and the 8×8 mid block): the general tcgen05 kernel (16×16: 13.5 vs
        // 14.3 µs on mma.sync)
        const bool pick = e->use_xattn_tc || (e->use_attn_tc && dh == 160);
        xtc = !xtc2 && pick && e->vt_cache && attention_tc_supported(dh, 128, C);
      }
      if (xtc2) {
        if constexpr (!std::is_same<AT, float>::value) {
          const int pi = e->prof.begin(PC_ATTN, st, 4.0 * R * heads * (double)P * e->uc.ctx_len * dh);
          xattention_tc2(q2, static_cast<const AT*>(e->kv_cache), e->U.kv_width, e->max_slots, k.koff,
                         static_cast<const AT*>(e->vt_cache), e->U.kv_width, e->vt_ld, k.voff, kv_index,
                         e->uc.ctx_len, o, R, heads, dh, C, P, st);
          e->prof.end(pi, st);
        }
      } else if (xtc) {
        if constexpr (!std::is_same<AT, float>::value) {
          const int pi = e->prof.begin(PC_ATTN, st, 4.0 * R * heads * (double)P * e->uc.ctx_len * dh);
          xattention_tc(q2, static_cast<const AT*>(e->kv_cache), e->U.kv_width, e->max_slots, k.koff,
                        static_cast<const AT*>(e->vt_cache), e->U.kv_width, e->vt_ld, k.voff, kv_index,
                        e->uc.ctx_len, o, R, heads, dh, C, P, st);
          e->prof.end(pi, st);
        }
      } else {
      AttnDescT<AT> cd{};
      cd.Q = q2;
      cd.ldq = C;
      cd.q_bstride = (long)P * C;
      cd.K = static_cast<const AT*>(e->kv_cache) + k.koff;
      cd.V = static_cast<const AT*>(e->kv_cache) + k.voff;
      cd.ldk = e->U.kv_width;
      cd.kv_bstride = e->slot_elems;
      cd.kv_index = kv_index;
      cd.O = o;
      cd.ldo = C;
      cd.o_bstride = (long)P * C;
      cd.rows = R;
      cd.heads = heads;
      cd.d = dh;
      cd.Lq = P;
      cd.Lk = e->uc.ctx_len;
      attn(cd);
      }
      AT* h3 = buf(T * C);
      linear(o, T, C, wt<AT>(k.wo2), C, k.bo2, h3, C, h2);
      AT* gg = buf(T * 4 * C);
      if (fold) {
        const float2* s3 = ln_st(h3, T, C);
        linear(h3, T, C, wt<AT>(k.wff1_f), 8 * C, k.bf_ff1, gg, 4 * C, nullptr, ACT_GEGLU, 0, PC_GEMM, nullptr, 0, s3,
               k.wb_ff1, 0);
      } else {
        ln(h3, n, T, C, k.l3g, k.l3b);
        linear(n, T, C, wt<AT>(k.wff1), 8 * C, k.bff1, gg, 4 * C, nullptr, ACT_GEGLU);
      }
      linear(gg, T, 4 * C, wt<AT>(k.wff2), C, k.bff2, hb, C, h3);  // block output → hb
      e->ws.reset(mb);
      std::swap(h, hb);
    }
    linear(h, T, C, wt<AT>(t.wpout), C, t.bpout, out, C, x, ACT_NONE, 0, PC_CONV1, out_gp, P);  // proj_out + the input
    split_P = 0;
    e->ws.reset(mk);
    return out;
  }
};

template <class AT>
static void unet_forward(Engine* e, cudaStream_t st, int R, int H, int W, const AT* x_in, const float* t_row,
                         const int* kv_index, float* eps_out) {
  const UNetCfg& c = e->uc;
  UNetW& U = e->U;
  Fwd<AT> f{e, st, R, nullptr, kv_index, nullptr};
  f.gn_ws = e->gn_ws;
  f.gn_epi = !std::is_same<AT, float>::value && gn_epilogue_on();
  const int T = c.temb_dim(), C0 = c.block_out[0];
  // time embedding: sinusoid → linear_1 → SiLU → linear_2 → SiLU (the ResBlocks consume SiLU(temb))
  AT* sinus = f.buf((long)R * C0);
  timestep_sinusoid(t_row, R, C0, sinus, st);
  AT* t1 = f.buf((long)R * T);
  f.linear(sinus, R, C0, wt<AT>(U.lin1_w), T, U.lin1_b, t1, T, nullptr, ACT_SILU);
  AT* t2 = f.buf((long)R * T);
  if (c.add_time_dim) {
    // SDXL: temb = linear_2(·) + aug[slot(row)] (the prompt's cached added embedding), then SiLU
    float* aug_rows = e->ws.get<float>((size_t)R * T);
    gather_rows_f32(e->aug_cache, kv_index, R, T, aug_rows, st);
    GemmDescT<AT> d;
    d.A = t1;
    d.M = R;
    d.K = T;
    d.lda = T;
    d.Bw[0] = wt<AT>(U.lin2_w);
    d.N = T;
    d.ldb = T;
    d.out = t2;
    d.ldo = T;
    d.bias = U.lin2_b;
    d.temb = aug_rows;
    d.ld_temb = T;
    d.rows_per_img = 1;
    d.act = ACT_SILU;
    const int pi = e->prof.begin(PC_GEMM, st, 2.0 * R * T * T);
    gemm(d, st);
    e->prof.end(pi, st);
  } else {
    f.linear(t1, R, T, wt<AT>(U.lin2_w), T, U.lin2_b, t2, T, nullptr, ACT_SILU);
  }
  float* temb_all = e->ws.get<float>((size_t)R * U.temb_all_n);
  f.linear(t2, R, T, wt<AT>(U.temb_all_w), U.temb_all_n, U.temb_all_b, temb_all, U.temb_all_n, nullptr, ACT_NONE, 1);
  f.temb_all = temb_all;

  int h = H, w = W;
  AT* x = f.buf((long)R * h * w * C0);
  float2* x_gp = f.gn_buf((long)R * h * w, C0);
  f.conv(x_in, h, w, 64, wt<AT>(U.conv_in_w), C0, U.conv_in_b, x, nullptr, nullptr, 0, 0, c.in_ch, 1, x_gp);
  struct Skip {
    AT* p;
    int C;
  };
  std::vector<Skip> skips;
  skips.push_back({x, C0});
  int C = C0;
  for (auto& d : U.down) {
    for (size_t j = 0; j < d.res.size(); ++j) {
      x = f.resblock(d.res[j], x, h, w);
      C = d.res[j].cout;
      if (!d.tf.empty()) x = f.transformer(d.tf[j], x, h, w);
      skips.push_back({x, C});
    }
    if (d.down) {
      const int ho = (h + 1) / 2, wo = (w + 1) / 2;
      const size_t mk = e->ws.mark();
      AT* out = f.buf((long)R * ho * wo * C);
      float2* out_gp = f.gn_buf((long)R * ho * wo, C);
      const size_t mk2 = e->ws.mark();
      if constexpr (!std::is_same<AT, float>::value) {
        // 3×3 / stride 2 / pad 1 as an implicit GEMM whose TMA boxes step 2 input pixels per output
        // pixel (element strides), so the taps are never materialised
        if (h % 2 || w % 2) throw std::invalid_argument("downsampler: odd spatial size");
        f.conv(x, ho, wo, C, wt<AT>(d.wdown), C, d.bdown, out, nullptr, nullptr, 0, 0, 0, 2, out_gp);
      } else {
        AT* cols = f.buf((long)R * ho * wo * 9 * C);
        im2col_s2(x, cols, R, h, w, C, st);
        f.linear(cols, (long)R * ho * wo, 9 * C, wt<AT>(d.wdown), C, d.bdown, out, C);
      }
      e->ws.reset(mk2);
      (void)mk;
      x = out;
      h = ho;
      w = wo;
      skips.push_back({x, C});
    }
  }
  x = f.resblock(U.mid0, x, h, w);
  x = f.transformer(U.midtf, x, h, w);
  x = f.resblock(U.mid1, x, h, w);
  for (auto& u : U.up) {
    for (size_t j = 0; j < u.res.size(); ++j) {
      Skip s = skips.back();
      skips.pop_back();
      if constexpr (!std::is_same<AT, float>::value) {
        x = f.resblock(u.res[j], x, h, w, s.p, s.C);  // concat [x | skip] read as two sources
      } else {  // fp32 parity mode: its SIMT GEMM takes one source
        const int Ccat = C + s.C;
        AT* cat = f.buf((long)R * h * w * Ccat);
        concat_channels(x, C, s.p, s.C, cat, (long)R * h * w, st);
        x = f.resblock(u.res[j], cat, h, w);
      }
      C = u.res[j].cout;
      if (!u.tf.empty()) x = f.transformer(u.tf[j], x, h, w);
    }
    if (u.up) {
      AT* upx = f.buf((long)R * 4 * h * w * C);
      upsample2x(x, upx, R, h, w, C, st);
      h *= 2;
      w *= 2;
      AT* out = f.buf((long)R * h * w * C);
      f.conv(upx, h, w, C, wt<AT>(u.wup), C, u.bup, out, nullptr, nullptr, 0, 0, 0, 1, f.gn_buf((long)R * h * w, C));
      x = out;
    }
  }
  AT* a = f.buf((long)R * h * w * C);
  f.gn(x, a, h * w, C, U.nout_g, U.nout_b, c.eps_res, true);
  f.conv(a, h, w, C, wt<AT>(U.conv_out_w), 4, U.conv_out_b, eps_out, nullptr, nullptr, 1, 4);
}

// ---------------------------------------------------------------------------------------------
// sampler coefficients (R4 / R5), fp64 on the host, passed as fp32
// ---------------------------------------------------------------------------------------------
struct Sched {
  double ac[1000];
  Sched() {
    const double a = sqrt(0.00085), b = sqrt(0.012);
    double prod = 1.0;
    for (int i = 0; i < 1000; ++i) {
      const double s = a + (b - a) * i / 999.0;
      prod *= 1.0 - s * s;
      ac[i] = prod;
    }
  }
};
static const Sched& sched() {
  static Sched s;
  return s;
}
static int t_of(int n, int i) { return (n - 1 - i) * (1000 / n) + 1; }
static double euler_sigma(int n, int i) {
  if (i >= n) return 0.0;
  const double a = sched().ac[t_of(n, i)];
  return sqrt((1.0 - a) / a);
}

void sampler_coefs(int sampler, int n, int i, float* t_out, float* c_in, float* A, float* Bc) {
  const Sched& s = sched();
  const int t = t_of(n, i);
  *t_out = (float)t;
  if (sampler == SD_SAMPLER_DDIM) {
    const int tp = t - 1000 / n;
    const double at = s.ac[t], ap = tp >= 0 ? s.ac[tp] : s.ac[0];
    *c_in = 1.f;
    *A = (float)sqrt(ap / at);
    *Bc = (float)(sqrt(1.0 - ap) - sqrt(ap) * sqrt(1.0 - at) / sqrt(at));
  } else {
    const double si = euler_sigma(n, i), sn = euler_sigma(n, i + 1);
    *c_in = (float)(1.0 / sqrt(si * si + 1.0));
    *A = 1.f;
    *Bc = (float)(sn - si);
  }
}

float init_sigma(int sampler, int n) {
  if (sampler == SD_SAMPLER_DDIM) return 1.f;
  const double s0 = euler_sigma(n, 0);
  return (float)sqrt(s0 * s0 + 1.0);
}

// ---------------------------------------------------------------------------------------------
// sd_step_batch
// ---------------------------------------------------------------------------------------------
// eps_dump (debug): run the gather and the UNet only, copy ε (fp32 NHWC [rows][h][w][4], rows in R26
// order) to eps_dump and leave the latents alone. eps_inject (debug): skip the UNet and apply the K12
// combine + sampler to the given ε (same layout). Both run eagerly (no graph).
// recompute the folded LayerNorm weights (W′ = W·diag(γ), w̄, b′ = b + W·β) of every transformer block, on
// the step's stream, when a weight changed since the last fold (build, sd_engine_set_weight)
template <class AT>
static void refold_t(Engine* e, cudaStream_t st) {
  auto fold_tf = [&](TfW& t) {
    const int C = t.C;
    for (BlkW& k : t.blk) {
      ln_fold(wt<AT>(k.wqkv), 3 * C, C, k.l1g, k.l1b, (const float*)nullptr, static_cast<AT*>(k.wqkv_f), k.wb_qkv,
              k.bf_qkv, st);
      ln_fold(wt<AT>(k.wq2), C, C, k.l2g, k.l2b, (const float*)nullptr, static_cast<AT*>(k.wq2_f), k.wb_q2, k.bf_q2,
              st);
      ln_fold(wt<AT>(k.wff1), 8 * C, C, k.l3g, k.l3b, k.bff1, static_cast<AT*>(k.wff1_f), k.wb_ff1, k.bf_ff1, st);
    }
  };
  for (auto& d : e->U.down)
    for (auto& t : d.tf) fold_tf(t);
  fold_tf(e->U.midtf);
  for (auto& u : e->U.up)
    for (auto& t : u.tf) fold_tf(t);
}
static void refold_if_dirty(Engine* e, cudaStream_t st) {
  if (!e->ln_fold || !e->fold_dirty) return;
  if (e->f16)
    refold_t<f16>(e, st);
  else
    refold_t<bf16>(e, st);
  e->fold_dirty = false;
}

void step_batch(Engine* e, const sd_batch* b, cudaStream_t st, float* eps_dump, const float* eps_inject) {
  refold_if_dirty(e, st);
  const int n = b->n_req, h = b->latent_h, w = b->latent_w, hw = h * w;
  std::vector<int> row_req, unc_row(n, -1);
  for (int r = 0; r < n; ++r) row_req.push_back(r);
  for (int r = 0; r < n; ++r)
    if (b->has_uncond[r]) {
      unc_row[r] = (int)row_req.size();
      row_req.push_back(r);
    }
  const int R = (int)row_req.size();
  // host metadata block → one H2D copy
  char* hb = e->meta_host.data();
  size_t off = 0;
  auto put = [&](const void* src, size_t bytes) {
    off = (off + 15) & ~size_t(15);
    const size_t o = off;
    memcpy(hb + o, src, bytes);
    off += bytes;
    return o;
  };
  std::vector<float> c_in(n), ga(n), A(n), Bc(n), t_row(R);
  std::vector<int> kv(R);
  std::vector<const float*> lat(n);
  for (int r = 0; r < n; ++r) {
    float t;
    sampler_coefs(e->cfg.sampler, b->n_steps[r], b->step[r], &t, &c_in[r], &A[r], &Bc[r]);
    ga[r] = b->guidance[r];
    lat[r] = b->latents[r];
    t_row[r] = t;
  }
  for (int k = 0; k < R; ++k) {
    const int r = row_req[k];
    t_row[k] = t_row[r];
    kv[k] = (k < n && b->ctx_slot) ? b->ctx_slot[r] : 0;
  }
  const size_t o_lat = put(lat.data(), n * sizeof(float*));
  const size_t o_cin = put(c_in.data(), n * 4);
  const size_t o_t = put(t_row.data(), R * 4);
  const size_t o_rr = put(row_req.data(), R * 4);
  const size_t o_ur = put(unc_row.data(), n * 4);
  const size_t o_g = put(ga.data(), n * 4);
  const size_t o_a = put(A.data(), n * 4);
  const size_t o_b = put(Bc.data(), n * 4);
  const size_t o_kv = put(kv.data(), R * 4);
  // the pinned staging buffer is reused: wait until the previous step's H2D copy consumed it
  const int par = e->meta_parity;
  e->meta_parity ^= 1;
  if (e->meta_ev_valid[par]) SD_CUDA(cudaEventSynchronize(e->meta_ev[par]));
  memcpy(e->meta_pinned[par], hb, off);
  char* db = e->meta_dev;
  RowMap m;
  m.latents = reinterpret_cast<const float* const*>(db + o_lat);
  m.c_in = reinterpret_cast<const float*>(db + o_cin);
  m.t_row = reinterpret_cast<const float*>(db + o_t);
  m.row_req = reinterpret_cast<const int*>(db + o_rr);
  m.unc_row = reinterpret_cast<const int*>(db + o_ur);
  m.guidance = reinterpret_cast<const float*>(db + o_g);
  m.coef_a = reinterpret_cast<const float*>(db + o_a);
  m.coef_b = reinterpret_cast<const float*>(db + o_b);
  const int* kv_dev = reinterpret_cast<const int*>(db + o_kv);

  // the metadata H2D runs on the caller's stream ahead of the step (outside the graph, so one graph
  // serves both staging buffers); the step itself — K11 gather → UNet → K12 combine + sampler — has
  // deterministic arena addresses for a given (n_req, rows, h, w): captured once, then replayed.
  SD_CUDA(cudaMemcpyAsync(e->meta_dev, e->meta_pinned[par], off, cudaMemcpyHostToDevice, st));
  auto run = [&](cudaStream_t s) {
    e->ws.reset(0);
    float* eps;
    if (eps_inject) {
      combine_update(m, n, hw, eps_inject, 4, reinterpret_cast<float* const*>(db + o_lat), s);
      return;
    }
    if (e->f32) {
      float* x_in = e->ws.get<float>((size_t)R * hw * 64);
      gather_rows(m, R, hw, 64, x_in, s);
      eps = e->ws.get<float>((size_t)R * hw * 4);
      unet_forward<float>(e, s, R, h, w, x_in, m.t_row, kv_dev, eps);
    } else if (e->f16) {
      f16* x_in = e->ws.get<f16>((size_t)R * hw * 64);
      gather_rows(m, R, hw, 64, x_in, s);
      eps = e->ws.get<float>((size_t)R * hw * 4);
      unet_forward<f16>(e, s, R, h, w, x_in, m.t_row, kv_dev, eps);
    } else {
      bf16* x_in = e->ws.get<bf16>((size_t)R * hw * 64);
      gather_rows(m, R, hw, 64, x_in, s);
      eps = e->ws.get<float>((size_t)R * hw * 4);
      unet_forward<bf16>(e, s, R, h, w, x_in, m.t_row, kv_dev, eps);
    }
    if (eps_dump) {
      SD_CUDA(cudaMemcpyAsync(eps_dump, eps, (size_t)R * hw * 4 * sizeof(float), cudaMemcpyDeviceToDevice, s));
      return;
    }
    combine_update(m, n, hw, eps, 4, reinterpret_cast<float* const*>(db + o_lat), s);
  };
  const bool use_graph = e->use_graphs && !eps_dump && !eps_inject;
  const bool prof = e->prof.on;
  if (!use_graph) {
    run(st);
  } else {
    // profiled graphs (event-record nodes around every launch) are cached separately
    auto& g = e->graphs[std::make_tuple(n, R, h, w, prof ? 1 : 0)];
    if (!g.seen) {
      run(st);  // first call runs eagerly (sets kernel attributes, validates), capture next time
      g.seen = true;
    } else {
      if (!g.exec) {
        cudaGraph_t graph;
        SD_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
        if (prof) e->prof.sink = &g.prof;
        try {
          run(e->cap_stream);
        } catch (...) {
          e->prof.sink = nullptr;
          cudaStreamEndCapture(e->cap_stream, &graph);
          throw;
        }
        e->prof.sink = nullptr;
        SD_CUDA(cudaStreamEndCapture(e->cap_stream, &graph));
        size_t nn = 0;
        SD_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        SD_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
        long kern = 0;
        for (auto nd : nodes) {
          cudaGraphNodeType ty;
          SD_CUDA(cudaGraphNodeGetType(nd, &ty));
          kern += ty == cudaGraphNodeTypeKernel;
        }
        ::sd::g_launches.fetch_sub(kern, std::memory_order_relaxed);  // capture executes nothing
        g.kernels = kern;
        SD_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
        SD_CUDA(cudaGraphDestroy(graph));
        ++e->graphs_built;
      }
      SD_CUDA(cudaGraphLaunch(g.exec, st));
      ::sd::g_launches.fetch_add(g.kernels ? g.kernels : 0, std::memory_order_relaxed);
      if (prof) e->prof.accumulate(g.prof);  // synchronises on this replay's events
    }
  }
  // the staging buffer `par` may be rewritten once this step's copy has run
  SD_CUDA(cudaEventRecord(e->meta_ev[par], st));
  e->meta_ev_valid[par] = true;
}

}  // namespace sd

namespace sd {
cudaEvent_t Prof::ev() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  SD_CUDA(cudaEventCreate(&e));
  return e;
}
// SD_NVTX=1: one NVTX range per kernel class around each launch (eager mode), so that ncu can select
// e.g. only the conv launches: ncu --nvtx --nvtx-include "conv/" …  (SD_NO_GRAPH=1)
static int nvtx_on() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("SD_NVTX");
    v = s && s[0] == '1';
  }
  return v;
}
static const char* const kClassName[] = {"conv", "gemm", "attn", "gn", "ln", "other", "vae", "other"};
int Prof::begin(int cls, cudaStream_t st, double work) {
  if (nvtx_on()) nvtxRangePushA(kClassName[cls & 7]);
  if (!on) return -1;
  std::vector<Rec>& dst = sink ? *sink : recs;
  Rec r{cls, ev(), ev(), work};
  // inside a stream capture the record must be an external event-record node to be readable later
  SD_CUDA(sink ? cudaEventRecordWithFlags(r.a, st, cudaEventRecordExternal) : cudaEventRecord(r.a, st));
  dst.push_back(r);
  return (int)dst.size() - 1;
}
void Prof::end(int idx, cudaStream_t st) {
  if (nvtx_on()) nvtxRangePop();
  if (idx < 0) return;
  std::vector<Rec>& dst = sink ? *sink : recs;
  SD_CUDA(sink ? cudaEventRecordWithFlags(dst[idx].b, st, cudaEventRecordExternal) : cudaEventRecord(dst[idx].b, st));
}
void Prof::accumulate(const std::vector<Rec>& rs) {
  for (auto& r : rs) {
    SD_CUDA(cudaEventSynchronize(r.b));
    float t = 0;
    SD_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    tot_ms[r.cls] += t;
    tot_n[r.cls] += 1;
    tot_work[r.cls] += r.work;
  }
}
void Prof::read(int cls, double* ms, long long* n, double* work) {
  accumulate(recs);
  for (auto& r : recs) {
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  recs.clear();
  *ms = tot_ms[cls];
  *n = tot_n[cls];
  *work = tot_work[cls];
}
void Prof::reset() {
  for (auto& r : recs) {
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  recs.clear();
  for (int i = 0; i < PC_N; ++i) {
    tot_ms[i] = 0;
    tot_n[i] = 0;
    tot_work[i] = 0;
  }
}
Prof::~Prof() {
  reset();
  for (auto e : pool) cudaEventDestroy(e);
}
}  // namespace sd
