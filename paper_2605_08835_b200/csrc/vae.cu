// Chunked VAE decode (SURVEY §8(a) a11; PAPER.md:162, :230 VAE Chunking; reading R7 V1
// "stage-synchronous halo tiles"). The decode is an ordered list of work items:
//   HEAD                 post_quant_conv, conv_in, mid block (res, d=512 attention, res) on the whole latent
//   GN_STATS / GN_APPLY  per row band: 128-pixel-chunk partials, merged in fixed order over ALL chunks
//   CONV / SHORTCUT      per row band of the output; the 1-row halo is read from the full input tensor
//                        by the TMA box (zero outside the image = the conv padding)
//   UPSAMPLE             per row band of the 2x output
// `c` chunks are `c` contiguous ranges of the list (min-max partition of the predicted item cost).
// Every item computes exactly what the whole-layer kernel computes for those rows, so any chunking
// is bitwise equal to the whole decode (I6).
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "engine.h"

namespace sd {

// query rows per chunk of the VAE mid-block attention: fp32 scores ≤ 2^24 elements (64 MB)
static size_t vae_attn_rows(size_t P) {
  size_t r = ((size_t)1 << 24) / P / 128 * 128;
  return std::max<size_t>(128, std::min(P, r));
}

enum { VOP_HEAD = 0, VOP_GN_STATS, VOP_GN_APPLY, VOP_CONV, VOP_SHORTCUT, VOP_UPSAMPLE, VOP_FINAL };
enum { NBUF = 6 };

struct DecodeState {
  int h = 0, w = 0, n_chunks = 0, next_chunk = 0;
  int nbands = 1;  // row bands per tail layer (band_rows)
  Arena ar;
  size_t buf_elems = 0;
  void* buf[NBUF];  // activation precision of the engine (bf16, or fp32 in the parity mode)
  float* img_nhwc = nullptr;
  void* gn_ws = nullptr;
  // GroupNorm statistics from the producing conv's epilogue (GemmDescT::gn_part), [P/32][C] per layer:
  // one buffer serves every layer — each GroupNorm's finalize (with its first band) is stream-ordered
  // before the next producer overwrites it
  float2* gn_part = nullptr;
  int head_gnf = 0;  // the head's last conv writes the statistics of the first tail GroupNorm
  std::vector<VItem> items;
  std::vector<int64_t> cost;
  std::vector<int> bounds;
  // recorded on the decode's stream when its last chunk has been enqueued and the state goes back to
  // the pool; the next owner (possibly on another stream) waits on it before touching the buffers
  cudaEvent_t done = nullptr;
};

// row bands of the tail layers: 32 rows (≥ 64-row layers) when the decode is chunked; one band per
// layer for a whole decode (fewer launches; same values — banding is bitwise neutral, I6)
// Row bands of the tail layers. The items only need to be fine enough for the min-max partition into
// c chunks to balance: with whole layers every item is ≤ ~3-5 % of an SD decode, so c ≤ 8 uses one
// band per layer (fewest launches); larger c splits every layer into ⌈c/8⌉ bands, in multiples of
// the minimum aligned band (32 rows at ≥ 64-row layers, else max(8, H/2): conv tile rows and GN
// 128-pixel chunks stay whole). Banding is bitwise neutral (I6). Measured (r01, SD VAE at latent
// 128², c = 4): 32-row bands everywhere cost 48.8 ms vs 14.7 ms for the whole decode.
static int bands_for(int n_chunks) { return std::min(4, std::max(1, (n_chunks + 7) / 8)); }
static int band_rows(int H, int nbands) {
  if (nbands <= 1) return H;
  const int unit = H >= 64 ? 32 : std::max(8, H / 2);
  const int rows = (H + nbands - 1) / nbands;
  return std::max(unit, (rows + unit - 1) / unit * unit);
}

template <class AT>
static AT* sb(DecodeState* s, int i) {
  return static_cast<AT*>(s->buf[i]);
}

template <class AT>
static void conv_desc(GemmDescT<AT>& d, const AT* x, int H, int W, int C, const AT* w, int N, const float* b, void* out,
                      const AT* res) {
  d.mode = GEMM_CONV3;
  d.xs[0] = x;
  d.cs[0] = C;
  d.B = 1;
  d.H = H;
  d.W = W;
  d.Bw[0] = w;
  d.N = N;
  d.out = out;
  d.ldo = N;
  d.bias = b;
  d.res = res;
  d.ldr = N;
}

// restrict a conv launch to output rows [y0, y1) of image 0: 128-pixel boxes of the tcgen05 kernel,
// output pixels of the fp32 kernel (kernels.h)
template <class T>
static void set_band(GemmDescT<T>& d, int H, int W, int y0, int y1) {
  int wt, ht, bt;
  conv3_tile_geometry(1, H, W, &wt, &ht, &bt);
  const int tx = cdiv(W, wt);
  if (y0 % ht || (y1 % ht && y1 != H)) throw CudaError("vae band not aligned to conv tile height");
  d.m_tile_begin = (y0 / ht) * tx;
  d.m_tile_count = cdiv(y1 - y0, ht) * tx;
}
static void set_band(GemmDescF& d, int H, int W, int y0, int y1) {
  (void)H;
  d.m_tile_begin = y0 * W;
  d.m_tile_count = (y1 - y0) * W;
}

template <class AT>
static void run_conv_band(Engine* e, const AT* x, int H, int W, int C, const AT* w, int N, const float* b, void* out,
                          const AT* res, int y0, int y1, int out_f32, cudaStream_t st, float2* gp = nullptr) {
  (void)e;
  GemmDescT<AT> d;
  conv_desc(d, x, H, W, C, w, N, b, out, res);
  d.out_f32 = out_f32;
  d.gn_part = gp;
  set_band(d, H, W, y0, y1);
  gemm(d, st);
}

// whether a conv layer of the tail (B = 1, output H × W × N, 16-bit) can write the GroupNorm statistics
// of its output (a function of the layer only: banding does not change it)
static bool vae_conv_gn_ok(const Engine* e, int H, int W, int C, int N) {
  if (e->f32 || !gn_epilogue_on()) return false;
  GemmDesc d;
  d.mode = GEMM_CONV3;
  d.cs[0] = C;
  d.B = 1;
  d.H = H;
  d.W = W;
  d.N = N;
  d.ldo = N;
  return gemm_gn_ok(d);
}

// whole-tensor resblock at the latent resolution (head)
template <class AT>
static void head_res(Engine* e, DecodeState* s, const ResW& r, AT* x, AT* out, AT* t1, AT* t2, int H, int W,
                     cudaStream_t st, float2* gp = nullptr) {
  const int P = H * W, G = e->vc.groups;
  group_norm(x, t1, 1, P, r.cin, G, r.n1g, r.n1b, e->vc.eps, true, s->gn_ws, st);
  run_conv_band(e, t1, H, W, r.cin, wt<AT>(r.w1), r.cout, r.b1, t2, (const AT*)nullptr, 0, H, 0, st);
  group_norm(t2, t1, 1, P, r.cout, G, r.n2g, r.n2b, e->vc.eps, true, s->gn_ws, st);
  run_conv_band(e, t1, H, W, r.cout, wt<AT>(r.w2), r.cout, r.b2, out, (const AT*)x, 0, H, 0, st, gp);
}

template <class AT>
static void run_head(Engine* e, DecodeState* s, const float* z, cudaStream_t st) {
  const int H = s->h, W = s->w, P = H * W;
  const int cm = e->vc.block_out.back();
  VAEW& V = e->V;
  size_t mk = s->ar.mark();
  AT* zin = s->ar.get<AT>((size_t)P * 64);
  latent_to_nhwc(z, P, 1.f / e->vc.sf, 64, zin, st);
  AT* hq = s->ar.get<AT>((size_t)P * 64);
  SD_CUDA(cudaMemsetAsync(hq, 0, (size_t)P * 64 * sizeof(AT), st));
  GemmDescT<AT> d;
  d.A = zin;
  d.M = P;
  d.K = 64;
  d.lda = 64;
  d.Bw[0] = wt<AT>(V.pq_w);
  d.N = 4;
  d.ldb = 64;
  d.out = hq;
  d.ldo = 64;
  d.bias = V.pq_b;
  gemm(d, st);
  AT* x0 = sb<AT>(s, 1);
  run_conv_band(e, (const AT*)hq, H, W, 64, wt<AT>(V.cin_w), cm, V.cin_b, x0, (const AT*)nullptr, 0, H, 0, st);
  AT* x1 = sb<AT>(s, 2);
  head_res(e, s, V.mid0, x0, x1, sb<AT>(s, 3), sb<AT>(s, 4), H, W, st);
  // single-head attention, d = cm
  AT* a = sb<AT>(s, 3);
  group_norm(x1, a, 1, P, cm, e->vc.groups, V.ag, V.ab, e->vc.eps, false, s->gn_ws, st);
  auto lin = [&](const AT* A, int M, int K, const AT* Wt, int N, const float* b, void* out, int ldo, const AT* res,
                 int bias_row, float alpha, int f32) {
    GemmDescT<AT> g;
    g.A = A;
    g.M = M;
    g.K = K;
    g.lda = K;
    g.Bw[0] = Wt;
    g.N = N;
    g.ldb = K;
    g.out = out;
    g.ldo = ldo;
    g.bias = b;
    g.bias_per_row = bias_row;
    g.res = res;
    g.ldr = ldo;
    g.alpha = alpha;
    g.out_f32 = f32;
    gemm(g, st);
  };
  AT* q = s->ar.get<AT>((size_t)P * cm);
  AT* k = s->ar.get<AT>((size_t)P * cm);
  AT* o = sb<AT>(s, 4);
  lin(a, P, cm, wt<AT>(V.wq), cm, V.bq, q, cm, nullptr, 0, 1.f, 0);
  lin(a, P, cm, wt<AT>(V.wk), cm, V.bk, k, cm, nullptr, 0, 1.f, 0);
  if constexpr (!std::is_same<AT, float>::value) {
    // via tcgen05 GEMMs: S = QKᵀ/√d (fp32), P = softmax(S), O = P·Vᵀᵀ
    // in query chunks of Pq rows, so the fp32 scores stay ≤ 64 MB (1024² = 16384 tokens: 16 chunks of
    // 1024 rows instead of one 1 GiB S and a 512 MiB P)
    const int Pq = (int)vae_attn_rows((size_t)P);
    AT* vt = s->ar.get<AT>((size_t)P * cm);
    float* S = s->ar.get<float>((size_t)Pq * P);
    AT* Pm = s->ar.get<AT>((size_t)Pq * P);
    lin(wt<AT>(V.wv), cm, cm, a, P, V.bv, vt, P, nullptr, 1, 1.f, 0);  // Vᵀ = Wv·aᵀ (+bv per row)
    for (int r0 = 0; r0 < P; r0 += Pq) {
      const int rq = std::min(Pq, P - r0);
      lin(q + (long)r0 * cm, rq, cm, k, P, nullptr, S, P, nullptr, 0, 1.f / sqrtf((float)cm), 1);
      softmax_rows(S, Pm, rq, P, st);
      lin(Pm, rq, P, vt, cm, nullptr, o + (long)r0 * cm, cm, nullptr, 0, 1.f, 0);
    }
  } else {
    // fp32 parity mode: V token-major and the fp32 attention kernel
    AT* v = s->ar.get<AT>((size_t)P * cm);
    lin(a, P, cm, wt<AT>(V.wv), cm, V.bv, v, cm, nullptr, 0, 1.f, 0);
    AttnDescT<AT> ad{};
    ad.Q = q;
    ad.ldq = cm;
    ad.q_bstride = (long)P * cm;
    ad.K = k;
    ad.V = v;
    ad.ldk = cm;
    ad.kv_bstride = (long)P * cm;
    ad.kv_index = nullptr;
    ad.O = o;
    ad.ldo = cm;
    ad.o_bstride = (long)P * cm;
    ad.rows = 1;
    ad.heads = 1;
    ad.d = cm;
    ad.Lq = P;
    ad.Lk = P;
    attention(ad, st);
  }
  AT* x2 = sb<AT>(s, 1);
  lin(o, P, cm, wt<AT>(V.wo), cm, V.bo, x2, cm, x1, 0, 1.f, 0);
  head_res(e, s, V.mid1, x2, sb<AT>(s, 0), sb<AT>(s, 3), sb<AT>(s, 4), H, W, st, s->head_gnf ? s->gn_part : nullptr);
  s->ar.reset(mk);
}

static int64_t conv_cost(long P, int C, int N) { return std::max<int64_t>(1, (int64_t)2 * P * C * 9 * N / 1000000); }

static void build_items(Engine* e, DecodeState* s) {
  const VAECfg& c = e->vc;
  auto& it = s->items;
  auto& cost = s->cost;
  it.clear();
  cost.clear();
  int H = s->h, W = s->w;
  it.push_back(VItem{VOP_HEAD});
  const int cm = c.block_out.back();
  s->head_gnf = vae_conv_gn_ok(e, H, W, cm, cm);
  int cur_gnf = s->head_gnf;  // statistics of `cur` were written by its producer
  cost.push_back(conv_cost((long)H * W, cm, cm) * 5 + (int64_t)H * W * H * W * cm * 4 / 1000000);
  int cur = 0;
  auto other = [&](std::initializer_list<int> used) {
    for (int b = 0; b < 5; ++b)
      if (std::find(used.begin(), used.end(), b) == used.end()) return b;
    return -1;
  };
  int gn_id = 0;
  for (auto& u : e->V.up) {
    for (auto& r : u.res) {
      const int t1 = other({cur});
      const int t2 = other({cur, t1});
      const int t3 = other({cur, t1, t2});
      const int y = other({cur, t1, t2, t3});
      const int br = band_rows(H, s->nbands);
      auto push_gn = [&](int src, int dst, const float* gam, const float* bet, int C, int gnf) {
        if (!gnf)
          for (int yy = 0; yy < H; yy += br) {
            VItem v{VOP_GN_STATS, src, dst, 0, gam, C, 0, H, W, yy, std::min(H, yy + br), gn_id, 1};
            it.push_back(v);
            cost.push_back(std::max<int64_t>(1, (int64_t)(v.y1 - v.y0) * W * C * 2 / 6000));
          }
        for (int yy = 0; yy < H; yy += br) {
          VItem v{VOP_GN_APPLY, src, dst, 0, gam, C, 0, H, W, yy, std::min(H, yy + br), gn_id, 1};
          v.p1 = bet;
          v.gnf = gnf;
          it.push_back(v);
          cost.push_back(std::max<int64_t>(1, (int64_t)(v.y1 - v.y0) * W * C * 4 / 6000));
        }
        ++gn_id;
      };
      push_gn(cur, t1, r.n1g, r.n1b, r.cin, cur_gnf);
      const int c1_gnf = vae_conv_gn_ok(e, H, W, r.cin, r.cout);
      for (int yy = 0; yy < H; yy += br) {
        VItem v{VOP_CONV, t1, t2, -1, &r, r.cin, r.cout, H, W, yy, std::min(H, yy + br), 1, 0};
        v.gnf = c1_gnf;
        it.push_back(v);
        cost.push_back(conv_cost((long)(v.y1 - v.y0) * W, r.cin, r.cout));
      }
      push_gn(t2, t1, r.n2g, r.n2b, r.cout, c1_gnf);
      int resb = cur;
      if (r.wsc) {
        for (int yy = 0; yy < H; yy += br) {
          VItem v{VOP_SHORTCUT, cur, t3, -1, &r, r.cin, r.cout, H, W, yy, std::min(H, yy + br), 0, 0};
          it.push_back(v);
          cost.push_back(std::max<int64_t>(1, conv_cost((long)(v.y1 - v.y0) * W, r.cin, r.cout) / 9));
        }
        resb = t3;
      }
      cur_gnf = vae_conv_gn_ok(e, H, W, r.cout, r.cout);
      for (int yy = 0; yy < H; yy += br) {
        VItem v{VOP_CONV, t1, y, resb, &r, r.cout, r.cout, H, W, yy, std::min(H, yy + br), 2, 0};
        v.gnf = cur_gnf;
        it.push_back(v);
        cost.push_back(conv_cost((long)(v.y1 - v.y0) * W, r.cout, r.cout));
      }
      cur = y;
    }
    if (u.up) {
      const int C = u.ch;
      H *= 2;
      W *= 2;
      const int br = band_rows(H, s->nbands);
      for (int yy = 0; yy < H; yy += br) {
        VItem v{VOP_UPSAMPLE, cur, 5, -1, nullptr, C, C, H, W, yy, std::min(H, yy + br), 0, 0};
        it.push_back(v);
        cost.push_back(std::max<int64_t>(1, (int64_t)(v.y1 - v.y0) * W * C * 3 / 6000));
      }
      const int y = other({cur});
      cur_gnf = vae_conv_gn_ok(e, H, W, C, C);
      for (int yy = 0; yy < H; yy += br) {
        VItem v{VOP_CONV, 5, y, -1, &u, C, C, H, W, yy, std::min(H, yy + br), 3, 0};
        v.gnf = cur_gnf;
        it.push_back(v);
        cost.push_back(conv_cost((long)(v.y1 - v.y0) * W, C, C));
      }
      cur = y;
    }
  }
  const int C0 = c.block_out[0];
  const int t1 = other({cur});
  {
    const int br = band_rows(H, s->nbands);
    if (!cur_gnf)
      for (int yy = 0; yy < H; yy += br) {
        VItem v{VOP_GN_STATS, cur, t1, 0, e->V.nout_g, C0, 0, H, W, yy, std::min(H, yy + br), gn_id, 1};
        it.push_back(v);
        cost.push_back(std::max<int64_t>(1, (int64_t)(v.y1 - v.y0) * W * C0 * 2 / 6000));
      }
    for (int yy = 0; yy < H; yy += br) {
      VItem v{VOP_GN_APPLY, cur, t1, 0, e->V.nout_g, C0, 0, H, W, yy, std::min(H, yy + br), gn_id, 1};
      v.p1 = e->V.nout_b;
      v.gnf = cur_gnf;
      it.push_back(v);
      cost.push_back(std::max<int64_t>(1, (int64_t)(v.y1 - v.y0) * W * C0 * 4 / 6000));
    }
    ++gn_id;
    for (int yy = 0; yy < H; yy += br) {
      VItem v{VOP_CONV, t1, -2, -1, nullptr, C0, 3, H, W, yy, std::min(H, yy + br), 4, 0};
      it.push_back(v);
      cost.push_back(conv_cost((long)(v.y1 - v.y0) * W, C0, 16));
    }
  }
  it.push_back(VItem{VOP_FINAL, 0, 0, 0, nullptr, 0, 0, H, W, 0, H, 0, 0});
  cost.push_back(1);
}

template <class AT>
static void run_item(Engine* e, DecodeState* s, const VItem& v, const float* z, float* image, cudaStream_t st) {
  const int G = e->vc.groups;
  switch (v.op) {
    case VOP_HEAD: run_head<AT>(e, s, z, st); break;
    case VOP_GN_STATS: {
      const int P = v.H * v.W;
      gn_stats_range(sb<AT>(s, v.a), P, v.C, G, v.y0 * v.W, v.y1 * v.W, s->gn_ws, st);
      break;
    }
    case VOP_GN_APPLY: {
      const int P = v.H * v.W;
      const float* gam = static_cast<const float*>(v.p0);
      if (v.gnf)
        gn_apply_range_parts(sb<AT>(s, v.a), sb<AT>(s, v.b), P, v.C, G, v.y0 * v.W, v.y1 * v.W, s->gn_part, gam,
                             static_cast<const float*>(v.p1), e->vc.eps, v.silu != 0, s->gn_ws, st);
      else
        gn_apply_range(sb<AT>(s, v.a), sb<AT>(s, v.b), P, v.C, G, v.y0 * v.W, v.y1 * v.W, gam,
                       static_cast<const float*>(v.p1), e->vc.eps, v.silu != 0, s->gn_ws, st);
      break;
    }
    case VOP_CONV: {
      const AT* res = v.c >= 0 ? sb<AT>(s, v.c) : nullptr;
      const AT* x = sb<AT>(s, v.a);
      float2* gp = v.gnf ? s->gn_part : nullptr;
      if (v.gn == 1) {
        const ResW* r = static_cast<const ResW*>(v.p0);
        run_conv_band(e, x, v.H, v.W, v.C, wt<AT>(r->w1), v.C2, r->b1, sb<AT>(s, v.b), res, v.y0, v.y1, 0, st, gp);
      } else if (v.gn == 2) {
        const ResW* r = static_cast<const ResW*>(v.p0);
        run_conv_band(e, x, v.H, v.W, v.C, wt<AT>(r->w2), v.C2, r->b2, sb<AT>(s, v.b), res, v.y0, v.y1, 0, st, gp);
      } else if (v.gn == 3) {
        const UpW* u = static_cast<const UpW*>(v.p0);
        run_conv_band(e, x, v.H, v.W, v.C, wt<AT>(u->wup), v.C2, u->bup, sb<AT>(s, v.b), res, v.y0, v.y1, 0, st, gp);
      } else {
        GemmDescT<AT> d;
        conv_desc(d, x, v.H, v.W, v.C, wt<AT>(e->V.cout_w), 3, e->V.cout_b, s->img_nhwc, (const AT*)nullptr);
        d.out_f32 = 1;
        d.ldo = 3;
        set_band(d, v.H, v.W, v.y0, v.y1);
        gemm(d, st);
      }
      break;
    }
    case VOP_SHORTCUT: {
      const ResW* r = static_cast<const ResW*>(v.p0);
      GemmDescT<AT> d;
      d.A = sb<AT>(s, v.a) + (long)v.y0 * v.W * v.C;
      d.M = (v.y1 - v.y0) * v.W;
      d.K = v.C;
      d.lda = v.C;
      d.Bw[0] = wt<AT>(r->wsc);
      d.N = v.C2;
      d.ldb = v.C;
      d.out = sb<AT>(s, v.b) + (long)v.y0 * v.W * v.C2;
      d.ldo = v.C2;
      d.bias = r->bsc;
      gemm(d, st);
      break;
    }
    case VOP_UPSAMPLE: {
      const int Wi = v.W / 2;
      upsample2x(sb<AT>(s, v.a) + (long)(v.y0 / 2) * Wi * v.C, sb<AT>(s, v.b) + (long)v.y0 * v.W * v.C, 1,
                 (v.y1 - v.y0) / 2, Wi, v.C, st);
      break;
    }
    case VOP_FINAL:
      nhwc_to_nchw3(s->img_nhwc, 3, (long)v.H * v.W, image, st);
      break;
  }
}

static std::vector<int> chunk_bounds(const std::vector<int64_t>& costs, int c);

static size_t decode_buf_elems(Engine* e, int h, int w) {
  // max P·C over the tail (incl. the 2x-upsampled tensors) and the head
  size_t m = (size_t)h * w * 64;
  int H = h, W = w;
  const int cm = e->vc.block_out.back();
  m = std::max(m, (size_t)H * W * cm);
  for (auto& u : e->V.up) {
    for (auto& r : u.res) m = std::max(m, (size_t)H * W * std::max(r.cin, r.cout));
    if (u.up) {
      H *= 2;
      W *= 2;
      m = std::max(m, (size_t)H * W * u.ch);
    }
  }
  return m;
}

static DecodeState* new_decode(Engine* e, int h, int w) {
  auto* s = new DecodeState();
  s->h = h;
  s->w = w;
  s->buf_elems = decode_buf_elems(e, h, w);
  const size_t P = (size_t)h * w;
  const int cm = e->vc.block_out.back();
  const size_t head = P * 64 * 2 * 2 + P * cm * 2 * 3 + vae_attn_rows(P) * P * 6 + ((size_t)8 << 20);
  const size_t img = (size_t)64 * P * 3 * 4;
  const size_t gnb = gn_workspace_bytes(1, (int)(64 * P), 64, 1024);
  const size_t gpb = (s->buf_elems / 32 + 64) * sizeof(float2);
  s->ar.init(NBUF * (s->buf_elems * e->esize + 4096) + head * (e->esize / 2) + img + gnb + gpb + ((size_t)16 << 20));
  for (int i = 0; i < NBUF; ++i) s->buf[i] = s->ar.alloc(s->buf_elems * e->esize);
  s->img_nhwc = s->ar.get<float>(64 * P * 3);
  s->gn_ws = s->ar.alloc(gnb);
  s->gn_part = s->ar.get<float2>(s->buf_elems / 32 + 64);

  build_items(e, s);
  return s;
}

void destroy_decode(Engine* e, DecodeState* d) {
  (void)e;
  if (d->done) cudaEventDestroy(d->done);
  d->ar.release();
  delete d;
}

void vae_decode_chunk(Engine* e, const float* z, int h, int w, int n_chunks, int chunk, DecodeState** state,
                      float* image, cudaStream_t st) {
  DecodeState* s = *state;
  if (chunk == 0) {
    if (s) throw std::logic_error("chunk 0 needs *state == NULL");
    {
      std::lock_guard<std::mutex> g(e->dmu);
      for (size_t i = 0; i < e->free_decodes.size(); ++i)
        if (e->free_decodes[i]->h == h && e->free_decodes[i]->w == w) {
          s = e->free_decodes[i];
          e->free_decodes.erase(e->free_decodes.begin() + i);
          break;
        }
    }
    if (!s)
      s = new_decode(e, h, w);
    else
      SD_CUDA(cudaStreamWaitEvent(st, s->done, 0));  // the previous owner's kernels may still run
    s->n_chunks = n_chunks;
    s->next_chunk = 0;
    if (s->nbands != bands_for(n_chunks)) {
      s->nbands = bands_for(n_chunks);
      build_items(e, s);
    }
    s->bounds = chunk_bounds(s->cost, n_chunks);
    *state = s;
  }
  if (!s || chunk != s->next_chunk || n_chunks != s->n_chunks || h != s->h || w != s->w)
    throw std::logic_error("VAE chunk out of order");
  const int nb = (int)s->bounds.size() - 1;
  if (chunk < nb)
    for (int i = s->bounds[chunk]; i < s->bounds[chunk + 1]; ++i) {
      if (e->f32)
        run_item<float>(e, s, s->items[i], z, image, st);
      else if (e->f16)
        run_item<f16>(e, s, s->items[i], z, image, st);
      else
        run_item<bf16>(e, s, s->items[i], z, image, st);
    }
  s->next_chunk++;
  if (s->next_chunk == n_chunks) {
    if (!s->done) SD_CUDA(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
    SD_CUDA(cudaEventRecord(s->done, st));
    std::lock_guard<std::mutex> g(e->dmu);
    e->free_decodes.push_back(s);
    *state = nullptr;
  }
}

// V2 independent-tile decode (R7 V2; oracle/vae.py decode_tiled): each
// tile × tile block of the latent is decoded on its own from its halo-padded window (clipped at the
// border) — tile-local GroupNorm and attention, an approximation of the whole decode — and its own
// image region is cut out and written into the output (disjoint writes, no blending). Windows are
// copied to a contiguous scratch latent; each window decode is a whole decode on the pooled states.
void vae_decode_tiled(Engine* e, const float* z, int h, int w, int tile, int halo, float* image, cudaStream_t st) {
  const int f = e->upscale();
  const int wmax = std::min(h, tile + 2 * halo), vmax = std::min(w, tile + 2 * halo);
  const size_t lat_elems = (size_t)4 * wmax * vmax, img_elems = (size_t)3 * f * wmax * f * vmax;
  // one scratch per engine, serialised across callers: a tiled decode enqueues under tile_mu, and the
  // next caller's stream waits on tile_ev (the previous decode's last enqueued work)
  std::unique_lock<std::mutex> tile_lock(e->tile_mu);
  if (!e->tile_ev) SD_CUDA(cudaEventCreateWithFlags(&e->tile_ev, cudaEventDisableTiming));
  else SD_CUDA(cudaStreamWaitEvent(st, e->tile_ev, 0));
  {
    const size_t need = (lat_elems + img_elems) * sizeof(float) + 256;
    if (e->tile_scratch_bytes < need) {
      if (e->tile_scratch) {
        SD_CUDA(cudaEventSynchronize(e->tile_ev));
        SD_CUDA(cudaStreamSynchronize(st));
        cudaFree(e->tile_scratch);
      }
      SD_CUDA(cudaMalloc(&e->tile_scratch, need));
      e->tile_scratch_bytes = need;
    }
  }
  float* win = reinterpret_cast<float*>(e->tile_scratch);
  float* timg = win + ((lat_elems + 63) & ~size_t(63));
  for (int y0 = 0; y0 < h; y0 += tile)
    for (int x0 = 0; x0 < w; x0 += tile) {
      const int y1 = std::min(h, y0 + tile), x1 = std::min(w, x0 + tile);
      const int a0 = std::max(0, y0 - halo), a1 = std::min(h, y1 + halo);
      const int b0 = std::max(0, x0 - halo), b1 = std::min(w, x1 + halo);
      const int wh = a1 - a0, ww = b1 - b0;
      for (int c = 0; c < 4; ++c)
        SD_CUDA(cudaMemcpy2DAsync(win + (size_t)c * wh * ww, (size_t)ww * 4, z + (size_t)c * h * w + (size_t)a0 * w + b0,
                                  (size_t)w * 4, (size_t)ww * 4, wh, cudaMemcpyDeviceToDevice, st));
      DecodeState* ds = nullptr;
      vae_decode_chunk(e, win, wh, ww, 1, 0, &ds, timg, st);
      const int H = f * h, W = f * w, TH = f * wh, TW = f * ww;
      for (int c = 0; c < 3; ++c)
        SD_CUDA(cudaMemcpy2DAsync(image + (size_t)c * H * W + (size_t)f * y0 * W + f * x0, (size_t)W * 4,
                                  timg + (size_t)c * TH * TW + (size_t)f * (y0 - a0) * TW + f * (x0 - b0), (size_t)TW * 4,
                                  (size_t)f * (x1 - x0) * 4, f * (y1 - y0), cudaMemcpyDeviceToDevice, st));
    }
  SD_CUDA(cudaEventRecord(e->tile_ev, st));
}

// min-max contiguous partition, boundaries placed as early as possible (oracle/vae.py chunk_ranges
// is the independent reference; the C-ABI sd_chunk_ranges exposes this function for the tests)
static int need(const std::vector<int64_t>& pre, int s, int n, int64_t cap) {
  if (s >= n) return 0;
  int cnt = 1, start = s;
  for (int k = s + 1; k <= n; ++k)
    if (pre[k] - pre[start] > cap) {
      start = k - 1;
      ++cnt;
    }
  return cnt;
}

static std::vector<int> chunk_bounds(const std::vector<int64_t>& costs, int c) {
  const int n = (int)costs.size();
  c = std::max(1, std::min(c, n));
  std::vector<int64_t> pre(n + 1, 0);
  int64_t mx = 0;
  for (int i = 0; i < n; ++i) {
    pre[i + 1] = pre[i] + costs[i];
    mx = std::max(mx, costs[i]);
  }
  int64_t lo = mx, hi = pre[n];
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (need(pre, 0, n, mid) <= c)
      hi = mid;
    else
      lo = mid + 1;
  }
  std::vector<int> b{0};
  for (int j = 1; j < c; ++j) {
    const int s = b.back();
    int e = s + 1;
    while (!(pre[e] - pre[s] <= lo && need(pre, e, n, lo) <= c - j && n - e >= c - j)) ++e;
    b.push_back(e);
  }
  b.push_back(n);
  return b;
}

std::vector<int> chunk_ranges_api(const std::vector<int64_t>& costs, int c) { return chunk_bounds(costs, c); }

}  // namespace sd
