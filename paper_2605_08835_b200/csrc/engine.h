// Engine internals: model definitions, device weights, workspaces, UNet / VAE forward.
#pragma once
#include <atomic>
#include <map>
#include <unordered_map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "kernels_ew.h"
#include "sd_api.h"

namespace sd {

struct UNetCfg {
  std::vector<int> block_out;
  std::vector<int> attn;
  int layers, groups, heads, ctx_dim, ctx_len;
  float eps_res = 1e-5f, eps_tf = 1e-6f, eps_ln = 1e-5f;
  int in_ch = 4;
  // SDXL generalisations (oracle/configs.py UNetConfig): transformer depth per level (empty → 1),
  // mid depth, head-dim heads (0 → `heads`), "text_time" added embedding dims (0 → none)
  std::vector<int> depth;
  int mid_depth = 1, head_dim = 0, add_time_dim = 0, pooled_dim = 0;
  int temb_dim() const { return 4 * block_out[0]; }
  int depth_at(int level) const { return attn[level] ? (depth.empty() ? 1 : depth[level]) : 0; }
  int heads_at(int C) const { return head_dim ? C / head_dim : heads; }
  int add_in() const { return 6 * add_time_dim + pooled_dim; }
};
struct VAECfg {
  std::vector<int> block_out;
  int layers, groups;
  float sf;
  float eps = 1e-6f;
};
UNetCfg unet_cfg(int model);
VAECfg vae_cfg(int model);

// Weight matrices are stored in the engine's activation precision: bf16 (SD_PREC_BF16) or fp32
// (SD_PREC_FP32 parity mode). `wptr` is the untyped device pointer; wt<T>(p) views it as T.
using wptr = void*;
template <class T>
static inline const T* wt(const void* p) {
  return static_cast<const T*>(p);
}

// bump allocator over one cudaMalloc'd block
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
  void init(size_t bytes);
  void release();
  void* alloc(size_t bytes);
  template <class T>
  T* get(size_t n) { return reinterpret_cast<T*>(alloc(n * sizeof(T))); }
  size_t mark() const { return used; }
  void reset(size_t m) { used = m; }
};

struct ResW {
  int cin, cout, temb_off;
  float *n1g, *n1b, *b1, *n2g, *n2b, *b2, *bsc = nullptr;
  wptr w1, w2, wsc = nullptr;
};
struct BlkW {  // one BasicTransformerBlock
  float *l1g, *l1b, *bo, *l2g, *l2b, *bo2, *l3g, *l3b, *bff1, *bff2;
  wptr wqkv, wo, wq2, wo2, wff1, wff2;
  int koff, voff;  // column offsets of this block's K / V in the text K/V cache rows
  // LayerNorm folded into the consumer GEMMs (Engine::ln_fold; norm.cu ln_fold): W′ = W·diag(γ) of the
  // LN1 → q|k|v, LN2 → q2 and LN3 → FF1 weights, their row sums w̄ and the folded biases b′
  wptr wqkv_f = nullptr, wq2_f = nullptr, wff1_f = nullptr;
  float *wb_qkv = nullptr, *bf_qkv = nullptr, *wb_q2 = nullptr, *bf_q2 = nullptr, *wb_ff1 = nullptr,
        *bf_ff1 = nullptr;
};
struct TfW {  // one Transformer2DModel: GN → proj_in → blocks → proj_out (+ x)
  int C;
  float *gng, *gnb, *bpin, *bpout;
  wptr wpin, wpout;
  std::vector<BlkW> blk;
};
struct DownW {
  std::vector<ResW> res;
  std::vector<TfW> tf;
  bool down;
  wptr wdown = nullptr;
  float* bdown = nullptr;
  int ch;
};
struct UpW {
  std::vector<ResW> res;
  std::vector<TfW> tf;
  bool up;
  wptr wup = nullptr;
  float* bup = nullptr;
  int ch;
};
struct UNetW {
  wptr conv_in_w;
  float* conv_in_b;
  wptr lin1_w, lin2_w, temb_all_w;
  float *lin1_b, *lin2_b, *temb_all_b;
  int temb_all_n = 0;
  std::vector<DownW> down;
  ResW mid0, mid1;
  TfW midtf;
  std::vector<UpW> up;
  float *nout_g, *nout_b, *conv_out_b;
  wptr conv_out_w;
  wptr kv_all_w;   // [kv_width][ctx_dim]: for each transformer block (forward order) K_j then V_j
  int kv_width = 0;
  // SDXL added embedding: Linear(add_in → T) → SiLU → Linear(T → T); per prompt slot, cached
  wptr add1_w = nullptr, add2_w = nullptr;
  float *add1_b = nullptr, *add2_b = nullptr;
};
struct VAEW {
  float *pq_b, *cin_b;
  wptr pq_w, cin_w;
  ResW mid0, mid1;
  float *ag, *ab, *bq, *bk, *bv, *bo;
  wptr wq, wk, wv, wo;
  std::vector<UpW> up;
  float *nout_g, *nout_b, *cout_b;
  wptr cout_w;
};

// one VAE work item: op over a band of output rows [y0, y1) (R7 V1)
// SD_GN_EPI=0: GroupNorm statistics by the separate statistics pass instead of the producers' conv /
// GEMM epilogues (gemm.cu gn_colstats)
inline bool gn_epilogue_on() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("SD_GN_EPI");
    v = !(s && s[0] == '0');
  }
  return v != 0;
}

struct VItem {
  int op;          // VOP_*
  int a, b, c;     // buffer ids (src, dst, extra)
  const void* p0;  // layer parameters
  int C, C2, H, W; // channels in/out, spatial size of the OUTPUT
  int y0, y1;
  int gn;          // GN layer index (partials slot)
  int silu;
  const void* p1 = nullptr;
  // GN_STATS / GN_APPLY: the statistics come from the producer's epilogue (DecodeState::gn_part; the
  // stats item is a no-op); CONV: this launch writes them for the next GroupNorm
  int gnf = 0;
};

struct DecodeState;

// Per-kernel-class device timing with CUDA events on the launching stream (bench roofline).
// PC_CONV1: the UNet's 1×1 convolutions (ResBlock shortcuts, transformer proj_in / proj_out) — dense
// GEMMs counted in SURVEY §8(d)'s UNet conv fraction together with PC_CONV
enum { PC_CONV = 0, PC_GEMM = 1, PC_ATTN = 2, PC_GN = 3, PC_LN = 4, PC_OTHER = 5, PC_VAE = 6, PC_CONV1 = 7, PC_N = 8 };
struct Prof {
  bool on = false;
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    double work;
  };
  std::vector<Rec> recs;            // eager launches since the last read
  std::vector<Rec>* sink = nullptr; // while capturing a profiled graph: that graph's records
  std::vector<cudaEvent_t> pool;
  double tot_ms[PC_N] = {0}, tot_work[PC_N] = {0};
  long long tot_n[PC_N] = {0};
  cudaEvent_t ev();
  int begin(int cls, cudaStream_t st, double work);
  void end(int idx, cudaStream_t st);
  void accumulate(const std::vector<Rec>& rs);
  void read(int cls, double* ms, long long* n, double* work);
  void reset();
  ~Prof();
};

struct Engine {
  Prof prof;
  sd_engine_config cfg{};
  int device = 0;
  UNetCfg uc;
  VAECfg vc;
  Arena warena;          // weights
  // canonical parameter name (diffusers naming, oracle/configs.py) → where and how it is stored
  // (sd_engine_set_weight rewrites a tensor through the same layout transform as the generator)
  std::unordered_map<std::string, WeightInit> wreg;
  Arena ws;              // UNet workspace (reset every step)
  UNetW U{};
  VAEW V{};
  bool f32 = false;       // SD_PREC_FP32: fp32 weights / activations, SIMT kernels (fp32.cu)
  bool f16 = false;       // SD_PREC_FP16: fp16 weights / activations on the same tcgen05 kernels
  size_t esize = 2;       // bytes per weight / activation element
  // text K/V cache (activation precision)
  void* kv_cache = nullptr;
  // text Vᵀ cache for the tcgen05 cross-attention: [kv_width][vt_ld], key j of slot s at column s·ctx_len + j
  // (rows of every layer's K and V projections; the kernel reads the V rows)
  void* vt_cache = nullptr;
  long vt_ld = 0;
  float* aug_cache = nullptr;  // SDXL: [max_slots][T] added embedding per prompt slot (fp32)
  // admission scratch (the activation-precision copy of a prompt embedding, the added-embedding
  // rows, the constant time ids): reused by every sd_ctx_register; the event orders reuse across
  // streams (no stream-ordered allocation on the admission path)
  char* reg_scratch = nullptr;
  void* gn_ws = nullptr;  // UNet GroupNorm workspace (partials + affine table), persistent
  // LayerNorm folded into its consumer GEMMs (16-bit modes, SD_LN_FOLD=1; off by default: measured slower):
  // the folded weights live in fold_mem and are recomputed before the next step whenever a weight changed
  bool ln_fold = false;
  bool fold_dirty = true;
  void* fold_mem = nullptr;
  float* time_ids = nullptr;
  cudaEvent_t reg_ev = nullptr;
  bool reg_ev_valid = false;
  std::mutex reg_mu;
  int max_slots = 0;
  long slot_elems = 0;
  std::vector<int> slot_used;
  // per-step metadata (device)
  char* meta_dev = nullptr;
  size_t meta_bytes = 0;
  std::vector<char> meta_host;
  char* meta_pinned[2] = {nullptr, nullptr};  // double-buffered pinned staging (graph H2D source)
  cudaEvent_t meta_ev[2] = {nullptr, nullptr};  // recorded after the step that read staging [i]
  bool meta_ev_valid[2] = {false, false};
  int meta_parity = 0;
  // CUDA graphs of the whole step keyed by (n_req, rows, h, w)
  struct GraphEntry {
    bool seen = false;
    cudaGraphExec_t exec = nullptr;
    long kernels = 0;
    std::vector<Prof::Rec> prof;  // event records of a profiled graph (read after every replay)
  };
  std::map<std::tuple<int, int, int, int, int>, GraphEntry> graphs;
  bool use_graphs = true;
  bool use_attn_tc = true;
  bool use_xattn_tc = true;   // tcgen05 cross-attention over the text K / Vᵀ caches (general kernel)
  bool use_xattn_tc2 = false; // the persistent tcgen05 cross-attention (xattention_tc.cu)  // tcgen05 flash attention where supported (SD_ATTN_TC=0 disables)
  int graphs_built = 0;
  cudaStream_t cap_stream = nullptr;
  int max_rows = 0;
  std::atomic<int64_t> launches{0};
  bool failed = false;
  std::mutex mu;
  // VAE decode slots
  std::vector<DecodeState*> free_decodes;
  std::mutex dmu;
  void* tile_scratch = nullptr;  // V2 tiled decode: window latent + window image (grown on demand)
  size_t tile_scratch_bytes = 0;
  cudaEvent_t tile_ev = nullptr;  // recorded after the last use of tile_scratch; the next user waits on it
  std::mutex tile_mu;             // one tiled decode enqueues at a time
  void* server = nullptr;  // serve_gpu.cu Server while serving
  int upscale() const { return 1 << ((int)vc.block_out.size() - 1); }
  ~Engine();
};

void build_engine(Engine* e);
void set_weight(Engine* e, const std::string& name, const float* host, size_t bytes);
void step_batch(Engine* e, const sd_batch* b, cudaStream_t st, float* eps_dump = nullptr,
                const float* eps_inject = nullptr);
int ctx_register(Engine* e, const float* emb, int len, int dim, const float* pooled, int pooled_dim, int slot,
                 cudaStream_t st);
void vae_decode_chunk(Engine* e, const float* z, int h, int w, int n_chunks, int chunk, DecodeState** state,
                      float* image, cudaStream_t st);
void destroy_decode(Engine* e, DecodeState* d);
void vae_decode_tiled(Engine* e, const float* z, int h, int w, int tile, int halo, float* image, cudaStream_t st);

}  // namespace sd

struct sd_engine {
  sd::Engine e;
};
