/* sd_api.h — C ABI of the SynerDiff B200 hot path (libsynerdiff.so).
 *
 * Paper: "SynerDiff: Synergetic Continuous Batching for Fast and Parallel Diffusion Model
 * Inference" (arXiv 2605.08835, /root/reference/PAPER.md, cited "P:<line>"). Blueprint:
 * SURVEY.md §8(b). Readings of the paper the ABI depends on: SURVEY.md §8(c) R1-R32, DESIGN.md.
 *
 * Conventions
 *  - Every call returns sd_status (int32). SD_OK = 0, errors are negative. Nothing throws or
 *    aborts across the ABI. SD_E_INVAL is returned by argument validation before anything is
 *    enqueued and leaves all state unchanged. A CUDA error puts the engine into a sticky FAILED
 *    state: every later call on it returns SD_E_STATE. sd_last_error() gives a per-thread
 *    message for the last non-OK status.
 *  - Ownership: the caller owns every buffer it passes; the library never frees caller memory.
 *    The engine owns its weights, workspaces, caches, decode states and completion images until
 *    sd_engine_destroy() / sd_release().
 *  - Device pointers are CUDA global-memory pointers on the engine's device. `stream` arguments
 *    are cudaStream_t passed as void* (NULL = legacy default stream). Data-plane calls are
 *    asynchronous on that stream unless stated otherwise.
 *  - Layouts: latents are fp32 [4][h][w] (NCHW, one request), images fp32 [3][8h][8w],
 *    text embeddings fp32 [len][dim] row-major.
 */
#ifndef SD_API_H
#define SD_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t sd_status;
enum {
  SD_OK = 0,
  SD_E_INVAL = -1,  /* invalid argument (validated before any work is enqueued)            */
  SD_E_NOMEM = -2,  /* device or host allocation failed                                      */
  SD_E_CUDA = -3,   /* CUDA runtime error (engine becomes FAILED)                            */
  SD_E_AGAIN = -4,  /* resource temporarily full (submit queue)                              */
  SD_E_STATE = -5,  /* call not valid in the current state (FAILED engine, out-of-order)     */
  SD_E_NOTSUP = -6  /* configuration not supported by this build                            */
};

/* R1: diffusers SD-1.5 / SDXL-base shapes (oracle/configs.py); tiny = CFG#1; tiny-XL = the SDXL code
 * paths (no attention at level 0, depth-2 transformers, head-dim heads, added embedding) at tiny size */
enum { SD_MODEL_TINY = 0, SD_MODEL_SD15 = 1, SD_MODEL_SDXL = 2, SD_MODEL_TINY_XL = 3 };
/* R19: SD_PREC_BF16 = the product path (bf16 weights / activations, fp32 accumulation and statistics,
 * tcgen05 tensor cores). SD_PREC_FP32 = the parity mode of SURVEY §8(c) ("fp32 mode: everything fp32",
 * rel-L2 ≤ 1e-4 vs the oracle): fp32 weights and activations, SIMT FP32 kernels (no tensor cores, no
 * split-K), same graph, same chunking; ~2x the weight memory. SD_PREC_FP16 = the bf16 path's kernels,
 * graph and layouts with fp16 operands and storage (fp32 accumulation and statistics unchanged): the
 * same tensor-core rate and bytes as bf16 with 3 more significand bits (the paper serves in FP16,
 * P:315); the weights are still the R20 bf16 values, held in fp16 (exact for |w| >= 2^-17). */
enum { SD_PREC_BF16 = 0, SD_PREC_FP32 = 1, SD_PREC_FP16 = 2 };
enum { SD_SAMPLER_DDIM = 0, SD_SAMPLER_EULER = 1 };      /* R4 / R5                                  */

typedef struct sd_engine sd_engine;
typedef struct sd_decode sd_decode;
typedef struct sd_table sd_table;
typedef struct sd_controller sd_controller;

/* ---- engine ---------------------------------------------------------------------------------
 * sd_engine_create: builds the UNet + VAE for `model` on `cuda_device`, allocates workspaces for
 * up to 2*b_max UNet rows at up to max_latent_hw x max_latent_hw, and initialises every weight
 * ON THE DEVICE from the counter-based generator keyed by (weight_seed, parameter name) (R20,
 * synth/__init__.py documents the generator). */
typedef struct {
  int32_t model;          /* SD_MODEL_* (SDXL: ~5.6 GB of bf16 weights)         */
  int32_t precision;      /* SD_PREC_BF16 | SD_PREC_FP16 | SD_PREC_FP32 (parity) */
  int32_t sampler;        /* SD_SAMPLER_*                                      */
  int32_t max_latent_hw;  /* e.g. 64 for 512x512 images                        */
  int32_t b_max;          /* max requests per UNet call (paper: BS = 8) */
  int32_t c_max;          /* max VAE chunks                            */
  uint64_t weight_seed;
} sd_engine_config;

sd_status sd_engine_create(const sd_engine_config* cfg, int32_t cuda_device, sd_engine** out);
sd_status sd_engine_destroy(sd_engine* e);
/* sd_engine_set_weight (parity tests): overwrite one parameter, named as in diffusers'
 * UNet2DConditionModel / AutoencoderKL decoder ("down_blocks.0.resnets.0.conv1.weight",
 * "decoder.mid_block.attentions.0.to_q.bias", ...; the list is oracle/configs.py's), from host fp32
 * values in that parameter's PyTorch layout ([O][I][3][3] conv, [O][I] linear, [C] norm / bias). The
 * engine converts them to its own layout and precision (bf16 RNE, or fp32) with the same transform as
 * its weight generator. Synchronous (the device is idle afterwards w.r.t. this call). Call it before
 * sd_ctx_register / sd_ctx_set_uncond: cached text K/V of registered prompts are NOT recomputed.
 * SD_E_INVAL: unknown name, or bytes != 4 x the parameter's element count. */
sd_status sd_engine_set_weight(sd_engine* e, const char* name, const void* host, size_t bytes);
const char* sd_last_error(void);
const char* sd_status_str(sd_status s);
/* Number of kernels this engine launched since creation (for the bench's gpu_launches claim). */
sd_status sd_engine_launch_count(sd_engine* e, int64_t* out);

/* Device timing per kernel class, CUDA events on the launching stream around every launch
 * (used by bench.py for the live roofline). enable != 0 starts recording (and clears old records).
 * Classes: 0 conv3x3 implicit GEMM, 1 dense GEMM, 2 attention, 3 GroupNorm, 4 LayerNorm, 5 other,
 * 6 VAE, 7 the UNet's 1x1 convolutions (shortcuts, proj_in / proj_out; dense GEMMs, not in class 1).
 * work_out = algorithmic FLOPs (classes 0-2) or bytes (3-4) of the recorded launches. Reading
 * synchronises on the recorded events. */
sd_status sd_engine_profile(sd_engine* e, int32_t enable);
sd_status sd_engine_profile_read(sd_engine* e, int32_t cls, double* ms_out, int64_t* launches_out, double* work_out);
/* Pre-builds what a server at latent h x w touches on first use, so no serving window pays for it:
 * the CUDA graph of every step shape (1..max_req requests, any number of Skip-CFG rows) and n_dec
 * pooled VAE decode states (whole and 2-chunk). Runs real kernels on scratch latents (ctx slot 0);
 * synchronous on `stream`. SD_E_INVAL on bad sizes; SD_E_CUDA on a CUDA error. */
sd_status sd_engine_warmup(sd_engine* e, int32_t h, int32_t w, int32_t max_req, int32_t n_dec, void* stream);

/* ---- data plane: one step-level batched denoising iteration ---------
 * sd_ctx_register: cache the cross-attention K/V of one prompt embedding (text_emb_dev: device
 * fp32 [len][dim], len = 77 / dim = 768 for SD-1.5). Text K/V do not depend on x or t, so they
 * are computed once at admission. Returns a slot id; slot 0 is the engine-global unconditional
 * embedding, registered with sd_ctx_set_uncond. */
sd_status sd_ctx_register(sd_engine* e, const float* text_emb_dev, int32_t len, int32_t dim, int32_t* slot_out,
                          void* stream);
sd_status sd_ctx_set_uncond(sd_engine* e, const float* text_emb_dev, int32_t len, int32_t dim, void* stream);
/* SDXL variants (SD_MODEL_SDXL / SD_MODEL_TINY_XL need them; the two calls above return SD_E_INVAL
 * for those models): pooled_dev = device fp32 [pooled_dim] pooled text embedding (1280 for SDXL).
 * Besides the text K/V, the slot caches the prompt's "text_time" added embedding (R27: time ids
 * (1024,1024,0,0,1024,1024), 256-d sinusoids ‖ pooled → Linear → SiLU → Linear, fp32 [1280]),
 * which every UNet row of that prompt adds to linear_2 of the time embedding. */
sd_status sd_ctx_register_pooled(sd_engine* e, const float* text_emb_dev, int32_t len, int32_t dim,
                                 const float* pooled_dev, int32_t pooled_dim, int32_t* slot_out, void* stream);
sd_status sd_ctx_set_uncond_pooled(sd_engine* e, const float* text_emb_dev, int32_t len, int32_t dim,
                                   const float* pooled_dev, int32_t pooled_dim, void* stream);
sd_status sd_ctx_release(sd_engine* e, int32_t slot);

/* One UNet step for n_req requests at one resolution (R22). Rows: one conditional row per
 * request, plus one unconditional row for requests with has_uncond = 1 (Adaptive Skip-CFG,
 * P:162; R3), ordered cond rows then uncond rows (R26). Then per request:
 *   eps~ = has_uncond ? eps_u + g (eps_c - eps_u) : eps_c                  (R2, R3)
 *   x    = DDIM / Euler update of x at step index step[r] of n_steps[r]     (R4, R5)
 * latents[r] are updated in place. All host arrays are copied at call time. */
typedef struct {
  int32_t n_req, latent_h, latent_w;
  float* const* latents;      /* [n_req] device ptrs, fp32 [4][h][w]                     */
  const int32_t* step;        /* [n_req] s_r: steps already done (index of this step)    */
  const int32_t* n_steps;     /* [n_req] n_r                                             */
  const uint8_t* has_uncond;  /* [n_req] 1 = CFG row present, 0 = Skip-CFG this step     */
  const float* guidance;      /* [n_req] g_r                                             */
  const int32_t* ctx_slot;    /* [n_req] from sd_ctx_register                            */
} sd_batch;
sd_status sd_step_batch(sd_engine* e, const sd_batch* b, void* stream);

/* Scheduler coefficients a request needs before its first step: x_T = init_sigma * z. */
sd_status sd_sampler_init_sigma(sd_engine* e, int32_t n_steps, float* out);

/* ---- chunked VAE decode (R7 "stage-synchronous halo tiles") -----------------------
 * Chunk j of n_chunks runs the j-th contiguous range of the decode work list. Chunk 0 allocates
 * *state (must be NULL), the last chunk writes image_dev (fp32 [3][8h][8w]) and frees *state
 * (set to NULL). Chunks must be issued in order on the same stream, else SD_E_STATE.
 * n_chunks == 1 is a whole-image decode. Any n_chunks gives the same image (I6). */
sd_status sd_vae_decode_chunked(sd_engine* e, const float* latent_dev, int32_t h, int32_t w, int32_t n_chunks,
                                int32_t chunk, sd_decode** state, float* image_dev, void* stream);
/* V2 independent-tile decode (reading R7 V2), the north star's literal "latent
 * split into halo-padded tiles, decoded tile by tile and stitched": every tile x tile block of the
 * latent is decoded on its own from its halo-padded window (clipped at the border), so GroupNorm and
 * the mid-block attention are tile-local (an APPROXIMATION of the whole decode, unlike the exact V1
 * sd_vae_decode_chunked); its own image region is written into image_dev [3][8h][8w] (disjoint
 * writes). h, w, tile, halo: multiples of 8. tile >= h, w or halo >= h, w reproduces the whole decode.
 * Asynchronous on `stream`; the engine owns the window scratch. */
sd_status sd_vae_decode_tiled(sd_engine* e, const float* latent_dev, int32_t h, int32_t w, int32_t tile,
                              int32_t halo, float* image_dev, void* stream);

/* ---- pure host control plane -------------------------------------------
 * Latency table: CSV "c,m,n,k,tau_us,delta_us" (integers, µs; R11). */
sd_status sd_table_load(const char* csv_path, sd_table** out);
sd_status sd_table_from_arrays(int32_t n, const int32_t* c, const int32_t* m, const int32_t* nn, const int32_t* k,
                               const int64_t* tau_us, const int64_t* delta_us, sd_table** out);
sd_status sd_table_free(sd_table* t);

/* Problem P (Eq. 3a-3f) for a window (M, N, K) at chunk granularity c. dp_mode 0 = exact
 * (Pareto labels, R10), 1 = Alg. 1 verbatim. T_lim = floor((1+a_num/a_den) tau_ref)
 * (R11, R13). Writes up to max_stages stages (m,n,k) into stages_out (3 ints each), the count
 * into *n_stages, and the objective cost / total time (µs) into cost_out / time_out. N = 0 gives
 * the single pure-UNet stage (M,0,0) (R8). */
sd_status sd_plan(const sd_table* t, int32_t M, int32_t N, int32_t K, int32_t c, int32_t a_num, int32_t a_den,
                  int32_t dp_mode, int32_t* stages_out, int32_t max_stages, int32_t* n_stages, int64_t* cost_out,
                  int64_t* time_out);

/* Feedback controller (R15). */
typedef struct {
  int32_t c_star, c_max, window, hysteresis;
  int32_t up_num, up_den;      /* theta_up   = up_num/up_den tasks per second   (default 1/2)  */
  int32_t down_num, down_den;  /* theta_down = down_num/down_den              (default -1/5) */
} sd_controller_config;
typedef struct {
  int32_t level;     /* 0 = no skip, 1 = s_min 0.7 n, 2 = s_min 0.5 n (R6) */
  int32_t c;         /* VAE chunk count                                   */
  int32_t changed;
} sd_directive;
sd_status sd_controller_create(const sd_controller_config* cfg, sd_controller** out);
sd_status sd_controller_decide(sd_controller* c, int64_t now_us, int32_t global_queue, sd_directive* out);
sd_status sd_controller_free(sd_controller* c);

/* Task mapping E of Problem P ("(S, E)"; R14) for the stages S of a window: each decode goes to
 * the stages in (arrival_us, id) order; the sum_t k_t Skip-CFG slots go to the eligible UNet tasks with
 * the largest s/n_steps (ties: smaller id), the other UNet slots to the remaining tasks in the given
 * (batch) order. Writes each UNet task's stage index and skip flag and each decode's stage index.
 * SD_E_INVAL if the stages do not cover the window (sum m = n_unet, sum n = n_dec, sum k <= #eligible)
 * or an array is NULL. Pure host function. */
sd_status sd_map_tasks(const int32_t* stages, int32_t n_stages, int32_t n_unet, const uint64_t* unet_id,
                       const int32_t* unet_s, const int32_t* unet_n, const uint8_t* unet_eligible, int32_t n_dec,
                       const uint64_t* dec_id, const int64_t* dec_arrival, int32_t* unet_stage_out,
                       uint8_t* unet_skip_out, int32_t* dec_stage_out);

/* Offline chunk-granularity selection (Eq. 1; P:248 the C_max rule; R31), from a profiled
 * table, for a window of m UNet requests and n decodes, over the candidate counts c_values[0..n_c):
 *   T_u(c) = tau^c(m, n, 0), T_v(c) = delta^c(m, n, 0)                     (Eq. 2, measured)
 *   T_u0(c) = c * tau^1(m, 0, 0)   the UNet alone over the same c rounds
 *   T_v0    = delta^1(0, n, 0)     the decodes alone (delta^1(n, n, 0) if the table has no decode-only row)
 *   L(c) = lam (T_u(c) - T_u0)/T_u0 + (1 - lam)(T_v(c) - T_v0)/T_v0,  lam = lam_num/lam_den (paper: 0.5)
 *   c* = argmin L(c), ties to the smaller c;  C_max = the largest c with tau^c(m,n,0)/c <= 1.05 tau^1(m,0,0)
 *   (else the smallest candidate). All comparisons are exact (integer µs, 128-bit rationals); cost_out
 * (may be NULL) receives L(c) per candidate as double, for reporting. SD_E_INVAL on a missing table row. */
sd_status sd_chunk_choice(const sd_table* t, int32_t m, int32_t n, const int32_t* c_values, int32_t n_c,
                          int32_t lam_num, int32_t lam_den, int32_t* c_max_out, int32_t* c_star_out, double* cost_out);

/* Saturation batch B_max ("identify the saturation batch size B_max based on the sub-linear
 * scaling of throughput"; SPEC find_b_max): throughput(m) = m / tau^1(m, 0, 0) from the profiled table;
 * B_max = the smallest m in [1, m_max) with throughput(m+1)/throughput(m) - 1 < eps (eps = eps_num /
 * eps_den, SPEC: 0.05), else m_max. Exact (128-bit integers). SD_E_INVAL if a (1, m, 0, 0) row is missing. */
sd_status sd_find_b_max(const sd_table* t, int32_t m_max, int32_t eps_num, int32_t eps_den, int32_t* b_max_out);

/* Min-max partition of the ordered VAE work list into c chunks (R7): boundaries[0..c]. */
sd_status sd_chunk_ranges(const int64_t* costs, int32_t n_items, int32_t c, int32_t* boundaries_out);

/* ---- serving: the paper's problem statement (P:289 Problem P, P:297 E2E = V_i - A_i) ----------
 * Continuous batching with step-level refill, the threshold-aware plan per window
 * (Eq. 3, Alg. 1 / exact DP), Skip-CFG and VAE chunking as planned, and the feedback
 * controller. Semantics: SURVEY §8(c) steps 1-5, DESIGN.md §2 (R6-R17). */
typedef struct {
  int32_t b_max;                /* max UNet batch (8)                                     */
  int32_t a_num, a_den;         /* throughput slack alpha (1/10)                          */
  int32_t dp_mode;              /* 0 exact, 1 Alg. 1 verbatim                                    */
  int32_t c_star;               /* offline chunk granularity c* (Eq. 1)                          */
  sd_controller_config ctl;     /* controller (R15); ctl.c_max = C_max                           */
  const sd_table* table;        /* tau/delta table for c = 1..C_max (owned by the caller)        */
  int32_t latent_hw;            /* GPU mode: one resolution per server (R22)                     */
  uint64_t trace_seed;          /* GPU mode: initial noise z ~ N(0,1) keyed by (trace_seed, id)  */
  int32_t n_max;                /* max decodes planned per window (0 = b_max); the table needs n ≤ n_max */
  int32_t policy;               /* SD_POLICY_*: SynerDiff, or a baseline of P:316-324           */
  int32_t ablation;             /* SD_ABL_* bits (SynerDiff only); no chunking = c_max 1 */
  int64_t dyn_window_us;        /* Dynamic Batching collection window (0 = 500 000)        */
  /* mixed resolutions: n_res tables, res_tables[i] profiled at latent res_hw[i];
   * a window plans with the table of the largest resolution among its batch and decode-pending
   * requests ("max multiplier"); n_res = 0: `table` for every request */
  int32_t n_res;
  const int32_t* res_hw;
  const sd_table* const* res_tables;
  /* SM partitioning of UNet ∥ VAE: 0 = the two streams differ only in priority
   * (UNet high, VAE low); > 0 = the VAE chunks run in a green context of vae_sms SMs (rounded up by the
   * driver, multiples of 8) and the UNet rounds in one of the remaining SMs (sd_sm_partition_create). */
  int32_t vae_sms;
} sd_serve_config;
/* Serving policies (§IV Baselines; semantics in oracle/serving.py):
 *  SYNERDIFF  the method: threshold-aware plan, Skip-CFG, VAE chunking, feedback controller;
 *  NAIVE      InstGenIE-like continuous batching with direct UNet-VAE concurrency: one stage
 *             (M, min(N, M), 0) per window, c = 1, no Skip-CFG, no controller;
 *  DYNAMIC    Dynamic Batching: 0.5 s collection window, lockstep until every member is done,
 *             synchronous release;
 *  SERIAL     Diffusers, BS = 1: denoise then decode, one request at a time. */
enum { SD_POLICY_SYNERDIFF = 0, SD_POLICY_NAIVE = 1, SD_POLICY_DYNAMIC = 2, SD_POLICY_SERIAL = 3 };
enum { SD_ABL_NO_SKIP = 1, SD_ABL_NO_CTL = 2 };
typedef struct {
  uint64_t id;
  int64_t arrival_us;           /* A_i, µs since sd_serve_start; not admitted before it          */
  int32_t n_steps;              /* n_i                                                           */
  float guidance;               /* g_i                                                           */
  const float* text_emb_host;   /* fp32 [emb_len][emb_dim], copied at submit                     */
  int32_t emb_len, emb_dim;
  const float* pooled_host;     /* SDXL: fp32 [pooled_dim] pooled text embedding (else NULL / 0) */
  int32_t pooled_dim;
  int32_t latent_hw;            /* this request's latent size (0 = the server's latent_hw); a
                                   multiple of 8, <= the engine's max_latent_hw, with a table when
                                   the server is mixed-resolution                                  */
} sd_request;
typedef struct {
  uint64_t id;
  int64_t arrival_us, denoise_done_us, decode_done_us;  /* A_i, U_i, V_i (µs)                     */
  int32_t n_skipped, h, w;      /* Skip-CFG steps taken; image is [3][h][w]                      */
  const float* image_host;      /* engine-owned pinned buffer, valid until sd_release(id)       */
  const int32_t* skipped_steps; /* [n_skipped] step indices run without the uncond row (audit)   */
} sd_completion;
/* GPU server: a thread per engine runs the loop; UNet rounds on a high-priority stream, VAE
 * chunks on a low-priority stream. */
sd_status sd_serve_start(sd_engine* e, const sd_serve_config* cfg);
sd_status sd_submit(sd_engine* e, const sd_request* r);    /* thread-safe; copies the embedding */
sd_status sd_poll(sd_engine* e, sd_completion* out, int32_t max, int32_t* n_out, int32_t timeout_ms);
/* sd_release: returns the completion's image buffer to the engine. Only ids already handed out by
 * sd_poll may be released (SD_E_INVAL otherwise: unknown id, or completed but not yet polled);
 * image_host / skipped_steps of that completion are invalid afterwards. */
sd_status sd_release(sd_engine* e, uint64_t id);
sd_status sd_serve_stop(sd_engine* e);                     /* drains nothing; stops the thread    */
/* Two streams on disjoint SM partitions (CUDA green contexts): vae_stream on vae_sms SMs (rounded up by
 * the driver to its granularity, 8 on sm_90+), unet_stream on the rest; the counts actually provisioned are
 * returned. Every kernel of the library sizes its persistent / cooperative grid by the SM count of the
 * stream it is launched on. The streams belong to the partition object (destroyed with it).
 * SD_E_INVAL / SD_E_CUDA if the driver has no green contexts or the split fails. */
typedef struct sd_partition sd_partition;
sd_status sd_sm_partition_create(int32_t cuda_device, int32_t vae_sms, sd_partition** out, void** unet_stream,
                                 void** vae_stream, int32_t* unet_sms, int32_t* vae_sms_out);
sd_status sd_sm_partition_destroy(sd_partition* p);
/* Controller trajectory (one record per planned window, in order): start / end µs, M, N, K, the level
 * and chunk count the window ran with, the waiting queue the controller then observed, its new level
 * and chunk count. Any output array may be NULL. Call before sd_serve_stop. */
sd_status sd_serve_window_log(sd_engine* e, int32_t max, int64_t* t_start, int64_t* t_end, int32_t* m, int32_t* n,
                              int32_t* k, int32_t* level, int32_t* c, int32_t* waiting, int32_t* level_after,
                              int32_t* c_after, int32_t* n_out);
/* The decision record of window `window` (T5 replay, "scheduler's batch/chunk decisions"): the
 * stages S the loop ran, and per task the inputs and output of the mapping E — UNet tasks in batch
 * order {id, s (steps done), n_steps, eligible (s >= s_min at the window's level), stage, skip}, and the
 * window's decodes in (A, id) order {id, A, stage} (stage -1: not planned in this window, naive policy).
 * Together with sd_serve_window_log's M, N, K, level and c, the plan can be recomputed from the table
 * and compared bit for bit; level_out / c_out (may be NULL) = the controller level and chunk count the
 * window ran with. SD_E_INVAL for an unknown window or arrays shorter than the record. */
typedef struct { uint64_t id; int32_t s, n_steps, eligible, stage, skip, pad_; } sd_logged_unet;
typedef struct { uint64_t id; int64_t arrival_us; int32_t stage, pad_; } sd_logged_decode;
sd_status sd_serve_window_plan(sd_engine* e, int32_t window, int32_t* stages_out, int32_t max_stages,
                               int32_t* n_stages, sd_logged_unet* unet_out, int32_t max_unet, int32_t* n_unet,
                               sd_logged_decode* dec_out, int32_t max_dec, int32_t* n_dec,
                               int32_t* level_out, int32_t* c_out);
/* loads = int32 [P][4] {waiting, decode-pending, active, completed} all-gathered over ranks (C1);
 * the controller then sums `waiting` over ranks. sd_get_load returns this rank's 4 counters. */
sd_status sd_set_global_load(sd_engine* e, const int32_t* loads, int32_t P, uint64_t epoch);
sd_status sd_get_load(sd_engine* e, int32_t* out4);
/* Virtual-clock twin of the loop (no GPU): round durations from the table. Fills U_i, V_i and
 * the number of Skip-CFG steps per request, and the number of windows. Bit-exact with
 * oracle/serving.py. */
sd_status sd_serve_simulate(const sd_serve_config* cfg, const sd_table* t, int32_t n, const uint64_t* ids,
                            const int64_t* arrival_us, const int32_t* n_steps, int64_t* U_out, int64_t* V_out,
                            int32_t* n_skips_out, int32_t* windows_out);
/* Stepping virtual-clock server: the same loop as sd_serve_start's, on the table's clock, advanced one
 * window at a time by the caller — so P of them (one per rank, each on its shard id mod P, R32) can run
 * in lockstep with the C1 all-gather of their loads between windows (tests). Policies
 * SynerDiff and naive. sd_vserve_window: *state_out = 1 a window ran, 0 nothing was admitted and the
 * clock jumped to the next arrival, -1 every request is done (no-op). sd_vserve_get_load: this server's
 * {waiting (arrived, not admitted), decode-pending, active, completed} now. sd_vserve_set_global_load:
 * the [P][4] snapshot; for P > 1 the controller then observes the snapshot's summed waiting queue (the
 * GPU server's rule). sd_vserve_results: U_i, V_i, Skip-CFG steps per request in creation order, the
 * clock and the window count. sd_vserve_trajectory: per window, the waiting queue the controller observed
 * and its level / chunk count after deciding. */
typedef struct sd_vserver sd_vserver;
sd_status sd_vserve_create(const sd_serve_config* cfg, const sd_table* t, int32_t n, const uint64_t* ids,
                           const int64_t* arrival_us, const int32_t* n_steps, sd_vserver** out);
sd_status sd_vserve_window(sd_vserver* v, int32_t* state_out);
sd_status sd_vserve_get_load(sd_vserver* v, int32_t* out4);
sd_status sd_vserve_set_global_load(sd_vserver* v, const int32_t* loads, int32_t P, uint64_t epoch);
sd_status sd_vserve_results(sd_vserver* v, int64_t* U_out, int64_t* V_out, int32_t* n_skips_out, int64_t* now_out,
                            int32_t* windows_out);
sd_status sd_vserve_trajectory(sd_vserver* v, int32_t max, int32_t* waiting, int32_t* level_after, int32_t* c_after,
                               int32_t* n_out);
sd_status sd_vserve_free(sd_vserver* v);
/* sd_serve_window_plan for the stepping virtual-clock server. */
sd_status sd_vserve_window_plan(sd_vserver* v, int32_t window, int32_t* stages_out, int32_t max_stages,
                                int32_t* n_stages, sd_logged_unet* unet_out, int32_t max_unet, int32_t* n_unet,
                                sd_logged_decode* dec_out, int32_t max_dec, int32_t* n_dec,
                                int32_t* level_out, int32_t* c_out);
/* The same with a latent size per request (mixed-resolution config: cfg->n_res tables). */
sd_status sd_serve_simulate_mixed(const sd_serve_config* cfg, int32_t n, const uint64_t* ids, const int64_t* arrival_us,
                                  const int32_t* n_steps, const int32_t* latent_hw, int64_t* U_out, int64_t* V_out,
                                  int32_t* n_skips_out, int32_t* windows_out);

/* ---- test-only exports (same library): single kernels on caller-owned device buffers --------- */
/* D[M][N] = A[M][K] · B[N][K]^T + bias[N] (bf16 in, fp32 accumulate, bf16 or fp32 out). */
sd_status sd_debug_gemm(const void* A, const void* B, const float* bias, void* D, int32_t M, int32_t N, int32_t K,
                        int32_t out_f32, int32_t act, void* stream);
/* D[M][N] = A·B^T + bias + res (res bf16 [M][ldr], may alias D when ldr == N): the residual
 * epilogue of the transformer projections. */
sd_status sd_debug_gemm_res(const void* A, const void* B, const float* bias, const void* res, int32_t ldr, void* D,
                            int32_t M, int32_t N, int32_t K, void* stream);
/* 3x3 / stride 1 / pad 1 conv over NHWC bf16 x [nb][h][w][cin] (+ optional second source x2 with
 * cin2 channels, concatenated after x), weights bf16 [cout][9][cin] (and [cout][9][cin2]),
 * bias fp32, optional temb fp32 [nb][cout], optional residual bf16 [nb][h][w][cout]. */
sd_status sd_debug_conv3x3(const void* x, int32_t cin, const void* x2, int32_t cin2, const void* w, const void* w2,
                           const float* bias, const float* temb, const void* res, void* y, int32_t nb, int32_t h,
                           int32_t wd, int32_t cout, void* stream);

/* Attention O = softmax(Q K^T / sqrt(d)) V; q,o bf16 [rows][Lq][heads*d], k,v bf16 [rows][Lk][heads*d]
 * (mma.sync flash kernel, any d <= 160, d % 8 == 0). */
sd_status sd_debug_attention(const void* q, const void* k, const void* v, void* o, int32_t rows, int32_t heads,
                             int32_t d, int32_t Lq, int32_t Lk, void* stream);
/* tcgen05 flash attention: qk [rows*P][2*heads*d] (q | k), vt [heads*d][rows*P] (V^T), o [rows*P][heads*d];
 * d in {40, 64, 80, 160}, P % 8 == 0 (ragged key blocks masked); use_f16 != 0: fp16 operands, else bf16. */
sd_status sd_debug_attention_tc(const void* qk, const void* vt, void* o, int32_t rows, int32_t heads, int32_t d,
                                int32_t P, int32_t use_f16, void* stream);
/* tcgen05 cross-attention over a text K / Vᵀ cache: q [rows*P][heads*d]; kc [n_slots*Lk][ldk]
 * with the K of head h at columns kcol + h*d; vtc [vt_rows][ld_keys] with Vᵀ of head h at rows vrow + h*d and
 * key j of slot s at column s*ceil8(Lk) + j (slot stride rounded up to 8 keys: 16-byte aligned TMA boxes); kv_index (device int32 [rows]) = slot per batch row; o [rows*P][heads*d].
 * f16 != 0: fp16 operands (SD_PREC_FP16), else bf16. d in {40, 64, 80, 160}; any Lk (masked in-kernel). */
sd_status sd_debug_xattention_tc(const void* q, const void* kc, int32_t ldk, int32_t n_slots, int32_t kcol,
                                 const void* vtc, int32_t vt_rows, int32_t ld_keys, int32_t vrow,
                                 const int32_t* kv_index, int32_t Lk, void* o, int32_t rows, int32_t heads, int32_t d,
                                 int32_t P, int32_t f16, void* stream);
/* GroupNorm(+SiLU) over x bf16 [nb][P][C] (NHWC), G groups, fp32 gamma/beta; LayerNorm over x [T][C]. */
sd_status sd_debug_groupnorm(const void* x, void* y, int32_t nb, int32_t P, int32_t C, int32_t G, const float* gamma,
                             const float* beta, float eps, int32_t silu, void* stream);
/* GroupNorm statistics from the producer's epilogue (fusions; the GroupNorm
 * definition PAPER.md:146-148 / SURVEY §2.4 K8 is unchanged — only where its sums are taken moves).
 * sd_debug_conv3x3_gn / sd_debug_gemm_gn: the conv (one source, optional residual) / dense GEMM of
 * sd_debug_conv3x3 / sd_debug_gemm_res, which also writes gn_part = device fp32 [nb][P/32][cout][2]:
 * (sum, sum of squares) of each channel over each 32-pixel slot of the STORED 16-bit output (conv: the
 * slot is a box of min(wt, 32) x 32/min(wt, 32) pixels of the conv tile geometry; dense: 32 consecutive
 * rows of one image of P rows). SD_E_INVAL if the launch cannot emit them (output channels % 32, a
 * slot straddling two images, split-K). sd_debug_groupnorm_parts: GroupNorm(+SiLU) of the channel concat
 * [x0 (C0) | x1 (C1), optional] from those statistics (one finalize launch + the apply; no statistics
 * pass), same output as sd_debug_groupnorm up to summation order. All buffers device, caller-owned. */
sd_status sd_debug_conv3x3_gn(const void* x, int32_t cin, const void* w, const float* bias, const void* res, void* y,
                              int32_t nb, int32_t h, int32_t wd, int32_t cout, float* gn_part, void* stream);
sd_status sd_debug_gemm_gn(const void* A, const void* B, const float* bias, const void* res, void* D, int32_t M,
                           int32_t N, int32_t K, int32_t P, float* gn_part, void* stream);
sd_status sd_debug_groupnorm_parts(const void* x0, int32_t C0, const float* part0, const void* x1, int32_t C1,
                                   const float* part1, void* y, int32_t nb, int32_t P, int32_t G, const float* gamma,
                                   const float* beta, float eps, int32_t silu, void* stream);
/* LayerNorm folded into the consumer GEMM ("LN into the GEMM"; the LayerNorm and
 * linear definitions of PAPER.md's UNet / SURVEY §2.4 K9 are unchanged — only where the normalisation is
 * applied moves): x 16-bit [T][K] (the raw hidden state), W 16-bit [N][K], gamma / beta / bias fp32 (bias
 * optional). cols = 0: D [T][N] (or [T][N/2] with act = 2, GEGLU over 128-column groups) = LN(x)·Wᵀ + b;
 * cols = 1: D [N][T] = W·LN(x)ᵀ + b (the Vᵀ projection: LN output as the B operand, bias per row). Computed
 * as W′ = W·diag(gamma) (16-bit), w̄ = row sums of W′, b′ = b + W·beta, per-token (μ, rstd), and the GEMM
 * epilogue v = rstd·(acc − μ·w̄) + b′. Device buffers, caller-owned; scratch is stream-ordered. */
sd_status sd_debug_gemm_ln(const void* x, int32_t T, const void* W, int32_t N, int32_t K, const float* gamma,
                           const float* beta, const float* bias, void* D, float eps, int32_t cols, int32_t act,
                           void* stream);
sd_status sd_debug_layernorm(const void* x, void* y, int32_t T, int32_t C, const float* gamma, const float* beta,
                             float eps, void* stream);
/* sd_debug_step_eps: the UNet part of sd_step_batch only (K11 gather → UNet), with the same rows as
 * sd_step_batch (cond rows in batch order, then uncond rows, R26): writes eps_dev = device fp32
 * [rows][h][w][4] (NHWC, the UNet's output layout) and leaves the latents unchanged. Lets the parity
 * tests compare ε_c and ε_u of every row on their own. Runs eagerly (no graph).
 * sd_debug_combine_update: the K12 kernel only — ε̃ = has_uncond ? ε_u + g(ε_c − ε_u) : ε_c, then the
 * DDIM / Euler update of latents[r] (R2-R5) — with an injected eps_dev in the same layout (rows as
 * sd_step_batch would form them; b->ctx_slot may be NULL). This is how the closed forms of SURVEY
 * §8(c) I7 (DDIM ε ≡ 0 telescoping; Euler constant ε) run through the GPU kernel. */
sd_status sd_debug_step_eps(sd_engine* e, const sd_batch* b, float* eps_dev, void* stream);
sd_status sd_debug_combine_update(sd_engine* e, const sd_batch* b, const float* eps_dev, void* stream);
/* fp16 (on != 0) instead of bf16 element type for sd_debug_gemm / _gemm_res / _conv3x3 / _conv3x3_s2 /
 * _groupnorm / _layernorm (the SD_PREC_FP16 instantiations of the same kernels); process-wide, tests only. */
sd_status sd_debug_set_f16(int32_t on);
/* GEMM tile mode for the tests: 0 = heuristic, 1 = 128-row CTA tiles, 2 = 256-row CTA-pair tiles. */
sd_status sd_debug_set_gemm_cg(int32_t cg);
/* 3x3 / stride 2 / pad 1 conv (the UNet downsamplers) by TMA boxes with element stride 2: x bf16
 * [nb][h_in][w_in][cin] (h_in, w_in even), weights bf16 [cout][9][cin], y bf16 [nb][h_in/2][w_in/2][cout]. */
sd_status sd_debug_conv3x3_s2(const void* x, int32_t cin, const void* w, const float* bias, void* y, int32_t nb,
                              int32_t h_in, int32_t w_in, int32_t cout, void* stream);
/* split-K of sd_debug_conv3x3: 0 = the production rule (conv layers of <= 64 pixels with >= 90 K
 * blocks of 64 channels take 3 splits), 1 = off, 2..8 = forced; partials summed in split order. A forced
 * count (2..8) also splits sd_debug_gemm_res (dense split-K: the engine's rule is 3 splits for the
 * transformer projections of <= 64-pixel levels with K >= 1280). */
sd_status sd_debug_set_conv_splits(int32_t splits);

#ifdef __cplusplus
}
#endif
#endif /* SD_API_H */
