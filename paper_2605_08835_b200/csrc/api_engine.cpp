// C ABI of the engine (include/sd_api.h: engine, data plane, chunked VAE decode).
#include <algorithm>
#include <vector>

#include "api_common.h"
#include "engine.h"

using namespace sd;

struct sd_decode {};  // opaque; the pointer is really a sd::DecodeState*

namespace sd {
float init_sigma(int sampler, int n);
}

#define ENGINE_GUARD(eng)                                               \
  SD_REQUIRE(eng, "null engine");                                       \
  if ((eng)->e.failed) {                                                \
    ::sd::set_error("engine is FAILED after an earlier CUDA error");    \
    return SD_E_STATE;                                                  \
  }

// run body; a CUDA error makes the engine FAILED (sticky)
#define ENGINE_BODY(eng, body)                      \
  try {                                             \
    SD_CUDA(cudaSetDevice((eng)->e.device));        \
    body;                                           \
  } catch (const ::sd::CudaError& ex) {             \
    (eng)->e.failed = true;                         \
    ::sd::set_error(ex.what());                     \
    return SD_E_CUDA;                               \
  } catch (const std::bad_alloc&) {                 \
    ::sd::set_error("out of memory");               \
    return SD_E_NOMEM;                              \
  } catch (const std::logic_error& ex) {            \
    ::sd::set_error(ex.what());                     \
    return SD_E_STATE;                              \
  } catch (const std::exception& ex) {              \
    ::sd::set_error(ex.what());                     \
    return SD_E_INVAL;                              \
  }                                                 \
  return SD_OK;

extern "C" sd_status sd_engine_create(const sd_engine_config* cfg, int32_t dev, sd_engine** out) {
  SD_REQUIRE(cfg && out, "sd_engine_create: null argument");
  SD_REQUIRE(cfg->model == SD_MODEL_TINY || cfg->model == SD_MODEL_SD15 || cfg->model == SD_MODEL_SDXL ||
                 cfg->model == SD_MODEL_TINY_XL,
             "sd_engine_create: unknown model");
  SD_REQUIRE(cfg->precision == SD_PREC_BF16 || cfg->precision == SD_PREC_FP32 ||
                 cfg->precision == SD_PREC_FP16, "sd_engine_create: precision");
  SD_REQUIRE(cfg->sampler == SD_SAMPLER_DDIM || cfg->sampler == SD_SAMPLER_EULER, "sd_engine_create: sampler");
  SD_REQUIRE(cfg->max_latent_hw >= 8 && cfg->max_latent_hw <= 256, "sd_engine_create: max_latent_hw");
  SD_REQUIRE(cfg->b_max >= 1 && cfg->b_max <= 32, "sd_engine_create: b_max");
  *out = nullptr;
  auto* h = new sd_engine();
  h->e.cfg = *cfg;
  h->e.device = dev;
  try {
    build_engine(&h->e);
  } catch (const CudaError& ex) {
    set_error(ex.what());
    delete h;
    return SD_E_CUDA;
  } catch (const std::bad_alloc&) {
    set_error("out of memory building the engine");
    delete h;
    return SD_E_NOMEM;
  } catch (const std::exception& ex) {
    set_error(ex.what());
    delete h;
    return SD_E_INVAL;
  }
  *out = h;
  return SD_OK;
}

extern "C" sd_status sd_engine_destroy(sd_engine* e) {
  if (!e) return SD_OK;
  if (e->e.server) sd_serve_stop(e);
  cudaSetDevice(e->e.device);
  cudaDeviceSynchronize();
  delete e;
  return SD_OK;
}

extern "C" sd_status sd_engine_set_weight(sd_engine* e, const char* name, const void* host, size_t bytes) {
  ENGINE_GUARD(e);
  SD_REQUIRE(name && host, "sd_engine_set_weight: null argument");
  ENGINE_BODY(e, set_weight(&e->e, name, static_cast<const float*>(host), bytes));
}

extern "C" sd_status sd_engine_launch_count(sd_engine* e, int64_t* out) {
  SD_REQUIRE(e && out, "bad args");
  *out = (int64_t)g_launches.load();
  return SD_OK;
}

extern "C" sd_status sd_ctx_register(sd_engine* e, const float* emb, int32_t len, int32_t dim, int32_t* slot_out,
                                     void* stream) {
  ENGINE_GUARD(e);
  SD_REQUIRE(emb && slot_out, "sd_ctx_register: null argument");
  SD_REQUIRE(len == e->e.uc.ctx_len && dim == e->e.uc.ctx_dim, "sd_ctx_register: embedding shape");
  SD_REQUIRE(!e->e.uc.add_time_dim, "sd_ctx_register: this model needs sd_ctx_register_pooled");
  ENGINE_BODY(e, { *slot_out = ctx_register(&e->e, emb, len, dim, nullptr, 0, -1, static_cast<cudaStream_t>(stream)); })
}

extern "C" sd_status sd_ctx_register_pooled(sd_engine* e, const float* emb, int32_t len, int32_t dim,
                                            const float* pooled, int32_t pooled_dim, int32_t* slot_out, void* stream) {
  ENGINE_GUARD(e);
  SD_REQUIRE(emb && pooled && slot_out, "sd_ctx_register_pooled: null argument");
  SD_REQUIRE(len == e->e.uc.ctx_len && dim == e->e.uc.ctx_dim, "sd_ctx_register_pooled: embedding shape");
  SD_REQUIRE(e->e.uc.add_time_dim && pooled_dim == e->e.uc.pooled_dim, "sd_ctx_register_pooled: pooled shape/model");
  ENGINE_BODY(e, {
    *slot_out = ctx_register(&e->e, emb, len, dim, pooled, pooled_dim, -1, static_cast<cudaStream_t>(stream));
  })
}

extern "C" sd_status sd_ctx_set_uncond_pooled(sd_engine* e, const float* emb, int32_t len, int32_t dim,
                                              const float* pooled, int32_t pooled_dim, void* stream) {
  ENGINE_GUARD(e);
  SD_REQUIRE(emb && pooled, "sd_ctx_set_uncond_pooled: null argument");
  SD_REQUIRE(len == e->e.uc.ctx_len && dim == e->e.uc.ctx_dim, "sd_ctx_set_uncond_pooled: embedding shape");
  SD_REQUIRE(e->e.uc.add_time_dim && pooled_dim == e->e.uc.pooled_dim, "sd_ctx_set_uncond_pooled: pooled shape/model");
  ENGINE_BODY(e, { ctx_register(&e->e, emb, len, dim, pooled, pooled_dim, 0, static_cast<cudaStream_t>(stream)); })
}

extern "C" sd_status sd_ctx_set_uncond(sd_engine* e, const float* emb, int32_t len, int32_t dim, void* stream) {
  ENGINE_GUARD(e);
  SD_REQUIRE(emb, "sd_ctx_set_uncond: null argument");
  SD_REQUIRE(len == e->e.uc.ctx_len && dim == e->e.uc.ctx_dim, "sd_ctx_set_uncond: embedding shape");
  SD_REQUIRE(!e->e.uc.add_time_dim, "sd_ctx_set_uncond: this model needs sd_ctx_set_uncond_pooled");
  ENGINE_BODY(e, { ctx_register(&e->e, emb, len, dim, nullptr, 0, 0, static_cast<cudaStream_t>(stream)); })
}

extern "C" sd_status sd_ctx_release(sd_engine* e, int32_t slot) {
  ENGINE_GUARD(e);
  SD_REQUIRE(slot >= 1 && slot < e->e.max_slots && e->e.slot_used[slot], "sd_ctx_release: bad slot");
  std::lock_guard<std::mutex> g(e->e.mu);
  e->e.slot_used[slot] = 0;
  return SD_OK;
}

static sd_status check_batch(sd_engine* e, const sd_batch* b, bool need_slots) {
  SD_REQUIRE(b && b->n_req >= 1 && b->n_req <= e->e.cfg.b_max, "sd_step_batch: n_req out of range [1, b_max]");
  SD_REQUIRE(b->latent_h >= 1 && b->latent_w >= 1 && b->latent_h <= e->e.cfg.max_latent_hw &&
                 b->latent_w <= e->e.cfg.max_latent_hw,
             "sd_step_batch: latent size");
  const int L = (int)e->e.uc.block_out.size();
  SD_REQUIRE(b->latent_h % (1 << (L - 1)) == 0 && b->latent_w % (1 << (L - 1)) == 0,
             "sd_step_batch: latent size must be divisible by 2^(levels-1)");
  SD_REQUIRE(b->latents && b->step && b->n_steps && b->has_uncond && b->guidance && (b->ctx_slot || !need_slots),
             "sd_step_batch: null array");
  for (int r = 0; r < b->n_req; ++r) {
    SD_REQUIRE(b->latents[r], "sd_step_batch: null latent");
    SD_REQUIRE(b->n_steps[r] >= 1 && b->n_steps[r] <= 1000, "sd_step_batch: n_steps");
    SD_REQUIRE(b->step[r] >= 0 && b->step[r] < b->n_steps[r], "sd_step_batch: step index");
    if (need_slots)
      SD_REQUIRE(b->ctx_slot[r] >= 0 && b->ctx_slot[r] < e->e.max_slots && e->e.slot_used[b->ctx_slot[r]],
                 "sd_step_batch: ctx slot not registered");
  }
  return SD_OK;
}

extern "C" sd_status sd_step_batch(sd_engine* e, const sd_batch* b, void* stream) {
  ENGINE_GUARD(e);
  const sd_status s = check_batch(e, b, true);
  if (s != SD_OK) return s;
  ENGINE_BODY(e, { step_batch(&e->e, b, static_cast<cudaStream_t>(stream)); })
}

extern "C" sd_status sd_debug_step_eps(sd_engine* e, const sd_batch* b, float* eps_dev, void* stream) {
  ENGINE_GUARD(e);
  const sd_status s = check_batch(e, b, true);
  if (s != SD_OK) return s;
  SD_REQUIRE(eps_dev, "sd_debug_step_eps: null eps");
  ENGINE_BODY(e, { step_batch(&e->e, b, static_cast<cudaStream_t>(stream), eps_dev, nullptr); })
}

extern "C" sd_status sd_debug_combine_update(sd_engine* e, const sd_batch* b, const float* eps_dev, void* stream) {
  ENGINE_GUARD(e);
  const sd_status s = check_batch(e, b, false);
  if (s != SD_OK) return s;
  SD_REQUIRE(eps_dev, "sd_debug_combine_update: null eps");
  ENGINE_BODY(e, { step_batch(&e->e, b, static_cast<cudaStream_t>(stream), nullptr, eps_dev); })
}

extern "C" sd_status sd_sampler_init_sigma(sd_engine* e, int32_t n_steps, float* out) {
  SD_REQUIRE(e && out && n_steps >= 1 && n_steps <= 1000, "sd_sampler_init_sigma: bad args");
  *out = init_sigma(e->e.cfg.sampler, n_steps);
  return SD_OK;
}

extern "C" sd_status sd_vae_decode_chunked(sd_engine* e, const float* z, int32_t h, int32_t w, int32_t n_chunks,
                                           int32_t chunk, sd_decode** state, float* image, void* stream) {
  ENGINE_GUARD(e);
  SD_REQUIRE(z && state && image, "sd_vae_decode_chunked: null argument");
  SD_REQUIRE(h >= 1 && w >= 1 && h <= e->e.cfg.max_latent_hw && w <= e->e.cfg.max_latent_hw,
             "sd_vae_decode_chunked: latent size");
  SD_REQUIRE(n_chunks >= 1 && n_chunks <= std::max(1, e->e.cfg.c_max) && chunk >= 0 && chunk < n_chunks,
             "sd_vae_decode_chunked: chunk index");
  ENGINE_BODY(e, {
    DecodeState* s = reinterpret_cast<DecodeState*>(*state);
    vae_decode_chunk(&e->e, z, h, w, n_chunks, chunk, &s, image, static_cast<cudaStream_t>(stream));
    *state = reinterpret_cast<sd_decode*>(s);
  })
}

extern "C" sd_status sd_vae_decode_tiled(sd_engine* e, const float* z, int32_t h, int32_t w, int32_t tile,
                                        int32_t halo, float* image, void* stream) {
  ENGINE_GUARD(e);
  SD_REQUIRE(z && image, "sd_vae_decode_tiled: null argument");
  SD_REQUIRE(h >= 8 && w >= 8 && h <= e->e.cfg.max_latent_hw && w <= e->e.cfg.max_latent_hw && h % 8 == 0 &&
                 w % 8 == 0,
             "sd_vae_decode_tiled: latent size (multiples of 8)");
  SD_REQUIRE(tile >= 8 && tile % 8 == 0 && halo >= 0 && halo % 8 == 0, "sd_vae_decode_tiled: tile / halo");
  ENGINE_BODY(e, { vae_decode_tiled(&e->e, z, h, w, tile, halo, image, static_cast<cudaStream_t>(stream)); })
}

extern "C" sd_status sd_engine_profile(sd_engine* e, int32_t enable) {
  ENGINE_GUARD(e);
  ENGINE_BODY(e, {
    e->e.prof.reset();
    e->e.prof.on = enable != 0;
  })
}

extern "C" sd_status sd_engine_profile_read(sd_engine* e, int32_t cls, double* ms, int64_t* n, double* work) {
  ENGINE_GUARD(e);
  SD_REQUIRE(cls >= 0 && cls < PC_N && ms && n && work, "sd_engine_profile_read: bad args");
  ENGINE_BODY(e, {
    long long c = 0;
    e->e.prof.read(cls, ms, &c, work);
    *n = c;
  })
}

// Pre-builds everything a server at latent h×w touches on its first use, so no serving window pays
// for it: the step graph of every batch shape (n_req ≤ max_req, any number of Skip-CFG rows; two
// calls each — the eager run, then the capture), and n_dec pooled decode states (whole and chunked).
// Runs real kernels on scratch latents; synchronous on `stream`.
static void warmup_impl(Engine* e, int h, int w, int max_req, int n_dec, cudaStream_t st) {
  const size_t lat_bytes = (size_t)4 * h * w * sizeof(float);
  const int nbuf = std::max(max_req, n_dec);
  std::vector<float*> lat(nbuf, nullptr);
  for (auto& p : lat) {
    SD_CUDA(cudaMallocAsync(&p, lat_bytes, st));
    SD_CUDA(cudaMemsetAsync(p, 0, lat_bytes, st));
  }
  std::vector<int32_t> step(max_req + 1, 0), nst(max_req + 1, 50), slot(max_req + 1, 0);
  std::vector<float> g(max_req + 1, 7.5f);
  for (int n = 1; n <= max_req; ++n)
    for (int k = 0; k <= n; ++k) {
      std::vector<uint8_t> hu(n, 1);
      for (int i = 0; i < k; ++i) hu[i] = 0;
      sd_batch b{n, h, w, lat.data(), step.data(), nst.data(), hu.data(), g.data(), slot.data()};
      for (int rep = 0; rep < 2; ++rep) step_batch(e, &b, st);
    }
  if (n_dec > 0) {
    float* img;
    const size_t img_elems = (size_t)3 * e->upscale() * h * e->upscale() * w;
    SD_CUDA(cudaMallocAsync(&img, img_elems * sizeof(float) * n_dec, st));
    for (int c = 1; c <= std::min(2, std::max(1, e->cfg.c_max)); ++c) {
      std::vector<DecodeState*> ds(n_dec, nullptr);
      for (int j = 0; j < c; ++j)
        for (int i = 0; i < n_dec; ++i) vae_decode_chunk(e, lat[i], h, w, c, j, &ds[i], img + i * img_elems, st);
    }
    SD_CUDA(cudaFreeAsync(img, st));
  }
  for (auto p : lat) SD_CUDA(cudaFreeAsync(p, st));
  SD_CUDA(cudaStreamSynchronize(st));
}

extern "C" sd_status sd_engine_warmup(sd_engine* e, int32_t h, int32_t w, int32_t max_req, int32_t n_dec,
                                      void* stream) {
  ENGINE_GUARD(e);
  SD_REQUIRE(h >= 8 && w >= 8 && h <= e->e.cfg.max_latent_hw && w <= e->e.cfg.max_latent_hw,
             "sd_engine_warmup: latent size");
  SD_REQUIRE(max_req >= 0 && max_req <= e->e.cfg.b_max && n_dec >= 0 && n_dec <= 64, "sd_engine_warmup: counts");
  ENGINE_BODY(e, { warmup_impl(&e->e, h, w, max_req, n_dec, static_cast<cudaStream_t>(stream)); })
}
