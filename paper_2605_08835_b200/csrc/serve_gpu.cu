// GPU server behind sd_serve_start / sd_submit / sd_poll (SURVEY §3 call stack 1-2): a thread per
// engine runs serve.h's Loop with the GPU executor. UNet rounds (sd_step_batch internals) run on a
// high-priority stream, VAE decode chunks on a low-priority stream ("tasks switching
// from UNet denoising to VAE decoding ... overlap with ongoing UNet batch iterations").
#include <math.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <condition_variable>
#include <deque>
#include <thread>

#include "api_common.h"
#include "engine.h"
#include "serve.h"

namespace sd {
float init_sigma(int sampler, int n);

static uint64_t mix64s(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t fnv(const std::string& s) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001B3ull;
  }
  return h;
}
// synth.initial_noise(trace_seed, id, h, w): Box-Muller over counters (2i, 2i+1), fp64 → fp32
static void initial_noise(uint64_t trace_seed, uint64_t id, int n, float* out) {
  const uint64_t seed = mix64s(fnv("noise/" + std::to_string(id)) ^ mix64s(trace_seed));
  for (int i = 0; i < n; ++i) {
    const uint64_t b1 = mix64s(seed + (uint64_t)(2 * i + 1) * 0x9E3779B97F4A7C15ull);
    const uint64_t b2 = mix64s(seed + (uint64_t)(2 * i + 2) * 0x9E3779B97F4A7C15ull);
    const double u1 = 1.0 - (double)(b1 >> 11) * 0x1.0p-53;
    const double u2 = (double)(b2 >> 11) * 0x1.0p-53;
    out[i] = (float)(sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2));
  }
}

struct Server;

struct GpuExec : Exec {
  Server* S;
  explicit GpuExec(Server* s) : S(s) {}
  int64_t now() override;
  void admit(STask* t) override;
  int64_t round(const std::vector<STask*>& step, const std::vector<uint8_t>& skip, const std::vector<STask*>& decs,
                int rho, int rounds, int64_t t0, int64_t tau, int64_t delta, std::vector<int64_t>* dd) override;
  void complete(STask* t) override;
  int64_t global_waiting(int64_t local) override;
};

struct Server {
  Engine* e;
  sd_serve_config cfg;
  Loop loop;
  GpuExec ex{this};
  std::thread th;
  std::mutex mu;
  std::condition_variable cv_sub, cv_done;
  bool stop = false;
  std::string error;
  std::vector<STask*> inbox;
  std::deque<STask*> completed;
  std::map<uint64_t, STask*> owned;
  std::chrono::steady_clock::time_point t0;
  cudaStream_t hi = nullptr, lo = nullptr;
  Partition* part = nullptr;  // cfg.vae_sms > 0: hi / lo are green-context streams on disjoint SMs
  cudaEvent_t ev_hi = nullptr, ev_lo = nullptr;
  int32_t counters[4] = {0, 0, 0, 0};  // waiting, decode-pending, active, completed
  std::vector<int32_t> global;
  int P = 0;
  float* pinned_noise = nullptr;
  float* pinned_emb = nullptr;
  float* emb_dev = nullptr;  // device copy of one admission's embedding (+ pooled)
  std::vector<int> res_hw;   // mixed resolutions: the latent sizes with a table (copied at start)
  std::vector<WindowLog> wlog;  // one entry per planned window (controller trajectory)
  // per-request buffers are recycled (cudaMalloc / cudaFree / cudaMallocHost in the loop would
  // stall it; cudaFree synchronises the whole device, i.e. the concurrent UNet round too)
  // keyed by buffer size (mixed resolutions)
  std::map<size_t, std::vector<float*>> pool_lat, pool_img, pool_host;
  float* take(std::map<size_t, std::vector<float*>>& pools, size_t bytes, bool host) {
    auto& pool = pools[bytes];
    if (!pool.empty()) {
      float* p = pool.back();
      pool.pop_back();
      return p;
    }
    float* p = nullptr;
    if (host)
      SD_CUDA(cudaMallocHost(&p, bytes));
    else
      SD_CUDA(cudaMalloc(&p, bytes));
    return p;
  }

  void run();
};

int64_t GpuExec::now() {
  return std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - S->t0).count();
}

void GpuExec::admit(STask* t) {
  Engine* e = S->e;
  const int hw = t->h * t->w;
  {
    std::lock_guard<std::mutex> g(S->mu);  // pool_host is refilled by sd_release
    t->lat = S->take(S->pool_lat, (size_t)4 * hw * 4, false);
    t->img_dev = S->take(S->pool_img, (size_t)3 * 64 * hw * 4, false);
    t->img_host = S->take(S->pool_host, (size_t)3 * 64 * hw * 4, true);
  }
  initial_noise(S->cfg.trace_seed, t->id, 4 * hw, S->pinned_noise);
  const float sig = init_sigma(e->cfg.sampler, t->n);
  for (int i = 0; i < 4 * hw; ++i) S->pinned_noise[i] *= sig;
  SD_CUDA(cudaMemcpyAsync(t->lat, S->pinned_noise, (size_t)4 * hw * 4, cudaMemcpyHostToDevice, S->hi));
  memcpy(S->pinned_emb, t->emb.data(), t->emb.size() * 4);
  if (!t->pooled.empty()) memcpy(S->pinned_emb + t->emb.size(), t->pooled.data(), t->pooled.size() * 4);
  const size_t nf = t->emb.size() + t->pooled.size();
  float* emb_dev = S->emb_dev;  // reused: admit ends with a stream synchronize
  SD_CUDA(cudaMemcpyAsync(emb_dev, S->pinned_emb, nf * 4, cudaMemcpyHostToDevice, S->hi));
  t->slot = ctx_register(e, emb_dev, t->emb_len, t->emb_dim, t->pooled.empty() ? nullptr : emb_dev + t->emb.size(),
                         (int)t->pooled.size(), -1, S->hi);
  SD_CUDA(cudaStreamSynchronize(S->hi));  // pinned staging is reused by the next admission
}

int64_t GpuExec::round(const std::vector<STask*>& step, const std::vector<uint8_t>& skip,
                       const std::vector<STask*>& decs, int rho, int rounds, int64_t, int64_t, int64_t,
                       std::vector<int64_t>* dd) {
  Engine* e = S->e;
  // one sd_step_batch per resolution group of the stepping tasks (ascending latent size; batch order
  // within a group) — a single group unless the server is mixed-resolution
  std::vector<int> sizes;
  for (STask* t : step)
    if (std::find(sizes.begin(), sizes.end(), t->h) == sizes.end()) sizes.push_back(t->h);
  std::sort(sizes.begin(), sizes.end());
  for (int hw : sizes) {
    std::vector<float*> lat;
    std::vector<int32_t> s, ns, slot;
    std::vector<uint8_t> hu;
    std::vector<float> g;
    for (size_t i = 0; i < step.size(); ++i) {
      if (step[i]->h != hw) continue;
      lat.push_back(step[i]->lat);
      s.push_back(step[i]->s);
      ns.push_back(step[i]->n);
      hu.push_back(skip[i] ? 0 : 1);
      g.push_back(step[i]->g);
      slot.push_back(step[i]->slot);
    }
    sd_batch b{(int)lat.size(), hw, hw, lat.data(), s.data(), ns.data(), hu.data(), g.data(), slot.data()};
    step_batch(e, &b, S->hi);
  }
  for (STask* t : decs) {
    DecodeState* ds = reinterpret_cast<DecodeState*>(t->decode);
    vae_decode_chunk(e, t->lat, t->h, t->w, rounds, rho, &ds, t->img_dev, S->lo);
    t->decode = ds;
  }
  SD_CUDA(cudaEventRecord(S->ev_lo, S->lo));
  SD_CUDA(cudaEventRecord(S->ev_hi, S->hi));
  if (!decs.empty() && rho == rounds - 1) {
    SD_CUDA(cudaEventSynchronize(S->ev_lo));  // Eq. 2: the decode does not wait for the UNet
    const int64_t td = now();
    for (size_t i = 0; i < decs.size(); ++i) (*dd)[i] = td;
  }
  SD_CUDA(cudaEventSynchronize(S->ev_hi));
  SD_CUDA(cudaEventSynchronize(S->ev_lo));
  return now();
}

void GpuExec::complete(STask* t) {
  const size_t bytes = (size_t)3 * 64 * t->h * t->w * 4;
  SD_CUDA(cudaMemcpyAsync(t->img_host, t->img_dev, bytes, cudaMemcpyDeviceToHost, S->lo));
  SD_CUDA(cudaStreamSynchronize(S->lo));
  {
    std::lock_guard<std::mutex> g(S->e->mu);
    if (t->slot > 0) S->e->slot_used[t->slot] = 0;
  }
  std::lock_guard<std::mutex> g(S->mu);
  S->pool_lat[(size_t)4 * t->h * t->w * 4].push_back(t->lat);
  S->pool_img[bytes].push_back(t->img_dev);
  t->lat = t->img_dev = nullptr;
  S->completed.push_back(t);
  S->counters[3]++;
  S->cv_done.notify_all();
}

int64_t GpuExec::global_waiting(int64_t local) {
  std::lock_guard<std::mutex> g(S->mu);
  S->counters[0] = (int32_t)local;
  S->counters[1] = (int32_t)S->loop.dec.size();
  S->counters[2] = (int32_t)S->loop.batch.size();
  if (S->P <= 1) return local;
  int64_t sum = 0;
  for (int r = 0; r < S->P; ++r) sum += S->global[4 * r];
  return sum;
}

void Server::run() {
  try {
    SD_CUDA(cudaSetDevice(e->device));
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu);
        for (STask* t : inbox) insert_pending(loop.pending, t);
        inbox.clear();
        if (stop) break;
      }
      if (!loop.window(ex)) {
        std::unique_lock<std::mutex> g(mu);
        const int64_t na = loop.next_event();
        const int64_t wait_us = na < 0 ? 2000 : std::max<int64_t>(0, na - ex.now());
        cv_sub.wait_for(g, std::chrono::microseconds(std::min<int64_t>(wait_us, 2000)),
                        [&] { return stop || !inbox.empty(); });
      }
    }
  } catch (const std::exception& ex_) {
    std::lock_guard<std::mutex> g(mu);
    error = ex_.what();
    e->failed = true;
    cv_done.notify_all();
  }
}

}  // namespace sd

using namespace sd;

static Server* server_of(sd_engine* e) { return reinterpret_cast<Server*>(e->e.server); }

extern "C" sd_status sd_serve_start(sd_engine* e, const sd_serve_config* cfg) {
  SD_REQUIRE(e && cfg && (cfg->table || cfg->n_res > 0), "sd_serve_start: bad args");
  SD_REQUIRE(cfg->n_res == 0 || (cfg->res_hw && cfg->res_tables), "sd_serve_start: mixed-resolution tables");
  SD_REQUIRE(!e->e.server, "sd_serve_start: already serving");
  SD_REQUIRE(cfg->b_max >= 1 && cfg->b_max <= e->e.cfg.b_max, "sd_serve_start: b_max exceeds the engine's");
  SD_REQUIRE(cfg->latent_hw >= 8 && cfg->latent_hw <= e->e.cfg.max_latent_hw, "sd_serve_start: latent_hw");
  SD_REQUIRE(cfg->c_star >= 1 && cfg->ctl.c_max >= cfg->c_star && cfg->ctl.c_max <= e->e.cfg.c_max,
             "sd_serve_start: chunk bounds");
  SD_API_BEGIN
  auto* S = new Server();
  S->e = &e->e;
  S->cfg = *cfg;
  S->loop.cfg.b_max = cfg->b_max;
  S->loop.cfg.n_max = cfg->n_max > 0 ? cfg->n_max : cfg->b_max;
  S->loop.cfg.a_num = cfg->a_num;
  S->loop.cfg.a_den = cfg->a_den;
  S->loop.cfg.dp_mode = cfg->dp_mode;
  S->loop.cfg.c_star = cfg->c_star;
  set_policy(S->loop.cfg, cfg);
  set_tables(S->loop, cfg);
  S->loop.log = &S->wlog;
  S->loop.log_mu = &S->mu;
  S->res_hw.assign(cfg->res_hw, cfg->res_hw + cfg->n_res);
  S->cfg.res_hw = nullptr;  // the caller's arrays need not outlive sd_serve_start (tables must)
  S->cfg.res_tables = nullptr;
  S->loop.table = &cfg->table->t;
  S->loop.ctl.cfg = cfg->ctl;
  S->loop.ctl.cfg.c_star = cfg->c_star;
  S->loop.ctl.c = cfg->c_star;
  SD_CUDA(cudaSetDevice(e->e.device));
  if (cfg->vae_sms > 0) {
    S->part = partition_create(e->e.device, cfg->vae_sms);
    S->lo = partition_stream(S->part, 0);
    S->hi = partition_stream(S->part, 1);
  } else {
    int lo_p, hi_p;
    SD_CUDA(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
    SD_CUDA(cudaStreamCreateWithPriority(&S->hi, cudaStreamNonBlocking, hi_p));
    SD_CUDA(cudaStreamCreateWithPriority(&S->lo, cudaStreamNonBlocking, lo_p));
  }
  SD_CUDA(cudaEventCreateWithFlags(&S->ev_hi, cudaEventDisableTiming));
  SD_CUDA(cudaEventCreateWithFlags(&S->ev_lo, cudaEventDisableTiming));
  const size_t hw = (size_t)e->e.cfg.max_latent_hw * e->e.cfg.max_latent_hw;  // any request resolution
  SD_CUDA(cudaMallocHost(&S->pinned_noise, 4 * hw * 4));
  SD_CUDA(cudaMallocHost(&S->pinned_emb, ((size_t)e->e.uc.ctx_len * e->e.uc.ctx_dim + e->e.uc.pooled_dim) * 4));
  SD_CUDA(cudaMalloc(&S->emb_dev, ((size_t)e->e.uc.ctx_len * e->e.uc.ctx_dim + e->e.uc.pooled_dim) * 4));
  S->t0 = std::chrono::steady_clock::now();
  e->e.server = S;
  S->th = std::thread([S] { S->run(); });
  SD_API_END
}

extern "C" sd_status sd_submit(sd_engine* e, const sd_request* r) {
  SD_REQUIRE(e && r && server_of(e), "sd_submit: not serving");
  SD_REQUIRE(r->n_steps >= 1 && r->n_steps <= 1000 && r->arrival_us >= 0, "sd_submit: bad request");
  SD_REQUIRE(r->text_emb_host && r->emb_len == e->e.uc.ctx_len && r->emb_dim == e->e.uc.ctx_dim,
             "sd_submit: embedding shape");
  SD_REQUIRE(e->e.uc.add_time_dim == 0 ? (r->pooled_dim == 0)
                                        : (r->pooled_host && r->pooled_dim == e->e.uc.pooled_dim),
             "sd_submit: pooled embedding (required for SDXL, absent otherwise)");
  Server* S = server_of(e);
  {
    const int hw = r->latent_hw > 0 ? r->latent_hw : S->cfg.latent_hw;
    const int L = (int)e->e.uc.block_out.size();
    SD_REQUIRE(hw >= 8 && hw <= e->e.cfg.max_latent_hw && hw % (1 << (L - 1)) == 0 && hw % 8 == 0,
               "sd_submit: latent_hw");
    bool ok = S->res_hw.empty() ? hw == S->cfg.latent_hw : false;
    for (int r : S->res_hw) ok = ok || r == hw;
    SD_REQUIRE(ok, "sd_submit: no latency table for this latent size");
  }
  if (e->e.failed) {
    set_error("engine FAILED: " + S->error);
    return SD_E_STATE;
  }
  auto* t = new STask();
  t->id = r->id;
  t->A = r->arrival_us;
  t->n = r->n_steps;
  t->g = r->guidance;
  t->h = t->w = r->latent_hw > 0 ? r->latent_hw : S->cfg.latent_hw;
  t->emb.assign(r->text_emb_host, r->text_emb_host + (size_t)r->emb_len * r->emb_dim);
  t->emb_len = r->emb_len;
  t->emb_dim = r->emb_dim;
  if (r->pooled_dim) t->pooled.assign(r->pooled_host, r->pooled_host + r->pooled_dim);
  std::lock_guard<std::mutex> g(S->mu);
  if (S->owned.count(r->id)) {
    delete t;
    set_error("sd_submit: duplicate id");
    return SD_E_INVAL;
  }
  S->owned[r->id] = t;
  S->inbox.push_back(t);
  S->cv_sub.notify_all();
  return SD_OK;
}

extern "C" sd_status sd_poll(sd_engine* e, sd_completion* out, int32_t max, int32_t* n_out, int32_t timeout_ms) {
  SD_REQUIRE(e && out && n_out && max >= 0 && server_of(e), "sd_poll: bad args");
  Server* S = server_of(e);
  std::unique_lock<std::mutex> g(S->mu);
  S->cv_done.wait_for(g, std::chrono::milliseconds(std::max(0, timeout_ms)),
                      [&] { return !S->completed.empty() || !S->error.empty(); });
  if (!S->error.empty()) {
    set_error("serving loop failed: " + S->error);
    return SD_E_CUDA;
  }
  int n = 0;
  while (n < max && !S->completed.empty()) {
    STask* t = S->completed.front();
    S->completed.pop_front();
    out[n].id = t->id;
    out[n].arrival_us = t->A;
    out[n].denoise_done_us = t->U;
    out[n].decode_done_us = t->V;
    out[n].n_skipped = (int32_t)t->skips.size();
    out[n].h = S->e->upscale() * t->h;
    out[n].w = S->e->upscale() * t->w;
    out[n].image_host = t->img_host;
    out[n].skipped_steps = t->skips.data();
    t->delivered = true;
    ++n;
  }
  *n_out = n;
  return SD_OK;
}

extern "C" sd_status sd_release(sd_engine* e, uint64_t id) {
  SD_REQUIRE(e && server_of(e), "sd_release: not serving");
  Server* S = server_of(e);
  std::lock_guard<std::mutex> g(S->mu);
  auto it = S->owned.find(id);
  // only a task sd_poll has handed out may be released: complete() pushed it to `completed` under mu
  // after its D2H finished, and sd_poll set `delivered` under mu, so nothing else still touches it
  // (V is written by the loop thread outside mu and is not a safe completion flag)
  SD_REQUIRE(it != S->owned.end() && it->second->delivered, "sd_release: unknown id, or not yet returned by sd_poll");
  if (it->second->img_host)
    S->pool_host[(size_t)3 * 64 * it->second->h * it->second->w * 4].push_back(it->second->img_host);
  delete it->second;
  S->owned.erase(it);
  return SD_OK;
}

extern "C" sd_status sd_serve_stop(sd_engine* e) {
  SD_REQUIRE(e && server_of(e), "sd_serve_stop: not serving");
  Server* S = server_of(e);
  {
    std::lock_guard<std::mutex> g(S->mu);
    S->stop = true;
    S->cv_sub.notify_all();
  }
  if (S->th.joinable()) S->th.join();
  cudaSetDevice(e->e.device);
  cudaDeviceSynchronize();
  for (auto& kv : S->owned) {
    STask* t = kv.second;
    if (t->lat) cudaFree(t->lat);
    if (t->img_dev) cudaFree(t->img_dev);
    if (t->img_host) cudaFreeHost(t->img_host);
    if (t->decode) destroy_decode(&e->e, reinterpret_cast<DecodeState*>(t->decode));
    delete t;
  }
  for (auto& kv : S->pool_lat)
    for (float* p : kv.second) cudaFree(p);
  for (auto& kv : S->pool_img)
    for (float* p : kv.second) cudaFree(p);
  for (auto& kv : S->pool_host)
    for (float* p : kv.second) cudaFreeHost(p);
  cudaFreeHost(S->pinned_noise);
  cudaFreeHost(S->pinned_emb);
  cudaFree(S->emb_dev);
  cudaEventDestroy(S->ev_hi);
  cudaEventDestroy(S->ev_lo);
  if (S->part) {
    partition_destroy(S->part);  // owns hi / lo
  } else {
    cudaStreamDestroy(S->hi);
    cudaStreamDestroy(S->lo);
  }
  const std::string err = S->error;
  delete S;
  e->e.server = nullptr;
  if (!err.empty()) {
    set_error(err);
    return SD_E_CUDA;
  }
  return SD_OK;
}

extern "C" sd_status sd_set_global_load(sd_engine* e, const int32_t* loads, int32_t P, uint64_t) {
  SD_REQUIRE(e && loads && P >= 1 && server_of(e), "sd_set_global_load: bad args");
  Server* S = server_of(e);
  std::lock_guard<std::mutex> g(S->mu);
  S->global.assign(loads, loads + 4 * P);
  S->P = P;
  return SD_OK;
}

extern "C" sd_status sd_get_load(sd_engine* e, int32_t* out4) {
  SD_REQUIRE(e && out4 && server_of(e), "sd_get_load: bad args");
  Server* S = server_of(e);
  std::lock_guard<std::mutex> g(S->mu);
  int32_t waiting = 0;
  for (auto* t : S->inbox) waiting += 1;
  for (int i = 0; i < 4; ++i) out4[i] = S->counters[i];
  out4[0] = std::max(out4[0], waiting);
  return SD_OK;
}

extern "C" sd_status sd_serve_window_plan(sd_engine* e, int32_t window, int32_t* stages_out, int32_t max_stages,
                                          int32_t* n_stages, sd_logged_unet* unet_out, int32_t max_unet,
                                          int32_t* n_unet, sd_logged_decode* dec_out, int32_t max_dec,
                                          int32_t* n_dec, int32_t* level_out, int32_t* c_out) {
  SD_REQUIRE(e && server_of(e) && stages_out && n_stages && unet_out && n_unet && dec_out && n_dec,
             "sd_serve_window_plan: bad args");
  Server* S = server_of(e);
  std::lock_guard<std::mutex> g(S->mu);
  SD_REQUIRE(window >= 0 && window < (int)S->wlog.size(), "sd_serve_window_plan: no such window");
  SD_API_BEGIN
  window_plan_copy(S->wlog[window], stages_out, max_stages, n_stages, unet_out, max_unet, n_unet, dec_out, max_dec,
                   n_dec, level_out, c_out);
  SD_API_END
}

// Controller trajectory of the running server (one record per planned window): window start / end
// (µs), M, N, K, the level and chunk count the window ran with, the waiting queue the controller then
// observed and its new level / chunk count. Call before sd_serve_stop; copies min(max, windows).
extern "C" sd_status sd_serve_window_log(sd_engine* e, int32_t max, int64_t* t_start, int64_t* t_end, int32_t* m,
                                         int32_t* n, int32_t* k, int32_t* level, int32_t* c, int32_t* waiting,
                                         int32_t* level_after, int32_t* c_after, int32_t* n_out) {
  SD_REQUIRE(e && server_of(e) && n_out && max >= 0, "sd_serve_window_log: bad args");
  Server* S = server_of(e);
  std::lock_guard<std::mutex> g(S->mu);
  const int cnt = std::min<int>(max, (int)S->wlog.size());
  for (int i = 0; i < cnt; ++i) {
    const WindowLog& w = S->wlog[i];
    if (t_start) t_start[i] = w.now;
    if (t_end) t_end[i] = w.end;
    if (m) m[i] = w.M;
    if (n) n[i] = w.N;
    if (k) k[i] = w.K;
    if (level) level[i] = w.level;
    if (c) c[i] = w.c;
    if (waiting) waiting[i] = w.waiting;
    if (level_after) level_after[i] = w.level_after;
    if (c_after) c_after[i] = w.c_after;
  }
  *n_out = cnt;
  return SD_OK;
}
