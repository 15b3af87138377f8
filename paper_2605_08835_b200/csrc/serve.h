// Continuous-batching serving loop (§8(c) steps 1-5): one loop,
// two executors — the GPU executor (real clock, sd_step_batch + chunked decodes on two streams) and
// the virtual-clock executor (round durations from the τ/δ table; bit-exact with oracle/serving.py).
#pragma once
#include <stdint.h>

#include <functional>
#include <mutex>
#include <vector>

#include "control.h"
#include "sd_api.h"

namespace sd {

struct STask {
  uint64_t id = 0;
  int64_t A = 0;
  int h = 0, w = 0, n = 0;
  float g = 7.5f;
  uint64_t noise_seed = 0;
  std::vector<float> emb;
  std::vector<float> pooled;  // SDXL added conditioning (empty otherwise)
  int emb_len = 0, emb_dim = 0;
  int s = 0;
  int64_t U = -1, V = -1;
  std::vector<int> skips;
  // GPU executor state
  float* lat = nullptr;
  int slot = -1;
  void* decode = nullptr;
  float* img_dev = nullptr;
  float* img_host = nullptr;
  bool delivered = false;  // handed out by sd_poll (under Server::mu); sd_release requires it
};

struct LoopCfg {
  int b_max = 8;
  int n_max = 8;  // decodes per window
  int a_num = 1, a_den = 10;
  int dp_mode = 0;
  int c_star = 1;
  sd_controller_config ctl{};
  // baseline policies and ablations (oracle/serving.py documents them)
  int policy = SD_POLICY_SYNERDIFF;
  bool no_skip = false, no_ctl = false;
  int64_t dyn_window_us = 500000;
};

struct WindowLog {
  int64_t now;
  int M, N, K, level, c;
  std::vector<std::array<int, 3>> stages;
  // the window's task records and the mapping E the loop ran (T5 replay): batch order / (A, id) order
  std::vector<MapTask> unet;
  std::vector<int> unet_stage, unet_skip;
  std::vector<uint64_t> dec_id;
  std::vector<int64_t> dec_A;
  std::vector<int> dec_stage;
  // after the window: its end, the waiting queue the controller observed, and its new state
  int64_t end = 0;
  int waiting = 0, level_after = 0, c_after = 0;
};

// Executor interface: the loop is identical for the GPU and the virtual clock.
struct Exec {
  virtual ~Exec() {}
  virtual int64_t now() = 0;
  virtual void admit(STask* t) = 0;
  // one round of a stage; step = tasks stepping this round, skip[i] = Skip-CFG for step[i];
  // decodes run chunk `rho` of `rounds`. Returns the round end time; fills dec_done (per decode,
  // completion time when rho == rounds-1).
  virtual int64_t round(const std::vector<STask*>& step, const std::vector<uint8_t>& skip,
                        const std::vector<STask*>& decs, int rho, int rounds, int64_t stage_t0, int64_t tau,
                        int64_t delta, std::vector<int64_t>* dec_done) = 0;
  virtual void complete(STask* t) = 0;
  virtual int64_t global_waiting(int64_t local) { return local; }
};

struct Loop {
  LoopCfg cfg;
  const Table* table = nullptr;
  std::vector<std::pair<int, const Table*>> res_tables;  // mixed resolutions: latent hw → table
  Controller ctl;
  std::vector<STask*> pending;  // sorted by (A, id)
  std::vector<STask*> batch, dec;
  std::vector<WindowLog>* log = nullptr;
  std::mutex* log_mu = nullptr;  // GPU server: the log is read by another thread
  // one window; returns false if there was nothing to do (the caller waits until next_event())
  bool window(Exec& ex);
  int64_t next_arrival() const { return pending.empty() ? -1 : pending.front()->A; }
  // earliest time window() can make progress when idle: the next arrival, or for Dynamic Batching
  // the dispatch time of the batch being collected
  int64_t next_event() const;

 private:
  // the table of the largest latent among `a` and `b` (mixed resolutions), else `table`
  const Table* table_for(const std::vector<STask*>& a, const std::vector<STask*>& b) const;
  bool serial_window(Exec& ex);
  bool dynamic_window(Exec& ex);
  int64_t dynamic_dispatch_time() const;
  int64_t stage_round(Exec& ex, const Table* tb, int m, int n, int k, const std::vector<STask*>& step,
                      const std::vector<uint8_t>& skip, const std::vector<STask*>& decs, std::vector<int64_t>* dd);
};

sd_status window_plan_copy(const WindowLog& w, int32_t* stages_out, int32_t max_stages, int32_t* n_stages,
                           sd_logged_unet* unet_out, int32_t max_unet, int32_t* n_unet, sd_logged_decode* dec_out,
                           int32_t max_dec, int32_t* n_dec, int32_t* level_out, int32_t* c_out);
void insert_pending(std::vector<STask*>& pending, STask* t);
void set_policy(LoopCfg& c, const sd_serve_config* cfg);
void set_tables(Loop& L, const sd_serve_config* cfg);

}  // namespace sd
