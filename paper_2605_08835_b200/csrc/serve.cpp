// Serving loop shared by the GPU server and the virtual-clock simulator (see serve.h).
// Semantics: SURVEY.md §8(c) steps 1-5 with readings R6, R8, R9, R13, R14, R16, R17;
// the independent reference is oracle/serving.py.
#include "serve.h"

#include <algorithm>
#include <stdexcept>

#include "api_common.h"
#include "common.cuh"

namespace sd {

void insert_pending(std::vector<STask*>& p, STask* t) {
  auto it = std::upper_bound(p.begin(), p.end(), t, [](const STask* a, const STask* b) {
    return a->A != b->A ? a->A < b->A : a->id < b->id;
  });
  p.insert(it, t);
}

static int s_min(int level, int n) {
  if (level <= 0) return n + 1;            // f = ∞: no step is eligible
  if (level == 1) return (7 * n + 9) / 10;  // ⌈0.7 n⌉
  return (n + 1) / 2;                       // ⌈0.5 n⌉
}

int64_t Loop::dynamic_dispatch_time() const {
  // the batch closes W after its oldest request, or when B_max requests have arrived
  const int64_t first = pending.front()->A;
  int64_t close = first + cfg.dyn_window_us;
  if ((int)pending.size() >= cfg.b_max) close = std::min(close, pending[cfg.b_max - 1]->A);
  return close;
}

int64_t Loop::next_event() const {
  if (pending.empty()) return -1;
  if (cfg.policy == SD_POLICY_DYNAMIC && batch.empty() && dec.empty()) return dynamic_dispatch_time();
  return next_arrival();
}

const Table* Loop::table_for(const std::vector<STask*>& a, const std::vector<STask*>& b) const {
  if (res_tables.empty()) return table;
  int r = 0;
  for (auto* t : a) r = std::max(r, t->h);
  for (auto* t : b) r = std::max(r, t->h);
  for (auto& kv : res_tables)
    if (kv.first == r) return kv.second;
  throw std::invalid_argument("no latency table for latent " + std::to_string(r));
}

// one c = 1 round of stage (m, n, k) with the given tasks; returns the round end
int64_t Loop::stage_round(Exec& ex, const Table* tb, int m, int n, int k, const std::vector<STask*>& step,
                          const std::vector<uint8_t>& skip, const std::vector<STask*>& decs,
                          std::vector<int64_t>* dd) {
  int64_t tau, delta;
  if (!tb->get(1, m, n, k, &tau, &delta))
    throw std::invalid_argument("latency table miss (c,m,n,k)=(1," + std::to_string(m) + "," + std::to_string(n) +
                                "," + std::to_string(k) + ")");
  dd->assign(decs.size(), -1);
  return ex.round(step, skip, decs, 0, 1, ex.now(), tau, delta, dd);
}

// Diffusers baseline: BS = 1, FCFS; every step a (1,0,0) round, then the whole decode
bool Loop::serial_window(Exec& ex) {
  const int64_t now = ex.now();
  if (batch.empty() && dec.empty()) {
    if (pending.empty() || pending.front()->A > now) return false;
    batch.push_back(pending.front());
    ex.admit(pending.front());
    pending.erase(pending.begin());
  }
  std::vector<int64_t> dd;
  if (!dec.empty()) {
    STask* t = dec.front();
    stage_round(ex, table_for({t}, {}), 0, 1, 0, {}, {}, {t}, &dd);
    t->V = dd[0];
    dec.clear();
    ex.complete(t);
    return true;
  }
  STask* t = batch.front();
  const int64_t end = stage_round(ex, table_for({t}, {}), 1, 0, 0, {t}, {0}, {}, &dd);
  if (++t->s == t->n) {
    t->U = end;
    batch.clear();
    dec.push_back(t);
  }
  return true;
}

// Dynamic Batching baseline: collect, step in lockstep until every member is done (finished
// members wait), decode in stages of ≤ n_max, release the whole batch together
bool Loop::dynamic_window(Exec& ex) {
  const int64_t now = ex.now();
  if (batch.empty() && dec.empty()) {
    if (pending.empty() || now < dynamic_dispatch_time()) return false;
    size_t taken = 0;
    while (taken < pending.size() && (int)batch.size() < cfg.b_max && pending[taken]->A <= now) {
      batch.push_back(pending[taken]);
      ex.admit(pending[taken]);
      ++taken;
    }
    pending.erase(pending.begin(), pending.begin() + taken);
  }
  std::vector<int64_t> dd;
  const Table* tb = table_for(batch, {});
  std::vector<STask*> active;
  for (auto* t : batch)
    if (t->s < t->n) active.push_back(t);
  if (!active.empty()) {
    const int64_t end =
        stage_round(ex, tb, (int)active.size(), 0, 0, active, std::vector<uint8_t>(active.size(), 0), {}, &dd);
    for (auto* t : active)
      if (++t->s == t->n) t->U = end;
    return true;
  }
  // all members done: decode the next ≤ n_max of them (dec holds the decoded ones)
  std::vector<STask*> todo;
  for (auto* t : batch)
    if (std::find(dec.begin(), dec.end(), t) == dec.end() && (int)todo.size() < cfg.n_max) todo.push_back(t);
  const int64_t end = stage_round(ex, tb, 0, (int)todo.size(), 0, {}, {}, todo, &dd);
  dec.insert(dec.end(), todo.begin(), todo.end());
  if (dec.size() == batch.size()) {  // synchronous release
    for (auto* t : batch) {
      t->V = end;
      ex.complete(t);
    }
    batch.clear();
    dec.clear();
  }
  return true;
}

bool Loop::window(Exec& ex) {
  if (cfg.policy == SD_POLICY_SERIAL) return serial_window(ex);
  if (cfg.policy == SD_POLICY_DYNAMIC) return dynamic_window(ex);
  const bool naive = cfg.policy == SD_POLICY_NAIVE;
  int64_t now = ex.now();
  size_t taken = 0;
  while (taken < pending.size() && pending[taken]->A <= now && (int)batch.size() < cfg.b_max) {
    batch.push_back(pending[taken]);
    ex.admit(pending[taken]);
    ++taken;
  }
  pending.erase(pending.begin(), pending.begin() + taken);
  if (batch.empty() && dec.empty()) return false;
  const int level = (naive || cfg.no_skip) ? 0 : ctl.level, c = naive ? 1 : ctl.c;
  const int M = (int)batch.size();
  std::vector<STask*> dq = dec;
  std::sort(dq.begin(), dq.end(), [](const STask* a, const STask* b) { return a->A != b->A ? a->A < b->A : a->id < b->id; });
  if ((int)dq.size() > std::min(cfg.b_max, cfg.n_max)) dq.resize(std::min(cfg.b_max, cfg.n_max));
  const int N = (int)dq.size();
  const Table* tb = table_for(batch, dq);  // mixed resolutions: the window's largest latent
  std::vector<uint8_t> elig(M);
  int K = 0;
  for (int i = 0; i < M; ++i) {
    elig[i] = batch[i]->s >= s_min(level, batch[i]->n);
    K += elig[i];
  }
  PlanOut plan;
  int tc = 1, rounds = 1;
  if (N == 0) {
    plan.stages.push_back({M, 0, 0});
  } else if (naive) {  // InstGenIE: the whole batch with the oldest decodes, no plan, no skip
    plan.stages.push_back({M, M ? std::min(N, M) : N, 0});
  } else {
    plan_window(*tb, M, N, K, c, cfg.a_num, cfg.a_den, cfg.dp_mode, &plan);
    tc = c;
    rounds = c;
  }
  // task mapping E (R14)
  std::vector<MapTask> mt(M);
  for (int i = 0; i < M; ++i) mt[i] = MapTask{batch[i]->id, batch[i]->s, batch[i]->n, elig[i] != 0};
  int n_planned = 0;  // naive policy: only min(N, M) decodes join the window
  for (auto& st : plan.stages) n_planned += st[1];
  const std::vector<StageMap> E = map_tasks(plan.stages, mt, n_planned);
  const std::vector<STask*> bsnap = batch;  // tasks leave `batch` as they finish below
  if (log) {
    WindowLog wl{now, M, N, K, level, c, plan.stages};
    wl.unet = mt;
    wl.unet_stage.assign(M, -1);
    wl.unet_skip.assign(M, 0);
    for (size_t t = 0; t < E.size(); ++t)
      for (size_t q = 0; q < E[t].unet.size(); ++q) {
        wl.unet_stage[E[t].unet[q]] = (int)t;
        wl.unet_skip[E[t].unet[q]] = E[t].skip[q];
      }
    for (auto* d : dq) {
      wl.dec_id.push_back(d->id);
      wl.dec_A.push_back(d->A);
    }
    wl.dec_stage.assign(N, -1);
    for (size_t t = 0; t < E.size(); ++t)
      for (int d : E[t].dec) wl.dec_stage[d] = (int)t;
    std::unique_lock<std::mutex> g;
    if (log_mu) g = std::unique_lock<std::mutex>(*log_mu);
    log->push_back(std::move(wl));
  }
  for (size_t ti = 0; ti < plan.stages.size(); ++ti) {
    const int m = plan.stages[ti][0], n = plan.stages[ti][1], k = plan.stages[ti][2];
    std::vector<STask*> u_ids, d_ids;
    std::vector<uint8_t> is_skip = E[ti].skip;
    for (int q : E[ti].unet) u_ids.push_back(bsnap[q]);
    for (int q : E[ti].dec) d_ids.push_back(dq[q]);
    int64_t tau, delta;
    if (!tb->get(tc, m, n, k, &tau, &delta))
      throw std::invalid_argument("latency table miss (c,m,n,k)=(" + std::to_string(tc) + "," + std::to_string(m) + "," +
                                  std::to_string(n) + "," + std::to_string(k) + ")");
    const int64_t t0 = ex.now();
    for (int rho = 0; rho < rounds; ++rho) {
      std::vector<STask*> step;
      std::vector<uint8_t> skip;
      for (size_t q = 0; q < u_ids.size(); ++q)
        if (u_ids[q]->s < u_ids[q]->n) {
          step.push_back(u_ids[q]);
          skip.push_back(is_skip[q]);
        }
      std::vector<int64_t> dd(d_ids.size(), -1);
      const int64_t end = ex.round(step, skip, d_ids, rho, rounds, t0, tau, delta, &dd);
      for (size_t q = 0; q < step.size(); ++q) {
        STask* t = step[q];
        if (skip[q]) t->skips.push_back(t->s);
        t->s += 1;
        if (t->s == t->n) {
          t->U = end;
          batch.erase(std::find(batch.begin(), batch.end(), t));
          dec.push_back(t);
        }
      }
      if (rho == rounds - 1) {
        for (size_t q = 0; q < d_ids.size(); ++q) {
          STask* t = d_ids[q];
          t->V = dd[q];
          dec.erase(std::find(dec.begin(), dec.end(), t));
          ex.complete(t);
        }
      }
    }
  }
  now = ex.now();
  int64_t waiting = 0;
  for (auto* t : pending)
    if (t->A <= now) ++waiting;
  const int64_t gw = ex.global_waiting(waiting);
  if (!(naive || cfg.no_ctl)) ctl.decide(now, (int32_t)gw);
  if (log) {
    std::unique_lock<std::mutex> g;
    if (log_mu) g = std::unique_lock<std::mutex>(*log_mu);
    WindowLog& w = log->back();
    w.end = now;
    w.waiting = (int)gw;
    w.level_after = ctl.level;
    w.c_after = ctl.c;
  }
  return true;
}

// ---- virtual clock ----------------------------------------------------------------------------
struct VirtualExec : Exec {
  int64_t t = 0;
  std::vector<STask*> done;
  int64_t now() override { return t; }
  void admit(STask*) override {}
  int64_t round(const std::vector<STask*>&, const std::vector<uint8_t>&, const std::vector<STask*>& decs, int rho,
                int rounds, int64_t t0, int64_t tau, int64_t delta, std::vector<int64_t>* dd) override {
    const int64_t per = tau / rounds, rem = tau % rounds;
    t += per + (rho == rounds - 1 ? rem : 0);
    for (size_t i = 0; i < decs.size(); ++i) (*dd)[i] = t0 + delta;
    return t;
  }
  void complete(STask* x) override { done.push_back(x); }
};

}  // namespace sd

namespace sd {
void set_tables(Loop& L, const sd_serve_config* cfg) {
  L.res_tables.clear();
  for (int i = 0; i < cfg->n_res; ++i) L.res_tables.push_back({cfg->res_hw[i], &cfg->res_tables[i]->t});
}

void set_policy(LoopCfg& c, const sd_serve_config* cfg) {
  c.policy = cfg->policy;
  c.no_skip = (cfg->ablation & SD_ABL_NO_SKIP) != 0;
  c.no_ctl = (cfg->ablation & SD_ABL_NO_CTL) != 0;
  c.dyn_window_us = cfg->dyn_window_us > 0 ? cfg->dyn_window_us : 500000;
}
}  // namespace sd

using namespace sd;


static sd_status simulate_impl(const sd_serve_config* cfg, const sd_table* table, int32_t n, const uint64_t* ids,
                               const int64_t* arrival_us, const int32_t* n_steps, const int32_t* latent_hw,
                               int64_t* U_out, int64_t* V_out, int32_t* n_skips_out, int32_t* windows_out) {
  SD_REQUIRE(cfg && (table || cfg->n_res > 0) && n >= 0 && (n == 0 || (ids && arrival_us && n_steps && U_out && V_out)),
             "sd_serve_simulate: bad args");
  SD_REQUIRE(cfg->b_max >= 1 && cfg->a_den > 0 && cfg->c_star >= 1 && cfg->ctl.c_max >= cfg->c_star,
             "sd_serve_simulate: bad config");
  SD_REQUIRE(cfg->n_res == 0 || (cfg->res_hw && cfg->res_tables && latent_hw), "sd_serve_simulate: mixed tables");
  for (int i = 0; i < n; ++i) SD_REQUIRE(n_steps[i] >= 1 && arrival_us[i] >= 0, "sd_serve_simulate: bad request");
  SD_API_BEGIN
  std::vector<STask> tasks(n);
  Loop L;
  L.cfg.b_max = cfg->b_max;
  L.cfg.n_max = cfg->n_max > 0 ? cfg->n_max : cfg->b_max;
  L.cfg.a_num = cfg->a_num;
  L.cfg.a_den = cfg->a_den;
  L.cfg.dp_mode = cfg->dp_mode;
  L.cfg.c_star = cfg->c_star;
  L.table = table ? &table->t : nullptr;
  L.ctl.cfg = cfg->ctl;
  L.ctl.cfg.c_star = cfg->c_star;
  L.ctl.c = cfg->c_star;
  set_policy(L.cfg, cfg);
  set_tables(L, cfg);
  for (int i = 0; i < n; ++i) {
    tasks[i].id = ids[i];
    tasks[i].A = arrival_us[i];
    tasks[i].n = n_steps[i];
    tasks[i].h = tasks[i].w = latent_hw ? latent_hw[i] : 0;
    insert_pending(L.pending, &tasks[i]);
  }
  VirtualExec ex;
  int windows = 0;
  while (!L.pending.empty() || !L.batch.empty() || !L.dec.empty()) {
    if (!L.window(ex)) {
      ex.t = std::max(ex.t, L.next_event());
      continue;
    }
    ++windows;
  }
  for (int i = 0; i < n; ++i) {
    U_out[i] = tasks[i].U;
    V_out[i] = tasks[i].V;
    if (n_skips_out) n_skips_out[i] = (int32_t)tasks[i].skips.size();
  }
  if (windows_out) *windows_out = windows;
  SD_API_END
}

extern "C" sd_status sd_serve_simulate(const sd_serve_config* cfg, const sd_table* table, int32_t n,
                                       const uint64_t* ids, const int64_t* arrival_us, const int32_t* n_steps,
                                       int64_t* U_out, int64_t* V_out, int32_t* n_skips_out, int32_t* windows_out) {
  SD_REQUIRE(table, "sd_serve_simulate: null table");
  return simulate_impl(cfg, table, n, ids, arrival_us, n_steps, nullptr, U_out, V_out, n_skips_out, windows_out);
}

extern "C" sd_status sd_serve_simulate_mixed(const sd_serve_config* cfg, int32_t n, const uint64_t* ids,
                                             const int64_t* arrival_us, const int32_t* n_steps,
                                             const int32_t* latent_hw, int64_t* U_out, int64_t* V_out,
                                             int32_t* n_skips_out, int32_t* windows_out) {
  SD_REQUIRE(cfg && cfg->n_res > 0, "sd_serve_simulate_mixed: the config needs n_res tables");
  return simulate_impl(cfg, nullptr, n, ids, arrival_us, n_steps, latent_hw, U_out, V_out, n_skips_out, windows_out);
}

// ---- stepping virtual-clock server (multi-rank tests of C1) ----------------------
namespace sd {
struct VServer;
struct VSExec : VirtualExec {
  VServer* S = nullptr;
  int64_t global_waiting(int64_t local) override;
};
struct VServer {
  sd_serve_config cfg;
  std::vector<STask> tasks;
  Loop L;
  VSExec ex;
  std::vector<int32_t> global;  // [P][4] snapshot (sd_vserve_set_global_load)
  int P = 0;
  int windows = 0;
  std::vector<WindowLog> wlog;
};
int64_t VSExec::global_waiting(int64_t local) {
  if (S->P <= 1) return local;
  int64_t sum = 0;
  for (int r = 0; r < S->P; ++r) sum += S->global[4 * r];
  return sum;
}
}  // namespace sd

extern "C" sd_status sd_vserve_create(const sd_serve_config* cfg, const sd_table* table, int32_t n, const uint64_t* ids,
                                      const int64_t* arrival_us, const int32_t* n_steps, sd_vserver** out) {
  SD_REQUIRE(cfg && table && out && n >= 0 && (n == 0 || (ids && arrival_us && n_steps)), "sd_vserve_create: bad args");
  SD_REQUIRE(cfg->b_max >= 1 && cfg->a_den > 0 && cfg->c_star >= 1 && cfg->ctl.c_max >= cfg->c_star,
             "sd_vserve_create: bad config");
  SD_REQUIRE(cfg->policy == SD_POLICY_SYNERDIFF || cfg->policy == SD_POLICY_NAIVE,
             "sd_vserve_create: SynerDiff or naive policy");
  for (int i = 0; i < n; ++i) SD_REQUIRE(n_steps[i] >= 1 && arrival_us[i] >= 0, "sd_vserve_create: bad request");
  SD_API_BEGIN
  auto* V = new VServer();
  V->cfg = *cfg;
  V->tasks.resize(n);
  Loop& L = V->L;
  L.cfg.b_max = cfg->b_max;
  L.cfg.n_max = cfg->n_max > 0 ? cfg->n_max : cfg->b_max;
  L.cfg.a_num = cfg->a_num;
  L.cfg.a_den = cfg->a_den;
  L.cfg.dp_mode = cfg->dp_mode;
  L.cfg.c_star = cfg->c_star;
  L.table = &table->t;
  L.ctl.cfg = cfg->ctl;
  L.ctl.cfg.c_star = cfg->c_star;
  L.ctl.c = cfg->c_star;
  set_policy(L.cfg, cfg);
  L.log = &V->wlog;
  for (int i = 0; i < n; ++i) {
    V->tasks[i].id = ids[i];
    V->tasks[i].A = arrival_us[i];
    V->tasks[i].n = n_steps[i];
    insert_pending(L.pending, &V->tasks[i]);
  }
  V->ex.S = V;
  *out = reinterpret_cast<sd_vserver*>(V);
  SD_API_END
}

extern "C" sd_status sd_vserve_window(sd_vserver* h, int32_t* state_out) {
  SD_REQUIRE(h && state_out, "sd_vserve_window: bad args");
  SD_API_BEGIN
  auto* V = reinterpret_cast<VServer*>(h);
  Loop& L = V->L;
  if (L.pending.empty() && L.batch.empty() && L.dec.empty()) {
    *state_out = -1;
  } else if (L.window(V->ex)) {
    ++V->windows;
    *state_out = 1;
  } else {
    V->ex.t = std::max(V->ex.t, L.next_event());
    *state_out = 0;
  }
  SD_API_END
}

extern "C" sd_status sd_vserve_get_load(sd_vserver* h, int32_t* out4) {
  SD_REQUIRE(h && out4, "sd_vserve_get_load: bad args");
  auto* V = reinterpret_cast<VServer*>(h);
  int32_t waiting = 0;
  for (auto* t : V->L.pending)
    if (t->A <= V->ex.t) ++waiting;
  out4[0] = waiting;
  out4[1] = (int32_t)V->L.dec.size();
  out4[2] = (int32_t)V->L.batch.size();
  out4[3] = (int32_t)V->ex.done.size();
  return SD_OK;
}

extern "C" sd_status sd_vserve_set_global_load(sd_vserver* h, const int32_t* loads, int32_t P, uint64_t) {
  SD_REQUIRE(h && loads && P >= 1, "sd_vserve_set_global_load: bad args");
  auto* V = reinterpret_cast<VServer*>(h);
  V->global.assign(loads, loads + 4 * P);
  V->P = P;
  return SD_OK;
}

extern "C" sd_status sd_vserve_results(sd_vserver* h, int64_t* U_out, int64_t* V_out, int32_t* n_skips_out,
                                       int64_t* now_out, int32_t* windows_out) {
  SD_REQUIRE(h, "sd_vserve_results: bad args");
  auto* V = reinterpret_cast<VServer*>(h);
  for (size_t i = 0; i < V->tasks.size(); ++i) {
    if (U_out) U_out[i] = V->tasks[i].U;
    if (V_out) V_out[i] = V->tasks[i].V;
    if (n_skips_out) n_skips_out[i] = (int32_t)V->tasks[i].skips.size();
  }
  if (now_out) *now_out = V->ex.t;
  if (windows_out) *windows_out = V->windows;
  return SD_OK;
}

extern "C" sd_status sd_vserve_trajectory(sd_vserver* h, int32_t max, int32_t* waiting, int32_t* level_after,
                                          int32_t* c_after, int32_t* n_out) {
  SD_REQUIRE(h && n_out && max >= 0, "sd_vserve_trajectory: bad args");
  auto* V = reinterpret_cast<VServer*>(h);
  const int cnt = std::min<int>(max, (int)V->wlog.size());
  for (int i = 0; i < cnt; ++i) {
    if (waiting) waiting[i] = V->wlog[i].waiting;
    if (level_after) level_after[i] = V->wlog[i].level_after;
    if (c_after) c_after[i] = V->wlog[i].c_after;
  }
  *n_out = cnt;
  return SD_OK;
}

namespace sd {
sd_status window_plan_copy(const WindowLog& w, int32_t* stages_out, int32_t max_stages, int32_t* n_stages,
                           sd_logged_unet* unet_out, int32_t max_unet, int32_t* n_unet, sd_logged_decode* dec_out,
                           int32_t max_dec, int32_t* n_dec, int32_t* level_out, int32_t* c_out) {
  if ((int)w.stages.size() > max_stages || (int)w.unet.size() > max_unet || (int)w.dec_id.size() > max_dec)
    throw std::invalid_argument("window plan: output arrays too small");
  for (size_t t = 0; t < w.stages.size(); ++t)
    for (int q = 0; q < 3; ++q) stages_out[3 * t + q] = w.stages[t][q];
  *n_stages = (int32_t)w.stages.size();
  for (size_t i = 0; i < w.unet.size(); ++i)
    unet_out[i] = sd_logged_unet{w.unet[i].id, w.unet[i].s, w.unet[i].n, w.unet[i].eligible ? 1 : 0,
                                 w.unet_stage[i], w.unet_skip[i], 0};
  *n_unet = (int32_t)w.unet.size();
  for (size_t i = 0; i < w.dec_id.size(); ++i) dec_out[i] = sd_logged_decode{w.dec_id[i], w.dec_A[i], w.dec_stage[i], 0};
  *n_dec = (int32_t)w.dec_id.size();
  if (level_out) *level_out = w.level;
  if (c_out) *c_out = w.c;
  return SD_OK;
}
}  // namespace sd

extern "C" sd_status sd_vserve_window_plan(sd_vserver* h, int32_t window, int32_t* stages_out, int32_t max_stages,
                                           int32_t* n_stages, sd_logged_unet* unet_out, int32_t max_unet,
                                           int32_t* n_unet, sd_logged_decode* dec_out, int32_t max_dec,
                                           int32_t* n_dec, int32_t* level_out, int32_t* c_out) {
  SD_REQUIRE(h && stages_out && n_stages && unet_out && n_unet && dec_out && n_dec, "sd_vserve_window_plan: bad args");
  auto* V = reinterpret_cast<VServer*>(h);
  SD_REQUIRE(window >= 0 && window < (int)V->wlog.size(), "sd_vserve_window_plan: no such window");
  SD_API_BEGIN
  window_plan_copy(V->wlog[window], stages_out, max_stages, n_stages, unet_out, max_unet, n_unet, dec_out, max_dec,
                   n_dec, level_out, c_out);
  SD_API_END
}

extern "C" sd_status sd_vserve_free(sd_vserver* h) {
  delete reinterpret_cast<VServer*>(h);
  return SD_OK;
}
