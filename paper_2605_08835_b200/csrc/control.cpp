// Host control plane (§III-C/§III-D): latency table, Problem P
// (Eq. 3a-3f) solved by an exact Pareto-label DP (reading R10) or by Alg. 1 verbatim
// (PAPER.md:327-349), and the load-adaptive feedback controller (reading R15).
// Integer µs arithmetic throughout (R11), so decisions are bit-exact against oracle/sched.py and
// oracle/controller.py (independent implementations).
#include <algorithm>
#include <array>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "api_common.h"
#include "common.cuh"
#include "control.h"

namespace sd {

// ---- table -------------------------------------------------------------------------------------
bool Table::get(int c, int m, int n, int k, int64_t* tau, int64_t* delta) const {
  auto it = e.find(key(c, m, n, k));
  if (it == e.end()) return false;
  *tau = it->second.first;
  *delta = it->second.second;
  return true;
}

// ---- Problem P ----------------------------------------------------------------------------------
struct Act {
  int m, n, k;
};

static std::vector<Act> actions(int i, int j, int u, int M, int N, int K) {
  std::vector<Act> out;
  const bool decode_only = N > M;
  for (int m = 0; m <= M - i; ++m)
    for (int n = 0; n <= N - j; ++n)
      for (int k = 0; k <= K - u; ++k) {
        if (m >= 1) {
          if (n <= m && k <= m) out.push_back({m, n, k});
        } else if (decode_only && n >= 1 && k == 0) {
          out.push_back({m, n, k});
        }
      }
  return out;
}

struct Label {
  int64_t cost, time;
  std::vector<std::array<int, 3>> seq;
};

static bool seq_less(const Label& a, const Label& b) {
  if (a.seq.size() != b.seq.size()) return a.seq.size() < b.seq.size();
  return a.seq < b.seq;
}
static bool key_less(const Label& a, const Label& b) {
  if (a.cost != b.cost) return a.cost < b.cost;
  if (a.time != b.time) return a.time < b.time;
  return seq_less(a, b);
}

static void insert_label(std::vector<Label>& lst, Label&& lab) {
  for (auto& x : lst) {
    if (x.cost <= lab.cost && x.time <= lab.time && (x.cost < lab.cost || x.time < lab.time)) return;
    if (x.cost == lab.cost && x.time == lab.time) {
      if (seq_less(lab, x)) x = std::move(lab);
      return;
    }
  }
  lst.erase(std::remove_if(lst.begin(), lst.end(),
                           [&](const Label& x) { return lab.cost <= x.cost && lab.time <= x.time; }),
            lst.end());
  lst.push_back(std::move(lab));
}

static std::vector<std::array<int, 3>> reference_plan(int M, int N, int K) {
  if (N <= M) return {{M, N, K}};
  if (M == 0) return {{0, N, 0}};
  return {{M, M, K}, {0, N - M, 0}};
}

int64_t t_lim(int64_t tau, int a_num, int a_den) { return (tau * a_den + tau * a_num) / a_den; }

bool plan_window(const Table& T, int M, int N, int K, int c, int a_num, int a_den, int mode, PlanOut* out) {
  out->stages.clear();
  out->cost = out->time = 0;
  if (M == 0 && N == 0) return true;
  auto tab = [&](int m, int n, int k, int64_t* tau, int64_t* d) {
    if (!T.get(c, m, n, k, tau, d))
      throw std::invalid_argument("latency table miss (c,m,n,k)=(" + std::to_string(c) + "," + std::to_string(m) +
                                  "," + std::to_string(n) + "," + std::to_string(k) + ")");
  };
  if (N == 0) {
    int64_t tau, d;
    tab(M, 0, 0, &tau, &d);
    out->stages.push_back({M, 0, 0});
    out->time = tau;
    return true;
  }
  int64_t tref = 0;
  for (auto& s : reference_plan(M, N, K)) {
    int64_t tau, d;
    tab(s[0], s[1], s[2], &tau, &d);
    tref += tau;
  }
  const int64_t lim = t_lim(tref, a_num, a_den);
  auto idx = [&](int i, int j, int u) { return (i * (N + 1) + j) * (K + 1) + u; };
  const int S = (M + 1) * (N + 1) * (K + 1);
  if (mode == 0) {
    std::vector<std::vector<Label>> L(S);
    L[idx(0, 0, 0)].push_back(Label{0, 0, {}});
    for (int i = 0; i <= M; ++i)
      for (int j = 0; j <= N; ++j)
        for (int u = 0; u <= K; ++u) {
          auto& cur = L[idx(i, j, u)];
          if (cur.empty()) continue;
          for (const Act& a : actions(i, j, u, M, N, K)) {
            int64_t tau, d;
            tab(a.m, a.n, a.k, &tau, &d);
            auto& nxt = L[idx(i + a.m, j + a.n, u + a.k)];
            for (const Label& lb : cur) {
              const int64_t tn = lb.time + tau;
              if (tn > lim) continue;
              const int64_t cn = lb.cost + (a.n > 0 ? (int64_t)a.n * (lb.time + d) : 0);
              Label nl{cn, tn, lb.seq};
              nl.seq.push_back({a.m, a.n, a.k});
              insert_label(nxt, std::move(nl));
            }
          }
        }
    const Label* best = nullptr;
    for (int u = 0; u <= K; ++u)
      for (const Label& lb : L[idx(M, N, u)])
        if (!best || key_less(lb, *best)) best = &lb;
    if (!best) {
      out->stages = reference_plan(M, N, K);
    } else {
      out->stages = best->seq;
    }
  } else {
    // Alg. 1 verbatim: one <cost,time> per state, relax on strictly smaller cost
    const int64_t INF = INT64_MAX;
    std::vector<int64_t> dc(S, INF), dt(S, 0);
    std::vector<std::array<int, 6>> par(S);
    dc[idx(0, 0, 0)] = 0;
    for (int i = 0; i <= M; ++i)
      for (int j = 0; j <= N; ++j)
        for (int u = 0; u <= K; ++u) {
          const int s = idx(i, j, u);
          if (dc[s] == INF) continue;
          for (const Act& a : actions(i, j, u, M, N, K)) {
            int64_t tau, d;
            tab(a.m, a.n, a.k, &tau, &d);
            const int64_t tn = dt[s] + tau;
            if (tn <= lim) {
              const int64_t cv = a.n > 0 ? dt[s] + d : 0;
              const int64_t cn = dc[s] + cv * a.n;
              const int ns = idx(i + a.m, j + a.n, u + a.k);
              if (cn < dc[ns]) {
                dc[ns] = cn;
                dt[ns] = tn;
                par[ns] = {i, j, u, a.m, a.n, a.k};
              }
            }
          }
        }
    int bu = -1;
    for (int u = 0; u <= K; ++u)
      if (dc[idx(M, N, u)] != INF && (bu < 0 || dc[idx(M, N, u)] < dc[idx(M, N, bu)])) bu = u;
    if (bu < 0) {
      out->stages = reference_plan(M, N, K);
    } else {
      std::vector<std::array<int, 3>> seq;
      int i = M, j = N, u = bu;
      while (!(i == 0 && j == 0 && u == 0)) {
        const auto& p = par[idx(i, j, u)];
        seq.push_back({p[3], p[4], p[5]});
        i = p[0];
        j = p[1];
        u = p[2];
      }
      std::reverse(seq.begin(), seq.end());
      out->stages = seq;
    }
  }
  // recompute (cost, time) of the chosen plan
  int64_t time = 0, cost = 0;
  for (auto& s : out->stages) {
    int64_t tau, d;
    tab(s[0], s[1], s[2], &tau, &d);
    if (s[1] > 0) cost += (int64_t)s[1] * (time + d);
    time += tau;
  }
  out->cost = cost;
  out->time = time;
  return true;
}

// ---- controller (R15) ------------------------------------------------------------------------
void Controller::observe(int64_t now, int32_t q) {
  if (!samples.empty() && now < samples.back().first) throw std::invalid_argument("time regression");
  samples.push_back({now, q});
  if ((int)samples.size() > cfg.window) samples.erase(samples.begin());
}

// slope = num/den in tasks per µs (den > 0), or false if undefined
bool Controller::slope(__int128* num, __int128* den) const {
  const int n = (int)samples.size();
  if (n < 2) return false;
  const int64_t t0 = samples[0].first;
  __int128 st = 0, sq = 0, stt = 0, stq = 0;
  for (auto& s : samples) {
    const __int128 t = s.first - t0;
    st += t;
    sq += s.second;
    stt += t * t;
    stq += t * s.second;
  }
  const __int128 d = (__int128)n * stt - st * st;
  if (d == 0) return false;
  *num = (__int128)n * stq - st * sq;
  *den = d;
  return true;
}

sd_directive Controller::decide(int64_t now, int32_t q) {
  observe(now, q);
  sd_directive r{level, c, 0};
  __int128 num, den;
  if (!slope(&num, &den)) return r;
  // slope > up_num/(up_den·1e6)  ⇔  num·up_den·1e6 > up_num·den   (den > 0)
  const __int128 M6 = 1000000;
  const bool up = num * cfg.up_den * M6 > (__int128)cfg.up_num * den;
  const bool down = num * cfg.down_den * M6 < (__int128)cfg.down_num * den;
  if (up) {
    ++n_up;
    n_down = 0;
  } else if (down) {
    ++n_down;
    n_up = 0;
  } else {
    n_up = n_down = 0;
  }
  if (n_up >= cfg.hysteresis) {
    n_up = 0;
    if (level < 2) {
      ++level;
      r.changed = 1;
    } else if (c < cfg.c_max) {
      ++c;
      r.changed = 1;
    }
  } else if (n_down >= cfg.hysteresis) {
    n_down = 0;
    if (c > cfg.c_star) {
      --c;
      r.changed = 1;
    } else if (level > 0) {
      --level;
      r.changed = 1;
    }
  }
  r.level = level;
  r.c = c;
  return r;
}

}  // namespace sd

// =============================== C ABI =========================================================
using namespace sd;

struct sd_controller {
  Controller c;
};

extern "C" sd_status sd_table_from_arrays(int32_t n, const int32_t* c, const int32_t* m, const int32_t* nn,
                                          const int32_t* k, const int64_t* tau, const int64_t* delta, sd_table** out) {
  SD_REQUIRE(out && n >= 0 && (n == 0 || (c && m && nn && k && tau && delta)), "sd_table_from_arrays: bad args");
  SD_API_BEGIN
  auto* t = new sd_table();
  for (int i = 0; i < n; ++i) {
    const uint64_t key = Table::key(c[i], m[i], nn[i], k[i]);
    if (t->t.e.count(key)) {
      delete t;
      throw std::invalid_argument("duplicate table key at row " + std::to_string(i));
    }
    if (tau[i] < 0 || delta[i] < 0) {
      delete t;
      throw std::invalid_argument("negative latency at row " + std::to_string(i));
    }
    t->t.e[key] = {tau[i], delta[i]};
  }
  *out = t;
  SD_API_END
}

extern "C" sd_status sd_table_load(const char* path, sd_table** out) {
  SD_REQUIRE(path && out, "sd_table_load: bad args");
  SD_API_BEGIN
  std::ifstream f(path);
  if (!f) throw std::invalid_argument(std::string("cannot open ") + path);
  std::string line;
  std::getline(f, line);
  if (line.rfind("c,m,n,k,tau_us,delta_us", 0) != 0) throw std::invalid_argument("bad header: " + line);
  std::vector<int32_t> c, m, n, k;
  std::vector<int64_t> tau, delta;
  int ln = 1;
  while (std::getline(f, line)) {
    ++ln;
    if (line.empty()) continue;
    std::stringstream ss(line);
    std::string tok;
    std::vector<long long> v;
    while (std::getline(ss, tok, ',')) {
      size_t pos = 0;
      long long x = std::stoll(tok, &pos);
      if (pos != tok.size()) throw std::invalid_argument("malformed row at line " + std::to_string(ln));
      v.push_back(x);
    }
    if (v.size() != 6) throw std::invalid_argument("malformed row at line " + std::to_string(ln));
    c.push_back((int32_t)v[0]);
    m.push_back((int32_t)v[1]);
    n.push_back((int32_t)v[2]);
    k.push_back((int32_t)v[3]);
    tau.push_back(v[4]);
    delta.push_back(v[5]);
  }
  sd_status s = sd_table_from_arrays((int32_t)c.size(), c.data(), m.data(), n.data(), k.data(), tau.data(),
                                     delta.data(), out);
  if (s != SD_OK) return s;
  SD_API_END
}

extern "C" sd_status sd_table_free(sd_table* t) {
  delete t;
  return SD_OK;
}

extern "C" sd_status sd_plan(const sd_table* t, int32_t M, int32_t N, int32_t K, int32_t c, int32_t a_num,
                             int32_t a_den, int32_t dp_mode, int32_t* stages_out, int32_t max_stages,
                             int32_t* n_stages, int64_t* cost_out, int64_t* time_out) {
  SD_REQUIRE(t && n_stages && M >= 0 && N >= 0 && K >= 0 && K <= M && a_den > 0 && a_num >= 0,
             "sd_plan: bad args");
  SD_REQUIRE(dp_mode == 0 || dp_mode == 1, "sd_plan: dp_mode must be 0 or 1");
  SD_REQUIRE(M <= 16 && N <= 16, "sd_plan: window too large (split by B_max first)");
  SD_API_BEGIN
  PlanOut p;
  plan_window(t->t, M, N, K, c, a_num, a_den, dp_mode, &p);
  if ((int)p.stages.size() > max_stages) throw std::invalid_argument("sd_plan: max_stages too small");
  for (size_t i = 0; i < p.stages.size(); ++i)
    for (int q = 0; q < 3; ++q) stages_out[3 * i + q] = p.stages[i][q];
  *n_stages = (int32_t)p.stages.size();
  if (cost_out) *cost_out = p.cost;
  if (time_out) *time_out = p.time;
  SD_API_END
}

std::vector<StageMap> sd::map_tasks(const std::vector<std::array<int, 3>>& stages, const std::vector<MapTask>& unet,
                                int n_dec) {
  std::vector<int> el;
  for (int i = 0; i < (int)unet.size(); ++i)
    if (unet[i].eligible) el.push_back(i);
  std::stable_sort(el.begin(), el.end(), [&](int a, int b) {
    const int64_t l = (int64_t)unet[a].s * unet[b].n, r = (int64_t)unet[b].s * unet[a].n;  // s_a/n_a vs s_b/n_b
    return l != r ? l > r : unet[a].id < unet[b].id;
  });
  int nskip = 0, nm = 0, nn = 0;
  for (auto& st : stages) nskip += st[2], nm += st[0], nn += st[1];
  if (nm != (int)unet.size() || nn != n_dec || nskip > (int)el.size())
    throw std::invalid_argument("map_tasks: stages do not cover the window (sum m = M, sum n = N, sum k <= K)");
  std::vector<int> skippers(el.begin(), el.begin() + nskip);
  std::vector<uint8_t> is_skipper(unet.size(), 0);
  for (int i : skippers) is_skipper[i] = 1;
  std::vector<int> rest;
  for (int i = 0; i < (int)unet.size(); ++i)
    if (!is_skipper[i]) rest.push_back(i);
  std::vector<StageMap> out;
  size_t si = 0, ri = 0;
  int di = 0;
  for (auto& st : stages) {
    StageMap sm;
    for (int q = 0; q < st[2]; ++q) {
      sm.unet.push_back(skippers[si++]);
      sm.skip.push_back(1);
    }
    for (int q = 0; q < st[0] - st[2]; ++q) {
      sm.unet.push_back(rest[ri++]);
      sm.skip.push_back(0);
    }
    for (int q = 0; q < st[1]; ++q) sm.dec.push_back(di++);
    out.push_back(std::move(sm));
  }
  return out;
}

// Task mapping E (R14) for given stages: decodes are ordered by (A_i, id) here; returns each task's
// stage index and skip flag.
extern "C" sd_status sd_map_tasks(const int32_t* stages, int32_t n_stages, int32_t n_unet, const uint64_t* unet_id,
                                  const int32_t* unet_s, const int32_t* unet_n, const uint8_t* unet_eligible,
                                  int32_t n_dec, const uint64_t* dec_id, const int64_t* dec_arrival,
                                  int32_t* unet_stage_out, uint8_t* unet_skip_out, int32_t* dec_stage_out) {
  SD_REQUIRE(n_stages >= 0 && n_unet >= 0 && n_dec >= 0 && (n_stages == 0 || stages), "sd_map_tasks: bad args");
  SD_REQUIRE(n_unet == 0 || (unet_id && unet_s && unet_n && unet_eligible && unet_stage_out && unet_skip_out),
             "sd_map_tasks: bad unet arrays");
  SD_REQUIRE(n_dec == 0 || (dec_id && dec_arrival && dec_stage_out), "sd_map_tasks: bad decode arrays");
  for (int i = 0; i < n_unet; ++i) SD_REQUIRE(unet_n[i] >= 1 && unet_s[i] >= 0, "sd_map_tasks: bad step counts");
  for (int t = 0; t < n_stages; ++t)
    SD_REQUIRE(stages[3 * t] >= 0 && stages[3 * t + 1] >= 0 && stages[3 * t + 2] >= 0 &&
                   stages[3 * t + 2] <= stages[3 * t],
               "sd_map_tasks: bad stage");
  SD_API_BEGIN
  std::vector<std::array<int, 3>> st(n_stages);
  for (int t = 0; t < n_stages; ++t) st[t] = {stages[3 * t], stages[3 * t + 1], stages[3 * t + 2]};
  std::vector<MapTask> u(n_unet);
  for (int i = 0; i < n_unet; ++i) u[i] = MapTask{unet_id[i], unet_s[i], unet_n[i], unet_eligible[i] != 0};
  std::vector<int> order(n_dec);
  for (int i = 0; i < n_dec; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return dec_arrival[a] != dec_arrival[b] ? dec_arrival[a] < dec_arrival[b] : dec_id[a] < dec_id[b];
  });
  const auto E = map_tasks(st, u, n_dec);
  for (int t = 0; t < n_stages; ++t) {
    for (size_t q = 0; q < E[t].unet.size(); ++q) {
      unet_stage_out[E[t].unet[q]] = t;
      unet_skip_out[E[t].unet[q]] = E[t].skip[q];
    }
    for (int d : E[t].dec) dec_stage_out[order[d]] = t;
  }
  SD_API_END
}

// Offline chunk selection (Eq. 1, P:248 the C_max 5 % rule, R31), exact in rationals.
extern "C" sd_status sd_chunk_choice(const sd_table* t, int32_t m, int32_t n, const int32_t* c_values, int32_t n_c,
                                     int32_t lam_num, int32_t lam_den, int32_t* c_max_out, int32_t* c_star_out,
                                     double* cost_out) {
  SD_REQUIRE(t && c_values && n_c >= 1 && c_max_out && c_star_out && m >= 1 && n >= 1 && n <= m,
             "sd_chunk_choice: bad args");
  SD_REQUIRE(lam_den > 0 && lam_num >= 0 && lam_num <= lam_den, "sd_chunk_choice: lambda must be in [0, 1]");
  for (int i = 0; i < n_c; ++i) SD_REQUIRE(c_values[i] >= 1, "sd_chunk_choice: c >= 1");
  SD_API_BEGIN
  int64_t tu1, dummy, tv0;
  if (!t->t.get(1, m, 0, 0, &tu1, &dummy)) throw std::invalid_argument("sd_chunk_choice: table lacks (1, m, 0, 0)");
  if (!t->t.get(1, 0, n, 0, &dummy, &tv0) && !t->t.get(1, n, n, 0, &dummy, &tv0))
    throw std::invalid_argument("sd_chunk_choice: table lacks (1, 0, n, 0) and (1, n, n, 0)");
  if (tu1 <= 0 || tv0 <= 0) throw std::invalid_argument("sd_chunk_choice: zero baseline");
  typedef __int128 i128;
  int best = -1, cmax = -1;
  i128 bn = 0, bd = 1;
  for (int i = 0; i < n_c; ++i) {
    const int c = c_values[i];
    int64_t tau, delta;
    if (!t->t.get(c, m, n, 0, &tau, &delta)) throw std::invalid_argument("sd_chunk_choice: table lacks (c, m, n, 0)");
    const i128 tu0 = (i128)c * tu1;  // the UNet alone over the same c rounds
    // L(c) = lam (Tu - Tu0)/Tu0 + (1 - lam)(Tv - Tv0)/Tv0 = num / den
    const i128 num = (i128)lam_num * (tau - tu0) * tv0 + (i128)(lam_den - lam_num) * (delta - tv0) * tu0;
    const i128 den = (i128)lam_den * tu0 * tv0;
    if (cost_out) cost_out[i] = (double)num / (double)den;
    if (best < 0 || num * bd < bn * den || (num * bd == bn * den && c < best)) {
      best = c;
      bn = num;
      bd = den;
    }
    // C_max: concurrent UNet round tau/c <= (1 + 5 %) solo round tu1
    if ((i128)tau * 100 <= (i128)c * tu1 * 105) cmax = std::max(cmax, c);
  }
  if (cmax < 0) cmax = *std::min_element(c_values, c_values + n_c);
  *c_max_out = cmax;
  *c_star_out = best;
  SD_API_END
}

// Saturation batch (SPEC find_b_max): smallest m with thr(m+1)/thr(m) − 1 < ε, thr(m) = m/τ(m,0,0)
extern "C" sd_status sd_find_b_max(const sd_table* t, int32_t m_max, int32_t eps_num, int32_t eps_den,
                                   int32_t* b_max_out) {
  SD_REQUIRE(t && b_max_out && m_max >= 1 && eps_den > 0 && eps_num > 0 && eps_num < eps_den,
             "sd_find_b_max: bad args (need 0 < eps < 1, m_max >= 1)");
  SD_API_BEGIN
  std::vector<int64_t> tau(m_max + 1, 0);
  for (int m = 1; m <= m_max; ++m) {
    int64_t d;
    if (!t->t.get(1, m, 0, 0, &tau[m], &d) || tau[m] <= 0)
      throw std::invalid_argument("sd_find_b_max: table lacks (1, m, 0, 0) for m = " + std::to_string(m));
  }
  int best = m_max;
  for (int m = 1; m < m_max; ++m) {
    // thr(m+1)/thr(m) − 1 < ε  ⇔  (m+1)·τ(m)·den < m·τ(m+1)·(den + num)   (all positive)
    typedef __int128 i128;
    if ((i128)(m + 1) * tau[m] * eps_den < (i128)m * tau[m + 1] * (eps_den + eps_num)) {
      best = m;
      break;
    }
  }
  *b_max_out = best;
  SD_API_END
}

extern "C" sd_status sd_controller_create(const sd_controller_config* cfg, sd_controller** out) {
  SD_REQUIRE(cfg && out && cfg->c_star >= 1 && cfg->c_max >= cfg->c_star && cfg->window >= 2 &&
                 cfg->hysteresis >= 1 && cfg->up_den > 0 && cfg->down_den > 0,
             "sd_controller_create: bad config");
  SD_API_BEGIN
  auto* c = new sd_controller();
  c->c.cfg = *cfg;
  c->c.c = cfg->c_star;
  *out = c;
  SD_API_END
}

extern "C" sd_status sd_controller_decide(sd_controller* c, int64_t now_us, int32_t q, sd_directive* out) {
  SD_REQUIRE(c && out, "sd_controller_decide: bad args");
  SD_API_BEGIN
  *out = c->c.decide(now_us, q);
  SD_API_END
}

extern "C" sd_status sd_controller_free(sd_controller* c) {
  delete c;
  return SD_OK;
}

namespace sd {
std::vector<int> chunk_ranges_api(const std::vector<int64_t>& costs, int c);
}

extern "C" sd_status sd_chunk_ranges(const int64_t* costs, int32_t n, int32_t c, int32_t* out) {
  SD_REQUIRE(costs && out && n >= 1 && c >= 1, "sd_chunk_ranges: bad args");
  for (int i = 0; i < n; ++i) SD_REQUIRE(costs[i] >= 0, "sd_chunk_ranges: negative cost");
  SD_API_BEGIN
  std::vector<int64_t> v(costs, costs + n);
  auto b = chunk_ranges_api(v, c);
  for (size_t i = 0; i < b.size(); ++i) out[i] = b[i];
  SD_API_END
}
