// Host control plane internals (control.cpp).
#pragma once
#include <stdint.h>

#include <array>
#include <unordered_map>
#include <utility>
#include <vector>

#include "sd_api.h"

namespace sd {

struct Table {
  std::unordered_map<uint64_t, std::pair<int64_t, int64_t>> e;  // (c,m,n,k) → (τ µs, δ µs)
  static uint64_t key(int c, int m, int n, int k) {
    return ((uint64_t)(uint16_t)c << 48) | ((uint64_t)(uint16_t)m << 32) | ((uint64_t)(uint16_t)n << 16) |
           (uint64_t)(uint16_t)k;
  }
  bool get(int c, int m, int n, int k, int64_t* tau, int64_t* delta) const;
};

struct PlanOut {
  std::vector<std::array<int, 3>> stages;
  int64_t cost = 0, time = 0;
};

int64_t t_lim(int64_t tau, int a_num, int a_den);
bool plan_window(const Table& T, int M, int N, int K, int c, int a_num, int a_den, int mode, PlanOut* out);

// Task mapping E of Problem P (R14). unet = the batch in batch order, dec = the window's
// decodes already ordered by (A_i, id). Skip slots go to the eligible tasks with the largest s/n
// (then id); the remaining UNet slots follow batch order. Per stage: indexes into unet (skippers
// first, in progress order, then the rest in batch order), their skip flags, and indexes into dec.
struct MapTask {
  uint64_t id;
  int s, n;
  bool eligible;
};
struct StageMap {
  std::vector<int> unet;
  std::vector<uint8_t> skip;
  std::vector<int> dec;
};
std::vector<StageMap> map_tasks(const std::vector<std::array<int, 3>>& stages, const std::vector<MapTask>& unet,
                                int n_dec);

struct Controller {
  sd_controller_config cfg{};
  int level = 0, c = 1, n_up = 0, n_down = 0;
  std::vector<std::pair<int64_t, int32_t>> samples;
  void observe(int64_t now, int32_t q);
  bool slope(__int128* num, __int128* den) const;
  sd_directive decide(int64_t now, int32_t q);
};

}  // namespace sd

struct sd_table {
  sd::Table t;
};
