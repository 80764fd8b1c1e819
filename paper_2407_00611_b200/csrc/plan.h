// plan.h -- the per-rank WallFacer plan (Alg. 2 / Alg. 3) used by the scheduler.
#pragma once
#include <string>
#include <vector>

namespace wf {

struct Plan {
  int P = 1, C = 1, T = 1, R = 1, W = 1;  // W = P / C units per extension slice
  bool paper = true;                      // C^2 <= P (Alg. 2/3) vs the C^2 > P extension
  std::vector<int> send, recv, next, last;
  // K/V team block held by rank r at forward ring step s: team of init_recv[last^s(r)].
  int block_at(int r, int s) const;
};

int get_init_send(int r_t, int r_a, int d_t, int d_a);
void get_p2p_config(int r_t, int r_a, int d_t, int d_a, int* next, int* last);
bool build_plan(int P, int C, Plan* p, std::string* err);

}  // namespace wf
