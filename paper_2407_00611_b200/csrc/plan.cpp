// plan.cpp -- WallFacer's Communication Configuration Generator (host, integer math).
//
//  get_init_send  : Alg. 2, PAPER.md:263-275 (§3.3)
//  get_init_recv  : "calculated similarly" -> the inverse permutation (reading c8)
//  get_p2p_config : Alg. 3; (r_t - 1) % g is the mathematical modulo (c6)
//  validity       : reading c2 -- C | P and (C^2 <= P => C^2 | P); C^2 > P is the extension
//                   regime (ours): R = 1, member a attends K/V slice a = units [aP/C,(a+1)P/C).
#include "plan.h"

#include <string>

namespace wf {

int get_init_send(int r_t, int r_a, int d_t, int d_a) {
  const int group_size = d_t / d_a;
  const int target_group = r_a;
  const int target_team = target_group * group_size + r_t / d_a;
  const int target_intra = r_t % d_a;
  return target_team * d_a + target_intra;
}

void get_p2p_config(int r_t, int r_a, int d_t, int d_a, int* next, int* last) {
  const int g = d_t / d_a;
  const int self_group = r_t / g;
  const int next_team = (r_t + 1) % g + g * self_group;
  const int last_team = ((r_t - 1) % g + g) % g + g * self_group;
  *next = r_a + next_team * d_a;
  *last = r_a + last_team * d_a;
}

bool build_plan(int P, int C, Plan* p, std::string* err) {
  if (P < 1 || C < 1) {
    if (err) *err = "P and C must be >= 1";
    return false;
  }
  if (C > P || P % C) {
    if (err) *err = "C=" + std::to_string(C) + " must divide P=" + std::to_string(P);
    return false;
  }
  if (C * C <= P && P % (C * C)) {
    if (err) *err = "C^2=" + std::to_string(C * C) + " must divide P=" + std::to_string(P) + " when C^2 <= P";
    return false;
  }
  p->P = P;
  p->C = C;
  p->T = P / C;
  p->paper = C * C <= P;
  p->R = p->paper ? P / (C * C) : 1;
  p->W = P / C;
  p->send.assign(P, 0);
  p->recv.assign(P, 0);
  p->next.assign(P, 0);
  p->last.assign(P, 0);
  for (int r = 0; r < P; ++r) {
    if (!p->paper) {
      p->send[r] = p->recv[r] = p->next[r] = p->last[r] = r;
      continue;
    }
    const int r_t = r / C, r_a = r % C;
    p->send[r] = get_init_send(r_t, r_a, p->T, C);
    get_p2p_config(r_t, r_a, p->T, C, &p->next[r], &p->last[r]);
  }
  if (p->paper) {
    std::vector<int> seen(P, 0);
    for (int r = 0; r < P; ++r) {
      if (p->send[r] < 0 || p->send[r] >= P || seen[p->send[r]]++) {
        if (err) *err = "init_send is not a permutation";
        return false;
      }
      p->recv[p->send[r]] = r;
    }
  }
  return true;
}

int Plan::block_at(int r, int s) const {
  int x = r;
  for (int i = 0; i < s; ++i) x = last[x];
  return recv[x] / C;
}

}  // namespace wf
