// cm_policy.cpp -- checkpoint sets of the baseline policies (Table 1,
// PAPER.md:103-125, 447-455; App. B; R3-R5).  Host code: a few
// hundred sets per sweep; the S matrices they imply are written on the device
// (cm_policy_sstar) and evaluated by the same kernels as rounded S*.
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "cm.h"

namespace {
thread_local std::string g_pol_err;
cm_status pol_fail(cm_status s, const char* m) {
  g_pol_err = m;
  return s;
}

// Articulation points of the undirected forward graph (nodes 0..L-1), Hopcroft-Tarjan
// low-link DFS, iterative (graphs of up to CM_NMAX nodes).
std::vector<char> articulation_points(int L, const std::vector<std::vector<int>>& adj) {
  std::vector<int> disc(L, -1), low(L, 0), parent(L, -1), it(L, 0), kids(L, 0);
  std::vector<char> ap(L, 0);
  int timer = 0;
  for (int root = 0; root < L; ++root) {
    if (disc[root] >= 0) continue;
    std::vector<int> stack{root};
    disc[root] = low[root] = timer++;
    while (!stack.empty()) {
      const int u = stack.back();
      if (it[u] < (int)adj[u].size()) {
        const int w = adj[u][it[u]++];
        if (disc[w] < 0) {
          parent[w] = u;
          ++kids[u];
          disc[w] = low[w] = timer++;
          stack.push_back(w);
        } else if (w != parent[u]) {
          low[u] = std::min(low[u], disc[w]);
        }
      } else {
        stack.pop_back();
        const int p = parent[u];
        if (p >= 0) {
          low[p] = std::min(low[p], low[u]);
          if (parent[p] >= 0 && low[u] >= disc[p]) ap[p] = 1;   // non-root cut vertex
        }
      }
    }
    if (kids[root] > 1) ap[root] = 1;                                // root with >1 DFS children
  }
  return ap;
}
}  // namespace

extern "C" {

const char* cm_policy_last_error(void) { return g_pol_err.c_str(); }

cm_status cm_policy_checkpoints(int32_t n, int32_t L, const int32_t* pred_ptr, const int32_t* pred_idx,
                                const int64_t* mem, int32_t policy, int64_t b, uint8_t* is_checkpoint) {
  if (n < 1 || n > CM_NMAX || L < 1 || L > n || !pred_ptr || !mem || !is_checkpoint)
    return pol_fail(CM_EINVAL, "bad arguments");
  if (policy < CM_POLICY_ALL || policy > CM_POLICY_AP_GREEDY) return pol_fail(CM_EINVAL, "unknown policy");
  std::vector<std::vector<int>> adj(L);
  for (int k = 0; k < L; ++k)
    for (int e = pred_ptr[k]; e < pred_ptr[k + 1]; ++e) {
      const int i = pred_idx[e];
      if (i < 0 || i >= k) return pol_fail(CM_ETOPO, "edge (i, k) with i >= k");
      adj[i].push_back(k);
      adj[k].push_back(i);
    }
  for (int v = 0; v < L; ++v) is_checkpoint[v] = 0;
  if (policy == CM_POLICY_ALL) {
    for (int v = 0; v < L; ++v) is_checkpoint[v] = 1;
    return CM_OK;
  }
  // candidates in topological order: every forward node (Chen / linearized), or the
  // articulation points plus the first and last forward node (AP, R5)
  std::vector<int> cand;
  if (policy == CM_POLICY_AP_SQRT || policy == CM_POLICY_AP_GREEDY) {
    const std::vector<char> ap = articulation_points(L, adj);
    for (int v = 0; v < L; ++v)
      if (ap[v] || v == 0 || v == L - 1) cand.push_back(v);
  } else {
    for (int v = 0; v < L; ++v) cand.push_back(v);
  }
  if (policy == CM_POLICY_SQRT || policy == CM_POLICY_AP_SQRT) {    // every s-th candidate
    const int s = (int)std::ceil(std::sqrt((double)cand.size()));
    for (size_t j = 0; j < cand.size(); ++j)
      if ((j + 1) % s == 0 && cand[j] != L - 1) is_checkpoint[cand[j]] = 1;
    return CM_OK;
  }
  if (b < 0) return pol_fail(CM_EINVAL, "greedy: b < 0");
  std::vector<char> is_cand(L, 0);
  for (int v : cand) is_cand[v] = 1;
  int64_t acc = 0;                                                  // DESIGN.md R4
  for (int v = 0; v < L; ++v) {
    acc += mem[v];
    if (is_cand[v] && acc >= b && v != L - 1) {
      is_checkpoint[v] = 1;
      acc = 0;
    }
  }
  return CM_OK;
}

}  // extern "C"
