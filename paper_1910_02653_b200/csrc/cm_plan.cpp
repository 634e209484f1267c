// cm_plan.cpp -- execution-plan emission for chosen schedules:
// Algorithm 1 "Generate execution plan" from a candidate's R / S masks,
// optionally with the code motion of PAPER.md:328 (spurious checkpoints deallocated at the
// start of their stage).  Host code: it runs for the few winners the GPU path selects.
#include <cstdint>
#include <string>
#include <vector>

#include "cm.h"

namespace {
thread_local std::string g_plan_err;
cm_status plan_fail(cm_status s, const char* msg) {
  g_plan_err = msg;
  return s;
}
inline bool bit(const uint64_t* rows, int W, int t, int i) { return (rows[(size_t)t * W + (i >> 6)] >> (i & 63)) & 1u; }
}  // namespace

extern "C" {

const char* cm_plan_last_error(void) { return g_plan_err.c_str(); }

cm_status cm_emit_plan(int32_t n, const int32_t* pred_ptr, const int32_t* pred_idx, const int64_t* mem,
                       int64_t mem_overhead, const uint64_t* r_mask, const uint64_t* s_mask, int32_t hoist,
                       cm_stmt* out, int64_t capacity, int64_t* n_out, int64_t* peak_out) {
  if (n < 1 || n > CM_NMAX || !pred_ptr || !mem || !r_mask || !s_mask || !n_out || capacity < 0 ||
      (capacity > 0 && !out))
    return plan_fail(CM_EINVAL, "bad arguments");
  const int E = pred_ptr[n];
  if (pred_ptr[0] != 0 || E < 0 || (E > 0 && !pred_idx)) return plan_fail(CM_EINVAL, "bad CSR");
  std::vector<std::vector<int>> deps(n), users(n);
  for (int k = 0; k < n; ++k) {
    if (pred_ptr[k + 1] < pred_ptr[k]) return plan_fail(CM_EINVAL, "bad CSR");
    for (int e = pred_ptr[k]; e < pred_ptr[k + 1]; ++e) {
      const int i = pred_idx[e];
      if (i < 0 || i >= k) return plan_fail(CM_ETOPO, "edge (i, k) with i >= k");
      deps[k].push_back(i);
      users[i].push_back(k);
    }
  }
  const int W = (n + 63) / 64;
  std::vector<int> regs(n, -1);        // REGS[i]: register of v_i's latest computation (Alg. 1)
  std::vector<char> resident(n, 0);
  int64_t count = 0, peak = INT64_MIN;
  int reg = 0;
  auto emit = [&](int32_t op, int32_t t, int32_t node, int32_t r) {
    if (count < capacity) out[count] = cm_stmt{op, t, node, r};
    ++count;
  };
  for (int t = 0; t < n; ++t) {                                     // stage t+1 of the paper
    auto S = [&](int tt, int i) { return tt < n && bit(s_mask, W, tt, i); };   // S_{n+1} = 0
    auto R = [&](int i) { return bit(r_mask, W, t, i); };
    // stage boundary: exactly the checkpoints S_t are resident (constraint (3) makes them so)
    int64_t cur = mem_overhead;
    for (int i = 0; i < n; ++i) {
      if (S(t, i)) {
        if (t == 0 || regs[i] < 0 || !resident[i]) return plan_fail(CM_EINVAL, "S violates constraint (3)");
        cur += mem[i];
      } else {
        resident[i] = 0;
      }
    }
    if (hoist) {
      std::vector<char> used(n, 0);
      for (int k = 0; k < n; ++k)
        if (R(k))
          for (int i : deps[k]) used[i] = 1;
      for (int i = 0; i < n; ++i)
        if (S(t, i) && !used[i] && !S(t + 1, i)) {
          emit(CM_OP_DEALLOC, t, i, regs[i]);
          resident[i] = 0;
          cur -= mem[i];
        }
    }
    for (int k = 0; k < n; ++k) {
      if (R(k)) {
        for (int i : deps[k])
          if (!resident[i]) return plan_fail(CM_EINVAL, "R violates constraint (2)");
        emit(CM_OP_COMPUTE, t, k, reg);
        regs[k] = reg++;
        resident[k] = 1;
        cur += mem[k];
        if (cur > peak) peak = cur;                                 // U_{t,k}: after the compute
        // FREE_{t,i,k} = R_{t,k} (1 - S_{t+1,i}) prod_{j in USERS(i), j > k} (1 - R_{t,j}),
        // i in DEPS(k) u {k} (Eqs. 8-9)
        auto try_free = [&](int i) {
          if (S(t + 1, i) || !resident[i]) return;
          for (int j : users[i])
            if (j > k && R(j)) return;
          emit(CM_OP_DEALLOC, t, i, regs[i]);
          resident[i] = 0;
          cur -= mem[i];
        };
        for (int i : deps[k]) try_free(i);
        try_free(k);
      }
    }
  }
  *n_out = count;
  if (peak_out) *peak_out = peak;
  if (count > capacity) return plan_fail(CM_ERANGE, "capacity too small: *n_out statements needed");
  return CM_OK;
}

}  // extern "C"
