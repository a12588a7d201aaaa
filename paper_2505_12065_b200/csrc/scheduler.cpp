// scheduler.cpp -- SearchAgent-X priority scheduling (§3.2; SURVEY.md
// §8(f)2).  Host code: it orders the LLM engine's waiting sequences before every generation
// step (Alg. 1 line 23, "ApplyPriorityScheduling").
//
//   Eq. 1  T_{M,k} = min(M) + (k/G)(max(M) - min(M)),  0 <= k < G,  M in {R, W, C}
//   Eq. 2  level_i = max{ j | R_i > T_{R,j} or W_i > T_{W,j} or C_i > T_{C,j} }, else 0
//   order: level descending, then W^cur descending, then request id ascending.
//
// Metrics are integers (retrieval counts, tokens, microseconds), so each test
// M_i > min + (j/G)(max - min) is evaluated exactly as G*(M_i - min) > j*(max - min) in
// 128-bit integers -- no rounding can move a sequence across a level boundary.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/sa.h"

namespace sa {
sa_status set_error(sa_status s, const std::string& msg);
}

namespace {

struct Range {
  int64_t lo, hi;
};

Range range_of(const int64_t* v, int64_t n) {
  Range r{v[0], v[0]};
  for (int64_t i = 1; i < n; ++i) {
    r.lo = std::min(r.lo, v[i]);
    r.hi = std::max(r.hi, v[i]);
  }
  return r;
}

// largest j in [0, G) with G*(x - lo) > j*(hi - lo), or -1
int top_level(int64_t x, const Range& r, int G) {
  const __int128 lhs = (__int128)G * (x - r.lo);
  const __int128 span = (__int128)(r.hi - r.lo);
  for (int j = G - 1; j >= 0; --j)
    if (lhs > (__int128)j * span) return j;
  return -1;
}

}  // namespace

extern "C" sa_status sa_priority_order(int64_t n, const int64_t* R, const int64_t* W_us,
                                       const int64_t* C, const int64_t* Wcur_us,
                                       const int64_t* ids, int32_t G, int32_t* out_level,
                                       int64_t* out_order) {
  if (n < 0 || G < 1) return sa::set_error(SA_ERR_INVALID_ARG, "n >= 0 and G >= 1 required");
  if (n == 0) return SA_OK;
  if (!R || !W_us || !C || !Wcur_us || !ids || !out_order)
    return sa::set_error(SA_ERR_INVALID_ARG, "null pointer");
  for (int64_t i = 0; i < n; ++i)
    if (R[i] < 0 || W_us[i] < 0 || C[i] < 0 || Wcur_us[i] < 0 || R[i] > (1ll << 50) ||
        W_us[i] > (1ll << 50) || C[i] > (1ll << 50))
      return sa::set_error(SA_ERR_INVALID_ARG, "metrics must be in [0, 2^50]");
  const Range rr = range_of(R, n), rw = range_of(W_us, n), rc = range_of(C, n);
  std::vector<int32_t> lv(n);
  for (int64_t i = 0; i < n; ++i) {
    int k = std::max({top_level(R[i], rr, G), top_level(W_us[i], rw, G), top_level(C[i], rc, G)});
    lv[i] = k < 0 ? 0 : k;  // "Requests that do not meet any threshold are assigned to level 0"
  }
  std::vector<int64_t> pos(n);
  std::iota(pos.begin(), pos.end(), 0);
  std::sort(pos.begin(), pos.end(), [&](int64_t a, int64_t b) {
    if (lv[a] != lv[b]) return lv[a] > lv[b];
    if (Wcur_us[a] != Wcur_us[b]) return Wcur_us[a] > Wcur_us[b];
    return ids[a] < ids[b];
  });
  std::copy(pos.begin(), pos.end(), out_order);
  if (out_level) std::copy(lv.begin(), lv.end(), out_level);
  return SA_OK;
}
