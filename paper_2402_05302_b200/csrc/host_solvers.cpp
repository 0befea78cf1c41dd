// Host solvers of the Cannikin hot path: the heterogeneous GNS estimator and the OptPerf split.
//
//   cannikin_gns_estimate   PAPER.md §4.4, Eq. 10, Theorem 1 / Eq. 11,
//                           B_noise = S/G.
//   cannikin_opt_split      PAPER.md §3 Eq. 3-7, optimality §3.3 / App. A
//                           (P:221-243), Alg. 1, integer batches.
//   cannikin_warmup_split   Eq. 8.
//
// Built with -ffp-contract=off: the integer split is decided by comparisons of per-node times
// evaluated under the frozen contract of cannikin.h, so no multiply-add may be fused.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "common.h"

namespace cannikin {

static thread_local std::string g_last_error;

void set_error_text(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
void clear_error() { g_last_error.clear(); }

}  // namespace cannikin

using cannikin::fail;

extern "C" const char* cannikin_last_error(void) { return cannikin::g_last_error.c_str(); }
extern "C" int cannikin_version(void) { return CANNIKIN_VERSION; }

// ============================================================================================
// GNS estimator
// ============================================================================================

// Solve M x = rhs (n x n, row-major, overwritten) by Gaussian elimination with partial pivoting.
static bool gepp_solve(std::vector<double>& M, std::vector<double>& rhs, int n) {
  for (int col = 0; col < n; ++col) {
    int piv = col;
    double best = std::fabs(M[col * n + col]);
    for (int r = col + 1; r < n; ++r) {
      double v = std::fabs(M[r * n + col]);
      if (v > best) { best = v; piv = r; }
    }
    if (!(best > 0.0) || !std::isfinite(best)) return false;
    if (piv != col) {
      for (int c = 0; c < n; ++c) std::swap(M[col * n + c], M[piv * n + c]);
      std::swap(rhs[col], rhs[piv]);
    }
    const double d = M[col * n + col];
    for (int r = col + 1; r < n; ++r) {
      const double f = M[r * n + col] / d;
      if (f == 0.0) continue;
      for (int c = col; c < n; ++c) M[r * n + c] -= f * M[col * n + c];
      rhs[r] -= f * rhs[col];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    double acc = rhs[r];
    for (int c = r + 1; c < n; ++c) acc -= M[r * n + c] * rhs[c];
    rhs[r] = acc / M[r * n + r];
    if (!std::isfinite(rhs[r])) return false;
  }
  return true;
}

// w = 1^T A^{-1} / (1^T A^{-1} 1)  (Eq. 11).  1^T A^{-1} is the transpose of the solution of
// A^T x = 1, so the elimination runs on A^T.
static bool theorem1_weights(const std::vector<double>& A, int n, double* w) {
  std::vector<double> At(n * n), x(n, 1.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) At[i * n + j] = A[j * n + i];
  if (!gepp_solve(At, x, n)) return false;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += x[i];
  if (!(sum != 0.0) || !std::isfinite(sum)) return false;
  for (int i = 0; i < n; ++i) w[i] = x[i] / sum;
  return true;
}

extern "C" cannikin_status cannikin_gns_estimate(const double* local_sq, double global_sq,
                                                 const int64_t* b, int n,
                                                 cannikin_gns_result* out) {
  if (!local_sq || !b || !out) return fail(CANNIKIN_ERR_INVALID, "gns_estimate: NULL argument");
  if (n < 2 || n > CANNIKIN_MAX_GNS_NODES)
    return fail(CANNIKIN_ERR_INVALID, "gns_estimate: n=%d outside [2, %d]", n,
                CANNIKIN_MAX_GNS_NODES);
  int64_t Bi = 0;
  for (int i = 0; i < n; ++i) {
    if (b[i] < 1) return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate: b[%d]=%lld < 1", i, (long long)b[i]);
    Bi += b[i];
  }
  for (int i = 0; i < n; ++i) {
    if (b[i] >= Bi)
      return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate: b[%d] = B (Eq. 10 divides by B - b_i)", i);
    if (!std::isfinite(local_sq[i])) return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate: local_sq[%d] not finite", i);
  }
  if (!std::isfinite(global_sq)) return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate: global_sq not finite");

  const double B = (double)Bi;
  std::memset(out, 0, sizeof *out);
  out->n = n;
  // Eq. 10
  for (int i = 0; i < n; ++i) {
    const double bi = (double)b[i];
    out->Gi[i] = (B * global_sq - bi * local_sq[i]) / (B - bi);
    out->Si[i] = bi * B / (B - bi) * (local_sq[i] - global_sq);
  }
  // Theorem 1 matrices as printed
  std::vector<double> AG(n * n), AS(n * n);
  for (int i = 0; i < n; ++i) {
    const double bi = (double)b[i];
    for (int j = 0; j < n; ++j) {
      const double bj = (double)b[j];
      if (i == j) {
        AG[i * n + j] = (B + 2.0 * bi) / (B * B - B * bi);
        AS[i * n + j] = B * bi / (B - bi);
      } else {
        AG[i * n + j] = (B * B - bi * bi - bj * bj) / (B * (B - bi) * (B - bj));
        AS[i * n + j] = bi * bj * (B - bi - bj) / ((B - bi) * (B - bj));
      }
    }
  }
  if (!theorem1_weights(AG, n, out->wG))
    return fail(CANNIKIN_ERR_SINGULAR, "gns_estimate: A_G singular");
  if (!theorem1_weights(AS, n, out->wS))
    return fail(CANNIKIN_ERR_SINGULAR, "gns_estimate: A_S singular");
  double G = 0.0, S = 0.0;
  for (int i = 0; i < n; ++i) {
    G += out->wG[i] * out->Gi[i];
    S += out->wS[i] * out->Si[i];
  }
  out->G2 = G;
  out->trS = S;
  out->B_noise = S / G;  // P:364; IEEE semantics when G == 0
  if (!(G > 0.0)) out->flags |= CANNIKIN_GNS_G_NONPOSITIVE;
  cannikin::clear_error();
  return CANNIKIN_OK;
}

// Corrected-covariance variant (reading Q31).  Under the paper's own
// model (Eq. 1: g_i = mean of b_i iid N(G, Sigma) samples; Eq. 9: g = sum r_j g_j) the exact
// covariance of the Eq. 10 estimators (Isserlis' theorem) satisfies A_G (B - b) = const and
// A_S (B - b) = const, so the minimum-variance weights are w_i = (B - b_i) / ((n - 1) B) for both
// G and S, independent of the unknown G and Sigma.
extern "C" cannikin_status cannikin_gns_estimate_corrected(const double* local_sq,
                                                           double global_sq, const int64_t* b,
                                                           int n, cannikin_gns_result* out) {
  if (!local_sq || !b || !out)
    return fail(CANNIKIN_ERR_INVALID, "gns_estimate_corrected: NULL argument");
  if (n < 2 || n > CANNIKIN_MAX_GNS_NODES)
    return fail(CANNIKIN_ERR_INVALID, "gns_estimate_corrected: n=%d outside [2, %d]", n,
                CANNIKIN_MAX_GNS_NODES);
  int64_t Bi = 0;
  for (int i = 0; i < n; ++i) {
    if (b[i] < 1)
      return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate_corrected: b[%d]=%lld < 1", i, (long long)b[i]);
    Bi += b[i];
  }
  for (int i = 0; i < n; ++i) {
    if (b[i] >= Bi)
      return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate_corrected: b[%d] = B (Eq. 10 divides by B - b_i)", i);
    if (!std::isfinite(local_sq[i]))
      return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate_corrected: local_sq[%d] not finite", i);
  }
  if (!std::isfinite(global_sq))
    return fail(CANNIKIN_ERR_DOMAIN, "gns_estimate_corrected: global_sq not finite");
  const double B = (double)Bi;
  std::memset(out, 0, sizeof *out);
  out->n = n;
  double G = 0.0, S = 0.0;
  for (int i = 0; i < n; ++i) {
    const double bi = (double)b[i];
    out->Gi[i] = (B * global_sq - bi * local_sq[i]) / (B - bi);       // Eq. 10
    out->Si[i] = bi * B / (B - bi) * (local_sq[i] - global_sq);
    out->wG[i] = out->wS[i] = (B - bi) / ((double)(n - 1) * B);
    G += out->wG[i] * out->Gi[i];
    S += out->wS[i] * out->Si[i];
  }
  out->G2 = G;
  out->trS = S;
  out->B_noise = S / G;
  if (!(G > 0.0)) out->flags |= CANNIKIN_GNS_G_NONPOSITIVE;
  cannikin::clear_error();
  return CANNIKIN_OK;
}

// ============================================================================================
// OptPerf split
// ============================================================================================
namespace {

struct Model {
  double q, s, k, m, gamma, t_o, t_u;
  // Two branches of the per-node time, as lines in b:
  //   compute-bound (Eq. 5): L1 = (q + k) b + (s + m + t_u)
  //   comm-bound    (Eq. 6): L2 = (q + gamma k) b + (s + gamma m + t_o + t_u)
  double s1, c1, s2, c2;
};

// Frozen evaluation contract (cannikin.h): f = (A + max(P, X)) + t_u.
inline double frozen_time(const Model& M, double b) {
  const double P = M.k * b + M.m;
  const double A = M.q * b + M.s;
  const double X = M.gamma * P + M.t_o;
  const double mx = (P < X) ? X : P;
  return (A + mx) + M.t_u;
}

inline double line_inverse(const Model& M, double T) {
  const double v1 = (T - M.c1) / M.s1;
  const double v2 = (T - M.c2) / M.s2;
  return v1 < v2 ? v1 : v2;
}

inline double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

inline double line_max(const Model& M, double b) {
  const double a = M.s1 * b + M.c1, c = M.s2 * b + M.c2;
  return a > c ? a : c;
}

// Relaxed optimum: T* with sum_i clamp(f_i^{-1}(T*), lo_i, cap_i) = B.  The sum is a continuous,
// nondecreasing, piecewise-linear function of T whose kinks are each node's clamp points and the
// crossing of its two branches; locate the segment holding B, then solve its linear equation.
void solve_real(const std::vector<Model>& Ms, const std::vector<double>& lo,
                const std::vector<double>& cap, double B, std::vector<double>& b_real) {
  const int n = (int)Ms.size();
  b_real.assign(n, 0.0);
  double sum_lo = 0.0;
  for (double v : lo) sum_lo += v;
  if (sum_lo >= B) {
    b_real = lo;
    return;
  }
  std::vector<double> bp;
  bp.reserve(3 * n);
  for (int i = 0; i < n; ++i) {
    const Model& M = Ms[i];
    bp.push_back(line_max(M, lo[i]));
    bp.push_back(line_max(M, cap[i]));
    if (M.s1 > M.s2) {
      const double bx = (M.c2 - M.c1) / (M.s1 - M.s2);  // branch crossing: (1-gamma)P = T_o
      if (bx > lo[i] && bx < cap[i]) bp.push_back(M.s1 * bx + M.c1);
    }
  }
  std::sort(bp.begin(), bp.end());
  auto H = [&](double T) {
    double h = 0.0;
    for (int i = 0; i < n; ++i) h += clampd(line_inverse(Ms[i], T), lo[i], cap[i]);
    return h;
  };
  // first breakpoint with H >= B (exists: at the largest one every node sits at its cap)
  size_t kb = 0;
  while (kb + 1 < bp.size() && H(bp[kb]) < B) ++kb;
  double T;
  if (kb == 0) {
    T = bp[0];
  } else {
    const double Ta = bp[kb - 1], Tb = bp[kb];
    const double Tm = 0.5 * (Ta + Tb);
    double cst = 0.0, num = 0.0, den = 0.0;
    for (int i = 0; i < n; ++i) {
      const Model& M = Ms[i];
      const double v1 = (Tm - M.c1) / M.s1, v2 = (Tm - M.c2) / M.s2;
      const bool use1 = v1 < v2;
      const double v = use1 ? v1 : v2;
      if (v <= lo[i]) {
        cst += lo[i];
      } else if (v >= cap[i]) {
        cst += cap[i];
      } else {
        const double sl = use1 ? M.s1 : M.s2, c = use1 ? M.c1 : M.c2;
        num += c / sl;
        den += 1.0 / sl;
      }
    }
    T = den > 0.0 ? (B - cst + num) / den : Tb;
    T = clampd(T, Ta, Tb);
  }
  for (int i = 0; i < n; ++i) b_real[i] = clampd(line_inverse(Ms[i], T), lo[i], cap[i]);
}

}  // namespace

extern "C" double cannikin_node_time(const cannikin_node_model* node,
                                     const cannikin_comm_model* cm, double b) {
  if (!node || !cm) return std::nan("");
  Model M{node->q, node->s, node->k, node->m, cm->gamma, cm->t_o, cm->t_u, 0, 0, 0, 0};
  return frozen_time(M, b);
}

extern "C" cannikin_status cannikin_opt_split(const cannikin_node_model* nodes, int n,
                                              const cannikin_comm_model* cm, int64_t B,
                                              const int64_t* lo_in, const int64_t* cap_in,
                                              unsigned flags, int64_t* b_out, double* b_real_out,
                                              double* t_out, int* label_out) {
  if (!nodes || !cm) return fail(CANNIKIN_ERR_INVALID, "opt_split: NULL nodes or comm model");
  if (n < 1) return fail(CANNIKIN_ERR_INVALID, "opt_split: n=%d < 1", n);
  if (B < 1) return fail(CANNIKIN_ERR_INVALID, "opt_split: B=%lld < 1", (long long)B);
  const double gamma = cm->gamma, t_o = cm->t_o, t_u = cm->t_u;
  if (!std::isfinite(gamma) || !std::isfinite(t_o) || !std::isfinite(t_u) || !(gamma >= 0.0) ||
      !(gamma < 1.0) || !(t_o >= 0.0) || !(t_u >= 0.0))
    return fail(CANNIKIN_ERR_DOMAIN, "opt_split: need 0 <= gamma < 1, t_o >= 0, t_u >= 0");
  std::vector<Model> Ms(n);
  std::vector<int64_t> lo(n), cap(n);
  int64_t sum_lo = 0, sum_cap = 0;
  for (int i = 0; i < n; ++i) {
    const cannikin_node_model& nd = nodes[i];
    if (!std::isfinite(nd.q) || !std::isfinite(nd.s) || !std::isfinite(nd.k) ||
        !std::isfinite(nd.m) || nd.q < 0 || nd.s < 0 || nd.k < 0 || nd.m < 0)
      return fail(CANNIKIN_ERR_DOMAIN, "opt_split: node %d has a negative/non-finite coefficient", i);
    Model& M = Ms[i];
    M = Model{nd.q, nd.s, nd.k, nd.m, gamma, t_o, t_u, 0, 0, 0, 0};
    M.s1 = nd.q + nd.k;
    M.c1 = (nd.s + nd.m) + t_u;
    M.s2 = nd.q + gamma * nd.k;
    M.c2 = ((nd.s + gamma * nd.m) + t_o) + t_u;
    if (!(M.s1 > 0.0) || !(M.s2 > 0.0))
      return fail(CANNIKIN_ERR_SINGULAR, "opt_split: node %d time does not grow with b", i);
    lo[i] = lo_in ? lo_in[i] : 1;
    cap[i] = cap_in ? cap_in[i] : B;
    if (lo[i] < 0 || lo[i] > cap[i])
      return fail(CANNIKIN_ERR_DOMAIN, "opt_split: node %d bounds lo=%lld cap=%lld", i,
                  (long long)lo[i], (long long)cap[i]);
    sum_lo += lo[i];
    sum_cap += std::min<int64_t>(cap[i], B);
  }
  if (sum_lo > B || sum_cap < B)
    return fail(CANNIKIN_ERR_INFEASIBLE, "opt_split: sum(lo)=%lld, sum(cap)=%lld, B=%lld",
                (long long)sum_lo, (long long)sum_cap, (long long)B);

  std::vector<double> lod(n), capd(n), b_real;
  for (int i = 0; i < n; ++i) {
    lod[i] = (double)lo[i];
    capd[i] = (double)std::min<int64_t>(cap[i], B);
  }
  solve_real(Ms, lod, capd, (double)B, b_real);

  // ---- integer split
  std::vector<int64_t> bi(n);
  if (flags & CANNIKIN_ROUND_PAPER) {
    // round the relaxed split -- largest remainder, ties to the lower index.
    int64_t s = 0;
    std::vector<double> rem(n);
    for (int i = 0; i < n; ++i) {
      bi[i] = (int64_t)std::floor(b_real[i]);
      rem[i] = b_real[i] - std::floor(b_real[i]);
      s += bi[i];
    }
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return rem[a] > rem[c]; });
    int64_t shortfall = B - s;
    for (int t = 0; shortfall > 0 && t < 4 * n; ++t) {
      const int i = order[t % n];
      if (bi[i] < cap[i]) { ++bi[i]; --shortfall; }
    }
    for (int t = n - 1; shortfall < 0 && t >= -3 * n; --t) {
      const int i = order[((t % n) + n) % n];
      if (bi[i] > lo[i]) { --bi[i]; ++shortfall; }
    }
  } else {
    // Exact integer optimum of Eq. 7 with the canonical tie-break: the greedy that hands out
    // samples one at a time to argmin_i (f_i(b_i + 1), i).  It chooses the K = B - sum(lo)
    // smallest marginal keys; every key at b <= f_i^{-1}(T*) - 1 lies strictly below T* and there
    // are at most K keys <= T*, so the greedy may start from floor(b_real) - 1 and finish the few
    // remaining steps (O(n^2) instead of O(n B)).
    int64_t s = 0;
    for (int i = 0; i < n; ++i) {
      const double x = b_real[i];
      double g = std::floor(x - 1e-9 * std::max(1.0, std::fabs(x))) - 1.0;
      int64_t v = (g <= (double)lo[i]) ? lo[i] : (int64_t)g;
      if (v > cap[i]) v = cap[i];
      bi[i] = v;
      s += v;
    }
    if (s > B) {
      for (int i = 0; i < n; ++i) bi[i] = lo[i];
      s = sum_lo;
    }
    for (int64_t step = s; step < B; ++step) {
      int best = -1;
      double best_t = 0.0;
      for (int i = 0; i < n; ++i) {
        if (bi[i] >= cap[i]) continue;
        const double t = frozen_time(Ms[i], (double)(bi[i] + 1));
        if (best < 0 || t < best_t) { best = i; best_t = t; }
      }
      ++bi[best];
    }
  }

  double T_real = 0.0, T_int = 0.0;
  for (int i = 0; i < n; ++i) {
    const double tr = frozen_time(Ms[i], b_real[i]);
    const double ti = frozen_time(Ms[i], (double)bi[i]);
    if (i == 0 || tr > T_real) T_real = tr;
    if (i == 0 || ti > T_int) T_int = ti;
  }
  for (int i = 0; i < n; ++i) {
    if (b_out) b_out[i] = bi[i];
    if (b_real_out) b_real_out[i] = b_real[i];
    if (label_out) label_out[i] = ((1.0 - gamma) * (Ms[i].k * b_real[i] + Ms[i].m) >= t_o) ? 1 : 0;
  }
  if (t_out) { t_out[0] = T_real; t_out[1] = T_int; }
  cannikin::clear_error();
  return CANNIKIN_OK;
}

extern "C" cannikin_status cannikin_warmup_split(const double* t_sample, int n, int64_t B,
                                                 double* b_real_out, int64_t* b_out) {
  if (!t_sample || n < 1 || B < 0) return fail(CANNIKIN_ERR_INVALID, "warmup_split: bad arguments");
  double tot = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!(t_sample[i] > 0.0) || !std::isfinite(t_sample[i]))
      return fail(CANNIKIN_ERR_DOMAIN, "warmup_split: t_sample[%d] must be > 0", i);
    tot += t_sample[i];
  }
  std::vector<double> w(n), br(n);
  double norm = 0.0;
  for (int i = 0; i < n; ++i) { w[i] = tot / t_sample[i]; norm += w[i]; }
  for (int i = 0; i < n; ++i) br[i] = w[i] / norm * (double)B;  // Eq. 8
  std::vector<int64_t> bi(n);
  std::vector<double> rem(n);
  int64_t s = 0;
  for (int i = 0; i < n; ++i) {
    bi[i] = (int64_t)std::floor(br[i]);
    rem[i] = br[i] - std::floor(br[i]);
    s += bi[i];
  }
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return rem[a] > rem[c]; });
  for (int64_t t = 0; t < B - s; ++t) ++bi[order[t % n]];
  for (int i = 0; i < n; ++i) {
    if (b_real_out) b_real_out[i] = br[i];
    if (b_out) b_out[i] = bi[i];
  }
  cannikin::clear_error();
  return CANNIKIN_OK;
}
