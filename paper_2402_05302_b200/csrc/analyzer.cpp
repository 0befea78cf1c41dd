// OptPerf analyzer: the measured-model loop around cannikin_opt_split.
//
//   parameter learning      PAPER.md §4.5: per node, fit a_i = q_i b + s_i and
//                           P_i = k_i b + m_i (Eq. 3) from >= 2 distinct local batch sizes (least
//                           squares; exact for two points)
//   overlap ratio           Eq. 12: inverse-variance weighting of the nodes' gamma_i
//   communication time      P:406: T = min_i T_i (the slowest node does not wait), for T_o and T_u
//   warm-up                 Eq. 8 P:317-324 (epoch 1), even split at epoch 0
//   plan                    epoch >= 2: OptPerf split from the learned models (cannikin_opt_split)
// Host-only, pure C++, -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "common.h"

using cannikin::fail;

extern "C" cannikin_status cannikin_fit_linear(const double* x, const double* y, int count,
                                               double* slope, double* intercept) {
  if (!x || !y || !slope || !intercept) return fail(CANNIKIN_ERR_INVALID, "fit_linear: NULL");
  if (count < 2) return fail(CANNIKIN_ERR_SINGULAR, "fit_linear: need >= 2 points");
  double mx = 0.0, my = 0.0;
  for (int i = 0; i < count; ++i) {
    if (!std::isfinite(x[i]) || !std::isfinite(y[i]))
      return fail(CANNIKIN_ERR_DOMAIN, "fit_linear: non-finite point %d", i);
    mx += x[i];
    my += y[i];
  }
  mx /= count;
  my /= count;
  double sxx = 0.0, sxy = 0.0;
  for (int i = 0; i < count; ++i) {
    sxx += (x[i] - mx) * (x[i] - mx);
    sxy += (x[i] - mx) * (y[i] - my);
  }
  if (!(sxx > 0.0)) return fail(CANNIKIN_ERR_SINGULAR, "fit_linear: all x equal");
  *slope = sxy / sxx;
  *intercept = my - *slope * mx;
  return CANNIKIN_OK;
}

extern "C" cannikin_status cannikin_ivw(const double* estimate, const double* variance, int n,
                                        double* out) {
  if (!estimate || !variance || !out || n < 1) return fail(CANNIKIN_ERR_INVALID, "ivw: bad arguments");
  // Eq. 12: sum_i (x_i / v_i) / sum_i (1 / v_i).  Nodes with v_i == 0 dominate (limit v -> 0):
  // if any exist, the result is their plain mean.  v_i < 0 or NaN -> DOMAIN.
  int nzero = 0;
  double zsum = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!(variance[i] >= 0.0) || !std::isfinite(estimate[i]))
      return fail(CANNIKIN_ERR_DOMAIN, "ivw: node %d has variance %g", i, variance[i]);
    if (variance[i] == 0.0) {
      ++nzero;
      zsum += estimate[i];
    }
  }
  if (nzero) {
    *out = zsum / nzero;
    return CANNIKIN_OK;
  }
  double num = 0.0, den = 0.0;
  for (int i = 0; i < n; ++i) {
    num += estimate[i] / variance[i];
    den += 1.0 / variance[i];
  }
  *out = num / den;
  return CANNIKIN_OK;
}

namespace {
struct Obs {
  int64_t iter, b;
  double a, P, gamma, t_o, t_u;
};
}  // namespace

struct OptPerfInitCache {
  std::vector<int64_t> cand;
  std::vector<double> T;
  std::vector<std::vector<int>> labels;
  bool valid = false;
};

struct cannikin_analyzer {
  int n = 0;
  int epoch = 0;  // number of plans issued
  std::vector<std::vector<Obs>> obs;
  OptPerfInitCache cache;
};

extern "C" cannikin_status cannikin_analyzer_create(int n, cannikin_analyzer** out) {
  if (!out || n < 1) return fail(CANNIKIN_ERR_INVALID, "analyzer_create: bad arguments");
  auto* an = new cannikin_analyzer();
  an->n = n;
  an->obs.resize(n);
  *out = an;
  return CANNIKIN_OK;
}

extern "C" cannikin_status cannikin_analyzer_destroy(cannikin_analyzer* an) {
  delete an;
  return CANNIKIN_OK;
}

extern "C" cannikin_status cannikin_analyzer_observe(cannikin_analyzer* an, int node, int64_t iter,
                                                     int64_t b, double a, double P, double gamma,
                                                     double t_o, double t_u) {
  if (!an || node < 0 || node >= an->n || b < 1)
    return fail(CANNIKIN_ERR_INVALID, "analyzer_observe: bad arguments");
  if (!(a >= 0.0) || !(P >= 0.0) || !std::isfinite(a) || !std::isfinite(P) || !std::isfinite(gamma) ||
      !std::isfinite(t_o) || !std::isfinite(t_u))
    return fail(CANNIKIN_ERR_DOMAIN, "analyzer_observe: non-finite or negative time");
  an->obs[node].push_back(Obs{iter, b, a, P, gamma, t_o, t_u});
  return CANNIKIN_OK;
}

static int distinct_b(const std::vector<Obs>& v) {
  std::vector<int64_t> bs;
  for (const Obs& o : v) bs.push_back(o.b);
  std::sort(bs.begin(), bs.end());
  return (int)(std::unique(bs.begin(), bs.end()) - bs.begin());
}

extern "C" cannikin_status cannikin_analyzer_models(cannikin_analyzer* an,
                                                    cannikin_node_model* nodes,
                                                    cannikin_comm_model* cm) {
  if (!an || !nodes || !cm) return fail(CANNIKIN_ERR_INVALID, "analyzer_models: NULL");
  const int n = an->n;
  std::vector<double> gmean(n), gvar(n);
  std::vector<double> to_i(n), tu_i(n);
  int with_var = 0;
  for (int i = 0; i < n; ++i) {
    const auto& v = an->obs[i];
    if (distinct_b(v) < 2)
      return fail(CANNIKIN_ERR_SINGULAR, "analyzer_models: node %d has < 2 distinct batch sizes", i);
    std::vector<double> x, ya, yp;
    double gs = 0.0, to = 0.0, tu = 0.0;
    for (const Obs& o : v) {
      x.push_back((double)o.b);
      ya.push_back(o.a);
      yp.push_back(o.P);
      gs += o.gamma;
      to += o.t_o;
      tu += o.t_u;
    }
    double q, s, k, m;
    cannikin_status st = cannikin_fit_linear(x.data(), ya.data(), (int)x.size(), &q, &s);
    if (st != CANNIKIN_OK) return st;
    st = cannikin_fit_linear(x.data(), yp.data(), (int)x.size(), &k, &m);
    if (st != CANNIKIN_OK) return st;
    // measurement noise can push a fitted coefficient below zero: the model's domain is >= 0
    // (Eq. 3 times are nonnegative and grow with b), so clamp (reading Q23)
    const double tiny = 1e-12;
    nodes[i] = cannikin_node_model{q > tiny ? q : tiny, s > 0.0 ? s : 0.0, k > tiny ? k : tiny,
                                   m > 0.0 ? m : 0.0};
    const double cnt = (double)v.size();
    gmean[i] = gs / cnt;
    to_i[i] = to / cnt;
    tu_i[i] = tu / cnt;
    if (v.size() >= 2) {
      double ss = 0.0;
      for (const Obs& o : v) ss += (o.gamma - gmean[i]) * (o.gamma - gmean[i]);
      gvar[i] = ss / (cnt - 1.0);  // sample variance of node i's gamma observations (Eq. 12)
      ++with_var;
    } else {
      gvar[i] = -1.0;
    }
  }
  // Eq. 12 over the nodes with a sample variance; T = min_i T_i
  std::vector<double> ge, gv;
  for (int i = 0; i < n; ++i)
    if (gvar[i] >= 0.0) {
      ge.push_back(gmean[i]);
      gv.push_back(gvar[i]);
    }
  double gamma;
  if (ge.empty()) {
    gamma = 0.0;
    for (int i = 0; i < n; ++i) gamma += gmean[i];
    gamma /= n;
  } else {
    cannikin_status st = cannikin_ivw(ge.data(), gv.data(), (int)ge.size(), &gamma);
    if (st != CANNIKIN_OK) return st;
  }
  gamma = std::min(std::max(gamma, 0.0), 0.999999);
  // per iteration T = min_i T_i (the slowest node did not wait); averaged over the
  // iterations every node reported.  Without a complete iteration: min over the node means.
  double t_o = 0.0, t_u = 0.0;
  {
    std::vector<int64_t> iters;
    for (const Obs& o : an->obs[0]) iters.push_back(o.iter);
    std::sort(iters.begin(), iters.end());
    iters.erase(std::unique(iters.begin(), iters.end()), iters.end());
    int complete = 0;
    for (int64_t it : iters) {
      double mo = INFINITY, mu = INFINITY;
      bool all = true;
      for (int i = 0; i < n && all; ++i) {
        bool found = false;
        for (const Obs& o : an->obs[i])
          if (o.iter == it) {
            mo = std::min(mo, o.t_o);
            mu = std::min(mu, o.t_u);
            found = true;
          }
        all = found;
      }
      if (all) {
        t_o += mo;
        t_u += mu;
        ++complete;
      }
    }
    if (complete) {
      t_o /= complete;
      t_u /= complete;
    } else {
      t_o = to_i[0];
      t_u = tu_i[0];
      for (int i = 1; i < n; ++i) {
        t_o = std::min(t_o, to_i[i]);
        t_u = std::min(t_u, tu_i[i]);
      }
    }
  }
  *cm = cannikin_comm_model{gamma, std::max(t_o, 0.0), std::max(t_u, 0.0)};
  return CANNIKIN_OK;
}

extern "C" cannikin_status cannikin_analyzer_plan(cannikin_analyzer* an, int64_t B,
                                                  const int64_t* cap, int64_t* b_out,
                                                  double* t_pred, int* phase_out) {
  if (!an || !b_out || B < an->n) return fail(CANNIKIN_ERR_INVALID, "analyzer_plan: bad arguments");
  const int n = an->n;
  bool have_obs = true, have_models = true;
  for (int i = 0; i < n; ++i) {
    if (an->obs[i].empty()) have_obs = false;
    if (distinct_b(an->obs[i]) < 2) have_models = false;
  }
  int phase;
  double pred = std::nan("");
  if (have_models) {
    // epoch >= 2: OptPerf from the learned models
    std::vector<cannikin_node_model> nodes(n);
    cannikin_comm_model cm;
    cannikin_status st = cannikin_analyzer_models(an, nodes.data(), &cm);
    if (st != CANNIKIN_OK) return st;
    double t[2];
    st = cannikin_opt_split(nodes.data(), n, &cm, B, nullptr, cap, 0, b_out, nullptr, t, nullptr);
    if (st != CANNIKIN_OK) return st;
    pred = t[1];
    phase = 2;
  } else if (have_obs) {
    // Eq. 8 from each node's per-sample compute time at its latest batch size
    std::vector<double> ts(n);
    for (int i = 0; i < n; ++i) {
      const int64_t bl = an->obs[i].back().b;
      double sum = 0.0;
      int cnt = 0;
      for (const Obs& o : an->obs[i])
        if (o.b == bl) {
          sum += (o.a + o.P) / (double)o.b;
          ++cnt;
        }
      ts[i] = sum / cnt;
    }
    cannikin_status st = cannikin_warmup_split(ts.data(), n, B, nullptr, b_out);
    if (st != CANNIKIN_OK) return st;
    for (int i = 0; i < n; ++i) if (b_out[i] < 1) b_out[i] = 1;  // every node keeps a sample
    int64_t s = 0;
    for (int i = 0; i < n; ++i) s += b_out[i];
    for (int i = 0; s > B && i < 4 * n; ++i)  // give back what the floor of 1 added
      if (b_out[i % n] > 1) { --b_out[i % n]; --s; }
    phase = 1;
  } else {
    // epoch 0: even split, the extra samples to the lowest ranks
    for (int i = 0; i < n; ++i) b_out[i] = B / n + (i < B % n ? 1 : 0);
    phase = 0;
  }
  if (cap && phase < 2) {  // respect per-node caps: move the excess to nodes with room
    int64_t excess = 0;
    for (int i = 0; i < n; ++i)
      if (b_out[i] > cap[i]) { excess += b_out[i] - cap[i]; b_out[i] = cap[i]; }
    for (int i = 0; excess > 0 && i < n; ++i) {
      const int64_t room = cap[i] - b_out[i];
      const int64_t give = room < excess ? room : excess;
      b_out[i] += give;
      excess -= give;
    }
    if (excess > 0) return fail(CANNIKIN_ERR_INFEASIBLE, "analyzer_plan: caps below B");
  }
  an->epoch++;
  if (t_pred) *t_pred = pred;
  if (phase_out) *phase_out = phase;
  return CANNIKIN_OK;
}

// ============================================================================================
// Adaptive total batch size: goodput = throughput x statistical efficiency
// (Pollux), B_noise from the heterogeneous GNS smoothed by an EMA of G and S
// separately (the ratio estimator is biased), OptPerf_init cache per candidate.
// ============================================================================================

extern "C" cannikin_status cannikin_gns_ema_update(cannikin_gns_ema* ema, double G2, double trS) {
  if (!ema || !(ema->decay >= 0.0) || !(ema->decay < 1.0))
    return fail(CANNIKIN_ERR_INVALID, "gns_ema_update: decay must be in [0, 1)");
  if (!std::isfinite(G2) || !std::isfinite(trS)) return fail(CANNIKIN_ERR_DOMAIN, "gns_ema_update: non-finite");
  if (G2 > 0.0) {  // a non-positive G snapshot is left out (reading Q26)
    if (ema->count == 0) {
      ema->G2 = G2;
      ema->trS = trS;
    } else {
      ema->G2 = ema->decay * ema->G2 + (1.0 - ema->decay) * G2;
      ema->trS = ema->decay * ema->trS + (1.0 - ema->decay) * trS;
    }
    ema->count++;
  }
  // B_noise = S / G of the averages
  ema->B_noise = ema->count ? ema->trS / ema->G2 : std::numeric_limits<double>::quiet_NaN();
  return CANNIKIN_OK;
}

extern "C" double cannikin_efficiency(int64_t B, int64_t B0, double B_noise) {
  // Pollux's statistical efficiency relative to the initial batch B0 (reading Q27)
  return (B_noise + (double)B0) / (B_noise + (double)B);
}

extern "C" cannikin_status cannikin_choose_batch(const cannikin_node_model* nodes, int n,
                                                 const cannikin_comm_model* cm,
                                                 const int64_t* candidates, int n_cand, int64_t B0,
                                                 double B_noise, int64_t* B_out,
                                                 double* T_out, double* goodput_out) {
  if (!nodes || !cm || !candidates || n_cand < 1 || !B_out || B0 < 1 || !(B_noise >= 0.0))
    return fail(CANNIKIN_ERR_INVALID, "choose_batch: bad arguments");
  double best = -1.0;
  std::vector<int64_t> b(n);
  for (int c = 0; c < n_cand; ++c) {
    double t[2];
    cannikin_status st =
        cannikin_opt_split(nodes, n, cm, candidates[c], nullptr, nullptr, 0, b.data(), nullptr, t,
                           nullptr);
    if (st != CANNIKIN_OK) return st;
    const double g = (double)candidates[c] / t[1] * cannikin_efficiency(candidates[c], B0, B_noise);
    if (T_out) T_out[c] = t[1];
    if (goodput_out) goodput_out[c] = g;
    if (g > best) {  // ties: the first (smallest) candidate
      best = g;
      *B_out = candidates[c];
    }
  }
  return CANNIKIN_OK;
}

extern "C" cannikin_status cannikin_analyzer_choose_batch(cannikin_analyzer* an,
                                                          const int64_t* candidates, int n_cand,
                                                          int64_t B0, double B_noise,
                                                          int64_t* B_out, int64_t* b_out,
                                                          double* t_pred, int* full_recompute) {
  if (!an || !candidates || n_cand < 1 || !B_out || !b_out)
    return fail(CANNIKIN_ERR_INVALID, "analyzer_choose_batch: bad arguments");
  const int n = an->n;
  std::vector<cannikin_node_model> nodes(n);
  cannikin_comm_model cm;
  cannikin_status st = cannikin_analyzer_models(an, nodes.data(), &cm);
  if (st != CANNIKIN_OK) return st;
  auto& C = an->cache;
  bool same_cands = C.valid && (int)C.cand.size() == n_cand;
  for (int c = 0; same_cands && c < n_cand; ++c) same_cands = C.cand[c] == candidates[c];
  std::vector<int64_t> bb(n);
  std::vector<int> lab(n);
  auto solve = [&](int c, double* T, std::vector<int>* labels) -> cannikin_status {
    double t[2];
    cannikin_status s2 = cannikin_opt_split(nodes.data(), n, &cm, candidates[c], nullptr, nullptr,
                                            0, bb.data(), nullptr, t, lab.data());
    if (s2 != CANNIKIN_OK) return s2;
    *T = t[1];
    if (labels) *labels = lab;
    return CANNIKIN_OK;
  };
  int recompute = 0;
  if (!same_cands) {  // OptPerf_init for every candidate
    C.cand.assign(candidates, candidates + n_cand);
    C.T.assign(n_cand, 0.0);
    C.labels.assign(n_cand, std::vector<int>(n));
    for (int c = 0; c < n_cand; ++c)
      if ((st = solve(c, &C.T[c], &C.labels[c])) != CANNIKIN_OK) return st;
    C.valid = true;
    recompute = 1;
  }
  for (int round = 0; round < 2; ++round) {
    int best = 0;
    double bestg = -1.0;
    for (int c = 0; c < n_cand; ++c) {
      const double g = (double)candidates[c] / C.T[c] * cannikin_efficiency(candidates[c], B0, B_noise);
      if (g > bestg) { bestg = g; best = c; }
    }
    // OptPerf of the chosen candidate from the updated models
    double T;
    std::vector<int> labels;
    if ((st = solve(best, &T, &labels)) != CANNIKIN_OK) return st;
    if (labels != C.labels[best] && round == 0) {
      // overlap pattern changed: start over for every candidate
      for (int c = 0; c < n_cand; ++c)
        if ((st = solve(c, &C.T[c], &C.labels[c])) != CANNIKIN_OK) return st;
      recompute = 1;
      continue;
    }
    C.T[best] = T;  // update OptPerf_init for this candidate
    C.labels[best] = labels;
    *B_out = candidates[best];
    for (int i = 0; i < n; ++i) b_out[i] = bb[i];
    if (t_pred) *t_pred = T;
    break;
  }
  if (full_recompute) *full_recompute = recompute;
  return CANNIKIN_OK;
}

// One host control step (the host half of a training step, replicated on every rank): the GNS
// estimate from the step's norm statistics, the EMA update, and the split for the next step.
extern "C" cannikin_status cannikin_control_step(const double* stats, const int64_t* b, int n,
                                                 cannikin_gns_ema* ema,
                                                 const cannikin_node_model* nodes,
                                                 const cannikin_comm_model* cm, int64_t B_next,
                                                 cannikin_gns_result* gns_out, int64_t* b_next,
                                                 double* t_next) {
  if (!stats || !b || !gns_out) return fail(CANNIKIN_ERR_INVALID, "control_step: NULL argument");
  cannikin_status st = CANNIKIN_OK;
  if (n >= 2) {
    st = cannikin_gns_estimate(stats, stats[n], b, n, gns_out);
    if (st != CANNIKIN_OK) return st;
    if (ema) {
      st = cannikin_gns_ema_update(ema, gns_out->G2, gns_out->trS);
      if (st != CANNIKIN_OK) return st;
    }
  }
  if (nodes && cm && b_next) {
    double t[2];
    st = cannikin_opt_split(nodes, n, cm, B_next, nullptr, nullptr, 0, b_next, nullptr, t, nullptr);
    if (st != CANNIKIN_OK) return st;
    if (t_next) *t_next = t[1];
  }
  return CANNIKIN_OK;
}
