// CPU ORACLE (test infrastructure only): More-Thuente strong-Wolfe line
// search, the published MINPACK-2 dcsrch/dcstep algorithm as used by
// proj/src/linesearch.cpp:13-214 (same safeguards and constants).
#include "oracle.hpp"

#include <algorithm>
#include <tuple>

namespace oracle {

namespace {

struct End {
  double t, f, g;  // step, value, derivative
};

// Cubic-interpolation minimiser between (a.t,a.f,a.g) and (t,f,g); `flip`
// selects the root orientation.
double cubic_min(const End& a, double t, double f, double g, bool use_g_of_a_first) {
  const double theta = 3.0 * (a.f - f) / (t - a.t) + a.g + g;
  const double s = std::max({std::abs(theta), std::abs(a.g), std::abs(g)});
  double gam = s * std::sqrt((theta / s) * (theta / s) - (a.g / s) * (g / s));
  (void)use_g_of_a_first;
  return gam;  // helper only returns gamma magnitude; callers orient it
}

// One safeguarded step (dcstep). `lo` holds the best point so far (stx),
// `hi` the other bracket end (sty). Returns the new trial step.
double safeguarded_step(End& lo, End& hi, double t, double f, double g, bool& bracketed, double tmin,
                        double tmax) {
  const double sgnd = g * (lo.g / std::abs(lo.g));
  double next = t;
  if (f > lo.f) {  // case 1: higher value -> minimum bracketed
    const double theta = 3.0 * (lo.f - f) / (t - lo.t) + lo.g + g;
    double gam = cubic_min(lo, t, f, g, true);
    if (t < lo.t) gam = -gam;
    const double p = (gam - lo.g) + theta;
    const double q = ((gam - lo.g) + gam) + g;
    const double tc = lo.t + (p / q) * (t - lo.t);
    const double tq = lo.t + ((lo.g / ((lo.f - f) / (t - lo.t) + lo.g)) / 2.0) * (t - lo.t);
    next = std::abs(tc - lo.t) < std::abs(tq - lo.t) ? tc : tc + (tq - tc) / 2.0;
    bracketed = true;
  } else if (sgnd < 0.0) {  // case 2: lower value, derivatives of opposite sign
    const double theta = 3.0 * (lo.f - f) / (t - lo.t) + lo.g + g;
    double gam = cubic_min(lo, t, f, g, false);
    if (t > lo.t) gam = -gam;
    const double p = (gam - g) + theta;
    const double q = ((gam - g) + gam) + lo.g;
    const double tc = t + (p / q) * (lo.t - t);
    const double tq = t + (g / (g - lo.g)) * (lo.t - t);
    next = std::abs(tc - t) > std::abs(tq - t) ? tc : tq;
    bracketed = true;
  } else if (std::abs(g) < std::abs(lo.g)) {  // case 3: derivative magnitude decreases
    const double theta = 3.0 * (lo.f - f) / (t - lo.t) + lo.g + g;
    const double s = std::max({std::abs(theta), std::abs(lo.g), std::abs(g)});
    double gam = s * std::sqrt(std::max(0.0, (theta / s) * (theta / s) - (lo.g / s) * (g / s)));
    if (t > lo.t) gam = -gam;
    const double p = (gam - g) + theta;
    const double q = (gam + (lo.g - g)) + gam;
    const double r = p / q;
    double tc;
    if (r < 0.0 && gam != 0.0) tc = t + r * (lo.t - t);
    else tc = t > lo.t ? tmax : tmin;
    const double tq = t + (g / (g - lo.g)) * (lo.t - t);
    if (bracketed) {
      next = std::abs(tc - t) < std::abs(tq - t) ? tc : tq;
      next = t > lo.t ? std::min(t + 0.66 * (hi.t - t), next) : std::max(t + 0.66 * (hi.t - t), next);
    } else {
      next = std::abs(tc - t) > std::abs(tq - t) ? tc : tq;
      next = std::clamp(next, tmin, tmax);
    }
  } else {  // case 4: derivative magnitude does not decrease
    if (bracketed) {
      const double theta = 3.0 * (f - hi.f) / (hi.t - t) + hi.g + g;
      const double s = std::max({std::abs(theta), std::abs(hi.g), std::abs(g)});
      double gam = s * std::sqrt((theta / s) * (theta / s) - (hi.g / s) * (g / s));
      if (t > hi.t) gam = -gam;
      const double p = (gam - g) + theta;
      const double q = ((gam - g) + gam) + hi.g;
      next = t + (p / q) * (hi.t - t);
    } else {
      next = t > lo.t ? tmax : tmin;
    }
  }
  // Interval update.
  if (f > lo.f) {
    hi = {t, f, g};
  } else {
    if (sgnd < 0.0) hi = lo;
    lo = {t, f, g};
  }
  return std::clamp(next, tmin, tmax);
}

}  // namespace

LineSearchResult more_thuente_search(const std::function<std::pair<double, double>(double)>& phi, double f0,
                                     double dphi0, double initial_step, const LineSearchConfig& cfg) {
  if (!(dphi0 < 0.0)) throw std::invalid_argument("more_thuente_search: direction is not a descent direction");
  LineSearchResult res;
  const double gtest = cfg.sufficient_decrease * dphi0;
  bool bracketed = false;
  bool stage_one = true;
  double width = cfg.step_max - cfg.step_min, width_prev = 2.0 * width;
  End lo{0.0, f0, dphi0}, hi{0.0, f0, dphi0};
  double t = std::clamp(initial_step, cfg.step_min, cfg.step_max);
  double tmin = 0.0, tmax = t + 4.0 * t;
  while (res.trials < cfg.max_trials) {
    double f, g;
    std::tie(f, g) = phi(t);
    ++res.trials;
    const double ftest = f0 + t * gtest;
    if (stage_one && f <= ftest && g >= 0.0) stage_one = false;
    if (f <= ftest && std::abs(g) <= cfg.curvature * (-dphi0)) {
      res.ok = true;
      res.step = t;
      res.f = f;
      res.dphi = g;
      return res;
    }
    if ((bracketed && (t <= tmin || t >= tmax)) || (bracketed && tmax - tmin <= cfg.step_tol * tmax) ||
        (t == cfg.step_max && f <= ftest && g <= gtest) || (t == cfg.step_min && (f > ftest || g >= gtest)))
      break;
    if (stage_one && f <= lo.f && f > ftest) {
      // Modified function psi(a) = phi(a) - phi(0) - ftol a phi'(0).
      End lm{lo.t, lo.f - lo.t * gtest, lo.g - gtest}, hm{hi.t, hi.f - hi.t * gtest, hi.g - gtest};
      t = safeguarded_step(lm, hm, t, f - t * gtest, g - gtest, bracketed, tmin, tmax);
      lo = {lm.t, lm.f + lm.t * gtest, lm.g + gtest};
      hi = {hm.t, hm.f + hm.t * gtest, hm.g + gtest};
    } else {
      t = safeguarded_step(lo, hi, t, f, g, bracketed, tmin, tmax);
    }
    if (bracketed) {
      if (std::abs(hi.t - lo.t) >= 0.66 * width_prev) t = lo.t + 0.5 * (hi.t - lo.t);
      width_prev = width;
      width = std::abs(hi.t - lo.t);
      tmin = std::min(lo.t, hi.t);
      tmax = std::max(lo.t, hi.t);
    } else {
      tmin = t + 1.1 * (t - lo.t);
      tmax = t + 4.0 * (t - lo.t);
    }
    t = std::clamp(t, cfg.step_min, cfg.step_max);
    if ((bracketed && (t <= tmin || t >= tmax)) || (bracketed && tmax - tmin <= cfg.step_tol * tmax)) t = lo.t;
  }
  res.ok = false;
  res.step = lo.t;
  res.f = lo.f;
  res.dphi = lo.g;
  return res;
}

}  // namespace oracle
