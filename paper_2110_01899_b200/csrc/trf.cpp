// NEXT-1 host side: the thresholds (ŝ−, ŝ+) of the ternary activation (Corollary 1, Algorithm 1 step 2,
// P:709-746).
//
// σ^ter(t) = −1·δ_{t<s−} + 1·δ_{t>s+} (Eq. (5)).  With a = s−/√τ, b = s+/√τ and φ the N(0,1) density, its
// weak-derivative Gaussian moments (Remark 2, via Stein's lemma) are
//   E[σ^ter'(√τξ)]  = (φ(a) + φ(b)) / √τ,      E[σ^ter''(√τξ)] = (aφ(a) + bφ(b)) / τ,
// so matching Theorem 1's d1 = E[σ']², d2 = E[σ'']²/4 of a target σ means solving
//   F1(a, b) = φ(a) + φ(b) − √(τ d1) = 0,     F2(a, b) = aφ(a) + bφ(b) − sign2·2τ√d2 = 0.
// (Eq. (8) as printed has other constants; reading R15.)  Feasible targets satisfy √(τ d1) ≤ 2φ(0)
// (the sign function) and |F2 target| ≤ 2φ(1).  Method: damped Newton from the symmetric solution
// (a = −b, 2φ(b) = √(τ d1), exact when d2 = 0: every odd σ), then multi-start Newton on a grid whose box is
// doubled from [−1, 1]² ("gradually enlarging the search range") if that fails.
#include <cmath>
#include <limits>

#include "../../include/rf.h"

namespace rfh {
namespace {

constexpr double kInvSqrt2Pi = 0.39894228040143267794;

inline double phi(double x) { return kInvSqrt2Pi * std::exp(-0.5 * x * x); }

struct Res {
  double f1, f2;
  double norm2() const { return f1 * f1 + f2 * f2; }
};

inline Res residual(double a, double b, double t1, double t2) {
  const double pa = phi(a), pb = phi(b);
  return {pa + pb - t1, a * pa + b * pb - t2};
}

// Damped Newton from (a, b); returns the final squared residual and updates a, b.
double newton(double& a, double& b, double t1, double t2, int iters = 100) {
  Res r = residual(a, b, t1, t2);
  for (int it = 0; it < iters && r.norm2() > 1e-32; ++it) {
    const double pa = phi(a), pb = phi(b);
    // J = [[dF1/da, dF1/db], [dF2/da, dF2/db]]
    const double j11 = -a * pa, j12 = -b * pb;
    const double j21 = pa * (1.0 - a * a), j22 = pb * (1.0 - b * b);
    const double det = j11 * j22 - j12 * j21;
    double da, db;
    if (std::fabs(det) > 1e-300) {
      da = (-r.f1 * j22 + r.f2 * j12) / det;
      db = (-r.f2 * j11 + r.f1 * j21) / det;
    } else {   // singular (e.g. a = b = 0 or a = −b with d2 target): gradient step on ½|F|²
      da = -(j11 * r.f1 + j21 * r.f2);
      db = -(j12 * r.f1 + j22 * r.f2);
    }
    double step = 1.0;
    bool moved = false;
    for (int ls = 0; ls < 60; ++ls, step *= 0.5) {
      const double na = a + step * da, nb = b + step * db;
      const Res nr = residual(na, nb, t1, t2);
      if (nr.norm2() < r.norm2()) {
        a = na;
        b = nb;
        r = nr;
        moved = true;
        break;
      }
    }
    if (!moved) break;
  }
  return r.norm2();
}

}  // namespace

// Returns 0 on success, 1 if the target is infeasible / not found.
int solve_ternary_thresholds(double d1, double d2, double tau, int sign2, double* s_minus, double* s_plus,
                             double* resid_out) {
  const double st = std::sqrt(tau);
  const double t1 = std::sqrt(tau * d1);
  const double t2 = (sign2 < 0 ? -2.0 : 2.0) * tau * std::sqrt(d2 > 0 ? d2 : 0.0);
  if (resid_out) *resid_out = std::numeric_limits<double>::infinity();
  if (t1 > 2.0 * phi(0.0) * (1.0 + 1e-15)) return 1;
  if (std::fabs(t2) > 2.0 * phi(1.0) * (1.0 + 1e-15)) return 1;
  double best = std::numeric_limits<double>::infinity(), ba = 0, bb = 0;
  auto consider = [&](double a, double b) {
    const double f = newton(a, b, t1, t2);
    if (f < best) {
      best = f;
      ba = a;
      bb = b;
    }
  };
  {   // symmetric start: 2φ(b) = t1
    const double q = t1 / (2.0 * phi(0.0));
    const double b0 = q >= 1.0 ? 0.0 : std::sqrt(-2.0 * std::log(q));
    consider(-b0, b0);
  }
  for (double R = 1.0; best > 1e-28 && R <= 64.0; R *= 2.0) {
    const int G = 8;
    for (int i = 0; i <= G && best > 1e-28; ++i)
      for (int j = i; j <= G && best > 1e-28; ++j) consider(-R + 2.0 * R * i / G, -R + 2.0 * R * j / G);
  }
  if (resid_out) *resid_out = std::sqrt(best);
  if (!(best <= 1e-24)) return 1;
  *s_minus = std::fmin(ba, bb) * st;
  *s_plus = std::fmax(ba, bb) * st;
  return 0;
}

}  // namespace rfh
