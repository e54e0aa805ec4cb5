// Φ2 — Gaussian moments at τ by Gauss–Hermite quadrature (host, fp64).
//   ⟨k,d⟩ = E[(√τ ξ)^k σ^(d)(√τ ξ)], ξ ~ N(0,1)  — the coefficients of EQ1; the paper says
//   which expectations are needed (draft P:193) but no method; the north star names Gauss–Hermite.
//   d0, d1, d2 as in Theorem 1.
// Nodes/weights by Golub–Welsch: the probabilists' Hermite Jacobi matrix (zero diagonal, off-diagonal
// √k) is diagonalised by implicit-shift QL; nodes = eigenvalues, weights = squared first components of
// the normalised eigenvectors (they sum to 1 for the N(0,1) density).
#include <map>
#include <mutex>
#include <cmath>
#include <cstring>
#include <vector>
#include <algorithm>

#include "../../include/rf.h"

namespace rfh {

// Implicit QL with Wilkinson-type shifts on a symmetric tridiagonal matrix (diag d, sub-diagonal e,
// e[n-1] unused); z carries the first row of the accumulated orthogonal transform.
static bool tridiag_ql_first_row(std::vector<double>& d, std::vector<double>& e, std::vector<double>& z) {
  const int n = (int)d.size();
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    for (;;) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1.1e-16 * dd) break;
      }
      if (m == l) break;
      if (++iter > 200) return false;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      int i = m - 1;
      bool deflated = false;
      for (; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[m] = 0.0;
          deflated = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        f = z[i + 1];
        z[i + 1] = s * z[i] + c * f;
        z[i] = c * z[i] - s * f;
      }
      if (deflated) continue;
      d[l] -= p;
      e[l] = g;
      e[m] = 0.0;
    }
  }
  return true;
}

static bool gauss_hermite_compute(int N, std::vector<double>& x, std::vector<double>& w) {
  std::vector<double> d(N, 0.0), e(N, 0.0), z(N, 0.0);
  for (int k = 0; k < N - 1; ++k) e[k] = std::sqrt((double)(k + 1));
  z[0] = 1.0;
  if (!tridiag_ql_first_row(d, e, z)) return false;
  std::vector<int> idx(N);
  for (int i = 0; i < N; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
  x.resize(N);
  w.resize(N);
  for (int i = 0; i < N; ++i) {
    x[i] = d[idx[i]];
    w[i] = z[idx[i]] * z[idx[i]];
  }
  // exact symmetry of the rule
  for (int i = 0; i < N / 2; ++i) {
    const double xs = 0.5 * (x[N - 1 - i] - x[i]);
    const double ws = 0.5 * (w[N - 1 - i] + w[i]);
    x[i] = -xs; x[N - 1 - i] = xs;
    w[i] = ws; w[N - 1 - i] = ws;
  }
  if (N & 1) x[N / 2] = 0.0;
  return true;
}

// The rules depend on N only: computed once per N (Golub–Welsch at N = 512 costs ≈ 10 ms) and cached.
static bool cached_rule(std::map<int, std::pair<std::vector<double>, std::vector<double>>>& cache, std::mutex& mu,
                        bool (*compute)(int, std::vector<double>&, std::vector<double>&), int N,
                        std::vector<double>& x, std::vector<double>& w) {
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(N);
    if (it != cache.end()) {
      x = it->second.first;
      w = it->second.second;
      return true;
    }
  }
  if (!compute(N, x, w)) return false;
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(N, std::make_pair(x, w));
  return true;
}

bool gauss_hermite(int N, std::vector<double>& x, std::vector<double>& w) {
  static std::map<int, std::pair<std::vector<double>, std::vector<double>>> cache;
  static std::mutex mu;
  return cached_rule(cache, mu, gauss_hermite_compute, N, x, w);
}

// σ, σ', σ'' of the north-star activations (analytic; sigmoid − ½ = ½ tanh(t/2)).
static inline void act_derivs(rf_act act, double t, double f[3]) {
  switch (act) {
    case RF_ACT_TANH: {
      const double th = std::tanh(t);
      f[0] = th;
      f[1] = 1.0 - th * th;
      f[2] = -2.0 * th * (1.0 - th * th);
      break;
    }
    case RF_ACT_ERF: {
      const double g = 1.1283791670955126 * std::exp(-t * t);   // 2/√π e^{−t²}
      f[0] = std::erf(t);
      f[1] = g;
      f[2] = -2.0 * t * g;
      break;
    }
    default: {
      const double th = std::tanh(0.5 * t);
      f[0] = 0.5 * th;
      f[1] = 0.25 * (1.0 - th * th);
      f[2] = -0.25 * th * (1.0 - th * th);
      break;
    }
  }
}

// table[0..14] = kd[k][d] (k-major), table[15] = E[σ²].  Returns false on a non-finite value.
static bool quad_table(rf_act act, double tau, const std::vector<double>& x, const std::vector<double>& w,
                       double table[16]) {
  std::memset(table, 0, 16 * sizeof(double));
  const double st = std::sqrt(tau);
  for (size_t q = 0; q < x.size(); ++q) {
    const double t = st * x[q];
    double f[3];
    act_derivs(act, t, f);
    if (!std::isfinite(f[0]) || !std::isfinite(f[1]) || !std::isfinite(f[2])) return false;
    double tk = w[q];
    for (int k = 0; k < 5; ++k) {
      for (int dd = 0; dd < 3; ++dd) table[k * 3 + dd] += tk * f[dd];
      tk *= t;
    }
    table[15] += w[q] * f[0] * f[0];
  }
  return true;
}

static bool trapezoid_table(rf_act act, double tau, double h, double table[16]) {
  const double L = 40.0;
  const int npts = (int)std::lround(2 * L / h) + 1;
  std::vector<double> x(npts), w(npts);
  for (int i = 0; i < npts; ++i) {
    x[i] = -L + h * i;
    w[i] = h * std::exp(-0.5 * x[i] * x[i]) * 0.3989422804014327;   // h·φ(x)
  }
  return quad_table(act, tau, x, w, table);
}

static void fill(const double table[16], double tau, rf_moments_t* out) {
  out->tau = tau;
  for (int k = 0; k < 5; ++k)
    for (int dd = 0; dd < 3; ++dd) out->kd[k][dd] = table[k * 3 + dd];
  out->e_sigma_sq = table[15];
  out->d0 = table[15] - table[0] * table[0] - tau * table[1] * table[1];
  out->d1 = table[1] * table[1];
  out->d2 = 0.25 * table[2] * table[2];
}

// ---------------------------------------------------------------------------------------------
// Parametrised Table-2 rows, registered at run time: ids RF_ACT_PARAM_BASE + k.  Entries are
// immutable once registered; the same coefficients give the same id.
struct ParamAct {
  int kind;        // 1: a₊max(0,t) + a₋max(0,−t) (a[0] = a₊, a[1] = a₋); 2: a₂t² + a₁t + a₀ (a[0..2] = a₀, a₁, a₂)
  double a[3];
};
static std::mutex g_param_mu;
static ParamAct g_param[RF_ACT_PARAM_MAX];
static int g_nparam = 0;

int register_param_act(int kind, const double a[3]) {
  std::lock_guard<std::mutex> lk(g_param_mu);
  for (int k = 0; k < g_nparam; ++k)
    if (g_param[k].kind == kind && g_param[k].a[0] == a[0] && g_param[k].a[1] == a[1] && g_param[k].a[2] == a[2])
      return RF_ACT_PARAM_BASE + k;
  if (g_nparam >= RF_ACT_PARAM_MAX) return -1;
  g_param[g_nparam] = ParamAct{kind, {a[0], a[1], a[2]}};
  return RF_ACT_PARAM_BASE + g_nparam++;
}
bool param_act(int id, int* kind, double a[3]) {
  const int k = id - RF_ACT_PARAM_BASE;
  std::lock_guard<std::mutex> lk(g_param_mu);
  if (k < 0 || k >= g_nparam) return false;
  *kind = g_param[k].kind;
  for (int i = 0; i < 3; ++i) a[i] = g_param[k].a[i];
  return true;
}

// NEXT-3 (Table-2 activations, weak derivatives by Stein): σ only.
static inline double act_value(rf_act act, double t) {
  int kind;
  double a[3];
  if ((int)act >= RF_ACT_PARAM_BASE && rfh::param_act((int)act, &kind, a))
    return kind == 1 ? a[0] * (t > 0.0 ? t : 0.0) + a[1] * (t < 0.0 ? -t : 0.0) : (a[2] * t + a[1]) * t + a[0];
  switch (act) {
    case RF_ACT_RELU: return t > 0.0 ? t : 0.0;
    case RF_ACT_ABS: return std::fabs(t);
    case RF_ACT_SIGN: return t > 0.0 ? 1.0 : (t < 0.0 ? -1.0 : 0.0);
    case RF_ACT_STEP: return t > 0.0 ? 1.0 : 0.0;
    case RF_ACT_COS: return std::cos(t);
    case RF_ACT_SIN: return std::sin(t);
    case RF_ACT_IDENT: return t;
    case RF_ACT_QUAD: return t * t;
    case RF_ACT_BUMP: return std::exp(-0.5 * t * t);
    default: return std::nan("");
  }
}

// Gauss–Legendre on [−1, 1] by Golub–Welsch (Jacobi matrix: zero diagonal, b_k = k/√(4k² − 1)); weights sum to 2.
static bool gauss_legendre_compute(int N, std::vector<double>& x, std::vector<double>& w) {
  std::vector<double> d(N, 0.0), e(N, 0.0), z(N, 0.0);
  for (int k = 1; k < N; ++k) e[k - 1] = k / std::sqrt(4.0 * k * k - 1.0);
  z[0] = 1.0;
  if (!tridiag_ql_first_row(d, e, z)) return false;
  x = d;
  w.resize(N);
  for (int i = 0; i < N; ++i) w[i] = 2.0 * z[i] * z[i];
  return true;
}

static bool gauss_legendre(int N, std::vector<double>& x, std::vector<double>& w) {
  static std::map<int, std::pair<std::vector<double>, std::vector<double>>> cache;
  static std::mutex mu;
  return cached_rule(cache, mu, gauss_legendre_compute, N, x, w);
}

// M_j = E[ξ^j σ(√τξ)], j = 0..6, and E[σ(√τξ)²]: composite Gauss–Legendre on [−L, 0] and [0, L] (the only kink /
// jump of these σ is at t = 0, so each half-line integrand is smooth).
static bool stein_table(rf_act act, double tau, double table[16]) {
  constexpr int kNodes = 24, kPanels = 48;
  constexpr double L = 12.0;
  std::vector<double> gx, gw;
  if (!gauss_legendre(kNodes, gx, gw)) return false;
  const double st = std::sqrt(tau), h = L / kPanels;
  double M[7] = {0, 0, 0, 0, 0, 0, 0}, S2 = 0.0;
  for (int side = -1; side <= 1; side += 2) {
    for (int pnl = 0; pnl < kPanels; ++pnl) {
      const double a = pnl * h;
      for (int q = 0; q < kNodes; ++q) {
        const double r = a + 0.5 * h * (gx[q] + 1.0);
        const double xi = side * r;
        const double wt = 0.5 * h * gw[q] * 0.3989422804014327 * std::exp(-0.5 * r * r);
        const double f = act_value(act, st * xi);
        if (!std::isfinite(f)) return false;
        double xp = wt;
        for (int j = 0; j < 7; ++j) {
          M[j] += xp * f;
          xp *= xi;
        }
        S2 += wt * f * f;
      }
    }
  }
  auto Mm = [&](int j) { return j >= 0 ? M[j] : 0.0; };
  for (int k = 0; k < 5; ++k) {
    table[k * 3 + 0] = std::pow(tau, 0.5 * k) * M[k];
    table[k * 3 + 1] = std::pow(tau, 0.5 * (k - 1)) * (M[k + 1] - k * Mm(k - 1));
    table[k * 3 + 2] = std::pow(tau, 0.5 * k - 1.0) * (M[k + 2] - (2 * k + 1) * M[k] + k * (k - 1) * Mm(k - 2));
  }
  table[15] = S2;
  return true;
}

// returns 0 ok, 1 non-finite, 2 eigen-solver failure
int compute_moments(rf_act act, double tau, int nodes, rf_moments_t* out) {
  if ((int)act >= RF_ACT_RELU) {
    double t[16];
    if (!stein_table(act, tau, t)) return 1;
    fill(t, tau, out);
    out->nodes = 2 * 48 * 24;
    out->method = 2;
    out->quad_err_est = 0.0;
    return 0;
  }
  std::vector<double> x, w;
  double cur[16], prev[16];
  if (nodes > 0) {
    if (!gauss_hermite(nodes, x, w)) return 2;
    if (!quad_table(act, tau, x, w, cur)) return 1;
    fill(cur, tau, out);
    out->nodes = nodes;
    out->method = 0;
    out->quad_err_est = 0.0;
    if (nodes >= 4) {
      std::vector<double> x2, w2;
      if (gauss_hermite(nodes / 2, x2, w2) && quad_table(act, tau, x2, w2, prev)) {
        double err = 0.0;
        for (int i = 0; i < 16; ++i) err = std::max(err, std::fabs(cur[i] - prev[i]));
        out->quad_err_est = err;
      }
    }
    return 0;
  }
  bool have_prev = false;
  for (int N = 64; N <= 512; N *= 2) {
    if (!gauss_hermite(N, x, w)) return 2;
    if (!quad_table(act, tau, x, w, cur)) return 1;
    if (have_prev) {
      double err = 0.0;
      for (int i = 0; i < 16; ++i) err = std::max(err, std::fabs(cur[i] - prev[i]));
      if (err < 1e-13) {
        fill(cur, tau, out);
        out->nodes = N;
        out->method = 0;
        out->quad_err_est = err;
        return 0;
      }
    }
    std::memcpy(prev, cur, sizeof(cur));
    have_prev = true;
  }
  // Gauss–Hermite did not converge (large τ for tanh: poles at ±iπ/(2√τ)) → composite trapezoid,
  // geometrically convergent for integrands analytic in a strip.
  double coarse[16];
  if (!trapezoid_table(act, tau, 0.05, cur)) return 1;
  if (!trapezoid_table(act, tau, 0.1, coarse)) return 1;
  double err = 0.0;
  for (int i = 0; i < 16; ++i) err = std::max(err, std::fabs(cur[i] - coarse[i]));
  fill(cur, tau, out);
  out->nodes = 1601;
  out->method = 1;
  out->quad_err_est = err;
  return 0;
}

}  // namespace rfh
