// Host-side coefficient fitter of libbf.so (bf_plan_create / bf_plan_get_info).
//
// Written from the paper (PAPER.md line numbers "P:n"); independent of the Python oracle.
//   range:   truncated trigonometric basis on [-T, T] with T = D (the
//            Case 1 substitution P:1215-1217, reading Q1), best N by raw |a_k| among the first
//            M = m_factor*N, ties to the smaller k, zeros pruned.
//   spatial: 2-D Haar coefficients (eq:Haar_2D_coefficients) of the square-truncated
//            K_s on [-(r+1/2), r+1/2]^2, best N_s by |c| (ties by canonical order), lowered to
//            integer-offset boxes with half-open cells (Appendix A; Q11), then
//            factored as fx(u) fy(v) for the separable GPU path.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "bf_internal.h"

namespace {

// ------------------------------------------------------------------ Gauss-Legendre nodes
struct GL {
  double x[16], w[16];
  GL() {
    const int n = 16;
    for (int i = 0; i < n; ++i) {
      double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
      for (int it = 0; it < 100; ++it) {
        double p0 = 1.0, p1 = z;
        for (int m = 2; m <= n; ++m) {
          double p2 = ((2.0 * m - 1.0) * z * p1 - (m - 1.0) * p0) / m;
          p0 = p1;
          p1 = p2;
        }
        double dp = n * (z * p1 - p0) / (z * z - 1.0);
        double dz = p1 / dp;
        z -= dz;
        if (std::fabs(dz) < 1e-16) break;
      }
      double p0 = 1.0, p1 = z;
      for (int m = 2; m <= n; ++m) {
        double p2 = ((2.0 * m - 1.0) * z * p1 - (m - 1.0) * p0) / m;
        p0 = p1;
        p1 = p2;
      }
      double dp = n * (z * p1 - p0) / (z * z - 1.0);
      x[i] = z;
      w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
  }
};

double range_kernel(int kind, double sigma, double t) {
  if (kind == BF_RANGE_GAUSSIAN) {
    if (std::isinf(sigma)) return 1.0;
    return std::exp(-t * t / (2.0 * sigma * sigma));
  }
  double u = t / sigma;  // Tukey biweight
  if (std::fabs(u) > 1.0) return 0.0;
  double v = 1.0 - u * u;
  return v * v;
}

// a_0 = 1/(2T) int f, a_j = 1/T int f cos(pi j x/T); composite 16-point
// Gauss-Legendre, >= 2 panels per cosine period, panels split at the kernel's kinks.
void range_coefficients(int kind, double sigma, double T, int M, std::vector<double>& a) {
  static const GL gl;
  std::vector<double> cuts = {-T, T};
  if (kind == BF_RANGE_TUKEY && sigma < T) {
    cuts.push_back(-sigma);
    cuts.push_back(sigma);
  }
  std::sort(cuts.begin(), cuts.end());
  const int n_panels = 2 * M + 64;
  std::vector<double> xs, ws;
  for (size_t s = 0; s + 1 < cuts.size(); ++s) {
    double lo = cuts[s], hi = cuts[s + 1];
    int m = std::max(1, (int)std::ceil(n_panels * (hi - lo) / (2.0 * T)));
    for (int p = 0; p < m; ++p) {
      double e0 = lo + (hi - lo) * p / m, e1 = lo + (hi - lo) * (p + 1) / m;
      double h = 0.5 * (e1 - e0), c = 0.5 * (e0 + e1);
      for (int i = 0; i < 16; ++i) {
        xs.push_back(c + h * gl.x[i]);
        ws.push_back(h * gl.w[i] * range_kernel(kind, sigma, c + h * gl.x[i]));
      }
    }
  }
  a.assign(M, 0.0);
  for (int j = 0; j < M; ++j) {
    double s = 0.0;
    const double om = M_PI * j / T;
    for (size_t i = 0; i < xs.size(); ++i) s += ws[i] * std::cos(om * xs[i]);
    a[j] = (j == 0) ? s / (2.0 * T) : s / T;
  }
}

// Best N-term selection: indices of the N largest |c| among candidates given in
// canonical order; |c| equal within 1e-12 relative -> smaller index; |c| <= 1e-14 max pruned.
std::vector<int> select_best(const std::vector<double>& c, int N) {
  double cmax = 0.0;
  for (double v : c) cmax = std::max(cmax, std::fabs(v));
  std::vector<int> alive;
  if (cmax == 0.0) return alive;
  for (int i = 0; i < (int)c.size(); ++i)
    if (std::fabs(c[i]) > 1e-14 * cmax) alive.push_back(i);
  if ((int)alive.size() <= N) return alive;
  std::vector<int> order = alive;
  std::stable_sort(order.begin(), order.end(), [&](int p, int q) { return std::fabs(c[p]) > std::fabs(c[q]); });
  const double vN = std::fabs(c[order[N - 1]]);
  std::vector<int> chosen;
  for (int i : alive)
    if (std::fabs(c[i]) > vN * (1.0 + 1e-12)) chosen.push_back(i);
  for (int i : alive) {
    if ((int)chosen.size() >= N) break;
    double m = std::fabs(c[i]);
    if (m >= vN * (1.0 - 1e-12) && m <= vN * (1.0 + 1e-12)) chosen.push_back(i);
  }
  std::sort(chosen.begin(), chosen.end());
  return chosen;
}

// ------------------------------------------------------------------ Haar functions
struct Haar1 {
  int j, k;  // j = -1 : scaling function phi; otherwise psi_{j,k}
};

// Canonical 1-D order: phi, psi_{0,0}, then psi_{j,k} by (j, k), k in K_j.
std::vector<Haar1> haar_index(int J) {
  std::vector<Haar1> v = {{-1, 0}, {0, 0}};
  for (int j = 1; j <= J; ++j) {
    int h = 1 << (j - 1);
    for (int k = -h; k <= h; ++k)
      if (k != 0) v.push_back({j, k});
  }
  return v;
}

struct Cell {
  double lo, hi, sign;
};

// phi = +1 on [-T, T]; psi_{j,k} = +1 on [2^-j(Z-T), 2^-j Z), -1 on [2^-j Z, 2^-j(Z+T)],
// Z = sign(k)(2|k|-1)T (eq:Haar_set P:285, Appendix A).
int haar_cells(const Haar1& h, double T, Cell out[2]) {
  if (h.j < 0) {
    out[0] = {-T, T, 1.0};
    return 1;
  }
  double Z = (h.k == 0) ? 0.0 : std::copysign((2.0 * std::abs(h.k) - 1.0) * T, (double)h.k);
  double s = std::ldexp(1.0, -h.j);
  out[0] = {s * (Z - T), s * Z, 1.0};
  out[1] = {s * Z, s * (Z + T), -1.0};
  return 2;
}

// int_lo^hi g for the 1-D factor of K_s on the square: Gaussian (erf) or box.
double factor_integral(int kind, double sigma, double lo, double hi) {
  if (kind == BF_SPATIAL_BOX) return hi - lo;
  const double c = sigma * std::sqrt(2.0);
  return sigma * std::sqrt(M_PI / 2.0) * (std::erf(hi / c) - std::erf(lo / c));
}

// 1-D coefficients c_0 = 1/(2T) int g phi, c_{jk} = 2^j/(2T) int g psi_{jk}.
double haar_coef(int kind, double sigma, double T, const Haar1& h) {
  Cell cs[2];
  int n = haar_cells(h, T, cs);
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += cs[i].sign * factor_integral(kind, sigma, cs[i].lo, cs[i].hi);
  double norm = (h.j < 0) ? 1.0 : std::ldexp(1.0, h.j);
  return norm * s / (2.0 * T);
}

// Integer offsets u with lo <= u < hi (half-open pixel cells, Q11).
void discretize(double lo, double hi, int& a, int& b) {
  a = (int)std::ceil(lo);
  b = (int)std::ceil(hi) - 1;
}

// Values of the Haar function on the integer offsets -r..r (index u + r).
void haar_values(const Haar1& h, double T, int r, std::vector<double>& v) {
  v.assign(2 * r + 1, 0.0);
  Cell cs[2];
  int n = haar_cells(h, T, cs);
  for (int i = 0; i < n; ++i) {
    int a, b;
    discretize(cs[i].lo, cs[i].hi, a, b);
    for (int u = std::max(a, -r); u <= std::min(b, r); ++u) v[u + r] += cs[i].sign;
  }
}

// Decompose a step function f on offsets -r..r into at most BF_MAX_AXIS_BOXES boxes
// sum_i w_i [lo_i, hi_i]: nested symmetric boxes when f is even, else its constant pieces.
bool step_to_boxes(const std::vector<double>& f, int r, int& nb, int lo[], int hi[], double w[]) {
  const int n = 2 * r + 1;
  double fmax = 0.0;
  for (double v : f) fmax = std::max(fmax, std::fabs(v));
  const double tol = 1e-13 * (fmax > 0 ? fmax : 1.0);
  bool sym = true;
  for (int i = 0; i < n; ++i)
    if (std::fabs(f[i] - f[n - 1 - i]) > tol) sym = false;
  nb = 0;
  if (sym) {
    // levels from the outside in: f(u) = sum over nested boxes [-e, e] of (value jumps)
    double prev = 0.0;
    for (int e = r; e >= 0; --e) {
      double v = f[e + r];
      if (std::fabs(v - prev) > tol) {
        if (nb >= BF_MAX_AXIS_BOXES) return false;
        lo[nb] = -e;
        hi[nb] = e;
        w[nb] = v - prev;
        ++nb;
        prev = v;
      }
    }
    return nb > 0;
  }
  int start = 0;
  for (int i = 1; i <= n; ++i) {
    if (i == n || std::fabs(f[i] - f[start]) > tol) {
      if (std::fabs(f[start]) > tol) {
        if (nb >= BF_MAX_AXIS_BOXES) return false;
        lo[nb] = start - r;
        hi[nb] = i - 1 - r;
        w[nb] = f[start];
        ++nb;
      }
      start = i;
    }
  }
  return nb > 0;
}

// Rank-2 box-pair form of a symmetric lowered kernel K (n x n, [v][u]): the elementary nested
// boxes of the x axis ([-e, e] at every edge of any row) and of the y axis, the weight matrix
// W with K(v, u) = sum_ij W_ij [|u| <= e_i][|v| <= f_j] (2-D differences of K at the box
// corners), then fx_s = [|u| <= e_s] and fy_s = sum_j W_sj [|v| <= f_j] for the (at most two)
// x boxes. Returns false if K is not of that form (checked exactly on every offset).
bool box_pair_rank2(const std::vector<double>& K, int r, bf_plan* p) {
  const int n = 2 * r + 1;
  double kmax = 0.0;
  for (double v : K) kmax = std::max(kmax, std::fabs(v));
  if (kmax == 0.0) return false;
  const double tol = 1e-12 * kmax;
  for (int v = 0; v < n; ++v)
    for (int u = 0; u < n; ++u)
      if (std::fabs(K[(size_t)v * n + u] - K[(size_t)(n - 1 - v) * n + (n - 1 - u)]) > tol ||
          std::fabs(K[(size_t)v * n + u] - K[(size_t)v * n + (n - 1 - u)]) > tol)
        return false;
  // edges e (box [-e, e]) where some row / column changes value going outwards
  std::vector<int> ex, ey;
  for (int e = r; e >= 0; --e) {
    bool cx = false, cy = false;
    for (int t = 0; t < n; ++t) {
      const double ox = (e == r) ? 0.0 : K[(size_t)t * n + (e + 1 + r)];   // value just outside, row t
      const double oy = (e == r) ? 0.0 : K[(size_t)(e + 1 + r) * n + t];
      if (std::fabs(K[(size_t)t * n + (e + r)] - ox) > tol) cx = true;
      if (std::fabs(K[(size_t)(e + r) * n + t] - oy) > tol) cy = true;
    }
    if (cx) ex.push_back(e);
    if (cy) ey.push_back(e);
  }
  const int nx = (int)ex.size(), ny = (int)ey.size();
  if (nx < 1 || ny < 1 || nx > 2 || ny > BF_MAX_AXIS_BOXES) return false;
  // M_ij = K(v = f_j, u = e_i) = sum_{i' <= i, j' <= j} W_i'j' (edges outermost first)
  std::vector<double> W((size_t)nx * ny);
  auto M = [&](int i, int j) { return (i < 0 || j < 0) ? 0.0 : K[(size_t)(ey[j] + r) * n + (ex[i] + r)]; };
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j) W[(size_t)i * ny + j] = M(i, j) - M(i - 1, j) - M(i, j - 1) + M(i - 1, j - 1);
  for (int v = -r; v <= r; ++v)
    for (int u = -r; u <= r; ++u) {
      double k = 0.0;
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j)
          if (std::abs(u) <= ex[i] && std::abs(v) <= ey[j]) k += W[(size_t)i * ny + j];
      if (std::fabs(k - K[(size_t)(v + r) * n + (u + r)]) > 1e-10 * kmax) return false;
    }
  p->ns = nx;
  for (int s = 0; s < nx; ++s) {
    p->snbx[s] = 1;
    p->slox[s][0] = -ex[s];
    p->shix[s][0] = ex[s];
    p->swx[s][0] = 1.0;
    p->snby[s] = 0;
    for (int j = 0; j < ny; ++j) {
      p->sloy[s][p->snby[s]] = -ey[j];
      p->shiy[s][p->snby[s]] = ey[j];
      p->swy[s][p->snby[s]] = W[(size_t)s * ny + j];   // zero weights kept: the states share taps
      ++p->snby[s];
    }
  }
  return true;
}

// Any step function on offsets -r..r as boxes sum_i w_i [lo_i, hi_i] (no count limit): nested
// symmetric boxes when f is even, else its constant pieces.
void step_boxes(const std::vector<double>& f, int r, std::vector<int>& lo, std::vector<int>& hi,
                std::vector<double>& w) {
  const int n = 2 * r + 1;
  double fmax = 0.0;
  for (double v : f) fmax = std::max(fmax, std::fabs(v));
  const double tol = 1e-13 * (fmax > 0 ? fmax : 1.0);
  bool sym = true;
  for (int i = 0; i < n; ++i)
    if (std::fabs(f[i] - f[n - 1 - i]) > tol) sym = false;
  lo.clear();
  hi.clear();
  w.clear();
  if (sym) {
    double prev = 0.0;
    for (int e = r; e >= 0; --e) {
      const double v = f[e + r];
      if (std::fabs(v - prev) > tol) {
        lo.push_back(-e);
        hi.push_back(e);
        w.push_back(v - prev);
        prev = v;
      }
    }
    return;
  }
  int start = 0;
  for (int i = 1; i <= n; ++i)
    if (i == n || std::fabs(f[i] - f[start]) > tol) {
      if (std::fabs(f[start]) > tol) {
        lo.push_back(start - r);
        hi.push_back(i - 1 - r);
        w.push_back(f[start]);
      }
      start = i;
    }
}

// General plans: K (n x n, [v][u]) is piecewise constant on a grid of cells (the Haar terms'
// breakpoints); its cell matrix C (rows: y cells, columns: x cells) is factored exactly as
// C = sum_s col_s row_s^T by Gaussian elimination with full pivoting (rank R <= min cells), so
// K~_s(v, u) = sum_s fx_s(u) fy_s(v) with step functions fx_s, fy_s; each becomes boxes
// (step_boxes) cut into groups of at most BF_MAX_AXIS_BOXES, one separable pass per pair of
// groups. Checked on every offset against K. Returns false if it needs more than
// BF_MAX_SP_PASSES passes.
bool general_passes(const std::vector<double>& K, int r, bf_plan* p) {
  const int n = 2 * r + 1;
  double kmax = 0.0;
  for (double v : K) kmax = std::max(kmax, std::fabs(v));
  if (kmax == 0.0) return false;
  const double tol = 1e-13 * kmax;
  std::vector<int> cx{0}, cy{0};   // first offset index of every cell
  for (int u = 1; u < n; ++u) {
    bool d = false;
    for (int v = 0; v < n && !d; ++v) d = std::fabs(K[(size_t)v * n + u] - K[(size_t)v * n + u - 1]) > tol;
    if (d) cx.push_back(u);
  }
  for (int v = 1; v < n; ++v) {
    bool d = false;
    for (int u = 0; u < n && !d; ++u) d = std::fabs(K[(size_t)v * n + u] - K[(size_t)(v - 1) * n + u]) > tol;
    if (d) cy.push_back(v);
  }
  const int nx = (int)cx.size(), ny = (int)cy.size();
  std::vector<double> C((size_t)ny * nx);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) C[(size_t)j * nx + i] = K[(size_t)cy[j] * n + cx[i]];
  std::vector<std::vector<double>> cols, rows;   // per rank term: y-cell values, x-cell values
  for (int it = 0; it < std::min(nx, ny); ++it) {
    int bj = 0, bi = 0;
    double best = 0.0;
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        if (std::fabs(C[(size_t)j * nx + i]) > best) {
          best = std::fabs(C[(size_t)j * nx + i]);
          bj = j;
          bi = i;
        }
    if (best <= 1e-12 * kmax) break;
    const double piv = C[(size_t)bj * nx + bi];
    std::vector<double> col(ny), row(nx);
    for (int j = 0; j < ny; ++j) col[j] = C[(size_t)j * nx + bi];
    for (int i = 0; i < nx; ++i) row[i] = C[(size_t)bj * nx + i] / piv;
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) C[(size_t)j * nx + i] -= col[j] * row[i];
    cols.push_back(col);
    rows.push_back(row);
  }
  p->rank = (int)cols.size();
  p->n_pass = 0;
  for (int s = 0; s < p->rank; ++s) {
    std::vector<double> fx(n), fy(n);
    for (int i = 0, c = 0; i < n; ++i) {
      while (c + 1 < nx && cx[c + 1] <= i) ++c;
      fx[i] = rows[s][c];
    }
    for (int i = 0, c = 0; i < n; ++i) {
      while (c + 1 < ny && cy[c + 1] <= i) ++c;
      fy[i] = cols[s][c];
    }
    std::vector<int> lx, hx, ly, hy;
    std::vector<double> wx, wy;
    step_boxes(fx, r, lx, hx, wx);
    step_boxes(fy, r, ly, hy, wy);
    for (size_t gx = 0; gx < lx.size(); gx += BF_MAX_AXIS_BOXES)
      for (size_t gy = 0; gy < ly.size(); gy += BF_MAX_AXIS_BOXES) {
        if (p->n_pass >= BF_MAX_SP_PASSES) return false;
        auto& P = p->pass[p->n_pass++];
        P.nbx = (int)std::min<size_t>(BF_MAX_AXIS_BOXES, lx.size() - gx);
        P.nby = (int)std::min<size_t>(BF_MAX_AXIS_BOXES, ly.size() - gy);
        for (int b = 0; b < P.nbx; ++b) {
          P.lox[b] = lx[gx + b];
          P.hix[b] = hx[gx + b];
          P.wx[b] = wx[gx + b];
        }
        for (int b = 0; b < P.nby; ++b) {
          P.loy[b] = ly[gy + b];
          P.hiy[b] = hy[gy + b];
          P.wy[b] = wy[gy + b];
        }
      }
  }
  // exact check on every offset
  for (int v = 0; v < n; ++v)
    for (int u = 0; u < n; ++u) {
      double k = 0.0;
      for (int q = 0; q < p->n_pass; ++q) {
        const auto& P = p->pass[q];
        double a = 0.0, b = 0.0;
        for (int i = 0; i < P.nbx; ++i)
          if (u - r >= P.lox[i] && u - r <= P.hix[i]) a += P.wx[i];
        for (int i = 0; i < P.nby; ++i)
          if (v - r >= P.loy[i] && v - r <= P.hiy[i]) b += P.wy[i];
        k += a * b;
      }
      if (std::fabs(k - K[(size_t)v * n + u]) > 1e-10 * kmax) return false;
    }
  return p->n_pass > 0;
}

}  // namespace

// ------------------------------------------------------------------ public entry points

extern "C" void bf_plan_options_default(bf_plan_options* opt) {
  if (!opt) return;
  opt->intensity_max = 255.0;
  opt->n_spatial_terms = 9;
  opt->input_dtype = BF_IN_F32;
  opt->m_factor = 20;
  opt->haar_levels = 4;
  opt->range_window = BF_RANGE_WINDOW_FULL;
}

extern "C" bf_status bf_plan_create(bf_plan** out, int ks, int kr, double sigma_s, double sigma_r, int radius,
                                    int n_terms, const bf_plan_options* opt_in) {
  if (!out) return BF_ERR_INVALID_ARG;
  *out = nullptr;
  bf_plan_options opt;
  bf_plan_options_default(&opt);
  if (opt_in) opt = *opt_in;
  if (ks != BF_SPATIAL_GAUSSIAN && ks != BF_SPATIAL_BOX) return BF_ERR_UNSUPPORTED;
  if (kr != BF_RANGE_GAUSSIAN && kr != BF_RANGE_TUKEY) return BF_ERR_UNSUPPORTED;
  if (opt.input_dtype != BF_IN_U8 && opt.input_dtype != BF_IN_F32) return BF_ERR_UNSUPPORTED;
  if (radius < 0 || radius > BF_MAX_RADIUS) return BF_ERR_INVALID_ARG;
  if (n_terms < 1 || n_terms > BF_MAX_TERMS) return BF_ERR_INVALID_ARG;
  if (!(sigma_r > 0.0) || (kr == BF_RANGE_TUKEY && std::isinf(sigma_r))) return BF_ERR_INVALID_ARG;
  if (ks == BF_SPATIAL_GAUSSIAN && !(sigma_s > 0.0 && std::isfinite(sigma_s))) return BF_ERR_INVALID_ARG;
  if (!(opt.intensity_max > 0.0 && std::isfinite(opt.intensity_max))) return BF_ERR_INVALID_ARG;
  if (opt.n_spatial_terms < 1 || opt.n_spatial_terms > BF_MAX_SPATIAL_TERMS) return BF_ERR_INVALID_ARG;
  if (opt.m_factor < 1 || opt.haar_levels < 0 || opt.haar_levels > 8) return BF_ERR_INVALID_ARG;
  if (opt.range_window != BF_RANGE_WINDOW_FULL && opt.range_window != BF_RANGE_WINDOW_LITERAL) return BF_ERR_INVALID_ARG;
  // literal window: T_r = K_r^{-1}(eps), eps = 0.01: Gaussian exp(-T^2/2s^2) = eps,
  // Tukey (1 - (T/s)^2)^2 = eps
  double Tr = opt.intensity_max;
  if (opt.range_window == BF_RANGE_WINDOW_LITERAL) {
    if (std::isinf(sigma_r)) return BF_ERR_INVALID_ARG;   // K_r == 1 has no truncation point
    Tr = (kr == BF_RANGE_GAUSSIAN) ? sigma_r * std::sqrt(-2.0 * std::log(0.01))
                                  : sigma_r * std::sqrt(1.0 - std::sqrt(0.01));
  }
  const int M = opt.m_factor * n_terms;
  if (M < n_terms) return BF_ERR_INVALID_ARG;

  bf_plan* p = new (std::nothrow) bf_plan();
  if (!p) return BF_ERR_NO_MEMORY;
  std::memset(p, 0, sizeof(*p));
  p->ks = ks;
  p->kr = kr;
  p->sigma_s = sigma_s;
  p->sigma_r = sigma_r;
  p->radius = radius;
  p->n_terms = n_terms;
  p->D = opt.intensity_max;
  p->T = Tr;
  p->literal = opt.range_window == BF_RANGE_WINDOW_LITERAL;
  p->input_dtype = opt.input_dtype;
  p->opt = opt;

  // ---- range fit on [-T, T] (T = D, or T_r for the literal window)
  std::vector<double> a;
  range_coefficients(kr, sigma_r, Tr, M, a);
  std::vector<int> sel = select_best(a, n_terms);
  if (sel.empty()) {
    delete p;
    return BF_ERR_NUMERIC;
  }
  p->n_k = (int)sel.size();
  for (int i = 0; i < p->n_k; ++i) {
    p->k[i] = sel[i];
    p->a[i] = a[sel[i]];
  }

  // ---- spatial fit on [-T_s, T_s]^2, T_s = r + 1/2
  const double T = radius + 0.5;
  std::vector<Haar1> idx = haar_index(opt.haar_levels);
  const int n1 = (int)idx.size();
  std::vector<double> c1(n1);
  for (int i = 0; i < n1; ++i) c1[i] = haar_coef(ks, sigma_s, T, idx[i]);
  // 2-D candidates in canonical order (family, j1, k1, j2, k2); the separable K_s makes each
  // 2-D integral the product of the two 1-D ones (P:312-318 with K_s(x,y) = g(x) g(y)).
  struct Cand {
    int fam, ia, ib;
    double c;
  };
  std::vector<Cand> cand;
  for (int ia = 0; ia < n1; ++ia)
    for (int ib = 0; ib < n1; ++ib) {
      int fam = (idx[ia].j < 0 ? 0 : 2) + (idx[ib].j < 0 ? 0 : 1);
      cand.push_back({fam, ia, ib, c1[ia] * c1[ib]});
    }
  std::stable_sort(cand.begin(), cand.end(), [](const Cand& p1, const Cand& p2) {
    if (p1.fam != p2.fam) return p1.fam < p2.fam;
    return p1.ia != p2.ia ? p1.ia < p2.ia : p1.ib < p2.ib;  // idx is already (j,k)-ordered
  });
  std::vector<double> cv(cand.size());
  for (size_t i = 0; i < cand.size(); ++i) cv[i] = cand[i].c;
  std::vector<int> ssel = select_best(cv, opt.n_spatial_terms);
  if (ssel.empty()) {
    delete p;
    return BF_ERR_NUMERIC;
  }
  p->n_sp = (int)ssel.size();
  for (int i = 0; i < p->n_sp; ++i) {
    const Cand& c = cand[ssel[i]];
    p->sp_family[i] = c.fam;
    p->sp_j1[i] = idx[c.ia].j;
    p->sp_k1[i] = idx[c.ia].k;
    p->sp_j2[i] = idx[c.ib].j;
    p->sp_k2[i] = idx[c.ib].k;
    p->sp_coef[i] = c.c;
  }
  // ---- separable factorisation of the lowered kernel K~_s(v, u) = sum_j c_j h_a(u) h_b(v)
  //      (eq:2D_box_N_terms evaluated on the integer offsets): K~_s = fy (x) fx iff the matrix is
  //      rank 1, in which case fx is its row and fy its column through the largest entry.
  {
    const int n = 2 * radius + 1;
    std::vector<double> K((size_t)n * n, 0.0), ha, hb;
    for (int i = 0; i < p->n_sp; ++i) {
      const Cand& c = cand[ssel[i]];
      haar_values(idx[c.ia], T, radius, ha);
      haar_values(idx[c.ib], T, radius, hb);
      for (int v = 0; v < n; ++v)
        if (hb[v] != 0.0)
          for (int u = 0; u < n; ++u) K[(size_t)v * n + u] += c.c * hb[v] * ha[u];
    }
    int vs = 0, us = 0;
    double kmax = 0.0;
    for (int v = 0; v < n; ++v)
      for (int u = 0; u < n; ++u)
        if (std::fabs(K[(size_t)v * n + u]) > kmax) {
          kmax = std::fabs(K[(size_t)v * n + u]);
          vs = v;
          us = u;
        }
    p->separable = kmax > 0.0 ? 1 : 0;
    std::vector<double> fx(n), fy(n);
    if (p->separable) {
      const double piv = K[(size_t)vs * n + us];
      for (int u = 0; u < n; ++u) fx[u] = K[(size_t)vs * n + u];
      for (int v = 0; v < n; ++v) fy[v] = K[(size_t)v * n + us] / piv;
      for (int v = 0; v < n && p->separable; ++v)
        for (int u = 0; u < n; ++u)
          if (std::fabs(fy[v] * fx[u] - K[(size_t)v * n + u]) > 1e-12 * kmax) {
            p->separable = 0;
            break;
          }
    }
    if (p->separable) {
      bool okx = step_to_boxes(fx, radius, p->nbx, p->lox, p->hix, p->wx);
      bool oky = step_to_boxes(fy, radius, p->nby, p->loy, p->hiy, p->wy);
      if (!okx || !oky) p->separable = 0;
    }
    if (!p->separable) p->nbx = p->nby = 0;
    p->ns = 0;
    if (p->separable) {
      p->ns = 1;
      p->snbx[0] = p->nbx;
      p->snby[0] = p->nby;
      for (int b = 0; b < p->nbx; ++b) {
        p->slox[0][b] = p->lox[b];
        p->shix[0][b] = p->hix[b];
        p->swx[0][b] = p->wx[b];
      }
      for (int b = 0; b < p->nby; ++b) {
        p->sloy[0][b] = p->loy[b];
        p->shiy[0][b] = p->hiy[b];
        p->swy[0][b] = p->wy[b];
      }
    } else if (box_pair_rank2(K, radius, p)) {
      // the same two terms as separable passes, for radii the rank-2 kernel cannot run
      p->rank = 2;
      p->n_pass = 2;
      for (int s = 0; s < 2; ++s) {
        auto& P = p->pass[s];
        P.nbx = p->snbx[s];
        P.nby = p->snby[s];
        for (int b = 0; b < P.nbx; ++b) {
          P.lox[b] = p->slox[s][b];
          P.hix[b] = p->shix[s][b];
          P.wx[b] = p->swx[s][b];
        }
        for (int b = 0; b < P.nby; ++b) {
          P.loy[b] = p->sloy[s][b];
          P.hiy[b] = p->shiy[s][b];
          P.wy[b] = p->swy[s][b];
        }
      }
    } else {
      p->ns = 0;
      // no GPU form -> bf_apply returns BF_ERR_UNSUPPORTED (also when the repair pass's fp64 factor
      // tables, 2 x passes x (2r + 1) doubles, would not fit its shared memory)
      if (!general_passes(K, radius, p) || p->n_pass * (2 * radius + 1) > 12288) p->n_pass = 0;
    }
  }
  *out = p;
  return BF_OK;
}

extern "C" bf_status bf_plan_destroy(bf_plan* plan) {
  delete plan;
  return BF_OK;
}

extern "C" bf_status bf_plan_get_info(const bf_plan* p, bf_plan_info* info) {
  if (!p || !info) return BF_ERR_INVALID_ARG;
  std::memset(info, 0, sizeof(*info));
  info->n_terms_eff = p->n_k;
  for (int i = 0; i < p->n_k; ++i) {
    info->k[i] = p->k[i];
    info->a[i] = p->a[i];
  }
  info->T_range = p->T;
  info->range_window = p->literal ? BF_RANGE_WINDOW_LITERAL : BF_RANGE_WINDOW_FULL;
  info->n_spatial_eff = p->n_sp;
  for (int i = 0; i < p->n_sp; ++i) {
    info->sp_family[i] = p->sp_family[i];
    info->sp_j1[i] = p->sp_j1[i];
    info->sp_k1[i] = p->sp_k1[i];
    info->sp_j2[i] = p->sp_j2[i];
    info->sp_k2[i] = p->sp_k2[i];
    info->sp_coef[i] = p->sp_coef[i];
  }
  info->separable = p->separable;
  info->spatial_rank = p->ns ? p->ns : p->rank;
  info->spatial_passes = p->ns ? 1 : p->n_pass;
  info->nbx = p->nbx;
  info->nby = p->nby;
  for (int i = 0; i < p->nbx; ++i) {
    info->box_lo_x[i] = p->lox[i];
    info->box_hi_x[i] = p->hix[i];
    info->box_w_x[i] = p->wx[i];
  }
  for (int i = 0; i < p->nby; ++i) {
    info->box_lo_y[i] = p->loy[i];
    info->box_hi_y[i] = p->hiy[i];
    info->box_w_y[i] = p->wy[i];
  }
  info->radius = p->radius;
  info->intensity_max = p->D;
  info->input_dtype = p->input_dtype;
  return BF_OK;
}

extern "C" bf_status bf_plan_spatial_kernel(const bf_plan* p, double* K, size_t n_values) {
  if (!p || !K) return BF_ERR_INVALID_ARG;
  const int r = p->radius, n = 2 * r + 1;
  if (n_values < (size_t)n * n) return BF_ERR_INVALID_ARG;
  if (p->ns == 0 && p->n_pass == 0) return BF_ERR_UNSUPPORTED;
  std::fill(K, K + (size_t)n * n, 0.0);
  const int nt = p->ns > 0 ? p->ns : p->n_pass;
  for (int t = 0; t < nt; ++t) {
    const bool gen = p->ns == 0;
    const int nbx = gen ? p->pass[t].nbx : p->snbx[t], nby = gen ? p->pass[t].nby : p->snby[t];
    std::vector<double> fx(n, 0.0), fy(n, 0.0);
    for (int b = 0; b < nbx; ++b) {
      const int lo = gen ? p->pass[t].lox[b] : p->slox[t][b], hi = gen ? p->pass[t].hix[b] : p->shix[t][b];
      for (int u = lo; u <= hi; ++u) fx[u + r] += gen ? p->pass[t].wx[b] : p->swx[t][b];
    }
    for (int b = 0; b < nby; ++b) {
      const int lo = gen ? p->pass[t].loy[b] : p->sloy[t][b], hi = gen ? p->pass[t].hiy[b] : p->shiy[t][b];
      for (int v = lo; v <= hi; ++v) fy[v + r] += gen ? p->pass[t].wy[b] : p->swy[t][b];
    }
    for (int v = 0; v < n; ++v)
      for (int u = 0; u < n; ++u) K[(size_t)v * n + u] += fy[v] * fx[u];
  }
  return BF_OK;
}

extern "C" const char* bf_status_string(bf_status s) {
  switch (s) {
    case BF_OK: return "BF_OK";
    case BF_ERR_INVALID_ARG: return "BF_ERR_INVALID_ARG: invalid argument";
    case BF_ERR_UNSUPPORTED: return "BF_ERR_UNSUPPORTED: unsupported kernel kind or plan shape";
    case BF_ERR_NO_MEMORY: return "BF_ERR_NO_MEMORY: host allocation failed";
    case BF_ERR_CUDA: return "BF_ERR_CUDA: CUDA launch or runtime error";
    case BF_ERR_NUMERIC: return "BF_ERR_NUMERIC: the fit produced no usable term";
    case BF_ERR_WORKSPACE: return "BF_ERR_WORKSPACE: the plan runs in several passes and needs a device workspace";
  }
  return "unknown bf_status";
}

extern "C" const char* bf_version(void) { return "bf-b200 0.2.0"; }
