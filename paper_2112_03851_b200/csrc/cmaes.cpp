// Stochastic transmission-coefficient optimisation (Section 4):
// CMA-ES (lambda samples of N(m, sigma^2 C), mu best, weighted mean, step size and
// covariance adaptation; population 25; stop at 7200 iterations / 5e-11)
// and the Fourier convergence-rate cost.  Host code; no CUDA.
//
// Samples use the symmetric square root of C (x = m + sigma C^{1/2} z), which is unique, so the
// trajectory does not depend on eigenvector sign or order; the standard normals z are supplied by
// the caller.  The small symmetric eigenproblems are solved by cyclic Jacobi rotations.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.h"

namespace osm {
extern thread_local std::string g_last_error;
}
using namespace osm;

namespace {

// Jacobi eigen-decomposition of a symmetric n x n matrix A (row-major): A = V diag(d) V^T.
void jacobi_eig(int n, std::vector<double> A, std::vector<double>& d, std::vector<double>& V) {
  V.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += A[i * n + j] * A[i * n + j];
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- J^T A J
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  d.resize(n);
  for (int i = 0; i < n; ++i) d[i] = A[i * n + i];
}

// symmetric C^{e} for e = +1/2 or -1/2
std::vector<double> sym_pow_half(int n, const std::vector<double>& C, bool inverse) {
  std::vector<double> d, V;
  jacobi_eig(n, C, d, V);
  std::vector<double> R(n * n, 0.0);
  for (int k = 0; k < n; ++k) {
    const double ev = std::max(d[k], 0.0);
    const double s = inverse ? (ev > 0 ? 1.0 / std::sqrt(ev) : 0.0) : std::sqrt(ev);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) R[i * n + j] += V[i * n + k] * s * V[j * n + k];
  }
  return R;
}

double rate_at(double k, double p1, double q1, double p2, double q2) {
  const double l1 = p1 + q1 * k * k, l2 = p2 + q2 * k * k;
  return std::fabs((l1 - k) / (l1 + k)) * std::fabs((l2 - k) / (l2 + k));
}

}  // namespace

struct osm_cmaes {
  int n, lam, mu, g = 0;
  std::vector<double> w, m, C, ps, pc, X, best_x, hist;
  double mueff, cs, ds, cc, c1, cmu, chin, sigma, best_f = INFINITY;
};

#define API_BEGIN try {
#define API_END                             \
  }                                         \
  catch (const Error& e) {                  \
    g_last_error = e.what();                \
    return e.status;                        \
  }                                         \
  catch (const std::exception& e) {         \
    g_last_error = e.what();                \
    return OSM_ERR_INVALID_ARG;             \
  }

extern "C" {

osm_status osm_rate_max(double p1, double q1, double p2, double q2, double kmin, double kmax, int nsamp,
                        double* rho, double* kargmax) {
  API_BEGIN
  if (!rho || !(kmin > 0) || !(kmax >= kmin) || nsamp < 1) fail(OSM_ERR_INVALID_ARG, "bad band");
  double best = -1.0, kb = kmin;
  for (int i = 0; i < nsamp; ++i) {  // geometric sampling, endpoints included
    const double k = nsamp == 1 ? kmin : kmin * std::pow(kmax / kmin, (double)i / (nsamp - 1));
    const double r = rate_at(k, p1, q1, p2, q2);
    if (r > best) {
      best = r;
      kb = k;
    }
  }
  *rho = best;
  if (kargmax) *kargmax = kb;
  return OSM_OK;
  API_END
}

osm_status osm_rate_curve(double p1, double q1, double p2, double q2, const double* k, int n, double* rho) {
  API_BEGIN
  if (!k || !rho || n < 0) fail(OSM_ERR_INVALID_ARG, "NULL array");
  for (int i = 0; i < n; ++i) rho[i] = rate_at(k[i], p1, q1, p2, q2);
  return OSM_OK;
  API_END
}

osm_status osm_cmaes_create(int n, int lambda, const double* mean, double sigma0, osm_cmaes** out) {
  API_BEGIN
  if (!out || !mean || n < 1 || n > 64 || lambda < 2 || !(sigma0 > 0)) fail(OSM_ERR_INVALID_ARG, "bad CMA-ES setup");
  auto* e = new osm_cmaes();
  e->n = n;
  e->lam = lambda;
  e->mu = lambda / 2;
  e->w.resize(e->mu);
  double sw = 0;
  for (int i = 0; i < e->mu; ++i) sw += (e->w[i] = std::log((lambda + 1) / 2.0) - std::log(i + 1.0));
  double sw2 = 0;
  for (double& x : e->w) {
    x /= sw;
    sw2 += x * x;
  }
  const double me = e->mueff = 1.0 / sw2;
  e->cs = (me + 2) / (n + me + 5);
  e->ds = 1 + 2 * std::max(0.0, std::sqrt((me - 1) / (n + 1)) - 1) + e->cs;
  e->cc = (4 + me / n) / (n + 4 + 2 * me / n);
  e->c1 = 2 / ((n + 1.3) * (n + 1.3) + me);
  e->cmu = std::min(1 - e->c1, 2 * (me - 2 + 1 / me) / ((n + 2.0) * (n + 2.0) + me));
  e->chin = std::sqrt((double)n) * (1 - 1.0 / (4 * n) + 1.0 / (21.0 * n * n));
  e->m.assign(mean, mean + n);
  e->sigma = sigma0;
  e->C.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) e->C[i * n + i] = 1.0;
  e->ps.assign(n, 0.0);
  e->pc.assign(n, 0.0);
  e->best_x = e->m;
  *out = e;
  return OSM_OK;
  API_END
}

void osm_cmaes_destroy(osm_cmaes* e) { delete e; }

void osm_cmaes_dims(const osm_cmaes* es, int* n, int* lambda) {
  if (n) *n = es ? es->n : 0;
  if (lambda) *lambda = es ? es->lam : 0;
}

osm_status osm_cmaes_ask(osm_cmaes* e, const double* z, double* x) {
  API_BEGIN
  if (!e || !z || !x) fail(OSM_ERR_INVALID_ARG, "NULL argument");
  const int n = e->n;
  const std::vector<double> R = sym_pow_half(n, e->C, false);
  e->X.assign((size_t)e->lam * n, 0.0);
  for (int k = 0; k < e->lam; ++k)
    for (int i = 0; i < n; ++i) {
      double s = 0;
      for (int j = 0; j < n; ++j) s += R[i * n + j] * z[k * n + j];
      e->X[k * n + i] = e->m[i] + e->sigma * s;
    }
  std::copy(e->X.begin(), e->X.end(), x);
  return OSM_OK;
  API_END
}

osm_status osm_cmaes_tell(osm_cmaes* e, const double* f_in) {
  API_BEGIN
  if (!e || !f_in || e->X.empty()) fail(OSM_ERR_STATE, "tell without ask");
  const int n = e->n, lam = e->lam, mu = e->mu;
  std::vector<double> f(f_in, f_in + lam);
  for (double& v : f)
    if (!std::isfinite(v)) v = INFINITY;  // non-finite -> worst rank
  std::vector<int> ord(lam);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return f[a] < f[b]; });
  if (f[ord[0]] < e->best_f) {
    e->best_f = f[ord[0]];
    e->best_x.assign(e->X.begin() + (size_t)ord[0] * n, e->X.begin() + (size_t)ord[0] * n + n);
  }
  const std::vector<double> m_old = e->m;
  for (int i = 0; i < n; ++i) {
    double s = 0;
    for (int k = 0; k < mu; ++k) s += e->w[k] * e->X[(size_t)ord[k] * n + i];
    e->m[i] = s;
  }
  std::vector<double> yw(n);
  for (int i = 0; i < n; ++i) yw[i] = (e->m[i] - m_old[i]) / e->sigma;
  const std::vector<double> Ci = sym_pow_half(n, e->C, true);
  const double a = std::sqrt(e->cs * (2 - e->cs) * e->mueff);
  for (int i = 0; i < n; ++i) {
    double s = 0;
    for (int j = 0; j < n; ++j) s += Ci[i * n + j] * yw[j];
    e->ps[i] = (1 - e->cs) * e->ps[i] + a * s;
  }
  e->g += 1;
  double nps = 0;
  for (double v : e->ps) nps += v * v;
  nps = std::sqrt(nps);
  const bool hs = nps / std::sqrt(1 - std::pow(1 - e->cs, 2.0 * e->g)) < (1.4 + 2.0 / (n + 1)) * e->chin;
  const double b = std::sqrt(e->cc * (2 - e->cc) * e->mueff);
  for (int i = 0; i < n; ++i) e->pc[i] = (1 - e->cc) * e->pc[i] + (hs ? b * yw[i] : 0.0);
  std::vector<double> Cn(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double rmu = 0;
      for (int k = 0; k < mu; ++k) {
        const double yi = (e->X[(size_t)ord[k] * n + i] - m_old[i]) / e->sigma;
        const double yj = (e->X[(size_t)ord[k] * n + j] - m_old[j]) / e->sigma;
        rmu += e->w[k] * yi * yj;
      }
      Cn[i * n + j] = (1 - e->c1 - e->cmu) * e->C[i * n + j] +
                      e->c1 * (e->pc[i] * e->pc[j] + (hs ? 0.0 : e->cc * (2 - e->cc)) * e->C[i * n + j]) +
                      e->cmu * rmu;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) e->C[i * n + j] = 0.5 * (Cn[i * n + j] + Cn[j * n + i]);
  e->sigma *= std::exp((e->cs / e->ds) * (nps / e->chin - 1));
  e->hist.push_back(f[ord[0]]);
  return OSM_OK;
  API_END
}

osm_status osm_cmaes_state(osm_cmaes* e, double* mean, double* sigma, double* cov, double* best_x, double* best_f,
                           int* generation) {
  API_BEGIN
  if (!e) fail(OSM_ERR_INVALID_ARG, "NULL handle");
  if (mean) std::copy(e->m.begin(), e->m.end(), mean);
  if (sigma) *sigma = e->sigma;
  if (cov) std::copy(e->C.begin(), e->C.end(), cov);
  if (best_x) std::copy(e->best_x.begin(), e->best_x.end(), best_x);
  if (best_f) *best_f = e->best_f;
  if (generation) *generation = e->g;
  return OSM_OK;
  API_END
}

osm_status osm_cmaes_should_stop(osm_cmaes* e, int max_iter, double ftol, int* stop) {
  API_BEGIN
  if (!e || !stop) fail(OSM_ERR_INVALID_ARG, "NULL argument");
  *stop = 0;
  if (e->g >= max_iter) *stop = 1;
  const int hl = 10 + (int)std::ceil(30.0 * e->n / e->lam);
  if ((int)e->hist.size() >= hl) {
    const auto b = e->hist.end() - hl;
    const double mx = *std::max_element(b, e->hist.end()), mn = *std::min_element(b, e->hist.end());
    if (mx - mn < ftol) *stop = 2;
  }
  std::vector<double> d, V;
  jacobi_eig(e->n, e->C, d, V);
  if (e->sigma * std::sqrt(*std::max_element(d.begin(), d.end())) < 1e-14) *stop = 3;
  return OSM_OK;
  API_END
}

}  // extern "C"
