// Host-side scalar math of the library (no device work):
//  * Chebyshev coefficients of the ideal low-pass + Jackson damping (§2.3-2.4)
//  * eigenvalue counts from Chebyshev moments and the lambda_k dichotomy (§3.2)
//  * largest eigenvalue of the Lanczos tridiagonal matrix (Sturm bisection)
#include <algorithm>
#include <cmath>
#include <vector>

#include "sc_internal.cuh"

namespace sc {

// h_{lambda_c}(lambda) = 1[lambda <= lambda_c] on [0, lambda_max]; x = 2 lambda/lambda_max - 1.
// Chebyshev series of the indicator of x <= a:  theta = arccos(a),
// c_0 = 1 - theta/pi (halved j=0 term), c_j = -2 sin(j theta) / (pi j).
// Jackson factors for M = order+1 terms:
// g_j = [(M - j + 1) cos(j q) + sin(j q) cot(q)] / (M + 1),  q = pi/(M+1).
void cheby_lowpass_coeffs(double lambda_c, double lambda_max, int order, bool jackson, double* out) {
  double a = 2.0 * lambda_c / lambda_max - 1.0;
  a = std::min(1.0, std::max(-1.0, a));
  const double theta = std::acos(a);
  const double pi = M_PI;
  out[0] = 1.0 - theta / pi;
  for (int j = 1; j <= order; ++j) out[j] = -2.0 * std::sin(j * theta) / (pi * j);
  if (jackson) {
    const double M = order + 1.0;
    const double q = pi / (M + 1.0);
    const double cotq = std::cos(q) / std::sin(q);
    for (int j = 0; j <= order; ++j) {
      const double gj = ((M - j + 1.0) * std::cos(j * q) + std::sin(j * q) * cotq) / (M + 1.0);
      out[j] *= gj;
    }
  }
}

// ||p(L~) X||_F^2 = sum_{j,l} d_j d_l <T_j X, T_l X> and T_j T_l = (T_{j+l} + T_{|j-l|})/2,
// so the count is sum_{j,l} d_j d_l (mu_{j+l} + mu_{|j-l|}) / 2.
double count_from_moments(const double* mu, int order, const double* d) {
  double tot = 0.0;
  for (int j = 0; j <= order; ++j) {
    double row = 0.0;
    for (int l = 0; l <= order; ++l) row += d[l] * (mu[j + l] + mu[j > l ? j - l : l - j]);
    tot += d[j] * row;
  }
  return 0.5 * tot;
}

int lambda_k_dichotomy(const double* mu, int order, int k, double lambda_max, bool jackson,
                       int max_iter, double rtol, double* lambda_k, double* count_k) {
  std::vector<double> d(order + 1);
  double lo = 0.0, hi = lambda_max, c_hi = NAN;
  for (int it = 0; it < max_iter; ++it) {
    const double mid = 0.5 * (lo + hi);
    cheby_lowpass_coeffs(mid, lambda_max, order, jackson, d.data());
    const double c = count_from_moments(mu, order, d.data());
    if (c >= k - 0.5) {
      hi = mid;
      c_hi = c;
    } else {
      lo = mid;
    }
    if (hi - lo <= rtol * lambda_max) break;
  }
  *lambda_k = hi;
  *count_k = c_hi;
  return SC_OK;
}

// number of eigenvalues of the symmetric tridiagonal (a, b) strictly below x
static int sturm_count(const std::vector<double>& a, const std::vector<double>& b, double x) {
  int cnt = 0;
  double q = 1.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double bb = i ? b[i - 1] * b[i - 1] : 0.0;
    q = a[i] - x - (i ? bb / q : 0.0);
    if (q == 0.0) q = -1e-300;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

double tridiag_max_eig(const std::vector<double>& a, const std::vector<double>& b) {
  const size_t m = a.size();
  if (m == 0) return 0.0;
  double lo = a[0], hi = a[0];
  for (size_t i = 0; i < m; ++i) {
    const double r = (i ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(1.0, std::fabs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (sturm_count(a, b, mid) >= (int)m) hi = mid;   // all eigenvalues below mid
    else lo = mid;
  }
  return hi;
}

}  // namespace sc
