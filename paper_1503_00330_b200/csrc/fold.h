// fold.h — host-side folding of LWPR receptive fields into device records.
//
// Restates FrozenLwpr.__init__ (lwpr.py:339-358) in float64 and extends it:
//   - log2(e) scaling of every exponent term and the 2^64 weight shift
//     (kExpShift) so the kernels use ex2 directly;
//   - a global linear shift g(x) = g0 + gs.x (the mean local model) folded
//     out of the local models so the kernels' one-pass variance does not
//     cancel (mean = g(x) + sum w (y - g) exactly in real arithmetic);
//   - three record layouts (common.cuh): per-field diagonal metric, per-field
//     full metric, and a metric shared by all fields of an axis.
#pragma once

#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace pi2 {

struct AxisRaw {
  int L = 0, d = 0;
  std::vector<double> centers, metrics, coefs, lvar;
};

inline bool axis_is_diagonal(const AxisRaw &a) {  // lwpr.py:348-349
  for (int l = 0; l < a.L; ++l)
    for (int i = 0; i < a.d; ++i)
      for (int j = 0; j < a.d; ++j)
        if (i != j && a.metrics[((size_t)l * a.d + i) * a.d + j] != 0.0) return false;
  return true;
}

inline bool axis_shares_metric(const AxisRaw &a) {
  const size_t n = (size_t)a.d * a.d;
  for (int l = 1; l < a.L; ++l)
    if (std::memcmp(&a.metrics[(size_t)l * n], &a.metrics[0], n * sizeof(double)) != 0) return false;
  return true;
}

inline int choose_layout(const AxisRaw *axes, int n_axes) {
  bool shared = true, diag = true;
  for (int i = 0; i < n_axes; ++i) {
    if (axes[i].L == 0) continue;
    shared = shared && axis_shares_metric(axes[i]);
    diag = diag && axis_is_diagonal(axes[i]);
  }
  return shared ? kLayShared : (diag ? kLayDiag : kLayFull);
}

inline int record_floats(int layout) {
  return layout == kLayShared ? kRecShared : (layout == kLayDiag ? kRecDiag : kRecFull);
}

// Append the records of one axis to `rec` and fill its header.
inline void fold_axis(const AxisRaw &a, int layout, std::vector<float> &rec, AxisHeader &h) {
  const int RS = record_floats(layout);
  const size_t base = rec.size();
  rec.resize(base + (size_t)a.L * RS, 0.0f);
  // shared metric: centre inputs on the mean field centre so the per-row
  // quadratic q(x~) stays small (the kernels may then drop it, see lwpr_kernel)
  double mu[4] = {0, 0, 0, 0};
  if (layout == kLayShared) {
    for (int l = 0; l < a.L; ++l)
      for (int i = 0; i < a.d; ++i) mu[i] += a.centers[(size_t)l * a.d + i];
    for (double &v : mu) v /= a.L;
  }
  std::vector<double> y0(a.L), s(4 * (size_t)a.L, 0.0);
  double g0 = 0.0, gs[4] = {0, 0, 0, 0};
  for (int l = 0; l < a.L; ++l) {
    double yy = a.coefs[(size_t)l * (a.d + 1)];
    for (int i = 0; i < a.d; ++i) {
      const double si = a.coefs[(size_t)l * (a.d + 1) + 1 + i];
      s[4 * (size_t)l + i] = si;
      yy -= si * (a.centers[(size_t)l * a.d + i] - mu[i]);  // y0 = coef0 - s.c (lwpr.py:355-357), in x~
    }
    y0[l] = yy;
    g0 += yy;
    for (int i = 0; i < 4; ++i) gs[i] += s[4 * (size_t)l + i];
  }
  g0 /= a.L;
  for (double &v : gs) v /= a.L;
  h = AxisHeader{};
  h.g0 = (float)g0;
  for (int i = 0; i < 4; ++i) {
    h.gs[i] = (float)gs[i];
    h.mu[i] = (float)mu[i];
  }
  h.num_fields = a.L;
  h.offset = (int64_t)base;
  double D0[4][4] = {{0}};
  for (int i = 0; i < a.d; ++i)
    for (int j = 0; j < a.d; ++j) D0[i][j] = a.metrics[(size_t)i * a.d + j];
  if (layout == kLayShared) {
    int q = 0;
    for (int i = 0; i < 4; ++i)
      for (int j = i; j < 4; ++j)
        h.qd[q++] = (float)((i == j ? -0.5 * D0[i][i] : -0.5 * (D0[i][j] + D0[j][i])) * kLog2e);
  }
  for (int l = 0; l < a.L; ++l) {
    double c[4] = {0, 0, 0, 0}, D[4][4] = {{0}};
    for (int i = 0; i < a.d; ++i) {
      c[i] = a.centers[(size_t)l * a.d + i] - mu[i];
      for (int j = 0; j < a.d; ++j) D[i][j] = a.metrics[((size_t)l * a.d + i) * a.d + j];
    }
    double dc[4], a0 = 0.0;
    for (int i = 0; i < 4; ++i) {  // dc = D c (lwpr.py:344)
      dc[i] = 0.0;
      for (int j = 0; j < 4; ++j) dc[i] += D[i][j] * c[j];
    }
    for (int i = 0; i < 4; ++i) a0 += dc[i] * c[i];
    a0 *= -0.5;  // lwpr.py:347
    float *f = rec.data() + base + (size_t)l * RS;
    if (layout == kLayDiag) {
      f[0] = (float)(a0 * kLog2e + kExpShift);
      for (int i = 0; i < 4; ++i) {
        f[1 + i] = (float)(-0.5 * D[i][i] * kLog2e);  // a1 (lwpr.py:345)
        f[5 + i] = (float)(dc[i] * kLog2e);           // a2 (lwpr.py:346)
        f[9 + i] = (float)(s[4 * (size_t)l + i] - gs[i]);
      }
      f[13] = (float)(y0[l] - g0);
      f[14] = (float)a.lvar[l];
    } else if (layout == kLayFull) {
      f[0] = (float)(a0 * kLog2e + kExpShift);
      int q = 1;
      for (int i = 0; i < 4; ++i)
        for (int j = i; j < 4; ++j)
          f[q++] = (float)((i == j ? -0.5 * D[i][i] : -0.5 * (D[i][j] + D[j][i])) * kLog2e);
      for (int i = 0; i < 4; ++i) {
        f[11 + i] = (float)(dc[i] * kLog2e);
        f[15 + i] = (float)(s[4 * (size_t)l + i] - gs[i]);
      }
      f[19] = (float)(y0[l] - g0);
      f[20] = (float)a.lvar[l];
    } else {
      f[0] = (float)(a0 * kLog2e + kExpShift);
      for (int i = 0; i < 4; ++i) {
        f[1 + i] = (float)(dc[i] * kLog2e);
        f[5 + i] = (float)(s[4 * (size_t)l + i] - gs[i]);
      }
      f[9] = (float)(y0[l] - g0);
      f[10] = (float)a.lvar[l];
    }
  }
}

}  // namespace pi2
