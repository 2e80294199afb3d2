// Device restatement of the reference element forms, operation for
// operation, so that with -fmad=false the GPU reproduces the reference's
// IEEE double results bit for bit:
//   TetFrame::from   element_forms.cpp:8-30 (Eigen 3x3 determinant by row-0
//                    cofactor expansion; inverse = adjugate * (1/det') with
//                    det' from column-0 cofactors — Eigen's InverseImpl.h)
//   element_l11      element_forms.cpp:49-73
//   element_l12/l21  element_forms.cpp:75-99
//   element_l22      element_forms.cpp:101-114
//   signed_tet_volume mesh.cpp:36-38
// Translation units including this header are compiled with -fmad=false.
#pragma once

#include <cuda_runtime.h>

namespace ect {

struct TetGeom {
  double g[4][3];  // barycentric gradients
  double vol;      // det / 6
  bool ok;         // det > 0 (TetFrame::from throws otherwise)
};

__device__ __forceinline__ void tet_frame(const double p[4][3], TetGeom& f) {
  // jac.col(c) = p[c+1] - p[0]  =>  m[r][c]
  double m[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) m[r][c] = p[c + 1][r] - p[0][r];
  // determinant(): m00*(m11 m22 - m12 m21) - m01*(m10 m22 - m12 m20) + m02*(m10 m21 - m11 m20)
  const double h0 = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]);
  const double h1 = m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]);
  const double h2 = m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  const double det = (h0 - h1) + h2;
  f.ok = det > 0.0;
  // inverse(): cof(i,j) = m(i1,j1) m(i2,j2) - m(i1,j2) m(i2,j1), i1=(i+1)%3 ...
  double cof[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      cof[i][j] = m[i1][j1] * m[i2][j2] - m[i1][j2] * m[i2][j1];
    }
  const double det_inv = (cof[0][0] * m[0][0] + cof[1][0] * m[1][0]) + cof[2][0] * m[2][0];
  const double invdet = 1.0 / det_inv;
  // inverse(r, c) = cof(c, r) * invdet ; grad[k+1] = row k of the inverse
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) f.g[k + 1][c] = cof[c][k] * invdet;
#pragma unroll
  for (int c = 0; c < 3; ++c) f.g[0][c] = -((f.g[1][c] + f.g[2][c]) + f.g[3][c]);
  f.vol = det / 6.0;
}

// Eigen dot on real 3-vectors: (a0 b0 + a1 b1) + a2 b2
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

// (b-a) x (c-a) . (d-a) / 6  (mesh.cpp:36-38)
__device__ __forceinline__ double signed_volume(const double p[4][3]) {
  double u[3], v[3], w[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    u[c] = p[1][c] - p[0][c];
    v[c] = p[2][c] - p[0][c];
    w[c] = p[3][c] - p[0][c];
  }
  const double cx = u[1] * v[2] - u[2] * v[1];
  const double cy = u[2] * v[0] - u[0] * v[2];
  const double cz = u[0] * v[1] - u[1] * v[0];
  return ((cx * w[0] + cy * w[1]) + cz * w[2]) / 6.0;
}

// Per-region coefficients exactly as the element routines form them.
struct RegionCoef {
  double mu_inv;      // 1.0 / mu                        (element_l11)
  double mt_inv;      // 1.0 / mu_tilde                  (element_l11)
  double mass_im;     // ((0,-1)*omega*sigma).imag = (-omega)*sigma
  double sigma;       // region sigma                    (l12/l21/l22 gauge)
  double neg_sigma;   // -sigma
  double stiff_im;    // sigma / omega                   (l22 stiff_coef)
  double gauge;       // delta_gauge * mu * sigma        (l22)
  double stiff_im_eps;  // sigma_eps / omega  (l22_use_sigma_eps branch)
};

}  // namespace ect
