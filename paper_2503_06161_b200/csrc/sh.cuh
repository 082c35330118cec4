// Real spherical-harmonic view-dependent colour, degree <= 3 (build extension).
//
// The reference is degree-0 only (colors() = clip(colors_raw, 0, 1),
// gaussians.py:63-64, rasterizer.py:181; SH > 0 reserved).  The
// extension keeps colors_raw as the degree-0 term and adds the higher bands:
//     colour = clip(colors_raw + sum_{k>=1} Y_k(d) * sh_rest[k-1], 0, 1),
//     d = normalize(mu_world - C_cam),   C_cam = -R^T t,
// so at degree 0 it reduces bit-exactly to the reference.  Y_k is the standard
// real SH basis (same constants as the usual 3DGS convention).
#pragma once

namespace fs4d {

template <typename T>
struct ShConst {
  static constexpr T C1 = T(0.4886025119029199);
  static constexpr T C2_0 = T(1.0925484305920792);
  static constexpr T C2_1 = T(-1.0925484305920792);
  static constexpr T C2_2 = T(0.31539156525252005);
  static constexpr T C2_3 = T(-1.0925484305920792);
  static constexpr T C2_4 = T(0.5462742152960396);
  static constexpr T C3_0 = T(-0.5900435899266435);
  static constexpr T C3_1 = T(2.890611442640554);
  static constexpr T C3_2 = T(-0.4570457994644658);
  static constexpr T C3_3 = T(0.3731763325901154);
  static constexpr T C3_4 = T(-0.4570457994644658);
  static constexpr T C3_5 = T(1.445305721320277);
  static constexpr T C3_6 = T(-0.5900435899266435);
};

// Y[k] for k = 1..(L+1)^2-1 (written to Y[0..n-1]) and, if dY != nullptr,
// dY[k][3] = dY_k/d(x,y,z) treating (x,y,z) as free variables.
template <typename T>
__host__ __device__ inline int sh_basis(int degree, T x, T y, T z, T* Y, T (*dY)[3]) {
  using C = ShConst<T>;
  int n = 0;
  if (degree >= 1) {
    Y[0] = -C::C1 * y;
    Y[1] = C::C1 * z;
    Y[2] = -C::C1 * x;
    if (dY) {
      dY[0][0] = 0; dY[0][1] = -C::C1; dY[0][2] = 0;
      dY[1][0] = 0; dY[1][1] = 0; dY[1][2] = C::C1;
      dY[2][0] = -C::C1; dY[2][1] = 0; dY[2][2] = 0;
    }
    n = 3;
  }
  if (degree >= 2) {
    T xx = x * x, yy = y * y, zz = z * z;
    Y[3] = C::C2_0 * x * y;
    Y[4] = C::C2_1 * y * z;
    Y[5] = C::C2_2 * (T(2) * zz - xx - yy);
    Y[6] = C::C2_3 * x * z;
    Y[7] = C::C2_4 * (xx - yy);
    if (dY) {
      dY[3][0] = C::C2_0 * y; dY[3][1] = C::C2_0 * x; dY[3][2] = 0;
      dY[4][0] = 0; dY[4][1] = C::C2_1 * z; dY[4][2] = C::C2_1 * y;
      dY[5][0] = C::C2_2 * (-T(2) * x); dY[5][1] = C::C2_2 * (-T(2) * y); dY[5][2] = C::C2_2 * (T(4) * z);
      dY[6][0] = C::C2_3 * z; dY[6][1] = 0; dY[6][2] = C::C2_3 * x;
      dY[7][0] = C::C2_4 * (T(2) * x); dY[7][1] = C::C2_4 * (-T(2) * y); dY[7][2] = 0;
    }
    n = 8;
  }
  if (degree >= 3) {
    T xx = x * x, yy = y * y, zz = z * z;
    Y[8] = C::C3_0 * y * (T(3) * xx - yy);
    Y[9] = C::C3_1 * x * y * z;
    Y[10] = C::C3_2 * y * (T(4) * zz - xx - yy);
    Y[11] = C::C3_3 * z * (T(2) * zz - T(3) * xx - T(3) * yy);
    Y[12] = C::C3_4 * x * (T(4) * zz - xx - yy);
    Y[13] = C::C3_5 * z * (xx - yy);
    Y[14] = C::C3_6 * x * (xx - T(3) * yy);
    if (dY) {
      dY[8][0] = C::C3_0 * (T(6) * x * y);
      dY[8][1] = C::C3_0 * (T(3) * xx - T(3) * yy);
      dY[8][2] = 0;
      dY[9][0] = C::C3_1 * y * z;
      dY[9][1] = C::C3_1 * x * z;
      dY[9][2] = C::C3_1 * x * y;
      dY[10][0] = C::C3_2 * (-T(2) * x * y);
      dY[10][1] = C::C3_2 * (T(4) * zz - xx - T(3) * yy);
      dY[10][2] = C::C3_2 * (T(8) * y * z);
      dY[11][0] = C::C3_3 * (-T(6) * x * z);
      dY[11][1] = C::C3_3 * (-T(6) * y * z);
      dY[11][2] = C::C3_3 * (T(6) * zz - T(3) * xx - T(3) * yy);
      dY[12][0] = C::C3_4 * (T(4) * zz - T(3) * xx - yy);
      dY[12][1] = C::C3_4 * (-T(2) * x * y);
      dY[12][2] = C::C3_4 * (T(8) * x * z);
      dY[13][0] = C::C3_5 * (T(2) * x * z);
      dY[13][1] = C::C3_5 * (-T(2) * y * z);
      dY[13][2] = C::C3_5 * (xx - yy);
      dY[14][0] = C::C3_6 * (T(3) * xx - T(3) * yy);
      dY[14][1] = C::C3_6 * (-T(6) * x * y);
      dY[14][2] = 0;
    }
    n = 15;
  }
  return n;
}

}  // namespace fs4d
