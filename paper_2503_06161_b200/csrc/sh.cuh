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

// Calls f(k, Y_k, dY_k/dx, dY_k/dy, dY_k/dz) for k = 0..(L+1)^2-2 (basis
// functions 1.. of the real SH, (x, y, z) treated as free variables), in
// increasing k.  A visitor instead of Y[15] / dY[15][3] arrays: with a runtime
// degree those arrays live in local memory (480 B per thread in the backward).
template <typename T, typename F>
__host__ __device__ __forceinline__ void sh_visit(int degree, T x, T y, T z, F&& f) {
  using C = ShConst<T>;
  const T o = T(0);
  if (degree >= 1) {
    f(0, -C::C1 * y, o, -C::C1, o);
    f(1, C::C1 * z, o, o, C::C1);
    f(2, -C::C1 * x, -C::C1, o, o);
  }
  if (degree >= 2) {
    const T xx = x * x, yy = y * y, zz = z * z;
    f(3, C::C2_0 * x * y, C::C2_0 * y, C::C2_0 * x, o);
    f(4, C::C2_1 * y * z, o, C::C2_1 * z, C::C2_1 * y);
    f(5, C::C2_2 * (T(2) * zz - xx - yy), C::C2_2 * (-T(2) * x), C::C2_2 * (-T(2) * y), C::C2_2 * (T(4) * z));
    f(6, C::C2_3 * x * z, C::C2_3 * z, o, C::C2_3 * x);
    f(7, C::C2_4 * (xx - yy), C::C2_4 * (T(2) * x), C::C2_4 * (-T(2) * y), o);
  }
  if (degree >= 3) {
    const T xx = x * x, yy = y * y, zz = z * z;
    f(8, C::C3_0 * y * (T(3) * xx - yy), C::C3_0 * (T(6) * x * y), C::C3_0 * (T(3) * xx - T(3) * yy), o);
    f(9, C::C3_1 * x * y * z, C::C3_1 * y * z, C::C3_1 * x * z, C::C3_1 * x * y);
    f(10, C::C3_2 * y * (T(4) * zz - xx - yy), C::C3_2 * (-T(2) * x * y), C::C3_2 * (T(4) * zz - xx - T(3) * yy),
      C::C3_2 * (T(8) * y * z));
    f(11, C::C3_3 * z * (T(2) * zz - T(3) * xx - T(3) * yy), C::C3_3 * (-T(6) * x * z), C::C3_3 * (-T(6) * y * z),
      C::C3_3 * (T(6) * zz - T(3) * xx - T(3) * yy));
    f(12, C::C3_4 * x * (T(4) * zz - xx - yy), C::C3_4 * (T(4) * zz - T(3) * xx - yy), C::C3_4 * (-T(2) * x * y),
      C::C3_4 * (T(8) * x * z));
    f(13, C::C3_5 * z * (xx - yy), C::C3_5 * (T(2) * x * z), C::C3_5 * (-T(2) * y * z), C::C3_5 * (xx - yy));
    f(14, C::C3_6 * x * (xx - T(3) * yy), C::C3_6 * (T(3) * xx - T(3) * yy), C::C3_6 * (-T(6) * x * y), o);
  }
}

}  // namespace fs4d
