// Periodic-grid stencil building blocks shared by the BVE kernels.
#pragma once

namespace sdv {

// Arakawa Jacobian J(a,b) ~ a_x b_y - a_y b_x from 3x3 neighbourhoods
// a[dy][dx], b[dy][dx] (dy, dx in {0,1,2} <-> offsets -1, 0, +1); returns 12 h^2 J.
__device__ __forceinline__ double arakawa12(const double a[3][3], const double b[3][3]) {
  const double jpp = (a[1][2] - a[1][0]) * (b[2][1] - b[0][1]) - (a[2][1] - a[0][1]) * (b[1][2] - b[1][0]);
  const double jpx = a[1][2] * (b[2][2] - b[0][2]) - a[1][0] * (b[2][0] - b[0][0]) -
                     a[2][1] * (b[2][2] - b[2][0]) + a[0][1] * (b[0][2] - b[0][0]);
  const double jxp = b[2][1] * (a[2][2] - a[2][0]) - b[0][1] * (a[0][2] - a[0][0]) -
                     b[1][2] * (a[2][2] - a[0][2]) + b[1][0] * (a[2][0] - a[0][0]);
  return jpp + jpx + jxp;
}
__device__ __forceinline__ double lap5(const double o[3][3]) {
  return o[1][0] + o[1][2] + o[0][1] + o[2][1] - 4.0 * o[1][1];
}

}  // namespace sdv
