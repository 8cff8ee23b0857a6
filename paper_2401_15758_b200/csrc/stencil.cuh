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


// 12 h^2 J(a, b) at two adjacent points from 3x4 windows (rows -1, 0, +1; the
// points' 3x3 neighbourhoods are columns 0..2 and 1..3), for a BASE field a
// and a per-vector field b. The Arakawa Jacobian is bilinear, so for a fixed a
// it is the 8-point stencil sum_k c_k(a) b_k (the centre coefficient is 0):
//   north/south: +-(a_x at this row + a_x at that row), a_x = a(.,+1) - a(.,-1)
//   east/west:   -+(a_y at this column + a_y at that column), a_y = a(+1,.) - a(-1,.)
//   corners:     differences of the two edge neighbours next to the corner.
// The column differences a_y and their pair sums are shared by the two
// points. ptxas finds most of this sharing in two inlined arakawa12 calls
// too (the instruction count falls ~1%), but this form keeps fewer values
// live: spills 24-120 -> 4-20 B per thread in the fused TLM stage kernels,
// their launches 2.4% faster (profiles/r2s4_ncu_stage_streaming.md). Same
// operator (antisymmetric in (a, b): J(b, a) = -J(a, b)); roundoff differs.
__device__ __forceinline__ void arakawa12_pair(const double a[3][4], const double b[3][4], double out[2]) {
  const double dy0 = a[2][0] - a[0][0], dy1 = a[2][1] - a[0][1], dy2 = a[2][2] - a[0][2], dy3 = a[2][3] - a[0][3];
  const double sy[3] = {dy0 + dy1, dy1 + dy2, dy2 + dy3};
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const double dx0 = a[0][p + 2] - a[0][p], dx1 = a[1][p + 2] - a[1][p], dx2 = a[2][p + 2] - a[2][p];
    const double cn = dx1 + dx2, cs = dx1 + dx0;  // b(+1, 0), -b(-1, 0)
    double r0 = cn * b[2][p + 1];
    double r1 = sy[p] * b[1][p];                   // b(0, -1)
    r0 = fma(-cs, b[0][p + 1], r0);
    r1 = fma(-sy[p + 1], b[1][p + 2], r1);        // b(0, +1)
    r0 = fma(a[1][p + 2] - a[2][p + 1], b[2][p + 2], r0);
    r1 = fma(a[0][p + 1] - a[1][p + 2], b[0][p + 2], r1);
    // (written as minus the opposite corner's difference of the diagonal
    // neighbour, so the unrolled row sweep reuses it: point (x, y)'s
    // north-east coefficient is minus point (x+1, y+1)'s south-west one)
    r0 = fma(-(a[1][p] - a[2][p + 1]), b[2][p], r0);
    r1 = fma(-(a[0][p + 1] - a[1][p]), b[0][p], r1);
    out[p] = r0 + r1;
  }
}

}  // namespace sdv
