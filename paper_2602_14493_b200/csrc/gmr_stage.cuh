// gmr_stage.cuh — the projection stage on its own (reference render.py:103-145
// project_cloud and :364-402 project_cloud_backward), for the drop-in stage
// functions of the same names.  The mesh path fuses the same math into K1
// (mesh_to_splats) and K5 (face_views_backward); these kernels take a
// Gaussian cloud and general (not necessarily symmetric) upstream cov2d
// gradients, as the reference's stage function does.
#pragma once

#include "gmr_kernels.cuh"

namespace gmr {

// project_cloud: thread per Gaussian.  Writes every Gaussian's screen
// quantities and a keep flag (depth window, render.py:108; 3-sigma screen
// box, :125-130); the host compacts the kept ones in cloud order.
template <typename S>
__global__ void __launch_bounds__(256) project_gaussians(const S* __restrict__ means, const S* __restrict__ cov3d,
                                                         int64_t K, const __grid_constant__ Cam<S> cam, int W, int H,
                                                         S* __restrict__ mean2d, S* __restrict__ cov2d,
                                                         S* __restrict__ conic, S* __restrict__ depth,
                                                         S* __restrict__ radius, S* __restrict__ t_cam,
                                                         uint8_t* __restrict__ kept) {
  pdl_wait();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  S m[3], t[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) m[i] = means[3 * k + i];
  cam_point(cam, m, t);
#pragma unroll
  for (int i = 0; i < 3; ++i) t_cam[3 * k + i] = t[i];
  depth[k] = t[2];
  uint8_t keep = 0;
  if (t[2] > cam.near_plane && t[2] < cam.far_plane) {
    S m2[2][3];
    cam_m2(cam, t, m2);
    const S* c = cov3d + 9 * k;
    S v[2][2];   // (M2 Sigma M2^T)[p][q] with the full 3x3 Sigma (render.py:115-116)
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        S acc = S(0);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const S mc = m2[p][0] * c[3 * 0 + i] + m2[p][1] * c[3 * 1 + i] + m2[p][2] * c[3 * 2 + i];
          acc += mc * m2[q][i];
        }
        v[p][q] = acc;
      }
    v[0][0] = add_rn(v[0][0], Const<S>::dilation());
    v[1][1] = add_rn(v[1][1], Const<S>::dilation());
    const S mx = add_rn(div_rn(mul_rn(cam.fx, t[0]), t[2]), cam.cx);
    const S my = add_rn(div_rn(mul_rn(cam.fy, t[1]), t[2]), cam.cy);
    S ca, cb, cc, r, ex, ey, tc;
    screen_shape(v[0][0], v[0][1], v[1][1], S(1), ca, cb, cc, r, ex, ey, tc);
    keep = add_rn(mx, r) >= S(-0.5) && sub_rn(mx, r) <= S(W) - S(0.5) && add_rn(my, r) >= S(-0.5) &&
           sub_rn(my, r) <= S(H) - S(0.5);
    mean2d[2 * k] = mx;
    mean2d[2 * k + 1] = my;
    cov2d[4 * k] = v[0][0];
    cov2d[4 * k + 1] = v[0][1];
    cov2d[4 * k + 2] = v[1][0];
    cov2d[4 * k + 3] = v[1][1];
    conic[3 * k] = ca;
    conic[3 * k + 1] = cb;
    conic[3 * k + 2] = cc;
    radius[k] = r;
  }
  kept[k] = keep;
}

// project_cloud_backward: thread per kept Gaussian, from its camera-space
// mean t (the forward's t_cam), its cov3d and the upstream (g_mean2d,
// g_cov2d) -> (g_mean3d, g_cov3d), render.py:364-402:
//   g_cov3d = M2^T G M2, g_M2 = (G + G^T) M2 Sigma, g_J = g_M2 R^T,
//   g_t through J and the mean projection, g_mean3d = g_t R.
template <typename S>
__global__ void __launch_bounds__(256) project_gaussians_backward(const S* __restrict__ t_cam,
                                                                  const S* __restrict__ cov3d, int64_t K,
                                                                  const __grid_constant__ Cam<S> cam,
                                                                  const S* __restrict__ g_mean2d,
                                                                  const S* __restrict__ g_cov2d,
                                                                  S* __restrict__ g_mean3d, S* __restrict__ g_cov3d) {
  pdl_wait();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  S t[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = t_cam[3 * k + i];
  S m2[2][3];
  cam_m2(cam, t, m2);
  const S* c = cov3d + 9 * k;
  const S G[2][2] = {{g_cov2d[4 * k], g_cov2d[4 * k + 1]}, {g_cov2d[4 * k + 2], g_cov2d[4 * k + 3]}};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      g_cov3d[9 * k + 3 * i + j] = G[0][0] * m2[0][i] * m2[0][j] + G[0][1] * m2[0][i] * m2[1][j] +
                                   G[1][0] * m2[1][i] * m2[0][j] + G[1][1] * m2[1][i] * m2[1][j];
  const S Gs[2][2] = {{G[0][0] + G[0][0], G[0][1] + G[1][0]}, {G[1][0] + G[0][1], G[1][1] + G[1][1]}};
  S ms[2][3];   // M2 Sigma
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) ms[r][j] = m2[r][0] * c[0 + j] + m2[r][1] * c[3 + j] + m2[r][2] * c[6 + j];
  S gM[2][3];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int j = 0; j < 3; ++j) gM[p][j] = Gs[p][0] * ms[0][j] + Gs[p][1] * ms[1][j];
  S gJ[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      gJ[r][j] = gM[r][0] * cam.R[3 * j] + gM[r][1] * cam.R[3 * j + 1] + gM[r][2] * cam.R[3 * j + 2];
  const S gm0 = g_mean2d[2 * k], gm1 = g_mean2d[2 * k + 1];
  const S iz = S(1) / t[2], iz2 = iz * iz;
  S gt0 = -cam.fx * iz2 * gJ[0][2] + gm0 * cam.fx * iz;
  S gt1 = -cam.fy * iz2 * gJ[1][2] + gm1 * cam.fy * iz;
  S gt2 = -cam.fx * iz2 * gJ[0][0] - cam.fy * iz2 * gJ[1][1] + S(2) * cam.fx * t[0] * iz2 * iz * gJ[0][2] +
          S(2) * cam.fy * t[1] * iz2 * iz * gJ[1][2] - gm0 * cam.fx * t[0] * iz2 - gm1 * cam.fy * t[1] * iz2;
#pragma unroll
  for (int j = 0; j < 3; ++j) g_mean3d[3 * k + j] = gt0 * cam.R[j] + gt1 * cam.R[3 + j] + gt2 * cam.R[6 + j];
}

}  // namespace gmr
