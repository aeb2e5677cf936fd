// gmr_eval.cuh — SURVEY §8f row 4: Gaussian export and evaluation metrics.
//
//   export_records   convert.py:444-532  export_gaussians (eigh -> scale/rotation, logit opacity, SH DC)
//   nn_partial/merge metrics.py:40-86    nearest surface sample (cKDTree query), Chamfer / normal consistency
//   surface_* etc.   mesh.py:560-622     sample_surface (area CDF, searchsorted, triangle fold)
//   ssim_* / sq_diff metrics.py:89-160   PSNR, SSIM (Gaussian windows, reflect borders)
//
// All float64, deterministic (fixed reduction orders, no atomics).
#pragma once

#include "gmr_common.cuh"

namespace gmr {

// ---------------------------------------------------------------------------
// export_gaussians
// ---------------------------------------------------------------------------

constexpr double kSz = 1e-6;              // convert.py:27
constexpr double kShDc = 0.28209479177387814;   // convert.py:29
constexpr double kOpacityClamp = 1e-6;    // convert.py:30

// Symmetric 3x3 eigendecomposition by cyclic Jacobi rotations (float64):
// a is overwritten, lam[k] / column k of v are an eigenpair.
__device__ __forceinline__ void jacobi_eigh3(double a[3][3], double lam[3], double v[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off == 0.0 || off <= 1e-300 || off <= scale * 1e-18) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = a[p][q];
      if (apq == 0.0) continue;
      const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
      const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
      for (int k = 0; k < 3; ++k) {   // A <- A J (columns p, q)
        const double akp = a[k][p], akq = a[k][q];
        a[k][p] = c * akp - s * akq;
        a[k][q] = s * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {   // A <- J^T A (rows p, q)
        const double apk = a[p][k], aqk = a[q][k];
        a[p][k] = c * apk - s * aqk;
        a[q][k] = s * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {   // V <- V J
        const double vkp = v[k][p], vkq = v[k][q];
        v[k][p] = c * vkp - s * vkq;
        v[k][q] = s * vkp + c * vkq;
      }
    }
  }
  lam[0] = a[0][0];
  lam[1] = a[1][1];
  lam[2] = a[2][2];
}

// Rotation matrix -> unit quaternion (w, x, y, z), w >= 0 (convert.py:444-481:
// branch on the trace / largest diagonal term).
__device__ __forceinline__ void rot_to_quat(const double m[3][3], double q[4]) {
  const double t = m[0][0] + m[1][1] + m[2][2];
  if (t > 0.0) {
    const double r = sqrt(1.0 + t) * 2.0;
    q[0] = 0.25 * r;
    q[1] = (m[2][1] - m[1][2]) / r;
    q[2] = (m[0][2] - m[2][0]) / r;
    q[3] = (m[1][0] - m[0][1]) / r;
  } else if (m[0][0] >= m[1][1] && m[0][0] >= m[2][2]) {
    const double r = sqrt(1.0 + m[0][0] - m[1][1] - m[2][2]) * 2.0;
    q[0] = (m[2][1] - m[1][2]) / r;
    q[1] = 0.25 * r;
    q[2] = (m[0][1] + m[1][0]) / r;
    q[3] = (m[0][2] + m[2][0]) / r;
  } else if (m[1][1] >= m[2][2]) {
    const double r = sqrt(1.0 + m[1][1] - m[0][0] - m[2][2]) * 2.0;
    q[0] = (m[0][2] - m[2][0]) / r;
    q[1] = (m[0][1] + m[1][0]) / r;
    q[2] = 0.25 * r;
    q[3] = (m[1][2] + m[2][1]) / r;
  } else {
    const double r = sqrt(1.0 + m[2][2] - m[0][0] - m[1][1]) * 2.0;
    q[0] = (m[1][0] - m[0][1]) / r;
    q[1] = (m[0][2] + m[2][0]) / r;
    q[2] = (m[1][2] + m[2][1]) / r;
    q[3] = 0.25 * r;
  }
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double sg = (q[0] / n < 0.0) ? -1.0 : 1.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = sg * (q[k] / n);
}

// One 56-byte little-endian record per Gaussian in the splat-viewer layout
// (convert.py:484-532): x y z, f_dc_0..2, opacity (logit), scale_0..2 (log),
// rot_0..3 -- all float32.
__global__ void __launch_bounds__(128) export_records(const double* __restrict__ means,
                                                      const double* __restrict__ cov3d,   // [n][3][3]
                                                      const double* __restrict__ colors,
                                                      const double* __restrict__ opacities, int64_t n,
                                                      float* __restrict__ rec) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a[3][3], lam[3], v[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) a[r][c] = cov3d[9 * i + 3 * r + c];
  // eigh reads the lower triangle: symmetrise from it
  a[0][1] = a[1][0];
  a[0][2] = a[2][0];
  a[1][2] = a[2][1];
  jacobi_eigh3(a, lam, v);
  // descending eigenvalues (convert.py:505-506)
  int ord[3] = {0, 1, 2};
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2 - x; ++y)
      if (lam[ord[y]] < lam[ord[y + 1]]) {
        const int t = ord[y];
        ord[y] = ord[y + 1];
        ord[y + 1] = t;
      }
  double R[3][3], L[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    L[k] = lam[ord[k]];
#pragma unroll
    for (int r = 0; r < 3; ++r) R[r][k] = v[r][ord[k]];
  }
  // proper rotation (convert.py:507-508)
  const double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
                     R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
                     R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
  if (det < 0.0) {
#pragma unroll
    for (int r = 0; r < 3; ++r) R[r][2] = -R[r][2];
  }
  double q[4];
  rot_to_quat(R, q);
  float* o = rec + 14 * i;
#pragma unroll
  for (int k = 0; k < 3; ++k) o[k] = (float)means[3 * i + k];
#pragma unroll
  for (int k = 0; k < 3; ++k) o[3 + k] = (float)((colors[3 * i + k] - 0.5) / kShDc);
  const double op = fmin(fmax(opacities[i], kOpacityClamp), 1.0 - kOpacityClamp);
  o[6] = (float)log(op / (1.0 - op));
#pragma unroll
  for (int k = 0; k < 3; ++k) o[7 + k] = (float)log(sqrt(fmax(L[k], kSz * kSz * 1e-2)));
#pragma unroll
  for (int k = 0; k < 4; ++k) o[10 + k] = (float)q[k];
}

// ---------------------------------------------------------------------------
// nearest sample (cKDTree(points).query(queries)): exact float64 brute force
// ---------------------------------------------------------------------------

constexpr int kNnThreads = 256;
constexpr int kNnQ = 2;          // queries per thread
constexpr int kNnTile = 512;     // points staged per smem round

// squared distance as cKDTree accumulates it: ((dx^2 + dy^2) + dz^2), no FMA
__device__ __forceinline__ double sqdist(double qx, double qy, double qz, double px, double py, double pz) {
  const double dx = __dsub_rn(qx, px), dy = __dsub_rn(qy, py), dz = __dsub_rn(qz, pz);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// grid (ceil(n / (256*2)), chunks): block y scans points [y*chunk, (y+1)*chunk)
// and writes its best (d2, index) per query; ties keep the lower index.
__global__ void __launch_bounds__(kNnThreads) nn_partial(const double* __restrict__ q, int64_t n,
                                                         const double* __restrict__ pts, int64_t m,
                                                         int64_t chunk, double* __restrict__ best_d,
                                                         int32_t* __restrict__ best_i) {
  pdl_wait();
  __shared__ double sx[kNnTile], sy[kNnTile], sz[kNnTile];
  const int64_t q0 = ((int64_t)blockIdx.x * kNnThreads) * kNnQ + threadIdx.x;
  double qx[kNnQ], qy[kNnQ], qz[kNnQ], bd[kNnQ];
  int32_t bi[kNnQ];
#pragma unroll
  for (int k = 0; k < kNnQ; ++k) {
    const int64_t qi = q0 + (int64_t)k * kNnThreads;
    const bool ok = qi < n;
    qx[k] = ok ? q[3 * qi] : 0.0;
    qy[k] = ok ? q[3 * qi + 1] : 0.0;
    qz[k] = ok ? q[3 * qi + 2] : 0.0;
    bd[k] = INFINITY;
    bi[k] = -1;
  }
  const int64_t p_lo = (int64_t)blockIdx.y * chunk, p_hi = min(m, p_lo + chunk);
  for (int64_t base = p_lo; base < p_hi; base += kNnTile) {
    const int cnt = (int)min((int64_t)kNnTile, p_hi - base);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kNnThreads) {
      sx[t] = pts[3 * (base + t)];
      sy[t] = pts[3 * (base + t) + 1];
      sz[t] = pts[3 * (base + t) + 2];
    }
    __syncthreads();
#pragma unroll 4
    for (int t = 0; t < cnt; ++t) {
      const double px = sx[t], py = sy[t], pz = sz[t];
#pragma unroll
      for (int k = 0; k < kNnQ; ++k) {
        const double d = sqdist(qx[k], qy[k], qz[k], px, py, pz);
        if (d < bd[k]) {
          bd[k] = d;
          bi[k] = (int32_t)(base + t);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kNnQ; ++k) {
    const int64_t qi = q0 + (int64_t)k * kNnThreads;
    if (qi < n) {
      best_d[(int64_t)blockIdx.y * n + qi] = bd[k];
      best_i[(int64_t)blockIdx.y * n + qi] = bi[k];
    }
  }
}

// merge the chunks in chunk order (strict <: the lowest index wins a tie),
// then per query: cKDTree's distance sqrt(d2), its square (metrics.py:48
// squares the returned distance), and |n_q . n_p| for normal consistency.
__global__ void __launch_bounds__(256) nn_merge(const double* __restrict__ best_d,
                                                const int32_t* __restrict__ best_i, int64_t n, int chunks,
                                                const double* __restrict__ qn, const double* __restrict__ pn,
                                                double* __restrict__ d2_out, double* __restrict__ cos_out,
                                                int32_t* __restrict__ idx_out) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double bd = best_d[i];
  int32_t bi = best_i[i];
  for (int c = 1; c < chunks; ++c) {
    const double d = best_d[(int64_t)c * n + i];
    if (d < bd) {
      bd = d;
      bi = best_i[(int64_t)c * n + i];
    }
  }
  const double dist = sqrt(bd);
  d2_out[i] = dist * dist;
  if (idx_out) idx_out[i] = bi;
  if (cos_out) {
    const double c = qn[3 * i] * pn[3 * (int64_t)bi] + qn[3 * i + 1] * pn[3 * (int64_t)bi + 1] +
                     qn[3 * i + 2] * pn[3 * (int64_t)bi + 2];
    cos_out[i] = fabs(c);
  }
}

// Deterministic sum of x[0..n) (fixed per-block order, then block sums in
// order by one block): out[0] = sum.
__global__ void __launch_bounds__(256) block_sums(const double* __restrict__ x, int64_t n,
                                                  double* __restrict__ partial) {
  pdl_wait();
  __shared__ double sh[256];
  double s = 0.0;
  const int64_t per = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += per) s += x[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void final_sum(const double* __restrict__ partial, int nb, double scale, double* __restrict__ out) {
  pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partial[b];
    *out = s * scale;
  }
}

// ---------------------------------------------------------------------------
// area-uniform surface samples (reference mesh.py:560-622), float64, with
// numpy's rounding: per-facet cross/norm/area/normal, the total as numpy's
// pairwise sum, the CDF as the sequential cumsum divided by the total, then
// per sample searchsorted(side='left') + the triangle fold.  The uniforms are
// the reference's Philox stream, drawn on the host.
// ---------------------------------------------------------------------------

constexpr double kDegenArea = 1e-12;   // mesh.py:15

__global__ void __launch_bounds__(256) surface_faces(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                                     int64_t F, double* __restrict__ area, double* __restrict__ nrm,
                                                     int32_t* __restrict__ fsorted) {
  pdl_wait();
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int32_t i0 = faces[3 * f], i1 = faces[3 * f + 1], i2 = faces[3 * f + 2];
  double e1[3], e2[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e1[k] = __dsub_rn(pos[3 * (int64_t)i1 + k], pos[3 * (int64_t)i0 + k]);
    e2[k] = __dsub_rn(pos[3 * (int64_t)i2 + k], pos[3 * (int64_t)i0 + k]);
  }
  const double c0 = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
  const double c1 = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
  const double c2 = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
  const double twice = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(c0, c0), __dmul_rn(c1, c1)), __dmul_rn(c2, c2)));
  const double a = 0.5 * twice;
  area[f] = a;
  if (a < kDegenArea) {   // placeholder normal (mesh.py:576)
    nrm[3 * f] = 0.0; nrm[3 * f + 1] = 0.0; nrm[3 * f + 2] = 1.0;
  } else {
    nrm[3 * f] = __ddiv_rn(c0, twice); nrm[3 * f + 1] = __ddiv_rn(c1, twice); nrm[3 * f + 2] = __ddiv_rn(c2, twice);
  }
  // np.sort(facets, axis=1)
  int32_t lo = min(i0, min(i1, i2)), hi = max(i0, max(i1, i2));
  fsorted[3 * f] = lo;
  fsorted[3 * f + 1] = i0 + i1 + i2 - lo - hi;
  fsorted[3 * f + 2] = hi;
}

// numpy pairwise_sum leaf (n <= 128): 8 accumulators, tree of the 8, tail
__device__ __forceinline__ double pw_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

constexpr int kPwMaxLeaves = 1 << 17;   // leaves hold >= 56 values: n <= 7M facets per call
constexpr int64_t kSurfaceMaxFaces = 7000000;
constexpr int kPwThreads = 1024;

// One block: (1) thread 0 walks numpy's split recursion and lists the
// leaves in order, (2) all threads sum the leaves, (3) thread 0 combines the
// leaf sums in the same recursion order.  out = total.
__global__ void __launch_bounds__(kPwThreads) pairwise_total(const double* __restrict__ a, int64_t n,
                                                             int64_t* __restrict__ leaf_off,
                                                             double* __restrict__ leaf_sum, double* __restrict__ out) {
  pdl_wait();
  __shared__ int nleaves;
  if (threadIdx.x == 0) {
    int cnt = 0;
    int64_t so[64], sn[64];
    int sp = 0;
    so[sp] = 0; sn[sp] = n; ++sp;
    while (sp) {
      --sp;
      const int64_t o = so[sp], m = sn[sp];
      if (m <= 128) {
        if (cnt < kPwMaxLeaves) leaf_off[cnt] = o;
        ++cnt;
        continue;
      }
      int64_t m2 = m / 2;
      m2 -= m2 % 8;
      // right pushed first so the left half is listed first
      so[sp] = o + m2; sn[sp] = m - m2; ++sp;
      so[sp] = o; sn[sp] = m2; ++sp;
    }
    nleaves = cnt;
  }
  __syncthreads();
  const int L = min(nleaves, kPwMaxLeaves);
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int64_t o = leaf_off[i], e = (i + 1 < L) ? leaf_off[i + 1] : n;
    leaf_sum[i] = pw_leaf(a + o, e - o);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // post-order combination: frame = (offset, n, state, left value)
    int64_t so[64], sn[64];
    int sstate[64];
    double sval[64];
    int sp = 0, leaf = 0;
    double ret = 0.0;
    so[0] = 0; sn[0] = n; sstate[0] = 0; sp = 1;
    while (sp) {
      const int t = sp - 1;
      const int64_t o = so[t], m = sn[t];
      if (m <= 128) {
        ret = leaf_sum[leaf++];
        --sp;
        continue;
      }
      int64_t m2 = m / 2;
      m2 -= m2 % 8;
      if (sstate[t] == 0) {            // descend left
        sstate[t] = 1;
        so[sp] = o; sn[sp] = m2; sstate[sp] = 0; ++sp;
      } else if (sstate[t] == 1) {     // left done: descend right
        sval[t] = ret;
        sstate[t] = 2;
        so[sp] = o + m2; sn[sp] = m - m2; sstate[sp] = 0; ++sp;
      } else {                         // both done
        ret = __dadd_rn(sval[t], ret);
        --sp;
      }
    }
    *out = ret;
  }
}

// prefix sums of area, sequential like np.cumsum (one thread: the rounding of
// every prefix depends on the previous one); the division by the total is
// elementwise and runs in parallel afterwards (cdf_divide)
__global__ void cumsum_seq(const double* __restrict__ area, int64_t n, double* __restrict__ cdf) {
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  int64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    const double4 v = *reinterpret_cast<const double4*>(area + i);   // 32-B aligned (workspace)
    double4 o;
    s = __dadd_rn(s, v.x); o.x = s;
    s = __dadd_rn(s, v.y); o.y = s;
    s = __dadd_rn(s, v.z); o.z = s;
    s = __dadd_rn(s, v.w); o.w = s;
    *reinterpret_cast<double4*>(cdf + i) = o;
  }
  for (; i < n; ++i) {
    s = __dadd_rn(s, area[i]);
    cdf[i] = s;
  }
}

__global__ void __launch_bounds__(256) cdf_divide(double* __restrict__ cdf, int64_t n,
                                                  const double* __restrict__ total) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cdf[i] = __ddiv_rn(cdf[i], *total);
}

__global__ void __launch_bounds__(256) surface_points(const double* __restrict__ pos,
                                                      const int32_t* __restrict__ fsorted,
                                                      const double* __restrict__ nrm, const double* __restrict__ cdf,
                                                      int64_t F, const double* __restrict__ u, int64_t n,
                                                      double* __restrict__ pts, double* __restrict__ out_n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double u0 = u[3 * i], u1 = u[3 * i + 1], u2 = u[3 * i + 2];
  // searchsorted(cdf, u0, side='left'): first index with cdf[k] >= u0
  int64_t lo = 0, hi = F;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] < u0) lo = mid + 1; else hi = mid;
  }
  const int64_t f = min(lo, F - 1);
  const bool fold = __dadd_rn(u1, u2) > 1.0;
  const double b1 = fold ? __dsub_rn(1.0, u1) : u1, b2 = fold ? __dsub_rn(1.0, u2) : u2;
  const int64_t a = fsorted[3 * f], b = fsorted[3 * f + 1], c = fsorted[3 * f + 2];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double pa = pos[3 * a + k];
    const double t = __dadd_rn(pa, __dmul_rn(b1, __dsub_rn(pos[3 * b + k], pa)));
    pts[3 * i + k] = __dadd_rn(t, __dmul_rn(b2, __dsub_rn(pos[3 * c + k], pa)));
    out_n[3 * i + k] = nrm[3 * f + k];
  }
}

// ---------------------------------------------------------------------------
// PSNR / SSIM (metrics.py:89-160)
// ---------------------------------------------------------------------------

constexpr int kSsimWin = 11;
constexpr int kSsimHalf = 5;

// scipy.ndimage 'reflect' (half-sample symmetric) index
__device__ __forceinline__ int reflect_idx(int i, int n) {
  if (n == 1) return 0;
  const int period = 2 * n;
  i %= period;
  if (i < 0) i += period;
  return i < n ? i : period - 1 - i;
}

// pass 1 (along rows of the image, axis 0 = v): for one channel, five maps
// x, y, x*x, y*y, x*y filtered along axis 0.  img [B,H,W,C]; tmp [B][5][H][W].
__global__ void __launch_bounds__(256) ssim_axis0(const double* __restrict__ a, const double* __restrict__ b,
                                                  int B, int H, int W, int C, int ch,
                                                  const double* __restrict__ kern, double* __restrict__ tmp) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t HW = (int64_t)H * W;
  if (idx >= (int64_t)B * HW) return;
  const int img = (int)(idx / HW);
  const int v = (int)((idx % HW) / W), u = (int)(idx % W);
  double s[5] = {0, 0, 0, 0, 0};
  for (int k = 0; k < kSsimWin; ++k) {
    const int vv = reflect_idx(v + k - kSsimHalf, H);
    const int64_t p = (((int64_t)img * H + vv) * W + u) * C + ch;
    const double x = a[p], y = b[p], w = kern[k];
    s[0] += w * x;
    s[1] += w * y;
    s[2] += w * (x * x);
    s[3] += w * (y * y);
    s[4] += w * (x * y);
  }
#pragma unroll
  for (int q = 0; q < 5; ++q) tmp[((int64_t)img * 5 + q) * HW + (int64_t)v * W + u] = s[q];
}

// pass 2 (axis 1 = u) + the SSIM map on the interior (border pixels whose
// window leaves the image are excluded, metrics.py:151); writes smap or 0.
__global__ void __launch_bounds__(256) ssim_axis1(const double* __restrict__ tmp, int B, int H, int W,
                                                  const double* __restrict__ kern, double c1, double c2,
                                                  double* __restrict__ smap) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t HW = (int64_t)H * W;
  if (idx >= (int64_t)B * HW) return;
  const int img = (int)(idx / HW);
  const int v = (int)((idx % HW) / W), u = (int)(idx % W);
  const bool interior = v >= kSsimHalf && v < H - kSsimHalf && u >= kSsimHalf && u < W - kSsimHalf;
  double out = 0.0;
  if (interior) {
    double s[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k < kSsimWin; ++k) {
      const int uu = reflect_idx(u + k - kSsimHalf, W);
      const double w = kern[k];
#pragma unroll
      for (int q = 0; q < 5; ++q) s[q] += w * tmp[((int64_t)img * 5 + q) * HW + (int64_t)v * W + uu];
    }
    const double mx = s[0], my = s[1];
    const double xx = s[2] - mx * mx, yy = s[3] - my * my, xy = s[4] - mx * my;
    const double num = (2 * mx * my + c1) * (2 * xy + c2);
    const double den = (mx * mx + my * my + c1) * (xx + yy + c2);
    out = num / den;
  }
  smap[idx] = out;
}

// per-image sums of `x` over [B][HW] (one block per image, fixed order)
__global__ void __launch_bounds__(256) image_sums(const double* __restrict__ x, int64_t HW, double scale,
                                                  double* __restrict__ out, int accumulate) {
  pdl_wait();
  __shared__ double sh[256];
  const double* p = x + (int64_t)blockIdx.x * HW;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < HW; i += blockDim.x) s += p[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (accumulate ? out[blockIdx.x] : 0.0) + sh[0] * scale;
}

// squared differences (for PSNR's MSE) into sq [B][H*W*C]
__global__ void __launch_bounds__(256) sq_diff(const double* __restrict__ a, const double* __restrict__ b,
                                               int64_t n, double* __restrict__ sq) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double d = a[i] - b[i];
    sq[i] = d * d;
  }
}

}  // namespace gmr
