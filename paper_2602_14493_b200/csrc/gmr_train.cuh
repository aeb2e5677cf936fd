// gmr_train.cuh — device-resident optimisation step.
//
//   edge_length_loss  losses.py:76-97   (per-edge lengths, mean detached)
//   laplacian_loss    losses.py:100-123 (uniform Laplacian, exact gradient)
//   VectorAdam        optim.py:29-81    (per-vertex shared second moment)
//   ScalarAdam        optim.py:84-126   (+ colour clip to [0, 1], optim.py:292)
//
// All parameters and optimiser state are float64 like the reference; the
// float32 render copies are refreshed by the update.  Scatter-adds run as
// fixed-order gathers over static CSR tables (built once per topology), and
// reductions are fixed trees, so every step is bit-reproducible.
#pragma once

#include "gmr_common.cuh"

namespace gmr {

constexpr int kTrainThreads = 256;

// fixed-tree block sum of one double; thread 0 writes it
__device__ __forceinline__ void block_sum1(double a, double* out) {
  __shared__ double sa[kTrainThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) sa[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < kTrainThreads / 32; ++w) x += sa[w];
    *out = x;
  }
}

// single block: out[0] = sum of part[0..n) in a fixed order
__global__ void __launch_bounds__(kTrainThreads) sum_partials(const double* __restrict__ part, int n,
                                                             double* __restrict__ out) {
  pdl_wait();
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += kTrainThreads) a += part[i];
  block_sum1(a, out);
}

// per edge: vector b - a and length; block partial sums of the lengths
__global__ void __launch_bounds__(kTrainThreads) edge_lengths(const double* __restrict__ pos,
                                                             const int32_t* __restrict__ edges, int64_t E,
                                                             double* __restrict__ vec4, double* __restrict__ part) {
  pdl_wait();
  const int64_t e = (int64_t)blockIdx.x * kTrainThreads + threadIdx.x;
  double len = 0.0;
  if (e < E) {
    const int32_t a = edges[2 * e], b = edges[2 * e + 1];
    const double x = pos[3 * b] - pos[3 * a], y = pos[3 * b + 1] - pos[3 * a + 1], z = pos[3 * b + 2] - pos[3 * a + 2];
    len = sqrt(x * x + y * y + z * z);
    vec4[4 * e] = x; vec4[4 * e + 1] = y; vec4[4 * e + 2] = z; vec4[4 * e + 3] = len;
  }
  block_sum1(len, part + blockIdx.x);
}

// per edge: dev = len - mean; coeff = (2/E) dev / max(len, 1e-12) -> vec4 = coeff * vec;
// block partial sums of dev^2
__global__ void __launch_bounds__(kTrainThreads) edge_terms(double* __restrict__ vec4, int64_t E,
                                                           const double* __restrict__ len_sum,
                                                           double* __restrict__ part) {
  pdl_wait();
  const int64_t e = (int64_t)blockIdx.x * kTrainThreads + threadIdx.x;
  double d2 = 0.0;
  if (e < E) {
    const double mean = *len_sum / (double)E;
    const double len = vec4[4 * e + 3];
    const double dev = len - mean;
    d2 = dev * dev;
    const double coeff = (2.0 / (double)E) * dev / fmax(len, 1e-12);
    vec4[4 * e] *= coeff; vec4[4 * e + 1] *= coeff; vec4[4 * e + 2] *= coeff;
  }
  block_sum1(d2, part + blockIdx.x);
}

// Laplacian per vertex over the sorted neighbour CSR (mesh.py:114-126):
// lap = v - mean(neighbours); scaled = lap / max(deg, 1); block sums |lap|^2
__global__ void __launch_bounds__(kTrainThreads) laplacian_terms(const double* __restrict__ pos,
                                                                const int32_t* __restrict__ adj_ptr,
                                                                const int32_t* __restrict__ adj, int64_t V,
                                                                double* __restrict__ lap4, double* __restrict__ part) {
  pdl_wait();
  const int64_t v = (int64_t)blockIdx.x * kTrainThreads + threadIdx.x;
  double l2 = 0.0;
  if (v < V) {
    const int32_t b = adj_ptr[v], e = adj_ptr[v + 1];
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (int32_t k = b; k < e; ++k) {
      const int32_t u = adj[k];
      sx += pos[3 * u]; sy += pos[3 * u + 1]; sz += pos[3 * u + 2];
    }
    const int deg = e - b;
    double lx = 0.0, ly = 0.0, lz = 0.0;
    if (deg > 0) {
      lx = pos[3 * v] - sx / deg; ly = pos[3 * v + 1] - sy / deg; lz = pos[3 * v + 2] - sz / deg;
    }
    l2 = lx * lx + ly * ly + lz * lz;
    const double inv = 1.0 / fmax((double)deg, 1.0);
    lap4[4 * v] = lx; lap4[4 * v + 1] = ly; lap4[4 * v + 2] = lz; lap4[4 * v + 3] = inv;
  }
  block_sum1(l2, part + blockIdx.x);
}

struct RegArgs {
  const int32_t* ve_ptr;    // vertex -> (edge, endpoint) CSR in np.add.at order
  const int32_t* ve_slot;   // slot = 2 * edge + endpoint (endpoint 1: +, endpoint 0: -)
  const int32_t* adj_ptr;
  const int32_t* adj;
  const double* evec4;      // per edge: coeff * vec
  const double* lap4;       // per vertex: lap, 1 / max(deg, 1)
  int64_t V;
  double w_edge, w_lap;
};

// edge-length gradient of vertex v (losses.py:93-97): the np.add.at
// contributions of its (edge, endpoint) slots in scatter order
__device__ __forceinline__ void edge_grad(const RegArgs& r, int64_t v, double g[3]) {
  double ex = 0.0, ey = 0.0, ez = 0.0;
  for (int32_t k = r.ve_ptr[v]; k < r.ve_ptr[v + 1]; ++k) {
    const int32_t s = r.ve_slot[k];
    const double sg = (s & 1) ? 1.0 : -1.0;
    const double* ev = r.evec4 + 4 * (s >> 1);
    ex += sg * ev[0]; ey += sg * ev[1]; ez += sg * ev[2];
  }
  g[0] = ex; g[1] = ey; g[2] = ez;
}

// Laplacian gradient of vertex v (losses.py:117-123)
__device__ __forceinline__ void lap_grad(const RegArgs& r, int64_t v, double g[3]) {
  double bx = 0.0, by = 0.0, bz = 0.0;
  for (int32_t k = r.adj_ptr[v]; k < r.adj_ptr[v + 1]; ++k) {
    const double* lu = r.lap4 + 4 * r.adj[k];
    const bool has = r.adj_ptr[r.adj[k] + 1] > r.adj_ptr[r.adj[k]];
    if (has) { bx += lu[0] * lu[3]; by += lu[1] * lu[3]; bz += lu[2] * lu[3]; }
  }
  const double c = 2.0 / (double)r.V;
  const double* lv = r.lap4 + 4 * v;
  g[0] = c * lv[0] - c * bx;
  g[1] = c * lv[1] - c * by;
  g[2] = c * lv[2] - c * bz;
}

// per vertex: w_e * g_edge + w_l * g_lap
__device__ __forceinline__ void reg_grad(const RegArgs& r, int64_t v, double g[3]) {
  double ge[3], gl[3];
  edge_grad(r, v, ge);
  lap_grad(r, v, gl);
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = r.w_edge * ge[k] + r.w_lap * gl[k];
}

// the two regulariser gradients as separate [V,3] arrays (either may be null)
__global__ void __launch_bounds__(kTrainThreads) reg_grads(RegArgs r, double* __restrict__ g_edge,
                                                          double* __restrict__ g_lap) {
  pdl_wait();
  const int64_t v = (int64_t)blockIdx.x * kTrainThreads + threadIdx.x;
  if (v >= r.V) return;
  double g[3];
  if (g_edge) {
    edge_grad(r, v, g);
    g_edge[3 * v] = g[0]; g_edge[3 * v + 1] = g[1]; g_edge[3 * v + 2] = g[2];
  }
  if (g_lap) {
    lap_grad(r, v, g);
    g_lap[3 * v] = g[0]; g_lap[3 * v + 1] = g[1]; g_lap[3 * v + 2] = g[2];
  }
}

// values (edge, laplacian) = (sum dev^2 / E, sum |lap|^2 / V)
__global__ void reg_values(const double* __restrict__ sums, int64_t E, int64_t V, double* __restrict__ out) {
  pdl_wait();
  out[0] = E ? sums[1] / (double)E : 0.0;
  out[1] = sums[2] / (double)V;
}

// Image losses of the drop-in color_loss / silhouette_loss (losses.py:43-73),
// float64 like the reference: kind 0 = mean squared error of x against t
// with grad 2 (x - t) / n; kind 1 = clamped binary cross-entropy of alpha x
// against mask t with the clamp-gated grad.  Block partial sums of the
// per-element terms (fixed tree), then sum_partials in block order.
__global__ void __launch_bounds__(kTrainThreads) image_loss_terms(int kind, const double* __restrict__ x,
                                                                 const double* __restrict__ t, int64_t n,
                                                                 double* __restrict__ grad,
                                                                 double* __restrict__ part) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * kTrainThreads + threadIdx.x;
  double term = 0.0;
  if (i < n) {
    const double a = x[i], m = t[i];
    if (kind == 0) {
      const double d = a - m;
      term = d * d;
      grad[i] = (2.0 / (double)n) * d;
    } else {
      const double eps = 1e-6;   // losses.py:20
      const double q = fmin(fmax(a, eps), 1.0 - eps);
      term = -(m * log(q) + (1.0 - m) * log1p(-q));
      const bool inside = a > eps && a < 1.0 - eps;
      grad[i] = inside ? (-m / q + (1.0 - m) / (1.0 - q)) / (double)n : 0.0;
    }
  }
  block_sum1(term, part + blockIdx.x);
}

__global__ void scale_value(double* __restrict__ v, double s) {
  pdl_wait(); v[0] *= s; }

struct AdamArgs {
  double* pos;        // [V,3] float64 parameters (updated)
  double* col;        // [V,3]
  float* pos_f;       // float32 render copies (or null)
  float* col_f;
  const float* g_img_pos;   // [V,3] image-term gradients from the render backward
  const float* g_img_col;
  double* m_pos;      // [V,3]
  double* v_pos;      // [V]
  double* m_col;      // [V,3]
  double* v_col;      // [V,3]
  int64_t* counts;    // [2]: accepted steps (positions, colours)
  int* bad;           // [2]: non-finite gradient flags of this step
  double lr_pos, lr_col, beta1, beta2, eps;
  int optimize_colors;
  RegArgs reg;
  // scheduled mode (replayable): learning rates lr_sched[2 it], [2 it + 1]
  // at it = *iter, read on the device; null = lr_pos / lr_col above
  const double* lr_sched;
  int64_t* iter;
  // the status of the render that produced g_img_* (or null): a step whose
  // render overflowed its entry capacity or met a non-finite splat has no
  // valid image gradient and is rejected whole (the host then re-runs)
  const DevStatus* render_status;
};

__device__ __forceinline__ bool render_failed(const DevStatus* st) {
  if (!st) return false;
  bool bad = st->overflow != 0u;
#pragma unroll
  for (int i = 0; i < 6; ++i) bad |= st->bad_item[i] != 0xffffffffu;
  return bad;
}

__device__ __forceinline__ double sched_lr_pos(const AdamArgs& a) { return a.lr_sched ? a.lr_sched[2 * *a.iter] : a.lr_pos; }
__device__ __forceinline__ double sched_lr_col(const AdamArgs& a) { return a.lr_sched ? a.lr_sched[2 * *a.iter + 1] : a.lr_col; }

// pass 1: total gradients (image + regularisers) -> stash, non-finite flags
__global__ void __launch_bounds__(kTrainThreads) fit_grads(AdamArgs a, double* __restrict__ gpos,
                                                          double* __restrict__ gcol) {
  pdl_wait();
  const int64_t v = (int64_t)blockIdx.x * kTrainThreads + threadIdx.x;
  bool bp = false, bc = false;
  if (v < a.reg.V) {
    double gr[3];
    reg_grad(a.reg, v, gr);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double gp = (double)a.g_img_pos[3 * v + k] + gr[k];
      const double gc = (double)a.g_img_col[3 * v + k];
      gpos[3 * v + k] = gp;
      gcol[3 * v + k] = gc;
      bp |= !isfinite(gp);
      bc |= !isfinite(gc);
    }
  }
  const bool failed = render_failed(a.render_status);
  if (__syncthreads_or(bp || failed) && threadIdx.x == 0) atomicOr(&a.bad[0], 1);
  if (__syncthreads_or(bc || failed) && threadIdx.x == 0) atomicOr(&a.bad[1], 1);
}

// pass 2: VectorAdam on positions, ScalarAdam + clip on colours; a step
// with any non-finite gradient is rejected whole (optim.py:55-60, :103-106)
__global__ void __launch_bounds__(kTrainThreads) fit_update(AdamArgs a, const double* __restrict__ gpos,
                                                           const double* __restrict__ gcol) {
  pdl_wait();
  const int64_t v = (int64_t)blockIdx.x * kTrainThreads + threadIdx.x;
  if (v >= a.reg.V) return;
  const double lr_pos = sched_lr_pos(a), lr_col = sched_lr_col(a);
  if (!a.bad[0]) {
    const double t = (double)(a.counts[0] + 1);
    const double g0 = gpos[3 * v], g1 = gpos[3 * v + 1], g2 = gpos[3 * v + 2];
    const double vv = a.beta2 * a.v_pos[v] + (1.0 - a.beta2) * (g0 * g0 + g1 * g1 + g2 * g2);
    a.v_pos[v] = vv;
    const double v_hat = vv / (1.0 - pow(a.beta2, t));
    const double den = sqrt(v_hat) + a.eps;
    const double c1 = 1.0 - pow(a.beta1, t);
    const double gg[3] = {g0, g1, g2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double m = a.beta1 * a.m_pos[3 * v + k] + (1.0 - a.beta1) * gg[k];
      a.m_pos[3 * v + k] = m;
      const double p = a.pos[3 * v + k] + (-lr_pos * (m / c1) / den);
      a.pos[3 * v + k] = p;
      if (a.pos_f) a.pos_f[3 * v + k] = (float)p;
    }
  }
  if (a.optimize_colors && !a.bad[1]) {
    const double t = (double)(a.counts[1] + 1);
    const double c1 = 1.0 - pow(a.beta1, t), c2 = 1.0 - pow(a.beta2, t);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double g = gcol[3 * v + k];
      const double m = a.beta1 * a.m_col[3 * v + k] + (1.0 - a.beta1) * g;
      const double vv = a.beta2 * a.v_col[3 * v + k] + (1.0 - a.beta2) * g * g;
      a.m_col[3 * v + k] = m;
      a.v_col[3 * v + k] = vv;
      const double c = fmin(fmax(a.col[3 * v + k] - lr_col * (m / c1) / (sqrt(vv / c2) + a.eps), 0.0), 1.0);
      a.col[3 * v + k] = c;
      if (a.col_f) a.col_f[3 * v + k] = (float)c;
    }
  }
}

// pass 3: step counters, flags reset, the iteration's loss report
// history[it] = (total, color, silhouette, edge, laplacian); in scheduled
// mode `history` is the [iterations][5] base, row it = *iter, the render's
// 64-byte status is kept in statuses[it] and the counter advances last.
__global__ void fit_finish(AdamArgs a, const double* __restrict__ img_sums, double inv_nc, double inv_na,
                           double w_color, double w_sil, const double* __restrict__ edge_sum, int64_t E,
                           const double* __restrict__ lap_sum, double* __restrict__ history,
                           const uint32_t* __restrict__ status_src, uint32_t* __restrict__ statuses) {
  pdl_wait();
  const int64_t it = a.iter ? *a.iter : 0;
  if (status_src && statuses && threadIdx.x < 16) statuses[16 * it + threadIdx.x] = status_src[threadIdx.x];
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (!a.bad[0]) a.counts[0] += 1;
  if (a.optimize_colors && !a.bad[1]) a.counts[1] += 1;
  a.bad[0] = a.bad[1] = 0;
  const double color = img_sums[0] * inv_nc, sil = img_sums[1] * inv_na;
  const double edge = E ? *edge_sum / (double)E : 0.0;
  const double lap = *lap_sum / (double)a.reg.V;
  double* h = history + 5 * it;
  h[0] = w_color * color + w_sil * sil + a.reg.w_edge * edge + a.reg.w_lap * lap;
  h[1] = color;
  h[2] = sil;
  h[3] = edge;
  h[4] = lap;
  if (a.iter) *a.iter = it + 1;
}

}  // namespace gmr
