// gmr_kernels.cuh — the GMR hot path as sm_100a CUDA kernels.
//
//   K1 mesh_to_splats      convert.py:239-276,321-326 + render.py:103-145
//   K1' pack_splats        render.py:168-188 (rasterize() stage input)
//   K2 depth sort -> count scan + entry emission -> tile sort -> tile_ranges
//                          render.py:200-229 (_RasterPlan)
//   K3 blend_forward       render.py:244-291
//   K4 blend_backward      render.py:294-361
//   K5 face_views_backward render.py:364-402 (+ conic->cov, :349-360)
//      face_convert_backward convert.py:393-425
//   K6 vertex_gather       convert.py:427-436 (np.add.at order, via CSR)
//
// Items: item = view * F + face (mesh path) or the splat index (splat path).
#pragma once

#include "gmr_common.cuh"
#include "radix_sort.cuh"

namespace gmr {

// ---------------------------------------------------------------------------
// status
// ---------------------------------------------------------------------------

__global__ void reset_status(DevStatus* st) {
  pdl_wait();
  st->entries = 0;
  st->kept = 0;
  for (int i = 0; i < 6; ++i) st->bad_item[i] = 0xffffffffu;
  st->overflow = 0;
  st->key_lo = 0xffffffffu;
  st->key_hi = 0u;
  st->max_bin = 0;
}

// min / max of the kept splats' 32-bit depth keys into the status (warp-
// aggregated); the global depth sort then runs only the passes their span
// needs (radix_sort.cuh KeyRange).  64-bit keys: no reduction.
__device__ __forceinline__ void note_key_range(DevStatus* st, uint32_t lo, uint32_t hi) {
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(&st->key_lo, lo);
    atomicMax(&st->key_hi, hi);
  }
}
__device__ __forceinline__ void note_key_range(DevStatus*, unsigned long long, unsigned long long) {}

__device__ __forceinline__ void flag_bad(DevStatus* st, int field, uint32_t item) {
  atomicMin(&st->bad_item[field], item);
}

// order-preserving key of a float / double (total order; -0 == +0)
__device__ __forceinline__ uint32_t order_key(float d) {
  if (d == 0.0f) d = 0.0f;
  uint32_t b = __float_as_uint(d);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ unsigned long long order_key(double d) {
  if (d == 0.0) d = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

// ---------------------------------------------------------------------------
// K1: facet -> Gaussian -> EWA projection -> cull -> screen record
// ---------------------------------------------------------------------------

// Facet geometry of the embed route, always in float64 like the reference
// (convert.py:239-276 runs in float64 whatever the render dtype; the render
// dtype only starts at projection, render.py:105,113).
struct FaceGeo {
  double e[3][3];      // e1 = b-a, e2 = c-a, e3 = c-b
  double n[3];         // unit normal (u / |u|, or u when degenerate)
  double nu;           // |u| (1 when degenerate)
  double area, kappa;
  double mean[3];
  bool degenerate, clamped;
};

template <typename S>
__device__ __forceinline__ void load_face(const S* __restrict__ pos, const int32_t* __restrict__ faces,
                                          int64_t f, int rescale, FaceGeo& g, int32_t idx[3]) {
  idx[0] = faces[3 * f + 0];
  idx[1] = faces[3 * f + 1];
  idx[2] = faces[3 * f + 2];
  double v[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int k = 0; k < 3; ++k) v[c][k] = (double)pos[3 * (int64_t)idx[c] + k];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g.e[0][k] = v[1][k] - v[0][k];
    g.e[1][k] = v[2][k] - v[0][k];
    g.e[2][k] = v[2][k] - v[1][k];
    g.mean[k] = (v[0][k] + v[1][k] + v[2][k]) / 3.0;
  }
  const double u0 = g.e[0][1] * g.e[1][2] - g.e[0][2] * g.e[1][1];
  const double u1 = g.e[0][2] * g.e[1][0] - g.e[0][0] * g.e[1][2];
  const double u2 = g.e[0][0] * g.e[1][1] - g.e[0][1] * g.e[1][0];
  const double nu = sqrt(u0 * u0 + u1 * u1 + u2 * u2);
  g.area = 0.5 * nu;
  g.degenerate = g.area < kDegenerateArea;
  g.nu = g.degenerate ? 1.0 : nu;
  g.n[0] = u0 / g.nu;
  g.n[1] = u1 / g.nu;
  g.n[2] = u2 / g.nu;
  const double det2d = g.area * g.area / 108.0;
  g.clamped = det2d < kDetEps;
  // convert.py:267 (== sqrt(108)/pi up to rounding when unclamped)
  g.kappa = rescale ? g.area / (kPi * sqrt(g.clamped ? kDetEps : det2d)) : 1.0;
}

// world cov3d (upper triangle xx,xy,xz,yy,yz,zz) of the embed route, float64
__device__ __forceinline__ void face_cov3d(const FaceGeo& g, double c[6]) {
  if (g.degenerate) {
    c[0] = c[3] = c[5] = kSz2;
    c[1] = c[2] = c[4] = 0.0;
    return;
  }
  const int ii[6] = {0, 0, 0, 1, 1, 2}, jj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const int i = ii[q], j = jj[q];
    const double c3 = (g.e[0][i] * g.e[0][j] + g.e[1][i] * g.e[1][j] + g.e[2][i] * g.e[2][j]) / 36.0;
    c[q] = g.kappa * c3 + kSz2 * g.n[i] * g.n[j];
  }
}

// cov2d = M2 Sigma M2^T in the render dtype (render.py:115-116)
template <typename S>
__device__ __forceinline__ void project_cov(const S m2[2][3], const S cv[6], S& a, S& b, S& c) {
  const S sg[3][3] = {{cv[0], cv[1], cv[2]}, {cv[1], cv[3], cv[4]}, {cv[2], cv[4], cv[5]}};
  S ms[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) ms[r][j] = m2[r][0] * sg[0][j] + m2[r][1] * sg[1][j] + m2[r][2] * sg[2][j];
  a = ms[0][0] * m2[0][0] + ms[0][1] * m2[0][1] + ms[0][2] * m2[0][2];
  b = ms[0][0] * m2[1][0] + ms[0][1] * m2[1][1] + ms[0][2] * m2[1][2];
  c = ms[1][0] * m2[1][0] + ms[1][1] * m2[1][1] + ms[1][2] * m2[1][2];
}

template <typename S>
__device__ __forceinline__ void cam_point(const Cam<S>& cam, const S p[3], S t[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    t[r] = cam.R[3 * r + 0] * p[0] + cam.R[3 * r + 1] * p[1] + cam.R[3 * r + 2] * p[2] + cam.t[r];
}

// M2 = J R (render.py:91-100,115)
template <typename S>
__device__ __forceinline__ void cam_m2(const Cam<S>& cam, const S t[3], S m2[2][3]) {
  const S iz = S(1) / t[2];
  const S j00 = cam.fx * iz, j02 = -cam.fx * t[0] * iz * iz;
  const S j11 = cam.fy * iz, j12 = -cam.fy * t[1] * iz * iz;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    m2[0][k] = j00 * cam.R[k] + j02 * cam.R[6 + k];
    m2[1][k] = j11 * cam.R[3 + k] + j12 * cam.R[6 + k];
  }
}

// Tiles of a splat's rectangle that its padded ellipse can reach (bit
// (ty - ty0) * w + (tx - tx0)), for rectangles of at most 32 tiles: a
// superset of the tiles whose blend coverage mask (tile_coverage, same rows,
// same padded half-widths) can be non-empty, so dropping the others changes
// no pixel and no gradient.  Entries of dropped tiles would be empty in both
// blend kernels anyway (the reference's _RasterPlan lists them,
// render.py:214-226; GMR_FLAG_FULL_TILE_LISTS keeps them).
constexpr int kMaskTiles = 32;
// sqrt for the conservative tile test only: float uses the MUFU
// approximation (relative error ~1e-7, far inside the 0.01 px extra padding)
__device__ __forceinline__ float mask_sqrt(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ double mask_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float mask_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ double mask_rcp(double x) { return 1.0 / x; }
template <typename S>
__device__ __forceinline__ uint32_t rect_tile_mask(const Splat<S>& sp, int tx0, int ty0, int tx1, int ty1) {
  const S mx = sp.a.x, my = sp.a.y, ca = sp.a.z, cb = sp.a.w, cc = sp.b.x, ex = sp.b.y, ey = sp.b.z, tau = sp.b.w;
  if (!(ex >= S(0)) || !(ca > S(0))) return 0u;   // never visible: tile_coverage marks nothing
  const int w = tx1 - tx0 + 1;
  const int area = w * (ty1 - ty0 + 1);
  const uint32_t full = area >= 32 ? 0xffffffffu : ((1u << area) - 1u);
  const S neg_det = cb * cb - ca * cc;
  if (!(neg_det < S(0)) || !(cc > S(0)) || !(tau >= S(0))) return full;   // not a proper ellipse: keep all
  // the rows tile_coverage solves: ceil(my - ey) .. floor(my + ey)
  const S y_lo = fmax(ceil(my - ey), S(ty0 * kTile)), y_hi = fmin(floor(my + ey), S(ty1 * kTile + kTile - 1));
  if (!(y_lo <= y_hi)) return 0u;
  const S inv_a = mask_rcp(ca);
  // Over a band of rows, the padded spans of tile_coverage lie inside
  // [Xmin - pad, Xmax + pad], where Xmin / Xmax are the extreme x of the
  // tau-ellipse clipped to the band.  The clipped ellipse is convex, so its
  // leftmost point is the ellipse's own leftmost point (row offset
  // dys = cb sqrt(tau / (det cc))) if inside the band, else on a band edge;
  // same for the right.  pad covers tile_coverage's 1.0005 h + 0.01, 0.01 px
  // more, and rounding; rows whose discriminant is only negative by
  // rounding are treated as touching.
  const S dys = cb * mask_sqrt(tau * mask_rcp(-neg_det * cc));
  const S pad = mask_sqrt(tau * inv_a) * S(0.0006) + S(0.03);
  const S x_min = S(tx0 * kTile), x_max = S(tx1 * kTile + kTile - 1);
  uint32_t m = 0;
  for (int tr = (int)y_lo >> 4; tr <= ((int)y_hi >> 4); ++tr) {
    const S ya = fmax(y_lo, S(tr * kTile)), yb = fmin(y_hi, S(tr * kTile + kTile - 1));
    S xl = S(INFINITY), xr = S(-INFINITY);
    auto probe = [&](S y, bool left, bool right) {
      const S dy = y - my;
      const S t1 = dy * dy * neg_det, t2 = ca * tau;
      const S disc = t1 + t2;
      if (!(disc >= S(-1e-5) * (fabs(t1) + fabs(t2)))) return;
      const S h = mask_sqrt(fmax(disc, S(0))) * inv_a;
      const S xc = mx - cb * dy * inv_a;
      if (left) xl = fmin(xl, xc - h);
      if (right) xr = fmax(xr, xc + h);
    };
    probe(ya, true, true);
    probe(yb, true, true);
    probe(fmin(fmax(my + dys, ya), yb), true, false);
    probe(fmin(fmax(my - dys, ya), yb), false, true);
    if (!(xl <= xr)) continue;                       // no row of the band meets the ellipse
    const S lo = fmax(ceil(xl - pad), x_min), hi = fmin(floor(xr + pad), x_max);
    if (!(lo <= hi)) continue;
    const int ta = ((int)lo >> 4) - tx0, tb = ((int)hi >> 4) - tx0;
    m |= ((0xffffffffu >> (31 - (tb - ta))) << ta) << ((tr - ty0) * w);
  }
  return m;
}

// per-item emitted-tile mask (bit = row-major index in the rectangle) of a
// rectangle of `area` tiles: all bits past 32 tiles, else culled or full;
// the entry count is item_count(mask, area)
template <typename S>
__device__ __forceinline__ uint32_t item_mask(const Splat<S>& sp, int tx0, int ty0, int tx1, int ty1, uint32_t area,
                                              bool cull) {
  if (area > (uint32_t)kMaskTiles) return 0xffffffffu;
  if (area == 1u || !cull) return 0xffffffffu >> (32 - area);
  return rect_tile_mask(sp, tx0, ty0, tx1, ty1);
}
__device__ __forceinline__ uint32_t item_count(uint32_t mask, uint32_t area) {
  return area > (uint32_t)kMaskTiles ? area : (uint32_t)__popc(mask);
}

// partial slot of an entry of `item` in tile (tx, ty): its rank among the
// item's emitted tiles (row-major over the rectangle)
__device__ __forceinline__ uint32_t entry_rank(uint2 rc, uint32_t mask, int tx, int ty) {
  const int tx0 = rc.x & 0xffff, ty0 = rc.x >> 16, tx1 = rc.y & 0xffff, ty1 = rc.y >> 16;
  const int w = tx1 - tx0 + 1;
  const uint32_t ri = (uint32_t)((ty - ty0) * w + (tx - tx0));
  if ((uint32_t)(w * (ty1 - ty0 + 1)) > (uint32_t)kMaskTiles) return ri;
  return (uint32_t)__popc(mask & ((1u << ri) - 1u));
}

template <typename S> struct MeshFwdArgs {
  const S* pos;
  const S* col;
  const int32_t* faces;
  int64_t F;
  int view0, nviews;
  int W, H, tiles_x, tiles_y;
  int rescale;
  Splat<S>* splat;
  V4<S>* col4;
  uint4* bin;        // [items]: (rect lo, rect hi, emitted-tile mask, entry count) -- one sector per gather
  uint32_t* count;   // [items]: entry count again, for the sequential readers
  typename KeyOf<S>::type* dkey;
  uint32_t* ditem;   // item ids for the global depth sort (null: per-tile depth order)
  int pack_shift;    // > 0: ditem = item | min(count, cmax) << pack_shift (cmax = all-ones above): scan_reduce needs no gather
  uint32_t* face_local;   // non-null (all views in this launch): the face's entries over all views, scanned per block
  uint32_t* face_bsum;    // ... and the block totals (what face_counts computes)
  int cull;          // drop tiles the splat cannot reach (not GMR_FLAG_FULL_TILE_LISTS)
  S* aux;   // optional [items][2] = (radius, depth)
  DevStatus* st;
};

template <typename S>
__global__ void __launch_bounds__(256) mesh_to_splats(MeshFwdArgs<S> p, const __grid_constant__ CamBatch<S> cams) {
  pdl_wait();
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = f < p.F;
  uint32_t kept = 0, fcnt = 0;
  typedef typename KeyOf<S>::type Key;
  Key klo = ~(Key)0, khi = 0;
  if (live) {
    FaceGeo g;
    int32_t idx[3];
    load_face(p.pos, p.faces, f, p.rescale, g, idx);
    if (p.view0 == 0) {
      V4<S> c;
      c.x = (p.col[3 * (int64_t)idx[0] + 0] + p.col[3 * (int64_t)idx[1] + 0] + p.col[3 * (int64_t)idx[2] + 0]) / S(3);
      c.y = (p.col[3 * (int64_t)idx[0] + 1] + p.col[3 * (int64_t)idx[1] + 1] + p.col[3 * (int64_t)idx[2] + 1]) / S(3);
      c.z = (p.col[3 * (int64_t)idx[0] + 2] + p.col[3 * (int64_t)idx[1] + 2] + p.col[3 * (int64_t)idx[2] + 2]) / S(3);
      c.w = S(1);  // opacity (convert.py:326)
      p.col4[f] = c;
    }
    // the float64 Gaussian, cast to the render dtype (render.py:105,113)
    double cov64[6];
    face_cov3d(g, cov64);
    S cov[6], mean[3];
#pragma unroll
    for (int q = 0; q < 6; ++q) cov[q] = (S)cov64[q];
#pragma unroll
    for (int q = 0; q < 3; ++q) mean[q] = (S)g.mean[q];
    for (int vv = 0; vv < p.nviews; ++vv) {
      const Cam<S>& cam = cams.cam[vv];
      const int64_t item = (int64_t)(p.view0 + vv) * p.F + f;
      S t[3];
      cam_point(cam, mean, t);
      Splat<S> rec;
      uint32_t cnt = 0, emask = 0;
      uint2 rc = make_uint2(0, 0);
      typename KeyOf<S>::type key = ~(typename KeyOf<S>::type)0;
      if (t[2] > cam.near_plane && t[2] < cam.far_plane) {
        S m2[2][3];
        cam_m2(cam, t, m2);
        S a, b, c;
        project_cov(m2, cov, a, b, c);
        a = add_rn(a, Const<S>::dilation());
        c = add_rn(c, Const<S>::dilation());
        const S mx = add_rn(div_rn(mul_rn(cam.fx, t[0]), t[2]), cam.cx);
        const S my = add_rn(div_rn(mul_rn(cam.fy, t[1]), t[2]), cam.cy);
        S ca, cb, cc, r, ex, ey, tc;
        screen_shape(a, b, c, S(1), ca, cb, cc, r, ex, ey, tc);
        const bool on = add_rn(mx, r) >= S(-0.5) && sub_rn(mx, r) <= S(p.W) - S(0.5) &&
                        add_rn(my, r) >= S(-0.5) && sub_rn(my, r) <= S(p.H) - S(0.5);
        rec.a.x = mx; rec.a.y = my; rec.a.z = ca; rec.a.w = cb;
        rec.b.x = cc; rec.b.y = ex; rec.b.z = ey; rec.b.w = tc;
        if (p.aux) {
          p.aux[2 * item] = r;
          p.aux[2 * item + 1] = t[2];
        }
        if (on) {
          int tx0, ty0, tx1, ty1;
          tile_rect(mx, my, r, p.tiles_x, p.tiles_y, tx0, ty0, tx1, ty1);
          const uint32_t area = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
          emask = item_mask(rec, tx0, ty0, tx1, ty1, area, p.cull != 0);
          cnt = item_count(emask, area);
          rc = make_uint2((uint32_t)tx0 | ((uint32_t)ty0 << 16), (uint32_t)tx1 | ((uint32_t)ty1 << 16));
          key = order_key(t[2]);
          klo = min(klo, key);
          khi = max(khi, key);
          ++kept;
          // render.py:191-197 on kept splats
          if (!(finite_s(mx) && finite_s(my))) flag_bad(p.st, 0, (uint32_t)item);
          if (!(finite_s(a) && finite_s(b) && finite_s(c))) flag_bad(p.st, 1, (uint32_t)item);
          if (!(finite_s(ca) && finite_s(cb) && finite_s(cc))) flag_bad(p.st, 2, (uint32_t)item);
          if (!finite_s(t[2])) flag_bad(p.st, 3, (uint32_t)item);
        }
      } else {
        rec.a.x = rec.a.y = rec.a.z = rec.a.w = S(0);
        rec.b.x = S(0); rec.b.y = rec.b.z = S(-1); rec.b.w = S(0);
        if (p.aux) {
          p.aux[2 * item] = S(NAN);
          p.aux[2 * item + 1] = t[2];
        }
      }
      p.splat[item] = rec;
      p.bin[item] = make_uint4(rc.x, rc.y, emask, cnt);
      p.count[item] = cnt;
      fcnt += cnt;
      p.dkey[item] = key;
      if (p.ditem)
        p.ditem[item] = p.pack_shift ? ((uint32_t)item | (min(cnt, 0xffffffffu >> p.pack_shift) << p.pack_shift))
                                     : (uint32_t)item;
    }
  }
  note_key_range(p.st, klo, khi);
  // warp-aggregated kept count
  uint32_t tot = kept;
#pragma unroll
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(&p.st->kept, (unsigned long long)tot);
  if (p.face_local) {   // face-major partial offsets, first step (face_counts fused)
    __shared__ uint32_t sw[8];
    uint32_t btot;
    const uint32_t ex = block_exclusive_scan_256(fcnt, sw, &btot);
    if (live) p.face_local[f] = ex;
    if (threadIdx.x == 0) p.face_bsum[blockIdx.x] = btot;
  }
}

// K1' — splat path: records from given (mean2d, cov2d, depth, color, opacity)
template <typename S> struct PackArgs {
  const S* mean2d;
  const S* cov2d;
  const S* depth;
  const S* color;
  const S* opacity;
  int64_t K;
  int tiles_x, tiles_y;
  Splat<S>* splat;
  V4<S>* col4;
  uint4* bin;
  uint32_t* count;
  typename KeyOf<S>::type* dkey;
  uint32_t* ditem;   // item ids for the global depth sort (null: per-tile depth order)
  int cull;
  DevStatus* st;
};

template <typename S>
__global__ void __launch_bounds__(256) pack_splats(PackArgs<S> p) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.K) return;
  const S mx = p.mean2d[2 * i], my = p.mean2d[2 * i + 1];
  const S a = p.cov2d[4 * i], b = p.cov2d[4 * i + 1], c = p.cov2d[4 * i + 3];
  const S o = p.opacity[i], d = p.depth[i];
  V4<S> col;
  col.x = p.color[3 * i]; col.y = p.color[3 * i + 1]; col.z = p.color[3 * i + 2]; col.w = o;
  S ca, cb, cc, r, ex, ey, tc;
  screen_shape(a, b, c, o, ca, cb, cc, r, ex, ey, tc);
  Splat<S> rec;
  rec.a.x = mx; rec.a.y = my; rec.a.z = ca; rec.a.w = cb;
  rec.b.x = cc; rec.b.y = ex; rec.b.z = ey; rec.b.w = tc;
  const uint32_t item = (uint32_t)i;
  if (!(finite_s(mx) && finite_s(my))) flag_bad(p.st, 0, item);
  if (!(finite_s(a) && finite_s(b) && finite_s(c) && finite_s(p.cov2d[4 * i + 2]))) flag_bad(p.st, 1, item);
  if (!(finite_s(ca) && finite_s(cb) && finite_s(cc))) flag_bad(p.st, 2, item);
  if (!finite_s(d)) flag_bad(p.st, 3, item);
  if (!(finite_s(col.x) && finite_s(col.y) && finite_s(col.z))) flag_bad(p.st, 4, item);
  if (!finite_s(o)) flag_bad(p.st, 5, item);
  int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
  if (finite_s(mx) && finite_s(my) && finite_s(r))
    tile_rect(mx, my, r, p.tiles_x, p.tiles_y, tx0, ty0, tx1, ty1);
  const bool has_rect = tx1 >= tx0 && ty1 >= ty0;
  const uint32_t area = has_rect ? (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1)) : 0u;
  const uint32_t emask = has_rect ? item_mask(rec, tx0, ty0, tx1, ty1, area, p.cull != 0) : 0u;
  const uint32_t cnt = has_rect ? item_count(emask, area) : 0u;
  p.splat[i] = rec;
  p.col4[i] = col;
  p.bin[i] = make_uint4((uint32_t)tx0 | ((uint32_t)ty0 << 16), (uint32_t)max(tx1, 0) | ((uint32_t)max(ty1, 0) << 16),
                        emask, cnt);
  p.count[i] = cnt;
  p.dkey[i] = order_key(d);
  if (p.ditem) p.ditem[i] = item;
  if (has_rect) atomicAdd(&p.st->kept, 1ull);
}

// ---------------------------------------------------------------------------
// K2: counts -> offsets -> entries -> (view, tile) sort -> ranges -> per-bin depth sort
// ---------------------------------------------------------------------------

constexpr int kScanTile = 256;   // one splat per thread

// Block totals of the entry counts, kScanTile items each, kReduceTiles tiles
// per block: every thread's loads are issued together (the reads are short
// and latency-bound), then each tile is summed by a fixed-order block tree.
constexpr int kReduceTiles = 4;
#ifndef GMR_EMIT_TILES
#define GMR_EMIT_TILES 2
#endif
constexpr int kEmitTiles = GMR_EMIT_TILES;
__global__ void __launch_bounds__(256) scan_reduce(const uint32_t* order, const uint32_t* order_alt,
                                                  const uint32_t* krange, int key_bits,
                                                  const uint32_t* __restrict__ count, uint32_t n,
                                                  uint32_t* __restrict__ bsum, int pack_shift) {
  pdl_wait();
  __shared__ uint32_t sw[kReduceTiles][8];
  if (krange) order = result_buffer(order, order_alt, krange, key_bits);
  uint32_t s[kReduceTiles];
#pragma unroll
  for (int t = 0; t < kReduceTiles; ++t) {
    const uint32_t i = (blockIdx.x * kReduceTiles + t) * (uint32_t)kScanTile + threadIdx.x;
    s[t] = 0u;
    if (i < n) {
      const uint32_t v = order ? order[i] : i;
      if (pack_shift && order) {   // the count rides in the sorted value (no gather) unless saturated
        const uint32_t c = v >> pack_shift, cmax = 0xffffffffu >> pack_shift;
        s[t] = c < cmax ? c : count[v & ((1u << pack_shift) - 1u)];
      } else {
        s[t] = count[v];
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < kReduceTiles; ++t) {
    uint32_t x = s[t];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sw[t][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < kReduceTiles) {
    const uint32_t tile = blockIdx.x * kReduceTiles + threadIdx.x;
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += sw[threadIdx.x][w];
    if ((uint64_t)tile * kScanTile < n) bsum[tile] = tot;
  }
}

// Exclusive scan of n uint32 in place by one 1024-thread block: thread t
// owns a contiguous run, one block scan of the run totals (64-bit carry).
// Returns the total (thread 0 of the caller's block sees it).
constexpr int kTopThreads = 1024;
__device__ __forceinline__ unsigned long long scan_runs_inplace(uint32_t* __restrict__ a, int n) {
  __shared__ unsigned long long wsum[kTopThreads / 32];
  // runs of a multiple of 4 elements: 16-byte loads and stores (a is
  // 16-byte aligned: workspace buffers are 256-byte aligned)
  const int per = (((n + kTopThreads - 1) / kTopThreads) + 3) & ~3;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  unsigned long long s = 0;
  int i = lo;
  for (; i + 4 <= hi; i += 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(a + i);
    s += (unsigned long long)v.x + v.y + v.z + v.w;
  }
  for (; i < hi; ++i) s += a[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  unsigned long long wp = 0, tot = 0;
  for (int w = 0; w < kTopThreads / 32; ++w) {
    const unsigned long long t = wsum[w];
    wp += (w < warp) ? t : 0ull;
    tot += t;
  }
  unsigned long long run = wp + x - s;
  i = lo;
  for (; i + 4 <= hi; i += 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(a + i);
    uint4 o;
    o.x = (uint32_t)run; run += v.x;
    o.y = (uint32_t)run; run += v.y;
    o.z = (uint32_t)run; run += v.z;
    o.w = (uint32_t)run; run += v.w;
    *reinterpret_cast<uint4*>(a + i) = o;
  }
  for (; i < hi; ++i) {
    const uint32_t v = a[i];
    a[i] = (uint32_t)run;
    run += v;
  }
  return tot;
}

__global__ void __launch_bounds__(kTopThreads) scan_top(uint32_t* __restrict__ bsum, int nb, DevStatus* st,
                                                       unsigned long long capacity, uint32_t* n_entries) {
  pdl_wait();
  const unsigned long long carry = scan_runs_inplace(bsum, nb);
  if (threadIdx.x == 0) {
    st->entries = carry;
    const bool over = carry > capacity || carry > 0xffffffffull;
    st->overflow = over ? 1u : 0u;
    *n_entries = over ? 0u : (uint32_t)carry;
  }
}

// Entry emission: per splat in `order` (item order when null; one per
// thread; block scan + the block's carry from scan_top), write its tile
// entries row-major over its rectangle (render.py:218-226): key = view * T +
// tile, value = item.  Skipped when the entries overflow.
__global__ void __launch_bounds__(256) scan_emit(const uint32_t* order, const uint32_t* order_alt,
                                                const uint32_t* krange, int key_bits,
                                                const uint4* __restrict__ bin, uint32_t n,
                                                const uint32_t* __restrict__ bsum,
                                                uint32_t items_per_view, int tiles_x,
                                                uint32_t tiles_per_view,
                                                const uint32_t* __restrict__ n_entries,
                                                uint32_t* __restrict__ key, uint32_t* __restrict__ val, int pack_shift) {
  pdl_wait();
  __shared__ uint32_t sw[8];
  if (krange) order = result_buffer(order, order_alt, krange, key_bits);
  // kEmitTiles tiles of kScanTile items per block: every tile's gathers are
  // issued before the first scan
  uint32_t items[kEmitTiles];
  uint4 bis[kEmitTiles];
#pragma unroll
  for (int t = 0; t < kEmitTiles; ++t) {
    const uint32_t i = (blockIdx.x * kEmitTiles + t) * (uint32_t)kScanTile + threadIdx.x;
    items[t] = i < n ? (order ? (pack_shift ? order[i] & ((1u << pack_shift) - 1u) : order[i]) : i) : 0u;
  }
#pragma unroll
  for (int t = 0; t < kEmitTiles; ++t) {
    const uint32_t i = (blockIdx.x * kEmitTiles + t) * (uint32_t)kScanTile + threadIdx.x;
    bis[t] = i < n ? bin[items[t]] : make_uint4(0, 0, 0, 0);
  }
  const uint32_t ne = *n_entries;
#pragma unroll
  for (int t = 0; t < kEmitTiles; ++t) {
    const uint32_t tile = blockIdx.x * kEmitTiles + t;
    if ((uint64_t)tile * kScanTile >= n) break;   // block-uniform
    const uint32_t i = tile * (uint32_t)kScanTile + threadIdx.x;
    const uint32_t item = items[t];
    const uint4 bi = bis[t];
    const uint32_t c = bi.w;
    const uint32_t run = bsum[tile] + block_exclusive_scan_256(c, sw, nullptr);
    if (i >= n || !c || ne == 0) continue;
    const uint2 rc = make_uint2(bi.x, bi.y);
    const int tx0 = rc.x & 0xffff, ty0 = rc.x >> 16, tx1 = rc.y & 0xffff, ty1 = rc.y >> 16;
    const int w = tx1 - tx0 + 1;
    const uint32_t vbase = (item / items_per_view) * tiles_per_view;
    if ((uint32_t)(w * (ty1 - ty0 + 1)) > (uint32_t)kMaskTiles) {
      int tx = tx0, ty = ty0;
      for (uint32_t e = 0; e < c; ++e) {
        key[run + e] = vbase + (uint32_t)(ty * tiles_x + tx);
        val[run + e] = item;
        if (++tx > tx1) { tx = tx0; ++ty; }
      }
    } else {
      // the rectangle's kept tiles, row-major (entry_rank order)
      uint32_t m = bi.z, e = 0;
      while (m) {
        const int ri = __ffs(m) - 1;
        m &= m - 1;
        key[run + e] = vbase + (uint32_t)((ty0 + ri / w) * tiles_x + tx0 + ri % w);
        val[run + e] = item;
        ++e;
      }
    }
  }
}

// Face-major layout of the per-entry gradient partials: all entries of face
// f (views 0..B-1, each row-major over its rectangle) are contiguous at
// entry_off[v * F + f], so K5 streams one range per face.
__global__ void __launch_bounds__(256) face_counts(const uint32_t* __restrict__ count, uint32_t F, int B,
                                                  uint32_t* __restrict__ face_local,
                                                  uint32_t* __restrict__ bsum) {
  pdl_wait();
  __shared__ uint32_t sw[8];
  const uint32_t f = blockIdx.x * 256u + threadIdx.x;
  uint32_t s = 0;
  if (f < F)
    for (int v = 0; v < B; ++v) s += count[(size_t)v * F + f];
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan_256(s, sw, &tot);
  if (f < F) face_local[f] = ex;
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// single-block exclusive scan in place
__global__ void __launch_bounds__(kTopThreads) scan_inplace(uint32_t* __restrict__ a, int n) {
  pdl_wait();
  scan_runs_inplace(a, n);
}

__global__ void __launch_bounds__(256) item_offsets(const uint32_t* __restrict__ count, uint32_t F, int B,
                                                   const uint32_t* __restrict__ face_local,
                                                   const uint32_t* __restrict__ bsum,
                                                   uint32_t* __restrict__ entry_off) {
  pdl_wait();
  const uint32_t f = blockIdx.x * 256u + threadIdx.x;
  if (f >= F) return;
  uint32_t run = bsum[blockIdx.x] + face_local[f];
  for (int v = 0; v < B; ++v) {
    const size_t item = (size_t)v * F + f;
    entry_off[item] = run;
    run += count[item];
  }
}

// bounds[g] = first entry with key >= g (searchsorted left, render.py:229)
__global__ void __launch_bounds__(256) tile_ranges(const uint32_t* __restrict__ key,
                                                  const uint32_t* n_dev, uint32_t n_host,
                                                  uint32_t num_bins, uint32_t* __restrict__ bounds,
                                                  uint32_t* __restrict__ sched_cnt) {
  pdl_wait();
  if (sched_cnt && blockIdx.x == 0)
    for (int i = threadIdx.x; i < 513; i += blockDim.x) sched_cnt[i] = 0u;
  // four positions per thread (one 16-byte load; key buffers are 256-B aligned)
  const uint32_t n = n_dev ? *n_dev : n_host;
  const uint32_t s0 = 4u * (blockIdx.x * blockDim.x + threadIdx.x);
  if (s0 > n) return;
  uint32_t k[4];
  if (s0 + 4 <= n) {
    const uint4 v = *reinterpret_cast<const uint4*>(key + s0);
    k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) k[q] = (s0 + q < n) ? key[s0 + q] : num_bins;
  }
  // bounds[g] = first position whose key >= g: position s starts every bin in
  // (key[s-1], key[s]] (keys past n read as num_bins)
  uint32_t prev_plus = s0 > 0 ? key[s0 - 1] + 1u : 0u;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t s = s0 + q;
    if (s > n) break;
    const uint32_t cur = min(k[q], num_bins);
    for (uint32_t g = prev_plus; g <= cur; ++g) bounds[g] = s;
    prev_plus = max(prev_plus, cur + 1u);
  }
}

// Blend schedule: bins ordered by decreasing entry count (bucketed), so the
// heaviest tiles start first and the last wave holds the lightest ones.
// The order within a bucket is arbitrary (atomics); every tile's result is
// independent of when it runs.
constexpr int kSchedThreads = 1024;
__device__ __forceinline__ uint32_t sched_bucket(uint32_t cnt) { return 255u - min(cnt >> 3, 255u); }

__global__ void __launch_bounds__(kSchedThreads) tile_schedule(const uint32_t* __restrict__ bounds, uint32_t bins,
                                                               uint32_t* __restrict__ order, DevStatus* st) {
  pdl_wait();
  __shared__ uint32_t hist[256];
  __shared__ uint32_t longest;
  for (int i = threadIdx.x; i < 256; i += kSchedThreads) hist[i] = 0;
  if (threadIdx.x == 0) longest = 0;
  __syncthreads();
  uint32_t mx = 0;
  for (uint32_t g = threadIdx.x; g < bins; g += kSchedThreads) {
    const uint32_t c = bounds[g + 1] - bounds[g];
    mx = max(mx, c);
    atomicAdd(&hist[sched_bucket(c)], 1u);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(&longest, mx);
  __syncthreads();
  if (threadIdx.x == 0) st->max_bin = longest;
  if (threadIdx.x < 32) {   // exclusive scan of the 256 buckets by one warp
    uint32_t v[8], s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { v[k] = hist[threadIdx.x * 8 + k]; s += v[k]; }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)threadIdx.x >= o) x += y;
    }
    uint32_t run = x - s;
#pragma unroll
    for (int k = 0; k < 8; ++k) { hist[threadIdx.x * 8 + k] = run; run += v[k]; }
  }
  __syncthreads();
  for (uint32_t g = threadIdx.x; g < bins; g += kSchedThreads)
    order[atomicAdd(&hist[sched_bucket(bounds[g + 1] - bounds[g])], 1u)] = g;
}

// The same schedule over the whole grid (many bins): sched_hist counts the
// bins per bucket and the longest list with global atomics, sched_place
// gives every bin its position (each block scans the 256 bucket counts
// itself; the order within a bucket is arbitrary, as above).  cnt[0..256)
// bucket counts, cnt[256..512) cursors, cnt[512] longest: zeroed by
// tile_ranges' first thread block.
__global__ void __launch_bounds__(256) sched_hist(const uint32_t* __restrict__ bounds, uint32_t bins,
                                                 uint32_t* __restrict__ cnt) {
  pdl_wait();
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t g = blockIdx.x * 256u + threadIdx.x;
  uint32_t c = 0;
  if (g < bins) {
    c = bounds[g + 1] - bounds[g];
    atomicAdd(&h[sched_bucket(c)], 1u);
  }
  c = __reduce_max_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicMax(&cnt[512], c);
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], h[threadIdx.x]);
}
__global__ void __launch_bounds__(256) sched_place(const uint32_t* __restrict__ bounds, uint32_t bins,
                                                  uint32_t* __restrict__ cnt, uint32_t* __restrict__ order,
                                                  DevStatus* st) {
  pdl_wait();
  __shared__ uint32_t start[256], h[256];
  h[threadIdx.x] = 0;
  if (threadIdx.x < 32) {   // exclusive scan of the 256 bucket counts (8 per lane)
    uint32_t v[8], s8 = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { v[k] = cnt[threadIdx.x * 8 + k]; s8 += v[k]; }
    uint32_t x = s8;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)threadIdx.x >= o) x += y;
    }
    uint32_t run = x - s8;
#pragma unroll
    for (int k = 0; k < 8; ++k) { start[threadIdx.x * 8 + k] = run; run += v[k]; }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) st->max_bin = cnt[512];
  const uint32_t g = blockIdx.x * 256u + threadIdx.x;
  uint32_t b = 0, r = 0;
  if (g < bins) {
    b = sched_bucket(bounds[g + 1] - bounds[g]);
    r = atomicAdd(&h[b], 1u);   // rank inside this block's share of the bucket
  }
  __syncthreads();
  if (h[threadIdx.x]) start[threadIdx.x] += atomicAdd(&cnt[256 + threadIdx.x], h[threadIdx.x]);
  __syncthreads();
  if (g < bins) order[start[b] + r] = g;
}

// ---------------------------------------------------------------------------
// K2'': per-bin depth order (render.py:227 lexsort by (tile, depth, source)).
// Entries are emitted in item order and the (view, tile) radix sort is
// stable, so every bin's list arrives in source order.  A stable LSD radix
// sort of each bin by its depth key then yields (tile, depth, source) — the
// order a global depth sort of all B*F items before emission gives
// (GMR_FLAG_TILE_DEPTH_SORT; the default is that global sort).  One CTA per
// bin.
// The digits are those of key - (the bin's smallest key), so a bin needs
// only as many passes as its depth range has bytes.  Bins of up to BinSortCap entries are ranked in
// shared memory; larger ones ping-pong through global scratch (the
// backward's partial buffer, unused until the backward) in chunks.
// ---------------------------------------------------------------------------

constexpr int kBinSortThreads = 256;   // thread t owns digit t
constexpr int kBinSortWarps = kBinSortThreads / 32;
template <typename K> struct BinSortCap { static constexpr int value = sizeof(K) == 4 ? 2048 : 1024; };

template <typename K> struct BinSortSmem {
  static constexpr int kCap = BinSortCap<K>::value;
  K key[2][kCap];
  uint32_t val[2][kCap];
  uint32_t cnt[kBinSortWarps][256];
  uint32_t sw[kBinSortWarps];
  K red_min[kBinSortWarps], red_max[kBinSortWarps];
};

// One stable pass on the 8-bit digit of (key - kmin) at `shift`: src -> dst
// (shared or global).  Chunks of up to kCap elements in order; in a chunk
// warp w ranks a contiguous segment (ballot-built digit groups; the group leader
// owns the warp's running digit count), so the output keeps the input order
// within each digit.
template <typename K>
__device__ __forceinline__ void bin_digit_pass(const K* sk, const uint32_t* sv, K* dk, uint32_t* dv, uint32_t n,
                                               int shift, K kmin, BinSortSmem<K>& sm) {
  constexpr int kCap = BinSortSmem<K>::kCap;
  constexpr int kGroups = kCap / kBinSortThreads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = lanemask_lt_sort();
  uint32_t run = 0;   // running output offset of digit tid
  const bool multi = n > (uint32_t)kCap;
  if (multi) {   // digit bases over the whole bin first
    sm.cnt[0][tid] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kBinSortThreads)
      atomicAdd(&sm.cnt[0][(uint32_t)((sk[i] - kmin) >> shift) & 255u], 1u);
    __syncthreads();
    run = block_exclusive_scan_256(sm.cnt[0][tid], sm.sw, nullptr);
  }
  for (uint32_t c0 = 0; c0 < n; c0 += kCap) {
    const uint32_t m = min((uint32_t)kCap, n - c0);
    const uint32_t seg = ((m + kBinSortThreads - 1) / kBinSortThreads) * 32;   // per warp, multiple of 32
#pragma unroll
    for (int w = 0; w < kBinSortWarps; ++w) sm.cnt[w][tid] = 0;
    __syncthreads();
    uint32_t dr[kGroups];   // digit << 16 | rank in the warp's digit run; ~0 = none
    const uint32_t w0 = c0 + warp * seg;
#pragma unroll
    for (int j = 0; j < kGroups; ++j) {
      dr[j] = 0xffffffffu;
      if (32u * j < seg) {   // warp-uniform
        const uint32_t i = w0 + 32 * j + lane;
        const bool valid = i < c0 + m;
        const uint32_t d = valid ? (uint32_t)((sk[i] - kmin) >> shift) & 255u : 256u;
        const unsigned peers = digit_peers_ballot(d);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (valid && lane == leader) {
          old = sm.cnt[warp][d];
          sm.cnt[warp][d] = old + (uint32_t)__popc(peers);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        __syncwarp();
        if (valid) dr[j] = (d << 16) | (old + (uint32_t)__popc(peers & lt));
      }
    }
    __syncthreads();
    uint32_t pre[kBinSortWarps], tot = 0;
#pragma unroll
    for (int w = 0; w < kBinSortWarps; ++w) { pre[w] = tot; tot += sm.cnt[w][tid]; }
    if (!multi) run = block_exclusive_scan_256(tot, sm.sw, nullptr);   // synchronises
#pragma unroll
    for (int w = 0; w < kBinSortWarps; ++w) sm.cnt[w][tid] = run + pre[w];
    run += tot;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kGroups; ++j) {
      if (dr[j] != 0xffffffffu) {
        const uint32_t i = w0 + 32 * j + lane;
        const uint32_t pos = sm.cnt[warp][dr[j] >> 16] + (dr[j] & 0xffffu);
        dk[pos] = sk[i];
        dv[pos] = sv[i];
      }
    }
    __syncthreads();
  }
}

template <typename K>
__global__ void __launch_bounds__(kBinSortThreads, 4) bin_depth_sort(const uint32_t* __restrict__ bounds,
                                                                  const uint32_t* __restrict__ sched,
                                                                  const K* __restrict__ dkey,
                                                                  uint32_t* __restrict__ entry_item,
                                                                  K* __restrict__ gk0, K* __restrict__ gk1,
                                                                  uint32_t* __restrict__ gv1) {
  pdl_wait();
  __shared__ BinSortSmem<K> sm;
  const uint32_t g = sched ? sched[blockIdx.x] : blockIdx.x;
  const uint32_t s = bounds[g], n = bounds[g + 1] - s;
  if (n < 2) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool in_smem = n <= (uint32_t)BinSortSmem<K>::kCap;
  K* k0 = in_smem ? sm.key[0] : gk0 + s;
  K* k1 = in_smem ? sm.key[1] : gk1 + s;
  uint32_t* v0 = in_smem ? sm.val[0] : entry_item + s;
  uint32_t* v1 = in_smem ? sm.val[1] : gv1 + s;
  K kmin = ~(K)0, kmax = 0;
  for (uint32_t i = tid; i < n; i += kBinSortThreads) {
    const uint32_t item = entry_item[s + i];
    const K k = dkey[item];
    if (in_smem) {
      sm.key[0][i] = k;
      sm.val[0][i] = item;
    } else {
      k0[i] = k;
    }
    kmin = min(kmin, k);
    kmax = max(kmax, k);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) { sm.red_min[warp] = kmin; sm.red_max[warp] = kmax; }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kBinSortWarps; ++w) { kmin = min(kmin, sm.red_min[w]); kmax = max(kmax, sm.red_max[w]); }
  // digits of (key - kmin): only as many passes as the bin's key range needs
  const K range = kmax - kmin;
  int cur = 0;
  if (in_smem) {   // separate call sites: shared-memory addressing (LDS/STS) here
    for (int shift = 0; shift < (int)(8 * sizeof(K)) && (range >> shift); shift += 8) {
      if (cur == 0) bin_digit_pass<K>(sm.key[0], sm.val[0], sm.key[1], sm.val[1], n, shift, kmin, sm);
      else bin_digit_pass<K>(sm.key[1], sm.val[1], sm.key[0], sm.val[0], n, shift, kmin, sm);
      cur ^= 1;
    }
  } else {
    for (int shift = 0; shift < (int)(8 * sizeof(K)) && (range >> shift); shift += 8) {
      if (cur == 0) bin_digit_pass<K>(k0, v0, k1, v1, n, shift, kmin, sm);
      else bin_digit_pass<K>(k1, v1, k0, v0, n, shift, kmin, sm);
      cur ^= 1;
    }
  }
  // the result goes back to entry_item[s, s+n)
  if (in_smem) {
    if (range) {
      const uint32_t* src = sm.val[cur];
      for (uint32_t i = tid; i < n; i += kBinSortThreads) entry_item[s + i] = src[i];
    }
  } else if (cur) {
    for (uint32_t i = tid; i < n; i += kBinSortThreads) entry_item[s + i] = v1[i];
  }
}

// ---------------------------------------------------------------------------
// K3 / K4: per-tile blending over exact per-pixel coverage lists
//
// One CTA per (view, 16x16 tile); warp w owns an 8x4 pixel block (tile_col /
// tile_row below), lane l one pixel of it, i.e. coverage bit 32w + l.  Entries
// are staged in shared memory in batches.  For each entry the loading
// thread solves, row by row, the (padded) ellipse alpha >= 1/255 and writes a
// 256-bit coverage mask of the tile.  A 32x32 bit transpose per warp turns
// 32 entry masks into, per lane, the bits of the entries covering its pixel,
// so every lane walks only its own pixel's candidates in front-to-back order
// (the exact per-pixel decisions of render.py:251-267 then run unchanged).
// ---------------------------------------------------------------------------

template <typename S> struct BlendArgs {
  const uint32_t* bounds;
  const uint32_t* entry_item;
  const Splat<S>* splat;
  const V4<S>* col4;
  const uint4* bin;          // per item: rect, emitted-tile mask, count
  const uint32_t* entry_off;
  uint32_t items_per_view;   // F (mesh) or K (splats)
  int tiles_x;
  uint32_t tiles_per_view;
  int W, H;
  S bg0, bg1, bg2;
  // forward outputs / backward inputs
  S* rgb;
  S* alpha;
  S* t_final;
  // backward
  const S* g_rgb;
  const S* g_alpha;
  S* partial;        // [E][8] at pre-sort slots
  S* partial_op;     // [E] (splat path only) or null
  // optional fused image losses (forward epilogue, losses.py:43-73,158-160)
  const S* target_rgb;     // [B,H,W,3] or null
  const S* target_mask;    // [B,H,W]
  double scale_rgb, scale_alpha;   // w_color / n, w_silhouette / n
  S* g_rgb_out;            // [B,H,W,3] dL/drgb (pre-scaled), read by K4
  S* g_alpha_out;          // [B,H,W]
  double* loss_tile;       // [bins][2]: sum of squared colour error, sum of BCE
  uint32_t* covbuf;        // [entries][8] coverage words: written by the forward, read by the backward (or null)
  // optional 8-bit images (dataset.py:59-61 `_save_png`); rgb/alpha may then be null
  uint8_t* rgb8;           // [B,H,W,3]
  uint8_t* alpha8;         // [B,H,W]
  const uint32_t* sched;   // launch order of the bins (tile_schedule) or null
};

// np.round(np.clip(float64(x), 0, 1) * 255).astype(uint8) (dataset.py:60-61):
// float64 clip and product, round half to even (rint); NaN maps to 0.
__device__ __forceinline__ uint8_t png_level(double x) {
  if (!(x == x)) return 0;
  return (uint8_t)rint(fmin(fmax(x, 0.0), 1.0) * 255.0);
}

constexpr double kBceClamp = 1e-6;   // losses.py:20

// Per-pixel colour MSE / clamped-BCE terms and their gradients, in float64
// like the reference (losses.py:43-73; image grads scaled by w/n, :158-160).
template <typename S>
__device__ __forceinline__ void pixel_loss(const BlendArgs<S>& p, size_t pix, const S rgb[3], S alpha,
                                           double& sq, double& bce) {
  const double nc = 3.0 * (double)p.W * (double)p.H, na = (double)p.W * (double)p.H;
  sq = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double d = (double)rgb[c] - (double)p.target_rgb[3 * pix + c];
    sq += d * d;
    p.g_rgb_out[3 * pix + c] = (S)((2.0 / nc) * d * p.scale_rgb);
  }
  const double a = (double)alpha, m = (double)p.target_mask[pix];
  const double q = fmin(fmax(a, kBceClamp), 1.0 - kBceClamp);
  bce = -(m * log(q) + (1.0 - m) * log1p(-q));
  const bool inside = a > kBceClamp && a < 1.0 - kBceClamp;
  p.g_alpha_out[pix] = (S)(inside ? ((-m / q + (1.0 - m) / (1.0 - q)) / na) * p.scale_alpha : 0.0);
}

// fixed-order block sum of two doubles (256 threads)
__device__ __forceinline__ void block_sum2(double a, double b, double* out2) {
  __shared__ double sa[8], sb[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sa[warp] = a; sb[warp] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < 8; ++w) { x += sa[w]; y += sb[w]; }
    out2[0] = x;
    out2[1] = y;
  }
}

// Sum the per-tile loss partials in tile order (single block, fixed tree).
__global__ void __launch_bounds__(256) loss_reduce(const double* __restrict__ tile, uint32_t bins,
                                                  double* __restrict__ out2) {
  pdl_wait();
  double a = 0.0, b = 0.0;
  for (uint32_t i = threadIdx.x; i < bins; i += 256) {
    a += tile[2 * i];
    b += tile[2 * i + 1];
  }
  block_sum2(a, b, out2);
}

// lane r holds row r of a 32x32 bit matrix (bit c = M[r][c]); transpose32
// returns column `lane` (bit r = M[r][lane]) in 5 shuffle stages.  Stage j
// exchanges j-bit groups with lane ^ j: a lane with (lane & j) keeps the high
// group of every 2j-bit block and takes its partner's high groups shifted
// down, the other lane keeps the low groups and takes the partner's low
// groups shifted up.  Per lane and stage that is one fixed byte permutation
// (j = 16, 8: PRMT) or a rotate by j or 32 - j plus a select mask (j < 8:
// SHF + LOP3), so the per-lane constants are made once per batch
// (TransposeLanes) and each stage costs 2-3 instructions.
struct TransposeLanes {
  uint32_t s16, s8, r4, r2, r1, m4, m2, m1;
  __device__ __forceinline__ explicit TransposeLanes(int lane) {
    s16 = (lane & 16) ? 0x3276u : 0x5410u;
    s8 = (lane & 8) ? 0x3715u : 0x6240u;
    r4 = (lane & 4) ? 4u : 28u;
    r2 = (lane & 2) ? 2u : 30u;
    r1 = (lane & 1) ? 1u : 31u;
    m4 = (lane & 4) ? 0x0F0F0F0Fu : 0xF0F0F0F0u;
    m2 = (lane & 2) ? 0x33333333u : 0xCCCCCCCCu;
    m1 = (lane & 1) ? 0x55555555u : 0xAAAAAAAAu;
  }
};
__device__ __forceinline__ uint32_t transpose32(uint32_t x, const TransposeLanes& k) {
  x = __byte_perm(x, __shfl_xor_sync(0xffffffffu, x, 16), k.s16);
  x = __byte_perm(x, __shfl_xor_sync(0xffffffffu, x, 8), k.s8);
  uint32_t y = __shfl_xor_sync(0xffffffffu, x, 4);
  x = (x & ~k.m4) | (__funnelshift_r(y, y, k.r4) & k.m4);
  y = __shfl_xor_sync(0xffffffffu, x, 2);
  x = (x & ~k.m2) | (__funnelshift_r(y, y, k.r2) & k.m2);
  y = __shfl_xor_sync(0xffffffffu, x, 1);
  x = (x & ~k.m1) | (__funnelshift_r(y, y, k.r1) & k.m1);
  return x;
}

// Opaque copies: the compiler must keep these per-thread constants in
// registers instead of re-deriving them from threadIdx.x in every loop trip
// (it does that under the occupancy's register cap; measured per variant).
__device__ __forceinline__ float pin(float x) { asm volatile("" : "+f"(x)); return x; }
__device__ __forceinline__ double pin(double x) { asm volatile("" : "+d"(x)); return x; }
__device__ __forceinline__ int pin(int x) { asm volatile("" : "+r"(x)); return x; }
#ifndef GMR_PIN_CONSTS
#define GMR_PIN_CONSTS 1
#endif
#ifndef GMR_PIN_FWD
#define GMR_PIN_FWD 1
#endif
#if GMR_PIN_CONSTS
#define GMR_PIN(x) pin(x)
#else
#define GMR_PIN(x) (x)
#endif
#if GMR_PIN_FWD
#define GMR_PIN_F(x) pin(x)
#else
#define GMR_PIN_F(x) (x)
#endif

// Pixel layout of a tile CTA: warp w owns the 8x4 block at columns
// 8 (w & 1) .. +7, rows 4 (w >> 1) .. +3; lane l is column l & 7, row l >> 3
// of it.  Square blocks keep a warp's lanes on nearly the same splats.
__device__ __forceinline__ int tile_col(int t) { return ((t >> 2) & 8) + (t & 7); }
__device__ __forceinline__ int tile_row(int t) { return ((t >> 4) & 12) + ((t >> 3) & 3); }

// Coverage of one splat in the tile with pixel origin (x0, y0), OR-ed row
// by row into 8 zeroed words `w`: word w holds warp w's 8x4 block, bit
// 8 (row & 3) + (col & 7) (shared memory, so the indices may be dynamic).
template <typename S>
__device__ __forceinline__ void tile_coverage(const V4<S>& a, const V4<S>& b, int x0, int y0, uint32_t* w) {
  const S mx = a.x, my = a.y, ca = a.z, cb = a.w, cc = b.x, ex = b.y, ey = b.z, tau = b.w;
  if (!(ex >= S(0)) || !(ca > S(0))) return;
  const int r0 = (int)fmax(S(0), ceil(my - ey) - S(y0));
  const int r1 = (int)fmin(S(15), floor(my + ey) - S(y0));
  const S mxr = mx - S(x0);
  const S neg_det = cb * cb - ca * cc;   // b^2 - ac < 0 for a positive definite conic
  const S inv_a = S(1) / ca;
#pragma unroll 1
  for (int r = r0; r <= r1; ++r) {
    const S dy = S(y0 + r) - my;
    const S disc = dy * dy * neg_det + ca * tau;
    if (!(disc >= S(0))) continue;
    const S hw = sqrt_s(disc) * inv_a * S(1.0005) + S(0.01);
    const S xc = mxr - cb * dy * inv_a;
    const S lo = fmax(ceil(xc - hw), S(0)), hi = fmin(floor(xc + hw), S(15));
    if (lo > hi) continue;
    const int ilo = (int)lo, ihi = (int)hi;
    const uint32_t bits = (0xffffu >> (15 - (ihi - ilo))) << ilo;
    const int wi = (r >> 2) << 1, sh = (r & 3) << 3;
    w[wi] |= (bits & 0xffu) << sh;
    w[wi + 1] |= (bits >> 8) << sh;
  }
}

#ifndef GMR_FAST_COVERAGE
#define GMR_FAST_COVERAGE 1
#endif
#if GMR_FAST_COVERAGE
// float: the same rows with approximate sqrt / reciprocal (relative error
// ~1e-7, far inside the 5e-4 + 0.01 px padding: the mask stays a superset of
// the alpha >= 1/255 pixels, so no result changes), integer rounding
// conversions, and the two words of a 4-row band built in registers and
// stored once: 45 SASS instructions per row instead of 58.
template <>
__device__ __forceinline__ void tile_coverage<float>(const V4<float>& a, const V4<float>& b, int x0, int y0,
                                                     uint32_t* w) {
  const float mx = a.x, my = a.y, ca = a.z, cb = a.w, cc = b.x, ex = b.y, ey = b.z, tau = b.w;
  if (!(ex >= 0.f) || !(ca > 0.f)) return;
  const int r0 = (int)fmaxf(0.f, ceilf(my - ey) - (float)y0);
  const int r1 = (int)fminf(15.f, floorf(my + ey) - (float)y0);
  const float mxr = mx - (float)x0;
  const float neg_det = cb * cb - ca * cc;
  float inv_a;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_a) : "f"(ca));
  const float k = inv_a * 1.0005f, cbi = cb * inv_a, ca_tau = ca * tau;
  float dy = (float)(y0 + r0) - my;
  uint32_t lo_w = 0u, hi_w = 0u;
#pragma unroll 1
  for (int r = r0; r <= r1; ++r, dy += 1.f) {
    const float disc = fmaf(dy * dy, neg_det, ca_tau);
    if (disc >= 0.f) {
      float sq;
      asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(disc));
      const float hw = fmaf(sq, k, 0.01f), xc = fmaf(-cbi, dy, mxr);
      const int ilo = max(__float2int_ru(xc - hw), 0), ihi = min(__float2int_rd(xc + hw), 15);
      if (ilo <= ihi) {
        const uint32_t bits = (0xffffu >> (15 - (ihi - ilo))) << ilo;
        const int sh = (r & 3) << 3;
        lo_w |= (bits & 0xffu) << sh;
        hi_w |= (bits >> 8) << sh;
      }
    }
    if ((r & 3) == 3 || r == r1) {   // last row of a band: its two words are final
      const int wi = (r >> 2) << 1;
      w[wi] = lo_w;
      w[wi + 1] = hi_w;
      lo_w = hi_w = 0u;
    }
  }
}
#endif

// 1 / (1 - alpha) with 1 - alpha >= 0.01 (alpha clamp): no denormal range
__device__ __forceinline__ float inv_om(float om) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(om));
  return r;
}
__device__ __forceinline__ double inv_om(double om) { return 1.0 / om; }

// Per-pixel alpha of a staged splat (render.py:251-256) from its conic in the
// form the evaluator wants (Eval<S>::prep: coefficients A, B, C) and its
// opacity o.  kOp = false: o == 1 (every mesh-path splat, convert.py:326),
// where o * e == e exactly, so the product is skipped without changing a bit.
//  double (parity path): the reference's expression and exp(), with each
//    operation rounded as numpy rounds it;
//  float (fast path): power * log2(e) as dx (A dx + B dy) + C dy^2 with the
//    coefficients folded at staging time, then ex2.approx.
template <typename S> struct Eval;
template <> struct Eval<double> {
  static __device__ __forceinline__ void prep(double ca, double cb, double cc, double& A, double& B, double& C) {
    A = ca; B = cb; C = cc;
  }
  template <bool kOp>
  static __device__ __forceinline__ double alpha(double dx, double dy, double A, double B, double C, double o,
                                                 double& ep, double& raw) {
    const double qq = add_rn(mul_rn(mul_rn(A, dx), dx), mul_rn(mul_rn(C, dy), dy));
    const double power = sub_rn(mul_rn(-0.5, qq), mul_rn(mul_rn(B, dx), dy));
    ep = exp(power);
    raw = kOp ? mul_rn(o, ep) : ep;
    return raw < 0.99 ? raw : 0.99;
  }
};
template <> struct Eval<float> {
  static __device__ __forceinline__ void prep(float ca, float cb, float cc, float& A, float& B, float& C) {
    const float l2e = 1.4426950408889634f;
    A = -0.5f * l2e * ca; B = -l2e * cb; C = -0.5f * l2e * cc;
  }
  template <bool kOp>
  static __device__ __forceinline__ float alpha(float dx, float dy, float A, float B, float C, float o, float& ep,
                                                float& raw) {
    const float p2 = __fmaf_rn(dx, __fmaf_rn(A, dx, __fmul_rn(B, dy)), __fmul_rn(__fmul_rn(C, dy), dy));
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(p2));
    ep = e;
    raw = kOp ? __fmul_rn(o, e) : e;
    return raw < 0.99f ? raw : 0.99f;
  }
};

// Warm L2 with the records of the next batch while the current one is
// processed: the gathers entry -> item -> record are otherwise exposed at
// every batch start.
template <typename S>
__device__ __forceinline__ void prefetch_records(const BlendArgs<S>& p, uint32_t item, uint32_t vbase_item) {
  if (item == 0xffffffffu) return;
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p.splat + item));
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p.col4 + (item - vbase_item)));
}

#ifndef GMR_BWD_BATCH
#define GMR_BWD_BATCH 128
#endif
#ifndef GMR_RQ_WORDS
#define GMR_RQ_WORDS 1
#endif
#ifndef GMR_BWD_TMA
// 1: the coverage rows of the next batch arrive by a 1-D bulk copy (TMA
// engine, UBLKCP + mbarrier) issued one batch ahead.  Measured slower
// (1.171 -> 1.274 ms at config 3): its 4 KB buffer comes out of the record
// buffer at 5 CTAs/SM, so batches are cut shorter.  Kept as the option.
#define GMR_BWD_TMA 0
#endif

#ifndef GMR_BWD_PAIR_BYTES
#if GMR_BWD_TMA
#define GMR_BWD_PAIR_BYTES 20224   // less the 4 KB coverage staging buffer
#else
#define GMR_BWD_PAIR_BYTES 24448   // 24 KB less 128 B: keeps BwdSmem<float> at 5 CTAs per SM
#endif
#endif
#ifndef GMR_BWD_MINB
#define GMR_BWD_MINB 5
#endif
#ifndef GMR_FWD_BATCH
#define GMR_FWD_BATCH 256
#endif
constexpr int kFwdBatch = GMR_FWD_BATCH;
constexpr int kBwdBatch = GMR_BWD_BATCH;

// A staged batch.  Per entry two 16-byte (float) records, read with two
// vector loads per (pixel, entry) pair:
//   ea = (mean_x, mean_y, A, B), eb = (C, r, g, b)
// plus the opacity (splat path only), the 8 coverage words (+1 pad:
// conflict-free transposes) and, per pixel, the covering entries of each
// 32-entry chunk.
template <typename S, int NB, bool kOp, bool kCov = true> struct StageSmem {
  V4<S> ea[NB];
  V4<S> eb[NB];
  S op[kOp ? NB : 1];
  uint32_t cov[kCov ? NB : 1][9];
  uint32_t tw[NB / 32][kBlendThreads];
};

// One entry of a batch: its records from the item's splat and colour.
template <typename S, int NB, bool kOp, bool kCov>
__device__ __forceinline__ void stage_entry(const BlendArgs<S>& p, StageSmem<S, NB, kOp, kCov>& sm, int i, uint32_t item,
                                            uint32_t vbase_item, Splat<S>& s) {
  s = p.splat[item];
  const V4<S> c = p.col4[item - vbase_item];
  V4<S> a, b;
  a.x = s.a.x; a.y = s.a.y;
  Eval<S>::prep(s.a.z, s.a.w, s.b.x, a.z, a.w, b.x);
  b.y = c.x; b.z = c.y; b.w = c.z;
  sm.ea[i] = a;
  sm.eb[i] = b;
  if constexpr (kOp) sm.op[i] = c.w;
}

// Stage one batch (forward): thread i < n loads entry base+i and solves its
// coverage rows (i >= n: empty mask), then every warp transposes its
// coverage words into per-pixel bit lists.
template <typename S, int NB, bool kOp>
__device__ __forceinline__ uint32_t stage_batch(const BlendArgs<S>& p, StageSmem<S, NB, kOp>& sm, uint32_t base,
                                                int n, uint32_t vbase_item, int x0, int y0,
                                                uint32_t item_hint = 0xffffffffu) {
  for (int i = threadIdx.x; i < NB; i += kBlendThreads) {
    uint32_t* w = sm.cov[i];
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = 0;
    if (i < n) {
      Splat<S> s;
      // item_hint: this thread's item, read during the previous batch
      stage_entry(p, sm, i, item_hint != 0xffffffffu ? item_hint : p.entry_item[base + i], vbase_item, s);
      tile_coverage(s.a, s.b, x0, y0, w);
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TransposeLanes tl(lane);
  uint32_t cmask = 0;   // chunks holding at least one candidate of this thread's pixel
#pragma unroll
  for (int c = 0; c < NB / 32; ++c)
    if (c * 32 < n) {
      const uint32_t x = transpose32(sm.cov[c * 32 + lane][warp], tl);
      sm.tw[c][threadIdx.x] = x;
      cmask |= (x != 0u) << c;
    }
  return cmask;
}

#ifndef GMR_WALK_HOIST
#define GMR_WALK_HOIST 1
#endif
#ifndef GMR_CW_HOIST
#define GMR_CW_HOIST 1
#endif
#ifndef GMR_FWD_LAZYCOL
#define GMR_FWD_LAZYCOL 1
#endif
// Iterator over a lane's covering entries of the staged batch, in order.
// `col` points at the lane's word of chunk 0 of the transposed candidate
// bits, chunk c at col[c * kStride]; `cmask` (bit c: chunk c holds a
// candidate of this lane, from the transposes) lets a refill jump straight
// to the next non-empty chunk.
template <int kStride>
struct BitWalk {
  const uint32_t* col;
  int base;
  uint32_t bits, cmask;
  __device__ __forceinline__ void start(const uint32_t* lane_col, uint32_t chunks, bool skip) {
    col = lane_col;
    cmask = skip ? 0u : chunks;
    bits = 0u;
    base = 0;
  }
  // Up to two candidates from the current chunk (has2 = false if it has
  // only one left; j2 is then meaningless); refills from the next non-empty
  // chunk only when the current one is exhausted, so the common path is
  // straight-line.  false = done.
  __device__ __forceinline__ bool pair(int& j1, int& j2, bool& has2) {
    if (__builtin_expect(bits == 0, 0)) {
      if (!cmask) return false;
      const int c = __ffs(cmask) - 1;
      cmask &= cmask - 1;
      bits = col[c * kStride];
      base = c << 5;
    }
    j1 = base + __ffs(bits) - 1;
    bits &= bits - 1;
    has2 = bits != 0u;
    j2 = has2 ? base + __ffs(bits) - 1 : j1;   // a valid index either way: the caller may load it unconditionally
    bits &= bits - 1;   // no-op when empty
    return true;
  }
  __device__ __forceinline__ void stop() { bits = 0; cmask = 0; }
};


#ifndef GMR_FWD_MINB
#define GMR_FWD_MINB 6   // 40 registers (measured: 6 CTAs/SM 0.550 ms vs 7 CTAs/SM at 32 registers 0.577 ms, config 3)
#endif
template <typename S, bool kOp>
__global__ void __launch_bounds__(kBlendThreads, sizeof(S) == 8 ? 4 : GMR_FWD_MINB) blend_forward(BlendArgs<S> p) {
  pdl_wait();
  __shared__ StageSmem<S, kFwdBatch, kOp> sm;
  const uint32_t g = p.sched ? p.sched[blockIdx.x] : blockIdx.x;
  const uint32_t view = g / p.tiles_per_view, t = g % p.tiles_per_view;
  const int tx = (int)(t % (uint32_t)p.tiles_x), ty = (int)(t / (uint32_t)p.tiles_x);
  const int x0 = tx * kTile, y0 = ty * kTile;
  const int px = x0 + tile_col(threadIdx.x), py = y0 + tile_row(threadIdx.x);
  const bool inside = px < p.W && py < p.H;
  const S fpx = GMR_PIN_F(S(px)), fpy = GMR_PIN_F(S(py));
  const S one = S(1);
  S T = one, ar = 0, ag = 0, ab = 0;
  bool done = !inside;
  const uint32_t start = p.bounds[g], end = p.bounds[g + 1];
  const uint32_t vbase_item = view * p.items_per_view;
  uint32_t item_next = 0xffffffffu;
  for (uint32_t base = start; base < end; base += kFwdBatch) {
    if (__syncthreads_count(done) == kBlendThreads) break;
    const int n = (int)min((uint32_t)kFwdBatch, end - base);
    const uint32_t chunks = stage_batch<S, kFwdBatch, kOp>(p, sm, base, n, vbase_item, x0, y0, item_next);
    __syncthreads();
    if (p.covbuf) {   // keep the coverage masks for the backward (coalesced 32-byte rows)
      for (int i = threadIdx.x; i < n; i += kBlendThreads) {
        const uint32_t* w = sm.cov[i];
        uint4* dst = reinterpret_cast<uint4*>(p.covbuf + (size_t)(base + i) * 8);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
    const uint32_t nxt_e = base + kFwdBatch + threadIdx.x;
    const uint32_t nxt = nxt_e < end ? p.entry_item[nxt_e] : 0xffffffffu;
    BitWalk<kBlendThreads> it;
    it.start(&sm.tw[0][threadIdx.x], chunks, done);
    // two candidates per trip: their alphas are independent, only the
    // transmittance update is sequential (front-to-back order kept)
    int j1, j2;
    bool has2;
    while (it.pair(j1, j2, has2)) {
#if GMR_FWD_LAZYCOL
      // alpha needs (mx, my, A, B) and C only: both candidates' five values
      // are loaded together, the colours only for included pairs
      const V4<S> a1 = sm.ea[j1], a2 = sm.ea[j2];
      const S c1 = reinterpret_cast<const S*>(&sm.eb[j1])[0], c2 = reinterpret_cast<const S*>(&sm.eb[j2])[0];
      S ep, raw;
      const S al1 = Eval<S>::template alpha<kOp>(sub_rn(fpx, a1.x), sub_rn(fpy, a1.y), a1.z, a1.w, c1,
                                                 kOp ? sm.op[j1] : one, ep, raw);
      S al2 = Eval<S>::template alpha<kOp>(sub_rn(fpx, a2.x), sub_rn(fpy, a2.y), a2.z, a2.w, c2,
                                           kOp ? sm.op[j2] : one, ep, raw);
      if (!has2) al2 = S(0);
      if (al1 >= Const<S>::contrib_floor()) {
        const S test = mul_rn(T, sub_rn(one, al1));
        if (test < Const<S>::t_stop()) goto fwd_stop;
        const V4<S> b1 = sm.eb[j1];
        const S w = mul_rn(al1, T);
        ar += w * b1.y;
        ag += w * b1.z;
        ab += w * b1.w;
        T = test;
      }
      if (al2 >= Const<S>::contrib_floor()) {
        const S test = mul_rn(T, sub_rn(one, al2));
        if (test < Const<S>::t_stop()) goto fwd_stop;
        const V4<S> b2 = sm.eb[j2];
        const S w = mul_rn(al2, T);
        ar += w * b2.y;
        ag += w * b2.z;
        ab += w * b2.w;
        T = test;
      }
#else
      const V4<S> a1 = sm.ea[j1], b1 = sm.eb[j1];
      S ep, raw;
      const S al1 = Eval<S>::template alpha<kOp>(sub_rn(fpx, a1.x), sub_rn(fpy, a1.y), a1.z, a1.w, b1.x,
                                                 kOp ? sm.op[j1] : one, ep, raw);
#if GMR_WALK_HOIST
      // the second candidate's loads and alpha unconditionally (j2 = j1 when
      // there is none): its shared-memory latency overlaps the first's
      const V4<S> a2 = sm.ea[j2], b2 = sm.eb[j2];
      S al2 = Eval<S>::template alpha<kOp>(sub_rn(fpx, a2.x), sub_rn(fpy, a2.y), a2.z, a2.w, b2.x,
                                           kOp ? sm.op[j2] : one, ep, raw);
      if (!has2) al2 = S(0);
#else
      V4<S> b2;
      S al2 = S(0);
      if (has2) {
        const V4<S> a2 = sm.ea[j2];
        b2 = sm.eb[j2];
        al2 = Eval<S>::template alpha<kOp>(sub_rn(fpx, a2.x), sub_rn(fpy, a2.y), a2.z, a2.w, b2.x,
                                           kOp ? sm.op[j2] : one, ep, raw);
      }
#endif
      // the transmittance stop is rare (T stays above 1e-4 on almost every
      // pixel): it leaves the walk by a jump, so no stop flag is carried
      if (al1 >= Const<S>::contrib_floor()) {
        const S test = mul_rn(T, sub_rn(one, al1));
        if (test < Const<S>::t_stop()) goto fwd_stop;
        const S w = mul_rn(al1, T);
        ar += w * b1.y;
        ag += w * b1.z;
        ab += w * b1.w;
        T = test;
      }
      if (al2 >= Const<S>::contrib_floor()) {
        const S test = mul_rn(T, sub_rn(one, al2));
        if (test < Const<S>::t_stop()) goto fwd_stop;
        const S w = mul_rn(al2, T);
        ar += w * b2.y;
        ag += w * b2.z;
        ab += w * b2.w;
        T = test;
      }
#endif
      continue;
    fwd_stop:
      done = true;
      it.stop();
      break;
    }
    prefetch_records(p, nxt, vbase_item);
    item_next = nxt;
    // no barrier here: the next batch's __syncthreads_count is one
  }
  double sq = 0.0, bce = 0.0;
  if (inside) {
    const size_t pix = ((size_t)view * p.H + py) * p.W + px;
    S out[3];
    out[0] = ar + T * p.bg0;
    out[1] = ag + T * p.bg1;
    out[2] = ab + T * p.bg2;
    if (p.rgb) {
      p.rgb[3 * pix + 0] = out[0];
      p.rgb[3 * pix + 1] = out[1];
      p.rgb[3 * pix + 2] = out[2];
      p.alpha[pix] = one - T;
    }
    if (p.rgb8) {
      p.rgb8[3 * pix + 0] = png_level((double)out[0]);
      p.rgb8[3 * pix + 1] = png_level((double)out[1]);
      p.rgb8[3 * pix + 2] = png_level((double)out[2]);
      p.alpha8[pix] = png_level((double)(one - T));
    }
    p.t_final[pix] = T;
    if (p.target_rgb) pixel_loss(p, pix, out, one - T, sq, bce);
  }
  if (p.target_rgb) block_sum2(sq, bce, p.loss_tile + 2 * (size_t)g);
}

// 1-D bulk copies (TMA engine, cp.async.bulk) completing on an mbarrier.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// One thread: arm the barrier with `bytes` and start the copy global -> shared.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of dst before the async write
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <typename S, bool kOpacity> struct RecOf { typedef V2<S> type; };
template <typename S> struct RecOf<S, true> { typedef V4<S> type; };

#ifndef GMR_BWD_PAIR_BYTES_F64
// float64 runs 3 CTAs/SM (register-bound): its 16-byte records get a buffer
// of the same record count as float's instead of half of it
#define GMR_BWD_PAIR_BYTES_F64 46080
#endif
template <typename S> struct BwdPairBytes { static constexpr int value = sizeof(S) == 8 ? GMR_BWD_PAIR_BYTES_F64 : GMR_BWD_PAIR_BYTES; };

template <typename S, bool kOpacity> struct BwdSmem {
  typedef typename RecOf<S, kOpacity>::type Rec;
  static constexpr int kCap = BwdPairBytes<S>::value / (int)(sizeof(Rec) + 1);
  StageSmem<S, kBwdBatch, kOpacity, false> st;
  uint2 cw[8][kBwdBatch];           // per warp block and entry: (coverage word, first record of its pixels)
  uint32_t rend[kBwdBatch];         // per entry: end of its records (they start at cw[0][j].y)
  uint32_t wsum[kBlendThreads / 32];
#if GMR_BWD_TMA
  uint4 covq[kBwdBatch][2];         // the batch's coverage rows (bulk copy of covbuf, issued one batch ahead)
  uint64_t bar;
#endif
  V4<S> pix[kBlendThreads];         // per tile pixel (col + 16 row): g_r, g_g, g_b
  Rec rec[kCap];                    // per (entry, covered pixel): (dp, w[, dL/dalpha * ep])
  uint8_t rq[(kCap + 3) & ~3];       // tile pixel (col + 16 row) of each record (whole words: read 4 at a time)
};

// Backward (render.py:294-361).  Per batch of staged entries:
//  - each staging thread takes one entry's records and the forward's
//    coverage words, counts its covered pixels per warp block, and a
//    scan over the batch gives every entry a contiguous record range
//    [cw[0][j].y, rend[j]) (the batch is cut where the ranges would overflow
//    shared memory), ordered by warp, then lane; the records are zeroed;
//  - pass 1 (lane = pixel) re-scans front to back with the forward's exact
//    decisions.  With C = g.(rgb - T_f bg) = sum_j (g.c_j) w_j the suffix is
//    S_k = C - sum_{j<=k} (g.c_j) w_j, so (render.py:327-334)
//      dL/dalpha_k = (g.c_k) T_k - (S_k + (g.bg - g_a) T_f) / (1 - alpha_k)
//    and each included pair writes (dp = dL/dalpha * alpha, 0 where the 0.99
//    clamp is active (:336-338), w = alpha T) to record
//    cw[warp][j].y + (rank of this lane among the warp's lanes covering j);
//  - pass 2 (two threads per entry, halves of its records) sums
//      [dp dx, dp dy, dp dx^2, dp dx dy, dp dy^2, w g_r, w g_g, w g_b]
//    in record order; the halves are combined in a fixed order.
//  No atomics, fixed orders: the result is deterministic.
template <typename S, bool kOpacity>
__global__ void __launch_bounds__(kBlendThreads, sizeof(S) == 8 ? 3 : GMR_BWD_MINB) blend_backward(BlendArgs<S> p) {
  pdl_wait();
  extern __shared__ __align__(32) unsigned char dyn[];
  typedef BwdSmem<S, kOpacity> Sm;
  typedef typename Sm::Rec Rec;
  Sm& sm = *reinterpret_cast<Sm*>(dyn);
  const uint32_t g = p.sched ? p.sched[blockIdx.x] : blockIdx.x;
  const uint32_t view = g / p.tiles_per_view, t = g % p.tiles_per_view;
  const int tx = (int)(t % (uint32_t)p.tiles_x), ty = (int)(t / (uint32_t)p.tiles_x);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int x0 = tx * kTile, y0 = ty * kTile;
  const int px = x0 + tile_col(threadIdx.x), py = y0 + tile_row(threadIdx.x);
  const bool inside = px < p.W && py < p.H;
  const S fpx = GMR_PIN(S(px)), fpy = GMR_PIN(S(py));
  const S one = S(1);
  const unsigned lt = lanemask_lt();
  S Ctot = 0, bterm = 0;
  V4<S> mypix;
  mypix.x = mypix.y = mypix.z = mypix.w = S(0);
  if (inside) {
    const size_t pix = ((size_t)view * p.H + py) * p.W + px;
    mypix.x = p.g_rgb[3 * pix]; mypix.y = p.g_rgb[3 * pix + 1]; mypix.z = p.g_rgb[3 * pix + 2];
    const S tf = p.t_final[pix];
    const S gbg = mypix.x * p.bg0 + mypix.y * p.bg1 + mypix.z * p.bg2;
    Ctot = mypix.x * p.rgb[3 * pix] + mypix.y * p.rgb[3 * pix + 1] + mypix.z * p.rgb[3 * pix + 2] - gbg * tf;
    bterm = (gbg - p.g_alpha[pix]) * tf;
  }
  // per-pixel data and record pixel ids use the natural tile index
  // col + 16 row (pass 2 recovers the offsets with two bit operations)
  const int my_pix = GMR_PIN(tile_col(tid) + 16 * tile_row(tid));
  {   // the fourth slot carries the pixel's tile column as a float (pass 2's dx)
    V4<S> pv = mypix;
    pv.w = S(tile_col(tid));
    sm.pix[my_pix] = pv;
  }
  S T = one, P = 0;
#ifndef GMR_SUFFIX_Q
#define GMR_SUFFIX_Q 1
#endif
#if GMR_SUFFIX_Q
  S Q = Ctot + bterm;
  (void)P;
#endif
  bool done = !inside;
  const uint32_t start = p.bounds[g], end = p.bounds[g + 1];
  const uint32_t vbase_item = view * p.items_per_view;
#if GMR_BWD_TMA
  uint32_t phase = 0;
  bool inflight = false;   // CTA-uniform: a coverage copy is outstanding
  if (tid == 0) {
    mbar_init(&sm.bar);
    if (start < end)
      bulk_load(sm.covq, p.covbuf + (size_t)start * 8, min((uint32_t)kBwdBatch, end - start) * 32u, &sm.bar);
  }
  inflight = start < end;
  __syncthreads();
#endif
  // pass 2: two threads per entry (halves of its records) for 128-entry
  // batches, one per entry for 256
  constexpr int kSplit = kBlendThreads / kBwdBatch;
  static_assert(kSplit == 1 || kSplit == 2, "backward batch must be 128 or 256 entries");
  const int je = kSplit == 2 ? tid >> 1 : tid, half = kSplit == 2 ? tid & 1 : 0;
  uint32_t base = start;
  uint32_t item_next = 0xffffffffu;   // this thread's entry of the next batch, read during this one
  while (base < end) {
    if (__syncthreads_count(done) == kBlendThreads) break;
    const int n_st = (int)min((uint32_t)kBwdBatch, end - base);
    // ---- stage records + the forward's coverage words; per-warp counts ----
    uint32_t ncov = 0;
    uint32_t wcnt[8];   // covered pixels of this entry in warp blocks before each warp
#pragma unroll
    for (int q = 0; q < 8; ++q) wcnt[q] = 0;
#if GMR_BWD_TMA
    mbar_wait(&sm.bar, phase);
    phase ^= 1u;
    inflight = false;
#endif
    if (tid < n_st) {
      Splat<S> s;
      stage_entry(p, sm.st, tid, item_next != 0xffffffffu ? item_next : p.entry_item[base + tid], vbase_item, s);
#if GMR_BWD_TMA
      const uint4 lo = sm.covq[tid][0], hi = sm.covq[tid][1];
#else
      const uint4* src = reinterpret_cast<const uint4*>(p.covbuf + (size_t)(base + tid) * 8);
      const uint4 lo = src[0], hi = src[1];
#endif
      const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        sm.cw[q][tid].x = w[q];
        wcnt[q] = ncov;
        ncov += __popc(w[q]);
      }
    }
    // exclusive scan of the covered counts over the batch (threads < 128)
    uint32_t x = ncov;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sm.wsum[warp] = x;
    __syncthreads();
    uint32_t excl = x - ncov;
    for (int w2 = 0; w2 < warp; ++w2) excl += sm.wsum[w2];
    const bool fits = tid < n_st && excl + ncov <= (uint32_t)Sm::kCap;

    if (fits) {
      sm.rend[tid] = excl + ncov;
#pragma unroll
      for (int q = 0; q < 8; ++q) sm.cw[q][tid].y = excl + wcnt[q];
    }
    const int n = __syncthreads_count(fits);          // entries taken this batch (prefix property)
#if GMR_BWD_TMA
    {   // every thread has read sm.covq (before the count barrier): fetch the next batch's rows
      const uint32_t nb = base + (uint32_t)n;
      if (nb < end) {
        if (tid == 0) bulk_load(sm.covq, p.covbuf + (size_t)nb * 8, min((uint32_t)kBwdBatch, end - nb) * 32u, &sm.bar);
        inflight = true;
      }
    }
#endif
    const uint32_t rec_end = n ? sm.rend[n - 1] : 0u;
    for (uint32_t r = tid; r < rec_end; r += kBlendThreads) {
      Rec z;
      z.x = z.y = S(0);
      if constexpr (kOpacity) { z.z = z.w = S(0); }
      sm.rec[r] = z;
    }
    // entries past n are re-staged next batch: their coverage reads as empty
    uint32_t chunks = 0;   // chunks holding at least one candidate of this thread's pixel
    {
      const TransposeLanes tl(lane);
#pragma unroll
      for (int c = 0; c < kBwdBatch / 32; ++c)
        if (c * 32 < n) {
          const uint32_t x = transpose32(c * 32 + lane < n ? sm.cw[warp][c * 32 + lane].x : 0u, tl);
          sm.st.tw[c][tid] = x;
          chunks |= (x != 0u) << c;
        }
    }
    __syncthreads();
    const uint32_t nxt_e = base + (uint32_t)n + threadIdx.x;
    const uint32_t nxt = (threadIdx.x < kBwdBatch && nxt_e < end) ? p.entry_item[nxt_e] : 0xffffffffu;
    // ---- pass 1: my pixel (two candidates per trip, sequential T) ----
    {
      BitWalk<kBlendThreads> it;
      it.start(&sm.st.tw[0][tid], chunks, done);
      int j1, j2;
      bool has2;
      while (it.pair(j1, j2, has2)) {
        int js[2] = {j1, j2};
#if GMR_CW_HOIST
        // both candidates' record bases now, overlapped with the alphas
        const uint2 cws[2] = {sm.cw[warp][j1], sm.cw[warp][j2]};
#endif
        S as[2], eps[2], raws[2];
        V4<S> bs[2];
        {
          const V4<S> a = sm.st.ea[j1];
          bs[0] = sm.st.eb[j1];
          as[0] = Eval<S>::template alpha<kOpacity>(sub_rn(fpx, a.x), sub_rn(fpy, a.y), a.z, a.w, bs[0].x,
                                                    kOpacity ? sm.st.op[j1] : one, eps[0], raws[0]);
        }
#if GMR_WALK_HOIST
        {   // unconditional (j2 = j1 when there is no second candidate)
          const V4<S> a = sm.st.ea[j2];
          bs[1] = sm.st.eb[j2];
          as[1] = Eval<S>::template alpha<kOpacity>(sub_rn(fpx, a.x), sub_rn(fpy, a.y), a.z, a.w, bs[1].x,
                                                    kOpacity ? sm.st.op[j2] : one, eps[1], raws[1]);
          if (!has2) as[1] = S(0);
        }
#else
        as[1] = S(0);
        if (has2) {
          const V4<S> a = sm.st.ea[j2];
          bs[1] = sm.st.eb[j2];
          as[1] = Eval<S>::template alpha<kOpacity>(sub_rn(fpx, a.x), sub_rn(fpy, a.y), a.z, a.w, bs[1].x,
                                                    kOpacity ? sm.st.op[j2] : one, eps[1], raws[1]);
        }
#endif
        // the rare transmittance stop leaves by a jump (no flag carried)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = js[u];
          const S a = as[u];
          if (!(a >= Const<S>::contrib_floor())) continue;
          const S om = sub_rn(one, a);
          const S test = mul_rn(T, om);
          if (test < Const<S>::t_stop()) goto bwd_stop;
          const S w = mul_rn(a, T);
          const S gdc = mypix.x * bs[u].y + mypix.y * bs[u].z + mypix.z * bs[u].w;
#if GMR_SUFFIX_Q
          Q -= gdc * w;   // Q = S_k + (g.bg - g_a) T_f, one update per pair
          const S d_alpha = gdc * T - Q * inv_om(om);
#else
          P += gdc * w;
          const S d_alpha = gdc * T - ((Ctot - P) + bterm) * inv_om(om);
#endif
          Rec s;
          s.x = raws[u] < Const<S>::alpha_clamp() ? d_alpha * a : S(0);
          s.y = w;
          if constexpr (kOpacity) {
            s.z = raws[u] < Const<S>::alpha_clamp() ? d_alpha * eps[u] : S(0);
            s.w = S(0);
          }
#if GMR_CW_HOIST
          const uint2 cwj = cws[u];
#else
          const uint2 cwj = sm.cw[warp][j];
#endif
          const uint32_t r = cwj.y + (uint32_t)__popc(cwj.x & lt);
          sm.rec[r] = s;
          sm.rq[r] = (uint8_t)my_pix;
          T = test;
        }
        continue;
      bwd_stop:
        done = true;
        it.stop();
        break;
      }
    }
    prefetch_records(p, nxt, vbase_item);
    item_next = nxt;   // the next batch's staging reuses it
#if !GMR_BWD_TMA
    if (nxt != 0xffffffffu)   // and the next batch's coverage words
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p.covbuf + (size_t)nxt_e * 8));
#endif
    __syncthreads();
    // ---- pass 2: my entry, my half of its records (pixel order) ----
    S acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = S(0);
    S aop = S(0);
    if (je < n) {
      const uint2 rr = make_uint2(sm.cw[0][je].y, sm.rend[je]);
      const uint32_t mid = kSplit == 2 ? rr.x + ((rr.y - rr.x + 1) >> 1) : rr.y;
      const uint32_t lo = half ? mid : rr.x, hi = half ? rr.y : mid;
      const V4<S> ea = sm.st.ea[je];
      const S ex0 = S(x0) - ea.x, ey0 = S(y0) - ea.y;
      auto add = [&](const Rec& s, int q, const V4<S>& pd) {
        const S dx = ex0 + pd.w, dy = ey0 + S(q >> 4);   // pd.w = S(q & 15)
        const S dpx = s.x * dx, dpy = s.x * dy;
        acc[0] += dpx;
        acc[1] += dpy;
        acc[2] += dpx * dx;
        acc[3] += dpx * dy;
        acc[4] += dpy * dy;
        acc[5] += s.y * pd.x;
        acc[6] += s.y * pd.y;
        acc[7] += s.y * pd.z;
        if constexpr (kOpacity) aop += s.z;
      };
      // not unrolled: measured 1.188 -> 1.171 ms at config 3 (the 4x unrolled
      // loop serialised its loads under the 48-register cap anyway)
#if GMR_RQ_WORDS
      // pixel ids four at a time (one 32-bit shared load per 4 records)
      const uint32_t* rq4 = reinterpret_cast<const uint32_t*>(sm.rq);
      uint32_t qw = lo < hi ? rq4[lo >> 2] : 0u;
#pragma unroll 1
      for (uint32_t r = lo; r < hi; ++r) {
        if ((r & 3u) == 0u) qw = rq4[r >> 2];
        const Rec s = sm.rec[r];
        const int q = (int)((qw >> ((r & 3u) << 3)) & 255u);
        add(s, q, sm.pix[q]);
      }
#else
#pragma unroll 1
      for (uint32_t r = lo; r < hi; ++r) {
        const Rec s = sm.rec[r];
        const int q = sm.rq[r];
        add(s, q, sm.pix[q]);
      }
#endif
    }
    // combine the two halves (fixed order) and store at the pre-sort slot
    if constexpr (kSplit == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 1);
      if (kOpacity) aop += __shfl_xor_sync(0xffffffffu, aop, 1);
    }
    if (half == 0 && je < n) {
      const uint32_t item_j = p.entry_item[base + je];
      const uint4 bi = p.bin[item_j];
      const uint32_t slot = p.entry_off[item_j] + entry_rank(make_uint2(bi.x, bi.y), bi.z, tx, ty);
      V4<S>* dst = reinterpret_cast<V4<S>*>(p.partial + (size_t)slot * 8);
      V4<S> lo, hi;
      lo.x = acc[0]; lo.y = acc[1]; lo.z = acc[2]; lo.w = acc[3];
      hi.x = acc[4]; hi.y = acc[5]; hi.z = acc[6]; hi.w = acc[7];
      dst[0] = lo;
      dst[1] = hi;
      if (kOpacity) p.partial_op[slot] = aop;
    }
    base += (uint32_t)n;
  }
#if GMR_BWD_TMA
  if (inflight) mbar_wait(&sm.bar, phase);   // no bulk copy may land after the CTA exits
#endif
  // the tile finished early: entries never loaded still own a partial slot,
  // which must hold zeros (every slot is written exactly once)
  for (uint32_t e = base + threadIdx.x; e < end; e += kBlendThreads) {
    const uint32_t item = p.entry_item[e];
    const uint4 bi = p.bin[item];
    const uint32_t slot = p.entry_off[item] + entry_rank(make_uint2(bi.x, bi.y), bi.z, tx, ty);
    V4<S>* dst = reinterpret_cast<V4<S>*>(p.partial + (size_t)slot * 8);
    V4<S> z;
    z.x = z.y = z.z = z.w = S(0);
    dst[0] = z;
    dst[1] = z;
    if (kOpacity) p.partial_op[slot] = S(0);
  }
}

// ---------------------------------------------------------------------------
// K5: per face — screen grads (summed over its entries, tile order) ->
// projection backward per view -> accumulate over views -> conversion backward
// ---------------------------------------------------------------------------

#ifndef GMR_K5_AHEAD
#define GMR_K5_AHEAD 4
#endif
template <typename S>
__device__ __forceinline__ void sum_entries(const S* __restrict__ partial, uint32_t off, uint32_t cnt,
                                            S acc[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = S(0);
  const V4<S>* src = reinterpret_cast<const V4<S>*>(partial + (size_t)off * 8);
  // loads of up to GMR_K5_AHEAD entries in flight, summed in entry (tile) order
  for (uint32_t e0 = 0; e0 < cnt; e0 += GMR_K5_AHEAD) {
    V4<S> lo[GMR_K5_AHEAD], hi[GMR_K5_AHEAD];
#pragma unroll
    for (int k = 0; k < GMR_K5_AHEAD; ++k)
      if (e0 + k < cnt) {
        lo[k] = src[2 * (e0 + k)];
        hi[k] = src[2 * (e0 + k) + 1];
      }
#pragma unroll
    for (int k = 0; k < GMR_K5_AHEAD; ++k)
      if (e0 + k < cnt) {
        acc[0] += lo[k].x; acc[1] += lo[k].y; acc[2] += lo[k].z; acc[3] += lo[k].w;
        acc[4] += hi[k].x; acc[5] += hi[k].y; acc[6] += hi[k].z; acc[7] += hi[k].w;
      }
  }
}

// conic sums -> (g_mean2d, g_cov2d) (render.py:344-360)
template <typename S>
__device__ __forceinline__ void conic_to_cov_grad(const S acc[8], S ca, S cb, S cc, S gm[2], S gcov[3]) {
  gm[0] = ca * acc[0] + cb * acc[1];
  gm[1] = cc * acc[1] + cb * acc[0];
  const S q00 = S(-0.5) * acc[2], q01 = S(-0.5) * acc[3], q11 = S(-0.5) * acc[4];
  // -M Q M with M = [[ca, cb], [cb, cc]], Q = [[q00, q01], [q01, q11]]
  const S mq00 = ca * q00 + cb * q01, mq01 = ca * q01 + cb * q11;
  const S mq10 = cb * q00 + cc * q01, mq11 = cb * q01 + cc * q11;
  gcov[0] = -(mq00 * ca + mq01 * cb);
  gcov[1] = -(mq00 * cb + mq01 * cc);
  gcov[2] = -(mq10 * cb + mq11 * cc);
}

template <typename S> struct FaceBwdArgs {
  const S* pos;
  const int32_t* faces;
  int64_t F;
  int view0, nviews;
  int rescale;
  const uint32_t* count;
  const uint32_t* entry_off;
  const Splat<S>* splat;
  const S* partial;
  double* face_acc;   // [F][12]: g_mean3 (3), g_cov3 sym (6), g_col (3), summed over views in float64
  S* corner;          // non-null on the last view group: write per-corner grads (convert_corners), not face_acc
  const DevStatus* st;   // the forward's status: after an entry overflow no partial was written
};

template <typename S>
__device__ __forceinline__ void convert_corners(const FaceGeo& g, const double a[12], int rescale, S* out);

template <typename S>
#ifndef GMR_K5_MINB
#define GMR_K5_MINB 4   // 128 registers: four partial runs in flight per face (latency-bound gathers)
#endif
__global__ void __launch_bounds__(128, GMR_K5_MINB) face_views_backward(FaceBwdArgs<S> p, const __grid_constant__ CamBatch<S> cams) {
  pdl_wait();
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.F) return;
  FaceGeo g;
  int32_t idx[3];
  load_face(p.pos, p.faces, f, p.rescale, g, idx);
  // the forward's float64 Gaussian in the render dtype (render.py:378)
  double cov64[6];
  face_cov3d(g, cov64);
  S cov[6], mean[3];
#pragma unroll
  for (int q = 0; q < 6; ++q) cov[q] = (S)cov64[q];
#pragma unroll
  for (int q = 0; q < 3; ++q) mean[q] = (S)g.mean[q];
  double acc[12];
  if (p.view0 == 0) {
#pragma unroll
    for (int q = 0; q < 12; ++q) acc[q] = 0.0;
  } else {
#pragma unroll
    for (int q = 0; q < 12; ++q) acc[q] = p.face_acc[f * 12 + q];
  }
  // the face's partials of consecutive views are one contiguous run
  // (item_offsets: face-major), so only the first offset is loaded; the
  // counts of a group of 8 views are loaded together, ahead of their use
  uint32_t off = p.entry_off[(int64_t)p.view0 * p.F + f];
  // An overflowed forward emitted no entries (scan_top), but the counts and
  // offsets still describe the full entry set, past the partial buffer: read
  // nothing and write zero gradients (the host reports GMR_ECAPACITY).
  const int nviews = p.st->overflow ? 0 : p.nviews;
  for (int v8 = 0; v8 < nviews; v8 += 8) {
   uint32_t cn[8], run = 0;
#pragma unroll
   for (int k = 0; k < 8; ++k) {
     cn[k] = (v8 + k < nviews) ? p.count[(int64_t)(p.view0 + v8 + k) * p.F + f] : 0u;
     run += cn[k];
   }
   // the group's partials are one contiguous run: start pulling it into L2
   {
     const char* b0 = reinterpret_cast<const char*>(p.partial + (size_t)off * 8);
     const char* b1 = reinterpret_cast<const char*>(p.partial + (size_t)(off + run) * 8);
     for (const char* q = b0; q < b1; q += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
   }
#pragma unroll
   for (int k = 0; k < 8; ++k) {
    const int vv = v8 + k;
    const uint32_t cnt = cn[k];
    if (!cnt) continue;
    const int64_t item = (int64_t)(p.view0 + vv) * p.F + f;
    const Splat<S> rec = p.splat[item];
    S s[8];
    sum_entries(p.partial, off, cnt, s);
    off += cnt;
    S gm[2], g2[3];
    conic_to_cov_grad(s, rec.a.z, rec.a.w, rec.b.x, gm, g2);
    const Cam<S>& cam = cams.cam[vv];
    S t[3], m2[2][3];
    cam_point(cam, mean, t);
    cam_m2(cam, t, m2);
    // g_cov3d += M2^T G M2 (render.py:382), G = [[g0, g1], [g1, g2]]
    const int ii[6] = {0, 0, 0, 1, 1, 2}, jj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int i = ii[q], j = jj[q];
      acc[3 + q] += (double)(m2[0][i] * (g2[0] * m2[0][j] + g2[1] * m2[1][j]) +
                             m2[1][i] * (g2[1] * m2[0][j] + g2[2] * m2[1][j]));
    }
    // g_M2 = (G + G^T) M2 Sigma (render.py:383-384)
    S ms[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      ms[r][0] = m2[r][0] * cov[0] + m2[r][1] * cov[1] + m2[r][2] * cov[2];
      ms[r][1] = m2[r][0] * cov[1] + m2[r][1] * cov[3] + m2[r][2] * cov[4];
      ms[r][2] = m2[r][0] * cov[2] + m2[r][1] * cov[4] + m2[r][2] * cov[5];
    }
    S gM[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      gM[0][k] = S(2) * (g2[0] * ms[0][k] + g2[1] * ms[1][k]);
      gM[1][k] = S(2) * (g2[1] * ms[0][k] + g2[2] * ms[1][k]);
    }
    // g_J = g_M2 R^T (render.py:385)
    S gJ[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        gJ[r][k] = gM[r][0] * cam.R[3 * k] + gM[r][1] * cam.R[3 * k + 1] + gM[r][2] * cam.R[3 * k + 2];
    const S iz = S(1) / t[2], iz2 = iz * iz;
    S gt0 = -cam.fx * iz2 * gJ[0][2] + gm[0] * cam.fx * iz;
    S gt1 = -cam.fy * iz2 * gJ[1][2] + gm[1] * cam.fy * iz;
    S gt2 = -cam.fx * iz2 * gJ[0][0] - cam.fy * iz2 * gJ[1][1] +
            S(2) * cam.fx * t[0] * iz2 * iz * gJ[0][2] + S(2) * cam.fy * t[1] * iz2 * iz * gJ[1][2] -
            gm[0] * cam.fx * t[0] * iz2 - gm[1] * cam.fy * t[1] * iz2;
    // g_mean3d = g_t R (render.py:401)
#pragma unroll
    for (int k = 0; k < 3; ++k) acc[k] += (double)(gt0 * cam.R[k] + gt1 * cam.R[3 + k] + gt2 * cam.R[6 + k]);
    acc[9] += (double)s[5];
    acc[10] += (double)s[6];
    acc[11] += (double)s[7];
   }
  }
  if (p.corner) {   // last view group: the conversion backward right here
    convert_corners<S>(g, acc, p.rescale, p.corner + f * 18);
  } else {
#pragma unroll
    for (int q = 0; q < 12; ++q) p.face_acc[f * 12 + q] = acc[q];
  }
}

// conversion backward per face (convert.py:393-425): the face's summed
// world-space grads a[12] = (g_mean3 (3), g_cov3 sym (6), g_col (3)) ->
// per-corner contributions out[c][6] = (g_pos xyz, g_col rgb)
template <typename S>
__device__ __forceinline__ void convert_corners(const FaceGeo& g, const double a[12], int rescale, S* out) {
  // G symmetric (xx,xy,xz,yy,yz,zz); gsym = 2G
  const double G[3][3] = {{a[3], a[4], a[5]}, {a[4], a[6], a[7]}, {a[5], a[7], a[8]}};
  double ge[3][3];   // g_e1, g_e2, g_e3 (float64 like convert.py:393-425)
  if (!g.degenerate) {
    const double sk = g.kappa * 2.0 / 36.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const double* e = g.e[i == 2 ? 2 : i];
        ge[i][r] = sk * (G[r][0] * e[0] + G[r][1] * e[1] + G[r][2] * e[2]);
      }
    }
    double d_area = 0.0;
    if (rescale && g.clamped) {
      double dk = 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          dk += G[r][c] * (g.e[0][r] * g.e[0][c] + g.e[1][r] * g.e[1][c] + g.e[2][r] * g.e[2][c]) / 36.0;
      d_area = dk / (kPi * sqrt(kDetEps));
    }
    double gn[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) gn[r] = kSz2 * 2.0 * (G[r][0] * g.n[0] + G[r][1] * g.n[1] + G[r][2] * g.n[2]);
    const double nd = g.n[0] * gn[0] + g.n[1] * gn[1] + g.n[2] * gn[2];
    double gu[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) gu[r] = (gn[r] - g.n[r] * nd) / g.nu + 0.5 * d_area * g.n[r];
    // g_e1 += e2 x g_u ; g_e2 += g_u x e1
    const double* e1 = g.e[0];
    const double* e2 = g.e[1];
    ge[0][0] += e2[1] * gu[2] - e2[2] * gu[1];
    ge[0][1] += e2[2] * gu[0] - e2[0] * gu[2];
    ge[0][2] += e2[0] * gu[1] - e2[1] * gu[0];
    ge[1][0] += gu[1] * e1[2] - gu[2] * e1[1];
    ge[1][1] += gu[2] * e1[0] - gu[0] * e1[2];
    ge[1][2] += gu[0] * e1[1] - gu[1] * e1[0];
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int r = 0; r < 3; ++r) ge[i][r] = 0.0;
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double third = a[r] / 3.0;
    out[0 + r] = (S)(third - ge[0][r] - ge[1][r]);
    out[6 + r] = (S)(third + ge[0][r] - ge[2][r]);
    out[12 + r] = (S)(third + ge[1][r] + ge[2][r]);
    const S gc = (S)(a[9 + r] / 3.0);
    out[3 + r] = gc;
    out[9 + r] = gc;
    out[15 + r] = gc;
  }
}

template <typename S>
__global__ void __launch_bounds__(128) face_convert_backward(const S* __restrict__ pos,
                                                             const int32_t* __restrict__ faces,
                                                             int64_t F, int rescale,
                                                             const double* __restrict__ face_acc,
                                                             S* __restrict__ corner) {
  pdl_wait();
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  FaceGeo g;
  int32_t idx[3];
  load_face(pos, faces, f, rescale, g, idx);
  double a[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) a[q] = face_acc[f * 12 + q];
  convert_corners<S>(g, a, rescale, corner + f * 18);
}

// K6: per vertex, sum its (face, corner) contributions in the reference's
// np.add.at order (all corner-0 faces ascending, then corner 1, then 2)
template <typename S>
__global__ void __launch_bounds__(256) vertex_gather(const uint32_t* __restrict__ vstart,
                                                    const uint32_t* __restrict__ slots, int64_t V,
                                                    int64_t F, const S* __restrict__ corner,
                                                    S* __restrict__ g_pos, S* __restrict__ g_col) {
  pdl_wait();
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  S gp[3] = {0, 0, 0}, gc[3] = {0, 0, 0};
  const uint32_t b = vstart[v], e = vstart[v + 1];
  const uint64_t F2 = 2 * (uint64_t)F;
  // four contributions in flight, summed in slot (np.add.at) order
  for (uint32_t k0 = b; k0 < e; k0 += 4) {
    S val[4][6];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (k0 + q < e) {
        const uint64_t sl = slots[k0 + q];   // corner * F + face
        const uint64_t c = sl >= F2 ? 2 : (sl >= (uint64_t)F ? 1 : 0);
        const S* src = corner + (sl - c * (uint64_t)F) * 18 + c * 6;
#pragma unroll
        for (int r = 0; r < 6; ++r) val[q][r] = src[r];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (k0 + q < e) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          gp[r] += val[q][r];
          gc[r] += val[q][3 + r];
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    g_pos[3 * v + r] = gp[r];
    g_col[3 * v + r] = gc[r];
  }
}

// splat path: per splat screen grads (render.py:338-360)
template <typename S>
__global__ void __launch_bounds__(256) splat_grads(const uint32_t* __restrict__ count,
                                                  const uint32_t* __restrict__ entry_off,
                                                  const Splat<S>* __restrict__ splat,
                                                  const S* __restrict__ partial,
                                                  const S* __restrict__ partial_op, int64_t K,
                                                  const DevStatus* __restrict__ st,
                                                  S* g_mean2d, S* g_cov2d, S* g_color, S* g_opacity) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  // after an entry overflow no partial exists (see face_views_backward)
  const uint32_t cnt = st->overflow ? 0u : count[i];
  S s[8];
  S op = S(0);
  if (cnt) {
    const uint32_t off = entry_off[i];
    sum_entries(partial, off, cnt, s);
    for (uint32_t e = 0; e < cnt; ++e) op += partial_op[off + e];
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = S(0);
  }
  const Splat<S> rec = splat[i];
  S gm[2], gc[3];
  conic_to_cov_grad(s, rec.a.z, rec.a.w, rec.b.x, gm, gc);
  if (!cnt) { gm[0] = gm[1] = gc[0] = gc[1] = gc[2] = S(0); }
  g_mean2d[2 * i] = gm[0];
  g_mean2d[2 * i + 1] = gm[1];
  g_cov2d[4 * i] = gc[0];
  g_cov2d[4 * i + 1] = gc[1];
  g_cov2d[4 * i + 2] = gc[1];
  g_cov2d[4 * i + 3] = gc[2];
  g_color[3 * i] = s[5];
  g_color[3 * i + 1] = s[6];
  g_color[3 * i + 2] = s[7];
  g_opacity[i] = op;
}

// topology: slot s = c * F + f -> key faces[3f + c]
__global__ void topo_keys(const int32_t* __restrict__ faces, int64_t F, uint32_t* key, uint32_t* val) {
  pdl_wait();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= 3 * F) return;
  const int64_t c = s / F, f = s - c * F;
  key[s] = (uint32_t)faces[3 * f + c];
  val[s] = (uint32_t)s;
}

// ---------------------------------------------------------------------------
// single-stage helpers (convert_mesh / convert_backward stage functions)
// ---------------------------------------------------------------------------

template <typename S>
__global__ void __launch_bounds__(128) convert_forward(const S* __restrict__ pos, const S* __restrict__ col,
                                                       const int32_t* __restrict__ faces, int64_t F,
                                                       int rescale, S* means, S* cov3d, S* colors,
                                                       uint8_t* degenerate) {
  pdl_wait();
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  FaceGeo g;
  int32_t idx[3];
  load_face(pos, faces, f, rescale, g, idx);
  double c[6];
  face_cov3d(g, c);
  const int map[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
#pragma unroll
  for (int k = 0; k < 9; ++k) cov3d[f * 9 + k] = (S)c[map[k]];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    means[3 * f + k] = (S)g.mean[k];
    colors[3 * f + k] = (col[3 * (int64_t)idx[0] + k] + col[3 * (int64_t)idx[1] + k] + col[3 * (int64_t)idx[2] + k]) / S(3);
  }
  if (degenerate) degenerate[f] = g.degenerate ? 1 : 0;
}

template <typename S>
__global__ void __launch_bounds__(256) pack_face_grads(const S* __restrict__ gm, const S* __restrict__ gcov,
                                                      const S* __restrict__ gcol, int64_t F,
                                                      double* __restrict__ face_acc) {
  pdl_wait();
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const S* G = gcov + f * 9;
  double* o = face_acc + f * 12;
  o[0] = gm[3 * f]; o[1] = gm[3 * f + 1]; o[2] = gm[3 * f + 2];
  // only (G + G^T)/2 matters (gsym and <G, c3> with c3 symmetric)
  o[3] = G[0];
  o[4] = 0.5 * ((double)G[1] + (double)G[3]);
  o[5] = 0.5 * ((double)G[2] + (double)G[6]);
  o[6] = G[4];
  o[7] = 0.5 * ((double)G[5] + (double)G[7]);
  o[8] = G[8];
  o[9] = gcol[3 * f]; o[10] = gcol[3 * f + 1]; o[11] = gcol[3 * f + 2];
}

}  // namespace gmr
