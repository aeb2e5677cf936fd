// gmr_common.cuh — shared device types and math for the GMR kernels (sm_100a).
//
// Constants and conventions follow the reference renderer
// (pkg/src/meshsplat/render.py:26-30, convert.py:27-28, mesh.py:15).
// Everything is templated on the scalar S (float = fast path, double =
// parity path).  Decision-relevant arithmetic (power, alpha, transmittance,
// tile rectangles) uses explicitly rounded ops (no FMA contraction) so it
// follows numpy's evaluation order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "../../include/gmr.h"

namespace gmr {

// Programmatic dependent launch (sm_90+): every kernel of the library waits
// here for its stream predecessor's completion and memory before touching
// anything, so a launch with the programmatic-serialization attribute can be
// processed while the predecessor drains (the inter-kernel gap shrinks;
// nothing runs early).  A no-op for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Host side: launch with the attribute (GMR_PDL=0 in the environment turns it
// off).  A failed launch is kept for the next GMR_LAUNCHED check.
inline thread_local cudaError_t g_launch_err = cudaSuccess;
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("GMR_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess && g_launch_err == cudaSuccess) g_launch_err = e;
}

constexpr int kTile = 16;
constexpr int kBlendThreads = 256;   // one CTA per 16x16 tile, one pixel per thread
constexpr int kMaxViewsPerLaunch = 64;

template <typename S> struct Const;
template <> struct Const<float> {
  static __device__ __forceinline__ float alpha_clamp() { return 0.99f; }
  static __device__ __forceinline__ float contrib_floor() { return (float)(1.0 / 255.0); }
  static __device__ __forceinline__ float t_stop() { return 1e-4f; }
  static __device__ __forceinline__ float dilation() { return 0.3f; }
};
template <> struct Const<double> {
  static __device__ __forceinline__ double alpha_clamp() { return 0.99; }
  static __device__ __forceinline__ double contrib_floor() { return 1.0 / 255.0; }
  static __device__ __forceinline__ double t_stop() { return 1e-4; }
  static __device__ __forceinline__ double dilation() { return 0.3; }
};

// conversion constants (convert.py:27-28, mesh.py:15), evaluated in S
constexpr double kSz2 = 1e-12;           // S_Z^2
constexpr double kDetEps = 1e-14;
constexpr double kDegenerateArea = 1e-12;
constexpr double kPi = 3.14159265358979323846;

// explicitly rounded arithmetic (no FMA contraction)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float exp_s(float x) { return expf(x); }
__device__ __forceinline__ double exp_s(double x) { return exp(x); }
__device__ __forceinline__ float sqrt_s(float x) { return sqrtf(x); }
__device__ __forceinline__ double sqrt_s(double x) { return sqrt(x); }
// C99 / numpy semantics: hypot(+-inf, y) = +inf even when y is NaN (an
// overflowed screen covariance keeps radius = inf, so the splat is kept and
// then reported as non-finite, render.py:84-88,125-133,191-197)
__device__ __forceinline__ float hypot_s(float a, float b) {
  return (isinf(a) || isinf(b)) ? INFINITY : hypotf(a, b);
}
__device__ __forceinline__ double hypot_s(double a, double b) {
  return (isinf(a) || isinf(b)) ? (double)INFINITY : hypot(a, b);
}
__device__ __forceinline__ float log_s(float x) { return logf(x); }
__device__ __forceinline__ double log_s(double x) { return log(x); }
__device__ __forceinline__ float floor_s(float x) { return floorf(x); }
__device__ __forceinline__ double floor_s(double x) { return floor(x); }
__device__ __forceinline__ bool finite_s(float x) { return isfinite(x); }
__device__ __forceinline__ bool finite_s(double x) { return isfinite(x); }

// Order-preserving unsigned key of a positive depth (depth > near > 0).
__device__ __forceinline__ uint32_t depth_key(float d) { return __float_as_uint(d); }
__device__ __forceinline__ unsigned long long depth_key(double d) {
  return (unsigned long long)__double_as_longlong(d);
}
template <typename S> struct KeyOf;
template <> struct KeyOf<float> { typedef uint32_t type; };
template <> struct KeyOf<double> { typedef unsigned long long type; };

template <typename S> struct V4 { S x, y, z, w; };
template <typename S> struct V2 { S x, y; };
template <> struct alignas(8) V2<float> { float x, y; };
template <> struct alignas(16) V2<double> { double x, y; };
template <> struct alignas(16) V4<float> { float x, y, z, w; };
template <> struct alignas(32) V4<double> { double x, y, z, w; };

// Per-item screen-space record read by the blend kernels:
//   a = (mean_x, mean_y, conic_a, conic_b), b = (conic_c, ext_x, ext_y, tau_cov)
// (see screen_shape: the coverage bound, used only to skip pairs).
template <typename S> struct Splat {
  V4<S> a, b;
};

// Camera converted to S.  Views of one launch are passed by value.
template <typename S> struct Cam {
  S R[9], t[3], fx, fy, cx, cy, near_plane, far_plane;
};
template <typename S> struct CamBatch {
  Cam<S> cam[kMaxViewsPerLaunch];
  int count;
};

// Device-side status words, at offset 0 of every workspace.
struct DevStatus {
  unsigned long long entries;    // sum of tile counts (may exceed capacity)
  unsigned long long kept;       // items with count > 0
  unsigned int bad_item[6];      // per field: min offending item (0xffffffff = none)
  unsigned int overflow;
  unsigned int key_lo, key_hi;   // float32 path: min / max depth key of the kept splats (KeyRange)
  unsigned int pad[2];
  unsigned int max_bin;          // longest (view, tile) list of the last forward (byte 60)
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Tile rectangle (render.py:214-217): floor((m -/+ r)/16) clipped, inclusive.
template <typename S>
__device__ __forceinline__ void tile_rect(S mx, S my, S r, int tiles_x, int tiles_y, int& tx0,
                                          int& ty0, int& tx1, int& ty1) {
  const S inv = S(1) / S(kTile);   // exact (power of two)
  auto clampi = [](S v, int hi) {
    S f = floor_s(v);
    // np.floor(...).astype(int64) then clip; the clip of huge magnitudes is
    // done in floating point first so the int conversion cannot overflow
    if (f < S(0)) return 0;
    if (f > S(hi)) return hi;
    return (int)f;
  };
  tx0 = clampi(mul_rn(sub_rn(mx, r), inv), tiles_x - 1);
  tx1 = clampi(mul_rn(add_rn(mx, r), inv), tiles_x - 1);
  ty0 = clampi(mul_rn(sub_rn(my, r), inv), tiles_y - 1);
  ty1 = clampi(mul_rn(add_rn(my, r), inv), tiles_y - 1);
}

// conic (render.py:76-81), 3-sigma radius (render.py:84-88,124) and the
// coverage bound of a screen covariance (a, b, c) with opacity o:
// alpha >= 1/255  <=>  o exp(-q/2) >= 1/255  <=>  q <= tau = 2 ln(255 o).
// `tau_cov` is tau padded (relative and absolute) so that the per-row
// coverage solve in the blend kernels is conservative; ext_* are the
// half-widths of that ellipse's box (negative = never visible).  Neither
// decides a pixel: they only let the kernels skip (pixel, splat) pairs
// that cannot reach alpha >= 1/255.
template <typename S>
__device__ __forceinline__ void screen_shape(S a, S b, S c, S o, S& ca, S& cb, S& cc, S& radius,
                                             S& ext_x, S& ext_y, S& tau_cov) {
  S det = sub_rn(mul_rn(a, c), mul_rn(b, b));
  ca = div_rn(c, det);
  cb = div_rn(-b, det);
  cc = div_rn(a, det);
  S half_sum = mul_rn(S(0.5), add_rn(a, c));
  S half_diff = mul_rn(S(0.5), sub_rn(a, c));
  radius = mul_rn(S(3), sqrt_s(add_rn(half_sum, hypot_s(half_diff, b))));
  S tau = S(2) * log_s(S(255) * o);
  if (!(tau > S(-1e-3))) {
    ext_x = ext_y = tau_cov = S(-1);
  } else {
    tau_cov = fmax(tau, S(0)) * S(1.004) + S(2e-3);
    ext_x = sqrt_s(tau_cov * a) * S(1.001) + S(0.02);
    ext_y = sqrt_s(tau_cov * c) * S(1.001) + S(0.02);
  }
}

}  // namespace gmr
