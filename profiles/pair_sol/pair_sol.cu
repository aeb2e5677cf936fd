// pair_sol.cu — arithmetic speed-of-light of the blend kernels (profiling
// infrastructure, not product code).
//
// The blend forward/backward (render.py:244-361) are bound by instruction
// issue and the shared-memory pipe, not HBM.  This microbenchmark measures
// what ONE (pixel, splat) pair costs when everything that is not the
// reference's per-pair arithmetic is taken away:
//   * every lane of every warp works (lane = pixel, all 32 lanes on the same
//     splat, every pair visible, no transmittance stop): no divergence;
//   * splat parameters come from shared memory as a broadcast (one
//     wavefront per load), staged once per CTA: no gathers, no coverage
//     masks, no depth-ordered batches, no barriers inside the loop;
//   * fwd: alpha (ex2.approx form of blend_forward), floor/stop tests,
//     weight, colour accumulation, transmittance update;
//   * bwd: the same plus g.c, the suffix recurrence, dL/dalpha (rcp.approx),
//     the clamp gate and the 8 gradient moments of the entry; the per-entry
//     sum over the pixels is a warp butterfly (amortised over 32 pairs) —
//     a lower bound on any per-entry reduction (records, atomics, ...).
// Result: ns per pair at full issue; times the config-3 pair count
// (pairs_c3.json) gives the floor of each blend kernel per view.
//
// Build/run: profiles/pair_sol/run.sh (nvcc -arch sm_100a, one GPU).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kThreads = 256;
constexpr int kEnt = 512;     // staged splats per CTA (the loop walks them L / kEnt times)

__device__ __forceinline__ float ex2(float x) { float r; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float rcpa(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

struct Ent { float4 a, b; };   // (mx, my, A, B), (C, r, g, b) as blend_forward stages them

__global__ void __launch_bounds__(kThreads) make_entries(Ent* e, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // far to the left of the tile and wide: alpha ~ 0.0067 .. 0.0094 on every
  // pixel (all visible, T stays above the stop over a 512-splat walk)
  const float l2e = 1.4426950408889634f;
  const float ca = 5.3e-5f * (1.f + 1e-4f * (i & 7)), cb = 1e-7f, cc = 1e-6f;
  e[i].a = make_float4(-420.f + 0.01f * (i & 3), 7.5f, -0.5f * l2e * ca, -l2e * cb);
  e[i].b = make_float4(-0.5f * l2e * cc, 0.2f, 0.5f, 0.7f);
}

// ops: per pair; L pairs per thread
__global__ void __launch_bounds__(kThreads) fwd_sol(const Ent* __restrict__ ent, int L, float* out) {
  __shared__ float4 sa[kEnt], sb[kEnt];
  for (int i = threadIdx.x; i < kEnt; i += kThreads) { sa[i] = ent[i].a; sb[i] = ent[i].b; }
  __syncthreads();
  const float fpx = (float)(threadIdx.x & 15), fpy = (float)(threadIdx.x >> 4);
  float T = 1.f, ar = 0.f, ag = 0.f, ab = 0.f;
  for (int k = 0; k < L; k += kEnt) {
#pragma unroll 4
    for (int j = 0; j < kEnt; ++j) {
      const float4 a = sa[j], b = sb[j];
      const float dx = fpx - a.x, dy = fpy - a.y;
      const float p2 = __fmaf_rn(dx, __fmaf_rn(a.z, dx, a.w * dy), (b.x * dy) * dy);
      float al = ex2(p2);
      al = al < 0.99f ? al : 0.99f;
      if (al >= (float)(1.0 / 255.0)) {
        const float test = T * (1.f - al);
        if (test < 1e-4f) break;
        const float w = al * T;
        ar += w * b.y; ag += w * b.z; ab += w * b.w;
        T = test;
      }
    }
    T = fmaxf(T, 0.5f);   // keep the walk alive for any L (values are irrelevant)
  }
  out[blockIdx.x * kThreads + threadIdx.x] = ar + ag + ab + T;
}

__global__ void __launch_bounds__(kThreads) bwd_sol(const Ent* __restrict__ ent, int L, float* out) {
  __shared__ float4 sa[kEnt], sb[kEnt];
  __shared__ float acc[kThreads / 32][8];
  for (int i = threadIdx.x; i < kEnt; i += kThreads) { sa[i] = ent[i].a; sb[i] = ent[i].b; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float fpx = (float)(threadIdx.x & 15), fpy = (float)(threadIdx.x >> 4);
  const float g0 = 0.3f + 0.001f * lane, g1 = -0.2f, g2 = 0.1f, Ctot = 0.05f, bterm = 0.01f;
  float T = 1.f, P = 0.f;
  float m[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) m[q] = 0.f;
  for (int k = 0; k < L; k += kEnt) {
#pragma unroll 2
    for (int j = 0; j < kEnt; ++j) {
      const float4 a = sa[j], b = sb[j];
      const float dx = fpx - a.x, dy = fpy - a.y;
      const float p2 = __fmaf_rn(dx, __fmaf_rn(a.z, dx, a.w * dy), (b.x * dy) * dy);
      const float raw = ex2(p2);
      const float al = raw < 0.99f ? raw : 0.99f;
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = 0.f;
      if (al >= (float)(1.0 / 255.0)) {
        const float om = 1.f - al;
        const float test = T * om;
        if (test < 1e-4f) break;
        const float w = al * T;
        const float gdc = g0 * b.y + g1 * b.z + g2 * b.w;
        P += gdc * w;
        const float d_alpha = gdc * T - ((Ctot - P) + bterm) * rcpa(om);
        const float dp = raw < 0.99f ? d_alpha * al : 0.f;
        const float dpx = dp * dx, dpy = dp * dy;
        v[0] = dpx; v[1] = dpy; v[2] = dpx * dx; v[3] = dpx * dy; v[4] = dpy * dy;
        v[5] = w * g0; v[6] = w * g1; v[7] = w * g2;
        T = test;
      }
      // per-entry sum over the warp's 32 pixels (butterfly), one lane keeps it
#pragma unroll
      for (int q = 0; q < 8; ++q) {
#pragma unroll
        for (int o = 16; o; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
      }
      if (lane == (j & 31)) {
#pragma unroll
        for (int q = 0; q < 8; ++q) m[q] += v[q];
      }
    }
    T = fmaxf(T, 0.5f);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) if (lane == 0) acc[warp][q] = m[q];
  out[blockIdx.x * kThreads + threadIdx.x] = m[0] + m[1] + m[2] + m[3] + m[4] + m[5] + m[6] + m[7] + T + acc[warp][lane & 7];
}

// bwd without the butterfly: the per-pixel part only (what pass 1 of a
// record-based design must do per pair), moments kept per lane
__global__ void __launch_bounds__(kThreads) bwd_pixel_sol(const Ent* __restrict__ ent, int L, float* out) {
  __shared__ float4 sa[kEnt], sb[kEnt];
  for (int i = threadIdx.x; i < kEnt; i += kThreads) { sa[i] = ent[i].a; sb[i] = ent[i].b; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float fpx = (float)(threadIdx.x & 15), fpy = (float)(threadIdx.x >> 4);
  const float g0 = 0.3f + 0.001f * lane, g1 = -0.2f, g2 = 0.1f, Ctot = 0.05f, bterm = 0.01f;
  float T = 1.f, P = 0.f, s0 = 0.f, s1 = 0.f;
  for (int k = 0; k < L; k += kEnt) {
#pragma unroll 4
    for (int j = 0; j < kEnt; ++j) {
      const float4 a = sa[j], b = sb[j];
      const float dx = fpx - a.x, dy = fpy - a.y;
      const float p2 = __fmaf_rn(dx, __fmaf_rn(a.z, dx, a.w * dy), (b.x * dy) * dy);
      const float raw = ex2(p2);
      const float al = raw < 0.99f ? raw : 0.99f;
      if (al >= (float)(1.0 / 255.0)) {
        const float om = 1.f - al;
        const float test = T * om;
        if (test < 1e-4f) break;
        const float w = al * T;
        const float gdc = g0 * b.y + g1 * b.z + g2 * b.w;
        P += gdc * w;
        const float d_alpha = gdc * T - ((Ctot - P) + bterm) * rcpa(om);
        const float dp = raw < 0.99f ? d_alpha * al : 0.f;
        s0 += dp * dx;   // stands in for the record write of (dp, w)
        s1 += w;
        T = test;
      }
    }
    T = fmaxf(T, 0.5f);
  }
  out[blockIdx.x * kThreads + threadIdx.x] = s0 + s1 + T;
}

int main(int argc, char** argv) {
  const double pairs_per_view = argc > 1 ? atof(argv[1]) : 14.8e6;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8;                  // 8 CTAs x 256 threads per SM
  const int L = 8 * kEnt;
  Ent* ent; float* out;
  cudaMalloc(&ent, kEnt * sizeof(Ent));
  cudaMalloc(&out, (size_t)blocks * kThreads * sizeof(float));
  make_entries<<<(kEnt + 255) / 256, 256>>>(ent, kEnt);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(const Ent*, int, float*)) {
    for (int w = 0; w < 3; ++w) k<<<blocks, kThreads>>>(ent, L, out);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      k<<<blocks, kThreads>>>(ent, L, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double pairs = (double)blocks * kThreads * L;
    const double ns = best * 1e6 / pairs;
    printf("{\"kernel\": \"%s\", \"pairs\": %.0f, \"ms\": %.4f, \"ns_per_pair\": %.6f, "
           "\"Gpairs_per_s\": %.2f, \"us_per_view_at_pairs\": %.2f, \"pairs_per_view\": %.0f}\n",
           name, pairs, best, ns, pairs / (best * 1e-3) / 1e9, ns * pairs_per_view / 1e3, pairs_per_view);
  };
  run("fwd_sol", fwd_sol);
  run("bwd_pixel_sol", bwd_pixel_sol);
  run("bwd_sol", bwd_sol);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
