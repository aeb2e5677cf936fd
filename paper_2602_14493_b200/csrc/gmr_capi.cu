// gmr_capi.cu — extern "C" entry points of libgmr.so (see include/gmr.h).
//
// Host-side sequencing of the kernels in gmr_kernels.cuh.  The library
// never allocates: every buffer lives in the caller's workspace, carved by
// `plan()` identically for the size query, the forward and the backward.
#include <math.h>
#include <stdlib.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <utility>
#include <vector>

#include "gmr_kernels.cuh"
#include "gmr_stage.cuh"
#include "gmr_train.cuh"
#include "gmr_eval.cuh"

using namespace gmr;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define GMR_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) return fail(GMR_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

thread_local long long g_launches = 0;   // kernels launched by this thread (bench evidence)

#define GMR_LAUNCHED()                                                                   \
  do {                                                                                   \
    ++g_launches;                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ == cudaSuccess) e_ = g_launch_err;                                            \
    g_launch_err = cudaSuccess;                                                          \
    if (e_ != cudaSuccess) return fail(GMR_ECUDA, "launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

// Optional per-stage CUDA-event timers (gmr_timing_enable / gmr_timing_read):
// events are recorded on the launching stream around each stage, so bench.py
// can attribute device time to kernels inside its own timed region.
enum Stage { kStProject = 0, kStDepthSort, kStEmit, kStTileSort, kStBlendFwd, kStBlendBwd, kStFaceBwd,
             kStVertex, kNumStages };
struct StageTimer {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[kNumStages];
  double ms[kNumStages] = {0};
  long long calls[kNumStages] = {0};
};
thread_local StageTimer g_timer;

struct StageScope {
  int stage;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  StageScope(int s, cudaStream_t stream) : stage(s), st(stream) {
    if (!g_timer.on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  ~StageScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    g_timer.pending[stage].emplace_back(a, b);
  }
};

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }
inline int ceil_log2(uint64_t x) {
  int b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}
inline unsigned grid_for(uint64_t n, unsigned block) { return (unsigned)std::max<uint64_t>(1, (n + block - 1) / block); }

// Workspace layout (byte offsets).
struct Layout {
  size_t status, splat, col4, bin, count, dkey[2], ditem[2], offs, fbsum, entry_off, bsum, nent;
  size_t ekey[2], eval[2], bounds, sched, schedcnt, covbuf, t_final, hist, partial, partial_op, face_acc, corner, aux, loss_tile;
  size_t total;
  uint64_t items, faces, bins, pixels, ecap;
  int views, tiles_x, tiles_y, tiles;
  int depth_bits, entry_bits;
};

Layout plan(uint64_t faces, int views, int W, int H, uint64_t ecap, int dtype, bool mesh) {
  Layout L{};
  const size_t s = dtype == GMR_F64 ? 8 : 4;
  L.faces = faces;
  L.views = views;
  L.items = faces * (uint64_t)views;
  L.tiles_x = (W + kTile - 1) / kTile;
  L.tiles_y = (H + kTile - 1) / kTile;
  L.tiles = L.tiles_x * L.tiles_y;
  L.bins = (uint64_t)L.tiles * views;
  L.pixels = (uint64_t)W * H * views;
  L.ecap = ecap;
  L.depth_bits = dtype == GMR_F64 ? 64 : 32;
  L.entry_bits = std::max(1, ceil_log2(L.bins));
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + std::max<size_t>(bytes, 1)); return r; };
  const size_t ks = dtype == GMR_F64 ? 8 : 4;
  L.status = take(sizeof(DevStatus));
  L.splat = take(L.items * 8 * s);
  L.col4 = take(faces * 4 * s);
  L.bin = take(L.items * 16);
  L.count = take(L.items * 4);
  L.dkey[0] = take(L.items * ks);
  L.dkey[1] = take(L.items * ks);
  L.ditem[0] = take(L.items * 4);
  L.ditem[1] = take(L.items * 4);
  L.offs = take(L.items * 4);
  L.fbsum = take(((faces + 255) / 256 + 1) * 4);
  L.entry_off = take(L.items * 4);
  L.bsum = take(((L.items + kScanTile - 1) / kScanTile + 1) * 4);
  L.nent = take(16);
  L.ekey[0] = take(ecap * 4);
  L.ekey[1] = take(ecap * 4);
  L.eval[0] = take(ecap * 4);
  L.eval[1] = take(ecap * 4);
  L.bounds = take((L.bins + 1) * 4);
  L.sched = take(L.bins * 4);
  L.schedcnt = take(513 * 4);
  L.covbuf = take(ecap * 32);
  L.t_final = take(L.pixels * s);
  L.hist = take(std::max(radix_hist_words((uint32_t)std::min<uint64_t>(L.items, 0xffffffffu)),
                         radix_hist_words((uint32_t)std::min<uint64_t>(ecap, 0xffffffffu))) * 4);
  L.partial = take(ecap * 8 * s);
  L.partial_op = take(mesh ? 0 : ecap * s);
  L.face_acc = take(mesh ? faces * 12 * 8 : 0);
  L.corner = take(mesh ? faces * 18 * s : 0);
  L.aux = take(mesh ? L.items * 2 * s : 0);
  L.loss_tile = take(L.bins * 16);
  L.total = o;
  return L;
}

template <typename T> inline T* at(void* ws, size_t off) { return reinterpret_cast<T*>((char*)ws + off); }

int check_raster(const GmrRaster* r) {
  if (!r) return fail(GMR_EINVAL, "raster settings are null");
  if (r->width < 1 || r->height < 1) return fail(GMR_EINVAL, "width and height must be >= 1");
  if ((int64_t)r->width > 16 * 65535 || (int64_t)r->height > 16 * 65535)
    return fail(GMR_EINVAL, "image too large");
  if (r->dtype != GMR_F32 && r->dtype != GMR_F64) return fail(GMR_EINVAL, "dtype must be GMR_F32 or GMR_F64");
  return GMR_OK;
}

template <typename S>
CamBatch<S> make_cams(const GmrCamera* cams, int v0, int nv) {
  CamBatch<S> b;
  memset(&b, 0, sizeof(b));
  b.count = nv;
  for (int i = 0; i < nv; ++i) {
    const GmrCamera& c = cams[v0 + i];
    Cam<S>& d = b.cam[i];
    for (int k = 0; k < 9; ++k) d.R[k] = (S)c.R[k];
    for (int k = 0; k < 3; ++k) d.t[k] = (S)c.t[k];
    d.fx = (S)c.fx; d.fy = (S)c.fy; d.cx = (S)c.cx; d.cy = (S)c.cy;
    d.near_plane = (S)c.near_plane; d.far_plane = (S)c.far_plane;
  }
  return b;
}

// optional fused losses of a forward
struct LossArgs {
  const void* target_rgb;
  const void* target_mask;
  double scale_rgb, scale_alpha;
  void* g_rgb;
  void* g_alpha;
  double* sums;   // device [2]
};

// optional 8-bit outputs of a forward (dataset rendering)
struct ImageArgs {
  uint8_t* rgb8;
  uint8_t* alpha8;
};

// Global depth order on the mesh path: K1 packs each item's entry count into
// the bits of its sort value above the item id (at least 4 of them), so the
// count scan after the depth sort reads them in order instead of gathering
// count[item].  Returns the item-id width, 0 = no packing.
inline int pack_shift_for(const Layout& L, const GmrRaster* r) {
  if (r->flags & GMR_FLAG_TILE_DEPTH_SORT) return 0;
  const int b = std::max(1, ceil_log2(L.items));
  return b <= 28 ? b : 0;
}

// Binning (K2) + blend forward (K3) over prepared item records.
template <typename S>
int bin_and_blend(const Layout& L, void* ws, const GmrRaster* r, void* rgb, void* alpha,
                  cudaStream_t st, bool unit_opacity, const LossArgs* la = nullptr, const ImageArgs* ia = nullptr,
                  void* status_host = nullptr, void* status_event = nullptr) {
  typedef typename KeyOf<S>::type K;
  const uint32_t items = (uint32_t)L.items;
  // (tile, depth, source) order (render.py:227), either way:
  //  default: stable depth sort of all items, entries emitted in depth
  //    order, stable (view, tile) sort;
  //  GMR_FLAG_TILE_DEPTH_SORT: entries emitted in item order, stable
  //    (view, tile) sort, then each tile list sorted by depth on its own.
  const bool tile_depth_sort = (r->flags & GMR_FLAG_TILE_DEPTH_SORT) != 0;
  // K1 packed the entry counts into the depth-sort values (mesh path only;
  // the splat path's values are plain item ids)
  const int packed = unit_opacity ? pack_shift_for(L, r) : 0;
  K* dk[2] = {at<K>(ws, L.dkey[0]), at<K>(ws, L.dkey[1])};
  const uint32_t* order = nullptr;
  // range-reduced global depth sort: the consumers pick the result buffer on
  // the device (order, order_alt, krange)
  const uint32_t* order_alt = nullptr;
  const uint32_t* krange = nullptr;
  if (!tile_depth_sort) {
    uint32_t* di[2] = {at<uint32_t>(ws, L.ditem[0]), at<uint32_t>(ws, L.ditem[1])};
    StageScope sc(kStDepthSort, st);
    // mesh path: K1 recorded the kept splats' depth-key span in the status
    const uint32_t* kr = unit_opacity ? &at<DevStatus>(ws, L.status)->key_lo : nullptr;
    bool reduced = false;
    const int cur = radix_sort_pairs<K>(dk, di, nullptr, items, items, L.depth_bits, at<uint32_t>(ws, L.hist), st,
                                        /*random_digits=*/true, kr, &reduced);
    g_launches += radix_sort_launches<K>((uint32_t)items, L.depth_bits) - 1;
    GMR_LAUNCHED();
    order = di[cur];
    if (reduced) {
      order = di[0];
      order_alt = di[1];
      krange = kr;
    }
  }
  StageScope* emit_scope = new StageScope(kStEmit, st);
  const uint32_t* count = at<uint32_t>(ws, L.count);
  const int nb = (int)((items + kScanTile - 1) / kScanTile);
  uint32_t* bsum = at<uint32_t>(ws, L.bsum);
  uint32_t* nent = at<uint32_t>(ws, L.nent);
  DevStatus* dst = at<DevStatus>(ws, L.status);
  if (items) {
    pdl_launch(scan_reduce, dim3((nb + kReduceTiles - 1) / kReduceTiles), dim3(256), 0, st, order, order_alt, krange, L.depth_bits, count, items, bsum,
               packed);
    GMR_LAUNCHED();
  }
  pdl_launch(scan_top, dim3(1), dim3(kTopThreads), 0, st, bsum, nb, dst, (unsigned long long)L.ecap, nent);
  GMR_LAUNCHED();
  // the status is final here (K1's non-finite items, the entry count and the
  // capacity verdict): publish it early so the host can validate the call
  // while the rest of the forward runs
  if (status_host) GMR_CUDA(cudaMemcpyAsync(status_host, dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  if (status_event) GMR_CUDA(cudaEventRecord((cudaEvent_t)status_event, st));
  uint32_t* ek[2] = {at<uint32_t>(ws, L.ekey[0]), at<uint32_t>(ws, L.ekey[1])};
  uint32_t* ev[2] = {at<uint32_t>(ws, L.eval[0]), at<uint32_t>(ws, L.eval[1])};
  if (items) {
    pdl_launch(scan_emit, dim3((nb + kEmitTiles - 1) / kEmitTiles), dim3(256), 0, st, order, order_alt, krange, L.depth_bits, at<uint4>(ws, L.bin), items, bsum,
                                  (uint32_t)L.faces,
                                  L.tiles_x, (uint32_t)L.tiles, nent, ek[0], ev[0], packed);
    GMR_LAUNCHED();
    // face-major partial offsets (bsum and offs are free again here)
    const int fb = (int)((L.faces + 255) / 256);
    // the mesh path's K1 already scanned each block of faces (one launch)
    const bool k1_scanned = unit_opacity && L.views <= kMaxViewsPerLaunch;
    uint32_t* fsum = k1_scanned ? at<uint32_t>(ws, L.fbsum) : bsum;
    if (!k1_scanned) {
      pdl_launch(face_counts, dim3(fb), dim3(256), 0, st, count, (uint32_t)L.faces, L.views, at<uint32_t>(ws, L.offs), bsum);
      GMR_LAUNCHED();
    }
    pdl_launch(scan_inplace, dim3(1), dim3(kTopThreads), 0, st, fsum, fb);
    GMR_LAUNCHED();
    pdl_launch(item_offsets, dim3(fb), dim3(256), 0, st, count, (uint32_t)L.faces, L.views, at<uint32_t>(ws, L.offs), fsum,
                                     at<uint32_t>(ws, L.entry_off));
    GMR_LAUNCHED();
  }
  delete emit_scope;
  const uint32_t ecap = (uint32_t)std::min<uint64_t>(L.ecap, 0xffffffffu);
  int ecur;
  {
    StageScope sc(kStTileSort, st);
    // entries emitted in depth order carry spatially random tile keys (ballot
    // ranking); in item order they are coherent (match_any)
    ecur = radix_sort_pairs<uint32_t>(ek, ev, nent, 0, ecap, L.entry_bits, at<uint32_t>(ws, L.hist), st,
                                      /*random_digits=*/!tile_depth_sort);
    g_launches += radix_sort_launches<uint32_t>(ecap, L.entry_bits);
    pdl_launch(tile_ranges, dim3(grid_for((uint64_t)ecap / 4 + 1, 256)), dim3(256), 0, st, ek[ecur], nent, 0, (uint32_t)L.bins,
               at<uint32_t>(ws, L.bounds), at<uint32_t>(ws, L.schedcnt));
    GMR_LAUNCHED();
    if (L.bins) {
      if (L.bins <= 4096) {   // few bins: one block
        pdl_launch(tile_schedule, dim3(1), dim3(kSchedThreads), 0, st, at<uint32_t>(ws, L.bounds), (uint32_t)L.bins,
                   at<uint32_t>(ws, L.sched), dst);
        GMR_LAUNCHED();
      } else {
        const unsigned nbs = (unsigned)((L.bins + 255) / 256);
        pdl_launch(sched_hist, dim3(nbs), dim3(256), 0, st, at<uint32_t>(ws, L.bounds), (uint32_t)L.bins,
                   at<uint32_t>(ws, L.schedcnt));
        GMR_LAUNCHED();
        pdl_launch(sched_place, dim3(nbs), dim3(256), 0, st, at<uint32_t>(ws, L.bounds), (uint32_t)L.bins,
                   at<uint32_t>(ws, L.schedcnt), at<uint32_t>(ws, L.sched), dst);
        GMR_LAUNCHED();
      }
    }
  }
  if (L.bins && tile_depth_sort) {
    StageScope sc(kStDepthSort, st);
    // heaviest bins first; bins over the shared-memory cap use the partial
    // buffer (free until the backward) as key/value scratch
    K* gk0 = at<K>(ws, L.partial);
    K* gk1 = gk0 + ecap;
    uint32_t* gv1 = reinterpret_cast<uint32_t*>(gk1 + ecap);
    pdl_launch(bin_depth_sort<K>, dim3((unsigned)L.bins), dim3(kBinSortThreads), 0, st, at<uint32_t>(ws, L.bounds),
                                                                    at<uint32_t>(ws, L.sched), dk[0], ev[ecur],
                                                                    gk0, gk1, gv1);
    GMR_LAUNCHED();
  }
  BlendArgs<S> a{};
  a.bounds = at<uint32_t>(ws, L.bounds);
  a.sched = at<uint32_t>(ws, L.sched);
  a.entry_item = ev[ecur];
  a.splat = at<Splat<S>>(ws, L.splat);
  a.col4 = at<V4<S>>(ws, L.col4);
  a.bin = at<uint4>(ws, L.bin);
  a.entry_off = at<uint32_t>(ws, L.entry_off);
  a.items_per_view = (uint32_t)L.faces;
  a.tiles_x = L.tiles_x;
  a.tiles_per_view = (uint32_t)L.tiles;
  a.W = r->width;
  a.H = r->height;
  a.bg0 = (S)r->background[0];
  a.bg1 = (S)r->background[1];
  a.bg2 = (S)r->background[2];
  a.rgb = (S*)rgb;
  a.alpha = (S*)alpha;
  a.t_final = at<S>(ws, L.t_final);
  if (la) {
    a.target_rgb = (const S*)la->target_rgb;
    a.target_mask = (const S*)la->target_mask;
    a.scale_rgb = la->scale_rgb;
    a.scale_alpha = la->scale_alpha;
    a.g_rgb_out = (S*)la->g_rgb;
    a.g_alpha_out = (S*)la->g_alpha;
    a.loss_tile = at<double>(ws, L.loss_tile);
  }
  // forwards that can be followed by a backward keep their coverage masks
  a.covbuf = ia ? nullptr : at<uint32_t>(ws, L.covbuf);
  if (ia) {
    a.rgb8 = ia->rgb8;
    a.alpha8 = ia->alpha8;
  }
  if (L.bins) {
    StageScope sc(kStBlendFwd, st);
    // all of the SM's unified L1/shared memory as shared memory: the
    // default carveout would cap residency below what registers allow
    // once per instantiation (thread-safe static init; also keeps it out of graph captures)
    static const cudaError_t attr_rc = [] {
      const cudaError_t e = cudaFuncSetAttribute(blend_forward<S, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                 (int)cudaSharedmemCarveoutMaxShared);
      return e != cudaSuccess ? e
                              : cudaFuncSetAttribute(blend_forward<S, true>,
                                                     cudaFuncAttributePreferredSharedMemoryCarveout,
                                                     (int)cudaSharedmemCarveoutMaxShared);
    }();
    GMR_CUDA(attr_rc);
    // mesh splats all have opacity 1 (convert.py:326): the evaluator skips the product
    if (unit_opacity) pdl_launch(blend_forward<S, false>, dim3((unsigned)L.bins), dim3(kBlendThreads), 0, st, a);
    else pdl_launch(blend_forward<S, true>, dim3((unsigned)L.bins), dim3(kBlendThreads), 0, st, a);
    GMR_LAUNCHED();
  }
  if (la && L.bins) {
    pdl_launch(loss_reduce, dim3(1), dim3(256), 0, st, at<double>(ws, L.loss_tile), (uint32_t)L.bins, la->sums);
    GMR_LAUNCHED();
  }
  return GMR_OK;
}

template <typename S>
int render_forward_t(const GmrMesh* m, const GmrCamera* cams, int B, const GmrRaster* r, void* rgb,
                     void* alpha, void* ws, const Layout& L, cudaStream_t st, const LossArgs* la = nullptr,
                     const ImageArgs* ia = nullptr, void* status_host = nullptr, void* status_event = nullptr) {
  pdl_launch(reset_status, dim3(1), dim3(1), 0, st, at<DevStatus>(ws, L.status));
  GMR_LAUNCHED();
  const uint64_t F = L.faces;
  for (int v0 = 0; v0 < B; v0 += kMaxViewsPerLaunch) {
    const int nv = std::min(kMaxViewsPerLaunch, B - v0);
    MeshFwdArgs<S> a{};
    a.pos = (const S*)m->positions;
    a.col = (const S*)m->colors;
    a.faces = m->faces;
    a.F = (int64_t)F;
    a.view0 = v0;
    a.nviews = nv;
    a.W = r->width;
    a.H = r->height;
    a.tiles_x = L.tiles_x;
    a.tiles_y = L.tiles_y;
    a.rescale = r->rescale;
    a.splat = at<Splat<S>>(ws, L.splat);
    a.col4 = at<V4<S>>(ws, L.col4);
    a.bin = at<uint4>(ws, L.bin);
    a.count = at<uint32_t>(ws, L.count);
    a.dkey = at<typename KeyOf<S>::type>(ws, L.dkey[0]);
    a.ditem = (r->flags & GMR_FLAG_TILE_DEPTH_SORT) ? nullptr : at<uint32_t>(ws, L.ditem[0]);
    a.pack_shift = pack_shift_for(L, r);
    // one launch covers every view: K1 also does face_counts' per-face scan
    a.face_local = B <= kMaxViewsPerLaunch ? at<uint32_t>(ws, L.offs) : nullptr;
    a.face_bsum = at<uint32_t>(ws, L.fbsum);
    a.cull = (r->flags & GMR_FLAG_FULL_TILE_LISTS) ? 0 : 1;
    a.aux = (r->flags & GMR_FLAG_DEBUG_AUX) ? at<S>(ws, L.aux) : nullptr;
    a.st = at<DevStatus>(ws, L.status);
    if (F) {
      StageScope sc(kStProject, st);
      pdl_launch(mesh_to_splats<S>, dim3(grid_for(F, 256)), dim3(256), 0, st, a, make_cams<S>(cams, v0, nv));
      GMR_LAUNCHED();
    }
  }
  return bin_and_blend<S>(L, ws, r, rgb, alpha, st, true, la, ia, status_host, status_event);
}

template <typename S, bool kOpacity>
int blend_backward_launch(const Layout& L, void* ws, const GmrRaster* r, const void* rgb,
                          const void* g_rgb, const void* g_alpha, cudaStream_t st) {
  const uint32_t ecur = (uint32_t)(((L.entry_bits + 7) / 8) & 1);
  BlendArgs<S> a{};
  a.bounds = at<uint32_t>(ws, L.bounds);
  a.sched = at<uint32_t>(ws, L.sched);
  a.covbuf = at<uint32_t>(ws, L.covbuf);   // the forward's coverage masks
  a.entry_item = at<uint32_t>(ws, L.eval[ecur]);
  a.splat = at<Splat<S>>(ws, L.splat);
  a.col4 = at<V4<S>>(ws, L.col4);
  a.bin = at<uint4>(ws, L.bin);
  a.entry_off = at<uint32_t>(ws, L.entry_off);
  a.items_per_view = (uint32_t)L.faces;
  a.tiles_x = L.tiles_x;
  a.tiles_per_view = (uint32_t)L.tiles;
  a.W = r->width;
  a.H = r->height;
  a.bg0 = (S)r->background[0];
  a.bg1 = (S)r->background[1];
  a.bg2 = (S)r->background[2];
  a.rgb = (S*)rgb;
  a.t_final = at<S>(ws, L.t_final);
  a.g_rgb = (const S*)g_rgb;
  a.g_alpha = (const S*)g_alpha;
  a.partial = at<S>(ws, L.partial);
  a.partial_op = kOpacity ? at<S>(ws, L.partial_op) : nullptr;
  const size_t dyn = sizeof(BwdSmem<S, kOpacity>);
  // the float mesh path's occupancy (GMR_BWD_MINB CTAs per SM) is what the
  // shared-memory layout is sized for: 228 KB per SM, allocated per CTA in
  // 128-byte units plus 1 KB reserved
  static_assert(((sizeof(BwdSmem<float, false>) + 127) / 128 * 128 + 1024) * GMR_BWD_MINB <= 228 * 1024,
                "blend_backward shared memory no longer fits GMR_BWD_MINB CTAs per SM");
  static_assert(((sizeof(BwdSmem<double, true>) + 127) / 128 * 128 + 1024) * 3 <= 228 * 1024,
                "float64 blend_backward shared memory no longer fits 3 CTAs per SM");
  // once per instantiation (thread-safe static init; also keeps it out of graph captures)
  static const cudaError_t attr_rc = [dyn] {
    const cudaError_t e = cudaFuncSetAttribute(blend_backward<S, kOpacity>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    return e != cudaSuccess ? e
                            : cudaFuncSetAttribute(blend_backward<S, kOpacity>,
                                                   cudaFuncAttributePreferredSharedMemoryCarveout,
                                                   (int)cudaSharedmemCarveoutMaxShared);
  }();
  GMR_CUDA(attr_rc);
  if (L.bins) {
    StageScope sc(kStBlendBwd, st);
    pdl_launch(blend_backward<S, kOpacity>, dim3((unsigned)L.bins), dim3(kBlendThreads), dyn, st, a);
    GMR_LAUNCHED();
  }
  return GMR_OK;
}

template <typename S>
int render_backward_t(const GmrMesh* m, const GmrCamera* cams, int B, const GmrRaster* r,
                      const void* rgb, const void* g_rgb, const void* g_alpha, void* g_pos,
                      void* g_col, const void* topo, void* ws, const Layout& L, cudaStream_t st) {
  int rc = blend_backward_launch<S, false>(L, ws, r, rgb, g_rgb, g_alpha, st);
  if (rc) return rc;
  const uint64_t F = L.faces, V = (uint64_t)m->num_vertices;
  for (int v0 = 0; v0 < B; v0 += kMaxViewsPerLaunch) {
    const int nv = std::min(kMaxViewsPerLaunch, B - v0);
    FaceBwdArgs<S> a{};
    a.pos = (const S*)m->positions;
    a.faces = m->faces;
    a.F = (int64_t)F;
    a.view0 = v0;
    a.nviews = nv;
    a.rescale = r->rescale;
    a.count = at<uint32_t>(ws, L.count);
    a.entry_off = at<uint32_t>(ws, L.entry_off);
    a.splat = at<Splat<S>>(ws, L.splat);
    a.partial = at<S>(ws, L.partial);
    a.face_acc = at<double>(ws, L.face_acc);
    // the last group also runs the conversion backward (face_acc stays in registers)
    a.corner = (v0 + nv == B) ? at<S>(ws, L.corner) : nullptr;
    a.st = at<DevStatus>(ws, L.status);
    if (F) {
      StageScope sc(kStFaceBwd, st);
      pdl_launch(face_views_backward<S>, dim3(grid_for(F, 128)), dim3(128), 0, st, a, make_cams<S>(cams, v0, nv));
      GMR_LAUNCHED();
    }
  }
  const uint32_t* vstart = (const uint32_t*)topo;
  const uint32_t* slots = vstart + align_up((V + 1) * 4) / 4;
  if (V) {
    StageScope sc(kStVertex, st);
    pdl_launch(vertex_gather<S>, dim3(grid_for(V, 256)), dim3(256), 0, st, vstart, slots, (int64_t)V, (int64_t)F,
                                                       at<S>(ws, L.corner), (S*)g_pos, (S*)g_col);
    GMR_LAUNCHED();
  }
  return GMR_OK;
}

int check_mesh(const GmrMesh* m) {
  if (!m) return fail(GMR_EINVAL, "mesh is null");
  if (m->num_faces < 0 || m->num_vertices < 0) return fail(GMR_EINVAL, "negative mesh sizes");
  if (m->num_faces > 0 && (!m->positions || !m->faces || !m->colors))
    return fail(GMR_EINVAL, "mesh buffers are null");
  if (m->num_vertices >= (1ll << 31) || 3 * m->num_faces >= (1ll << 31))
    return fail(GMR_EINVAL, "mesh too large for 32-bit indices");
  return GMR_OK;
}

template <typename S>
int rasterize_forward_t(const GmrSplats* sp, const GmrRaster* r, void* rgb, void* alpha, void* ws,
                        const Layout& L, cudaStream_t st) {
  pdl_launch(reset_status, dim3(1), dim3(1), 0, st, at<DevStatus>(ws, L.status));
  GMR_LAUNCHED();
  PackArgs<S> a{};
  a.mean2d = (const S*)sp->mean2d;
  a.cov2d = (const S*)sp->cov2d;
  a.depth = (const S*)sp->depth;
  a.color = (const S*)sp->color;
  a.opacity = (const S*)sp->opacity;
  a.K = sp->count;
  a.tiles_x = L.tiles_x;
  a.tiles_y = L.tiles_y;
  a.splat = at<Splat<S>>(ws, L.splat);
  a.col4 = at<V4<S>>(ws, L.col4);
  a.bin = at<uint4>(ws, L.bin);
  a.count = at<uint32_t>(ws, L.count);
  a.dkey = at<typename KeyOf<S>::type>(ws, L.dkey[0]);
  a.ditem = (r->flags & GMR_FLAG_TILE_DEPTH_SORT) ? nullptr : at<uint32_t>(ws, L.ditem[0]);
  a.cull = (r->flags & GMR_FLAG_FULL_TILE_LISTS) ? 0 : 1;
  a.st = at<DevStatus>(ws, L.status);
  if (sp->count) {
    pdl_launch(pack_splats<S>, dim3(grid_for(sp->count, 256)), dim3(256), 0, st, a);
    GMR_LAUNCHED();
  }
  return bin_and_blend<S>(L, ws, r, rgb, alpha, st, false);
}

int check_splats(const GmrSplats* sp) {
  if (!sp || sp->count < 0) return fail(GMR_EINVAL, "bad splats");
  if (sp->count && (!sp->mean2d || !sp->cov2d || !sp->depth || !sp->color || !sp->opacity))
    return fail(GMR_EINVAL, "splat buffers are null");
  if (sp->count >= (1ll << 31)) return fail(GMR_EINVAL, "too many splats");
  return GMR_OK;
}

template <typename S>
int rasterize_backward_t(const GmrSplats* sp, const GmrRaster* r, const void* rgb, const void* g_rgb,
                         const void* g_alpha, void* gm, void* gc, void* gcol, void* gop, void* ws,
                         const Layout& L, cudaStream_t st) {
  int rc = blend_backward_launch<S, true>(L, ws, r, rgb, g_rgb, g_alpha, st);
  if (rc) return rc;
  if (sp->count) {
    pdl_launch(splat_grads<S>, dim3(grid_for(sp->count, 256)), dim3(256), 0, st,
        at<uint32_t>(ws, L.count), at<uint32_t>(ws, L.entry_off), at<Splat<S>>(ws, L.splat),
        at<S>(ws, L.partial), at<S>(ws, L.partial_op), sp->count, at<DevStatus>(ws, L.status), (S*)gm, (S*)gc,
        (S*)gcol, (S*)gop);
    GMR_LAUNCHED();
  }
  return GMR_OK;
}

template <typename S>
int convert_backward_t(const GmrMesh* m, int rescale, const void* gm, const void* gc, const void* gcol, void* gp,
                       void* gcv, const void* topo, void* scratch, cudaStream_t st) {
  const int64_t F = m->num_faces, V = m->num_vertices;
  double* acc = (double*)scratch;
  S* corner = (S*)((char*)scratch + align_up(F * 12 * 8));
  if (F) {
    pdl_launch(pack_face_grads<S>, dim3(grid_for(F, 256)), dim3(256), 0, st, (const S*)gm, (const S*)gc, (const S*)gcol, F, acc);
    GMR_LAUNCHED();
    pdl_launch(face_convert_backward<S>, dim3(grid_for(F, 128)), dim3(128), 0, st, (const S*)m->positions, m->faces, F, rescale, acc, corner);
    GMR_LAUNCHED();
  }
  const uint32_t* vstart = (const uint32_t*)topo;
  const uint32_t* slots = vstart + align_up((V + 1) * 4) / 4;
  if (V) {
    pdl_launch(vertex_gather<S>, dim3(grid_for(V, 256)), dim3(256), 0, st, vstart, slots, V, F, corner, (S*)gp, (S*)gcv);
    GMR_LAUNCHED();
  }
  return GMR_OK;
}

}  // namespace

extern "C" {

const char* gmr_last_error(void) { return g_err.c_str(); }

void gmr_timing_enable(int32_t on) { g_timer.on = on != 0; }

int64_t gmr_launch_count(void) { return g_launches; }

int gmr_timing_read(double* ms, int64_t* launches, int32_t n, int32_t reset) {
  for (int s = 0; s < kNumStages; ++s) {
    for (auto& ev : g_timer.pending[s]) {
      float t = 0.f;
      GMR_CUDA(cudaEventSynchronize(ev.second));
      GMR_CUDA(cudaEventElapsedTime(&t, ev.first, ev.second));
      g_timer.ms[s] += t;
      g_timer.calls[s] += 1;
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
    g_timer.pending[s].clear();
  }
  for (int s = 0; s < n && s < kNumStages; ++s) {
    if (ms) ms[s] = g_timer.ms[s];
    if (launches) launches[s] = g_timer.calls[s];
  }
  if (reset)
    for (int s = 0; s < kNumStages; ++s) g_timer.ms[s] = 0, g_timer.calls[s] = 0;
  return kNumStages;
}
const char* gmr_version(void) { return "gmr-b200 0.1 (sm_100a)"; }

int gmr_render_workspace_size(int64_t F, int32_t B, int32_t W, int32_t H, int64_t ecap, int32_t dtype,
                              size_t* bytes) {
  if (!bytes || F < 0 || B < 1 || W < 1 || H < 1 || ecap < 0) return fail(GMR_EINVAL, "bad workspace sizes");
  if (ecap > 0xffffffffll)
    return fail(GMR_EINVAL, "%lld tile entries: a call is limited to 2^32 - 1 (render fewer views per call)",
                (long long)ecap);
  if ((uint64_t)F * B >= 0xffffffffull) return fail(GMR_EINVAL, "faces*views must be < 2^32");
  if (dtype != GMR_F32 && dtype != GMR_F64) return fail(GMR_EINVAL, "bad dtype");
  *bytes = plan((uint64_t)F, B, W, H, (uint64_t)ecap, dtype, true).total;
  return GMR_OK;
}

int gmr_render_forward(const GmrMesh* mesh, const GmrCamera* cams, int32_t B, const GmrRaster* r,
                       void* rgb, void* alpha, void* ws, size_t ws_bytes, int64_t ecap, void* stream) {
  int rc = check_mesh(mesh);
  if (rc) return rc;
  if ((rc = check_raster(r))) return rc;
  if (!cams || B < 1 || B > GMR_MAX_VIEWS_PER_CALL) return fail(GMR_EINVAL, "need 1..%d cameras", GMR_MAX_VIEWS_PER_CALL);
  if (!rgb || !alpha || !ws) return fail(GMR_EINVAL, "output or workspace pointer is null");
  if ((uint64_t)mesh->num_faces * B >= 0xffffffffull) return fail(GMR_EINVAL, "faces*views must be < 2^32");
  const Layout L = plan((uint64_t)mesh->num_faces, B, r->width, r->height, (uint64_t)ecap, r->dtype, true);
  if (ws_bytes < L.total) return fail(GMR_EWORKSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
  cudaStream_t st = (cudaStream_t)stream;
  if (r->dtype == GMR_F64) return render_forward_t<double>(mesh, cams, B, r, rgb, alpha, ws, L, st);
  return render_forward_t<float>(mesh, cams, B, r, rgb, alpha, ws, L, st);
}

int gmr_render_forward_ex(const GmrMesh* mesh, const GmrCamera* cams, int32_t B, const GmrRaster* r, void* rgb,
                          void* alpha, void* ws, size_t ws_bytes, int64_t ecap, void* status_host,
                          void* status_event, void* stream) {
  int rc = check_mesh(mesh);
  if (rc) return rc;
  if ((rc = check_raster(r))) return rc;
  if (!cams || B < 1 || B > GMR_MAX_VIEWS_PER_CALL) return fail(GMR_EINVAL, "need 1..%d cameras", GMR_MAX_VIEWS_PER_CALL);
  if (!rgb || !alpha || !ws) return fail(GMR_EINVAL, "output or workspace pointer is null");
  if ((uint64_t)mesh->num_faces * B >= 0xffffffffull) return fail(GMR_EINVAL, "faces*views must be < 2^32");
  const Layout L = plan((uint64_t)mesh->num_faces, B, r->width, r->height, (uint64_t)ecap, r->dtype, true);
  if (ws_bytes < L.total) return fail(GMR_EWORKSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
  cudaStream_t st = (cudaStream_t)stream;
  if (r->dtype == GMR_F64)
    return render_forward_t<double>(mesh, cams, B, r, rgb, alpha, ws, L, st, nullptr, nullptr, status_host, status_event);
  return render_forward_t<float>(mesh, cams, B, r, rgb, alpha, ws, L, st, nullptr, nullptr, status_host, status_event);
}

int gmr_render_forward_loss(const GmrMesh* mesh, const GmrCamera* cams, int32_t B, const GmrRaster* r,
                            const void* target_rgb, const void* target_mask, double scale_rgb,
                            double scale_alpha, void* rgb, void* alpha, void* g_rgb, void* g_alpha,
                            double* loss_sums, void* ws, size_t ws_bytes, int64_t ecap, void* stream) {
  int rc = check_mesh(mesh);
  if (rc) return rc;
  if ((rc = check_raster(r))) return rc;
  if (!cams || B < 1 || B > GMR_MAX_VIEWS_PER_CALL) return fail(GMR_EINVAL, "need 1..%d cameras", GMR_MAX_VIEWS_PER_CALL);
  if (!rgb || !alpha || !ws || !target_rgb || !target_mask || !g_rgb || !g_alpha || !loss_sums)
    return fail(GMR_EINVAL, "null pointer argument");
  if ((uint64_t)mesh->num_faces * B >= 0xffffffffull) return fail(GMR_EINVAL, "faces*views must be < 2^32");
  const Layout L = plan((uint64_t)mesh->num_faces, B, r->width, r->height, (uint64_t)ecap, r->dtype, true);
  if (ws_bytes < L.total) return fail(GMR_EWORKSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
  LossArgs la{target_rgb, target_mask, scale_rgb, scale_alpha, g_rgb, g_alpha, loss_sums};
  cudaStream_t st = (cudaStream_t)stream;
  if (r->dtype == GMR_F64) return render_forward_t<double>(mesh, cams, B, r, rgb, alpha, ws, L, st, &la);
  return render_forward_t<float>(mesh, cams, B, r, rgb, alpha, ws, L, st, &la);
}

int gmr_render_images_u8(const GmrMesh* mesh, const GmrCamera* cams, int32_t B, const GmrRaster* r,
                         uint8_t* rgb8, uint8_t* alpha8, void* ws, size_t ws_bytes, int64_t ecap, void* stream) {
  int rc = check_mesh(mesh);
  if (rc) return rc;
  if ((rc = check_raster(r))) return rc;
  if (!cams || B < 1 || B > GMR_MAX_VIEWS_PER_CALL) return fail(GMR_EINVAL, "need 1..%d cameras", GMR_MAX_VIEWS_PER_CALL);
  if (!rgb8 || !alpha8 || !ws) return fail(GMR_EINVAL, "output or workspace pointer is null");
  if ((uint64_t)mesh->num_faces * B >= 0xffffffffull) return fail(GMR_EINVAL, "faces*views must be < 2^32");
  const Layout L = plan((uint64_t)mesh->num_faces, B, r->width, r->height, (uint64_t)ecap, r->dtype, true);
  if (ws_bytes < L.total) return fail(GMR_EWORKSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
  ImageArgs ia{rgb8, alpha8};
  cudaStream_t st = (cudaStream_t)stream;
  if (r->dtype == GMR_F64) return render_forward_t<double>(mesh, cams, B, r, nullptr, nullptr, ws, L, st, nullptr, &ia);
  return render_forward_t<float>(mesh, cams, B, r, nullptr, nullptr, ws, L, st, nullptr, &ia);
}

int gmr_fit_scratch_size(int64_t V, int64_t E, size_t* bytes) {
  if (!bytes || V < 0 || E < 0) return fail(GMR_EINVAL, "bad sizes");
  const size_t nbe = (E + kTrainThreads - 1) / kTrainThreads + 1, nbv = (V + kTrainThreads - 1) / kTrainThreads + 1;
  *bytes = align_up(E * 32) + align_up(V * 32) + 2 * align_up(V * 24) + align_up((2 * nbe + nbv) * 8) + align_up(64);
  return GMR_OK;
}

namespace {
// The regulariser terms shared by gmr_fit_step and gmr_mesh_regularizers:
// per-edge coeff * vec, per-vertex Laplacian, and sums[0..2] = (sum of edge
// lengths, sum of dev^2, sum of |lap|^2), all in `scratch` (gmr_fit_scratch_size).
struct RegScratch {
  double *evec4, *lap4, *gpos, *gcol, *sums;
};

int reg_terms(const double* pos, const GmrMeshGraph* gr, int64_t V, void* scratch, cudaStream_t st,
              RegScratch* out) {
  const int64_t E = gr->num_edges;
  const int nbe = (int)((E + kTrainThreads - 1) / kTrainThreads), nbv = (int)((V + kTrainThreads - 1) / kTrainThreads);
  char* o = (char*)scratch;
  double* evec4 = (double*)o; o += align_up(E * 32);
  double* lap4 = (double*)o; o += align_up(V * 32);
  double* gpos = (double*)o; o += align_up(V * 24);
  double* gcol = (double*)o; o += align_up(V * 24);
  double* part = (double*)o; o += align_up((2 * (nbe + 1) + nbv + 1) * 8);
  double* sums = (double*)o;   // [0] sum len, [1] sum dev^2, [2] sum |lap|^2
  double* part_len = part;
  double* part_dev = part + nbe + 1;
  double* part_lap = part + 2 * (nbe + 1);
  if (E) {
    pdl_launch(edge_lengths, dim3(nbe), dim3(kTrainThreads), 0, st, pos, gr->edges, E, evec4, part_len);
    GMR_LAUNCHED();
    pdl_launch(sum_partials, dim3(1), dim3(kTrainThreads), 0, st, part_len, nbe, sums);
    GMR_LAUNCHED();
    pdl_launch(edge_terms, dim3(nbe), dim3(kTrainThreads), 0, st, evec4, E, sums, part_dev);
    GMR_LAUNCHED();
    pdl_launch(sum_partials, dim3(1), dim3(kTrainThreads), 0, st, part_dev, nbe, sums + 1);
    GMR_LAUNCHED();
  } else {
    GMR_CUDA(cudaMemsetAsync(sums, 0, 16, st));
  }
  pdl_launch(laplacian_terms, dim3(nbv), dim3(kTrainThreads), 0, st, pos, gr->adj_ptr, gr->adj, V, lap4, part_lap);
  GMR_LAUNCHED();
  pdl_launch(sum_partials, dim3(1), dim3(kTrainThreads), 0, st, part_lap, nbv, sums + 2);
  GMR_LAUNCHED();
  *out = RegScratch{evec4, lap4, gpos, gcol, sums};
  return GMR_OK;
}

int fit_step_impl(const GmrFitState* s, const GmrMeshGraph* gr, int64_t V, const float* grad_img_pos,
                  const float* grad_img_col, const double* img_loss_sums, double inv_nc, double inv_na,
                  double w_color, double w_sil, double w_edge, double w_lap, double lr_pos, double lr_col,
                  const double* lr_sched, int64_t* iter, double beta1, double beta2, double eps,
                  int32_t optimize_colors, double* history_row, const void* status_src, void* statuses,
                  void* scratch, size_t scratch_bytes, void* stream) {
  if (!s || !gr || V <= 0 || !grad_img_pos || !grad_img_col || !img_loss_sums || !history_row || !scratch)
    return fail(GMR_EINVAL, "null or empty argument");
  const int64_t E = gr->num_edges;
  size_t need;
  int rc = gmr_fit_scratch_size(V, E, &need);
  if (rc) return rc;
  if (scratch_bytes < need) return fail(GMR_EWORKSPACE, "fit scratch has %zu bytes, needs %zu", scratch_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  const int nbv = (int)((V + kTrainThreads - 1) / kTrainThreads);
  RegScratch rs;
  if ((rc = reg_terms(s->positions, gr, V, scratch, st, &rs))) return rc;
  double *evec4 = rs.evec4, *lap4 = rs.lap4, *gpos = rs.gpos, *gcol = rs.gcol, *sums = rs.sums;
  AdamArgs a{};
  a.pos = s->positions; a.col = s->colors; a.pos_f = s->positions_f32; a.col_f = s->colors_f32;
  a.g_img_pos = grad_img_pos; a.g_img_col = grad_img_col;
  a.m_pos = s->m_pos; a.v_pos = s->v_pos; a.m_col = s->m_col; a.v_col = s->v_col;
  a.counts = s->step_counts; a.bad = s->flags;
  a.lr_pos = lr_pos; a.lr_col = lr_col; a.beta1 = beta1; a.beta2 = beta2; a.eps = eps;
  a.lr_sched = lr_sched; a.iter = iter;
  a.optimize_colors = optimize_colors;
  a.render_status = (const DevStatus*)status_src;
  a.reg.ve_ptr = gr->ve_ptr; a.reg.ve_slot = gr->ve_slot; a.reg.adj_ptr = gr->adj_ptr; a.reg.adj = gr->adj;
  a.reg.evec4 = evec4; a.reg.lap4 = lap4; a.reg.V = V; a.reg.w_edge = w_edge; a.reg.w_lap = w_lap;
  pdl_launch(fit_grads, dim3(nbv), dim3(kTrainThreads), 0, st, a, gpos, gcol);
  GMR_LAUNCHED();
  pdl_launch(fit_update, dim3(nbv), dim3(kTrainThreads), 0, st, a, gpos, gcol);
  GMR_LAUNCHED();
  pdl_launch(fit_finish, dim3(1), dim3(32), 0, st, a, img_loss_sums, inv_nc, inv_na, w_color, w_sil, sums + 1, E, sums + 2, history_row,
                               (const uint32_t*)status_src, (uint32_t*)statuses);
  GMR_LAUNCHED();
  return GMR_OK;
}
}  // namespace

int gmr_fit_step(const GmrFitState* s, const GmrMeshGraph* gr, int64_t V, const float* grad_img_pos,
                 const float* grad_img_col, const double* img_loss_sums, double inv_nc, double inv_na,
                 double w_color, double w_sil, double w_edge, double w_lap, double lr_pos, double lr_col,
                 double beta1, double beta2, double eps, int32_t optimize_colors, double* history_row,
                 void* scratch, size_t scratch_bytes, void* stream) {
  return fit_step_impl(s, gr, V, grad_img_pos, grad_img_col, img_loss_sums, inv_nc, inv_na, w_color, w_sil, w_edge,
                       w_lap, lr_pos, lr_col, nullptr, nullptr, beta1, beta2, eps, optimize_colors, history_row,
                       nullptr, nullptr, scratch, scratch_bytes, stream);
}

int gmr_fit_step_scheduled(const GmrFitState* s, const GmrMeshGraph* gr, int64_t V, const float* grad_img_pos,
                           const float* grad_img_col, const double* img_loss_sums, double inv_nc, double inv_na,
                           double w_color, double w_sil, double w_edge, double w_lap, const double* lr_schedule,
                           int64_t* iteration, double beta1, double beta2, double eps, int32_t optimize_colors,
                           double* history, const void* render_status, void* statuses, void* scratch,
                           size_t scratch_bytes, void* stream) {
  if (!lr_schedule || !iteration) return fail(GMR_EINVAL, "schedule and iteration counter are required");
  return fit_step_impl(s, gr, V, grad_img_pos, grad_img_col, img_loss_sums, inv_nc, inv_na, w_color, w_sil, w_edge,
                       w_lap, 0.0, 0.0, lr_schedule, iteration, beta1, beta2, eps, optimize_colors, history,
                       render_status, statuses, scratch, scratch_bytes, stream);
}

int gmr_mesh_regularizers(const double* positions, const GmrMeshGraph* gr, int64_t V, double* values,
                          double* grad_edge, double* grad_laplacian, void* scratch, size_t scratch_bytes,
                          void* stream) {
  if (!positions || !gr || V <= 0 || !values || !scratch) return fail(GMR_EINVAL, "null or empty argument");
  size_t need;
  int rc = gmr_fit_scratch_size(V, gr->num_edges, &need);
  if (rc) return rc;
  if (scratch_bytes < need) return fail(GMR_EWORKSPACE, "regulariser scratch has %zu bytes, needs %zu", scratch_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  RegScratch rs;
  if ((rc = reg_terms(positions, gr, V, scratch, st, &rs))) return rc;
  pdl_launch(reg_values, dim3(1), dim3(1), 0, st, rs.sums, gr->num_edges, V, values);
  GMR_LAUNCHED();
  if (grad_edge || grad_laplacian) {
    RegArgs r{};
    r.ve_ptr = gr->ve_ptr; r.ve_slot = gr->ve_slot; r.adj_ptr = gr->adj_ptr; r.adj = gr->adj;
    r.evec4 = rs.evec4; r.lap4 = rs.lap4; r.V = V; r.w_edge = 1.0; r.w_lap = 1.0;
    pdl_launch(reg_grads, dim3((unsigned)((V + kTrainThreads - 1) / kTrainThreads)), dim3(kTrainThreads), 0, st, r, grad_edge,
                                                                                          grad_laplacian);
    GMR_LAUNCHED();
  }
  return GMR_OK;
}

int gmr_image_loss_scratch_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return fail(GMR_EINVAL, "bad sizes");
  *bytes = align_up(((n + kTrainThreads - 1) / kTrainThreads + 1) * 8);
  return GMR_OK;
}

int gmr_image_loss(int32_t kind, const double* x, const double* target, int64_t n, double* grad, double* value,
                   void* scratch, size_t scratch_bytes, void* stream) {
  if (kind != 0 && kind != 1) return fail(GMR_EINVAL, "kind must be 0 (colour MSE) or 1 (silhouette BCE)");
  if (n <= 0 || !x || !target || !grad || !value || !scratch) return fail(GMR_EINVAL, "null or empty argument");
  size_t need;
  int rc = gmr_image_loss_scratch_size(n, &need);
  if (rc) return rc;
  if (scratch_bytes < need) return fail(GMR_EWORKSPACE, "loss scratch has %zu bytes, needs %zu", scratch_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)((n + kTrainThreads - 1) / kTrainThreads);
  double* part = (double*)scratch;
  pdl_launch(image_loss_terms, dim3(nb), dim3(kTrainThreads), 0, st, kind, x, target, n, grad, part);
  GMR_LAUNCHED();
  pdl_launch(sum_partials, dim3(1), dim3(kTrainThreads), 0, st, part, nb, value);
  GMR_LAUNCHED();
  pdl_launch(scale_value, dim3(1), dim3(1), 0, st, value, 1.0 / (double)n);
  GMR_LAUNCHED();
  return GMR_OK;
}

int gmr_status(const void* ws, GmrStatus* out, void* stream) {
  if (!ws || !out) return fail(GMR_EINVAL, "null argument");
  DevStatus h;
  GMR_CUDA(cudaMemcpyAsync(&h, ws, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  GMR_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  out->entries = (int64_t)h.entries;
  out->kept = (int64_t)h.kept;
  out->overflow = (int32_t)h.overflow;
  out->entry_capacity = -1;
  out->nonfinite_field = -1;
  out->nonfinite_item = -1;
  for (int i = 0; i < 6; ++i)
    if (h.bad_item[i] != 0xffffffffu) {
      out->nonfinite_field = i;
      out->nonfinite_item = h.bad_item[i];
      break;
    }
  if (out->nonfinite_field >= 0)
    return fail(GMR_ENONFINITE, "non-finite splat parameter (field %d) at item %lld", out->nonfinite_field,
                (long long)out->nonfinite_item);
  if (h.overflow)
    return fail(GMR_ECAPACITY, "%llu tile entries exceed the capacity", (unsigned long long)h.entries);
  return GMR_OK;
}

int gmr_topology_size(int64_t F, int64_t V, size_t* bytes) {
  if (!bytes || F < 0 || V < 0) return fail(GMR_EINVAL, "bad topology sizes");
  const uint64_t n = 3 * (uint64_t)F;
  size_t o = align_up((V + 1) * 4) + align_up(n * 4);            // vstart, slots (result)
  o += 4 * align_up(n * 4) + align_up(radix_hist_words((uint32_t)n) * 4);  // sort scratch
  *bytes = o;
  return GMR_OK;
}

int gmr_topology_build(const int32_t* faces, int64_t F, int64_t V, void* topo, size_t bytes, void* stream) {
  size_t need;
  int rc = gmr_topology_size(F, V, &need);
  if (rc) return rc;
  if (bytes < need) return fail(GMR_EWORKSPACE, "topology buffer has %zu bytes, needs %zu", bytes, need);
  if (F > 0 && !faces) return fail(GMR_EINVAL, "faces is null");
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t n = 3 * (uint64_t)F;
  char* base = (char*)topo;
  uint32_t* vstart = (uint32_t*)base;
  uint32_t* slots = (uint32_t*)(base + align_up((V + 1) * 4));
  char* scratch = (char*)slots + align_up(n * 4);
  uint32_t* k[2] = {(uint32_t*)scratch, (uint32_t*)(scratch + align_up(n * 4))};
  uint32_t* v[2] = {(uint32_t*)(scratch + 2 * align_up(n * 4)), (uint32_t*)(scratch + 3 * align_up(n * 4))};
  uint32_t* hist = (uint32_t*)(scratch + 4 * align_up(n * 4));
  if (n) {
    pdl_launch(topo_keys, dim3(grid_for(n, 256)), dim3(256), 0, st, faces, F, k[0], v[0]);
    GMR_LAUNCHED();
  }
  const int bits = std::max(1, ceil_log2((uint64_t)std::max<int64_t>(V, 1)));
  int cur = radix_sort_pairs<uint32_t>(k, v, nullptr, (uint32_t)n, (uint32_t)n, bits, hist, st);
  GMR_LAUNCHED();
  pdl_launch(tile_ranges, dim3(grid_for(n / 4 + 1, 256)), dim3(256), 0, st, k[cur], nullptr, (uint32_t)n, (uint32_t)V, vstart,
             nullptr);
  GMR_LAUNCHED();
  GMR_CUDA(cudaMemcpyAsync(slots, v[cur], n * 4, cudaMemcpyDeviceToDevice, st));
  return GMR_OK;
}

int gmr_render_backward(const GmrMesh* mesh, const GmrCamera* cams, int32_t B, const GmrRaster* r,
                        const void* rgb, const void* g_rgb, const void* g_alpha, void* g_pos, void* g_col,
                        const void* topo, void* ws, size_t ws_bytes, int64_t ecap, void* stream) {
  int rc = check_mesh(mesh);
  if (rc) return rc;
  if ((rc = check_raster(r))) return rc;
  if (!cams || B < 1 || B > GMR_MAX_VIEWS_PER_CALL) return fail(GMR_EINVAL, "need 1..%d cameras", GMR_MAX_VIEWS_PER_CALL);
  if (!rgb || !g_rgb || !g_alpha || !g_pos || !g_col || !topo || !ws) return fail(GMR_EINVAL, "null pointer argument");
  const uint64_t F = (uint64_t)mesh->num_faces;
  const Layout L = plan(F, B, r->width, r->height, (uint64_t)ecap, r->dtype, true);
  if (ws_bytes < L.total) return fail(GMR_EWORKSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
  cudaStream_t st = (cudaStream_t)stream;
  if (r->dtype == GMR_F64)
    return render_backward_t<double>(mesh, cams, B, r, rgb, g_rgb, g_alpha, g_pos, g_col, topo, ws, L, st);
  return render_backward_t<float>(mesh, cams, B, r, rgb, g_rgb, g_alpha, g_pos, g_col, topo, ws, L, st);
}

// ---- projection stage (project_cloud / project_cloud_backward) ------------

int gmr_project(const void* means, const void* cov3d, int64_t K, const GmrCamera* cam, int32_t W, int32_t H,
                int32_t dtype, void* mean2d, void* cov2d, void* conic, void* depth, void* radius, void* t_cam,
                uint8_t* kept, void* stream) {
  if (K < 0 || !cam || W < 1 || H < 1) return fail(GMR_EINVAL, "bad projection arguments");
  if (dtype != GMR_F32 && dtype != GMR_F64) return fail(GMR_EINVAL, "bad dtype");
  if (K == 0) return GMR_OK;
  if (!means || !cov3d || !mean2d || !cov2d || !conic || !depth || !radius || !t_cam || !kept)
    return fail(GMR_EINVAL, "null pointer argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == GMR_F64) {
    pdl_launch(project_gaussians<double>, dim3(grid_for(K, 256)), dim3(256), 0, st, 
        (const double*)means, (const double*)cov3d, K, make_cams<double>(cam, 0, 1).cam[0], W, H, (double*)mean2d,
        (double*)cov2d, (double*)conic, (double*)depth, (double*)radius, (double*)t_cam, kept);
  } else {
    pdl_launch(project_gaussians<float>, dim3(grid_for(K, 256)), dim3(256), 0, st, 
        (const float*)means, (const float*)cov3d, K, make_cams<float>(cam, 0, 1).cam[0], W, H, (float*)mean2d,
        (float*)cov2d, (float*)conic, (float*)depth, (float*)radius, (float*)t_cam, kept);
  }
  GMR_LAUNCHED();
  return GMR_OK;
}

int gmr_project_backward(const void* t_cam, const void* cov3d, int64_t K, const GmrCamera* cam, int32_t dtype,
                         const void* g_mean2d, const void* g_cov2d, void* g_mean3d, void* g_cov3d, void* stream) {
  if (K < 0 || !cam) return fail(GMR_EINVAL, "bad projection arguments");
  if (dtype != GMR_F32 && dtype != GMR_F64) return fail(GMR_EINVAL, "bad dtype");
  if (K == 0) return GMR_OK;
  if (!t_cam || !cov3d || !g_mean2d || !g_cov2d || !g_mean3d || !g_cov3d) return fail(GMR_EINVAL, "null pointer argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == GMR_F64) {
    pdl_launch(project_gaussians_backward<double>, dim3(grid_for(K, 256)), dim3(256), 0, st, 
        (const double*)t_cam, (const double*)cov3d, K, make_cams<double>(cam, 0, 1).cam[0], (const double*)g_mean2d,
        (const double*)g_cov2d, (double*)g_mean3d, (double*)g_cov3d);
  } else {
    pdl_launch(project_gaussians_backward<float>, dim3(grid_for(K, 256)), dim3(256), 0, st, 
        (const float*)t_cam, (const float*)cov3d, K, make_cams<float>(cam, 0, 1).cam[0], (const float*)g_mean2d,
        (const float*)g_cov2d, (float*)g_mean3d, (float*)g_cov3d);
  }
  GMR_LAUNCHED();
  return GMR_OK;
}

// ---- splat path ----------------------------------------------------------

int gmr_raster_workspace_size(int64_t K, int32_t W, int32_t H, int64_t ecap, int32_t dtype, size_t* bytes) {
  if (!bytes || K < 0 || W < 1 || H < 1 || ecap < 0) return fail(GMR_EINVAL, "bad workspace sizes");
  if (ecap > 0xffffffffll) return fail(GMR_EINVAL, "%lld tile entries: a call is limited to 2^32 - 1", (long long)ecap);
  if (K >= 0xffffffffll) return fail(GMR_EINVAL, "splats must be < 2^32");
  if (dtype != GMR_F32 && dtype != GMR_F64) return fail(GMR_EINVAL, "bad dtype");
  *bytes = plan((uint64_t)K, 1, W, H, (uint64_t)ecap, dtype, false).total;
  return GMR_OK;
}

int gmr_rasterize_forward(const GmrSplats* sp, const GmrRaster* r, void* rgb, void* alpha, void* ws,
                          size_t ws_bytes, int64_t ecap, void* stream) {
  int rc = check_splats(sp);
  if (rc) return rc;
  if ((rc = check_raster(r))) return rc;
  if (!rgb || !alpha || !ws) return fail(GMR_EINVAL, "output or workspace pointer is null");
  const Layout L = plan((uint64_t)sp->count, 1, r->width, r->height, (uint64_t)ecap, r->dtype, false);
  if (ws_bytes < L.total) return fail(GMR_EWORKSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
  cudaStream_t st = (cudaStream_t)stream;
  if (r->dtype == GMR_F64) return rasterize_forward_t<double>(sp, r, rgb, alpha, ws, L, st);
  return rasterize_forward_t<float>(sp, r, rgb, alpha, ws, L, st);
}

int gmr_rasterize_backward(const GmrSplats* sp, const GmrRaster* r, const void* rgb, const void* g_rgb,
                           const void* g_alpha, void* gm, void* gc, void* gcol, void* gop, void* ws,
                           size_t ws_bytes, int64_t ecap, void* stream) {
  int rc = check_splats(sp);
  if (rc) return rc;
  if ((rc = check_raster(r))) return rc;
  if (!rgb || !g_rgb || !g_alpha || !gm || !gc || !gcol || !gop || !ws) return fail(GMR_EINVAL, "null pointer argument");
  const uint64_t K = (uint64_t)sp->count;
  const Layout L = plan(K, 1, r->width, r->height, (uint64_t)ecap, r->dtype, false);
  if (ws_bytes < L.total) return fail(GMR_EWORKSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
  cudaStream_t st = (cudaStream_t)stream;
  if (r->dtype == GMR_F64) return rasterize_backward_t<double>(sp, r, rgb, g_rgb, g_alpha, gm, gc, gcol, gop, ws, L, st);
  return rasterize_backward_t<float>(sp, r, rgb, g_rgb, g_alpha, gm, gc, gcol, gop, ws, L, st);
}

// ---- inspection ------------------------------------------------------------

int gmr_copy_entries(const void* ws, int64_t items_per_view, int32_t views, const GmrRaster* r, int64_t ecap,
                     int32_t mesh_path, uint32_t* entry_items, uint32_t* bounds, void* stream) {
  int rc = check_raster(r);
  if (rc) return rc;
  if (!ws || !entry_items || !bounds || views < 1) return fail(GMR_EINVAL, "bad arguments");
  const Layout L = plan((uint64_t)items_per_view, views, r->width, r->height, (uint64_t)ecap, r->dtype, mesh_path != 0);
  DevStatus h;
  cudaStream_t st = (cudaStream_t)stream;
  GMR_CUDA(cudaMemcpyAsync(&h, ws, sizeof(h), cudaMemcpyDeviceToHost, st));
  GMR_CUDA(cudaStreamSynchronize(st));
  if (h.overflow) return fail(GMR_ECAPACITY, "forward overflowed its entry capacity");
  const uint32_t ecur = (uint32_t)(((L.entry_bits + 7) / 8) & 1);
  if (h.entries)
    GMR_CUDA(cudaMemcpyAsync(entry_items, (const char*)ws + L.eval[ecur], h.entries * 4, cudaMemcpyDeviceToDevice, st));
  GMR_CUDA(cudaMemcpyAsync(bounds, (const char*)ws + L.bounds, (L.bins + 1) * 4, cudaMemcpyDeviceToDevice, st));
  return GMR_OK;
}

int gmr_copy_splats(const void* ws, int64_t items_per_view, int32_t views, const GmrRaster* r, int64_t ecap,
                    int32_t mesh_path, void* records, void* rects, uint32_t* counts, void* aux, void* stream) {
  int rc = check_raster(r);
  if (rc) return rc;
  if (!ws || !records || !rects || !counts || views < 1) return fail(GMR_EINVAL, "bad arguments");
  const Layout L = plan((uint64_t)items_per_view, views, r->width, r->height, (uint64_t)ecap, r->dtype, mesh_path != 0);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t s = r->dtype == GMR_F64 ? 8 : 4;
  GMR_CUDA(cudaMemcpyAsync(records, (const char*)ws + L.splat, L.items * 8 * s, cudaMemcpyDeviceToDevice, st));
  // rects = the first 8 bytes of each 16-byte bin record
  if (L.items)
    GMR_CUDA(cudaMemcpy2DAsync(rects, 8, (const char*)ws + L.bin, 16, 8, L.items, cudaMemcpyDeviceToDevice, st));
  GMR_CUDA(cudaMemcpyAsync(counts, (const char*)ws + L.count, L.items * 4, cudaMemcpyDeviceToDevice, st));
  if (aux && mesh_path)
    GMR_CUDA(cudaMemcpyAsync(aux, (const char*)ws + L.aux, L.items * 2 * s, cudaMemcpyDeviceToDevice, st));
  return GMR_OK;
}

// ---- single stages ---------------------------------------------------------

int gmr_convert(const GmrMesh* mesh, int32_t rescale, int32_t dtype, void* means, void* cov3d, void* colors,
                uint8_t* degenerate, void* stream) {
  int rc = check_mesh(mesh);
  if (rc) return rc;
  if (dtype != GMR_F32 && dtype != GMR_F64) return fail(GMR_EINVAL, "bad dtype");
  if (!means || !cov3d || !colors) return fail(GMR_EINVAL, "null output");
  const int64_t F = mesh->num_faces;
  if (!F) return GMR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == GMR_F64)
    pdl_launch(convert_forward<double>, dim3(grid_for(F, 128)), dim3(128), 0, st, (const double*)mesh->positions, (const double*)mesh->colors,
                                                              mesh->faces, F, rescale, (double*)means, (double*)cov3d,
                                                              (double*)colors, degenerate);
  else
    pdl_launch(convert_forward<float>, dim3(grid_for(F, 128)), dim3(128), 0, st, (const float*)mesh->positions, (const float*)mesh->colors,
                                                             mesh->faces, F, rescale, (float*)means, (float*)cov3d,
                                                             (float*)colors, degenerate);
  GMR_LAUNCHED();
  return GMR_OK;
}

int gmr_convert_scratch_size(int64_t F, int32_t dtype, size_t* bytes) {
  if (!bytes || F < 0) return fail(GMR_EINVAL, "bad sizes");
  const size_t s = dtype == GMR_F64 ? 8 : 4;
  *bytes = align_up(F * 12 * 8) + align_up(F * 18 * s);
  return GMR_OK;
}

int gmr_convert_backward(const GmrMesh* mesh, int32_t rescale, int32_t dtype, const void* gm, const void* gc,
                         const void* gcol, void* gp, void* gcv, const void* topo, void* scratch, size_t scratch_bytes,
                         void* stream) {
  int rc = check_mesh(mesh);
  if (rc) return rc;
  size_t need;
  if ((rc = gmr_convert_scratch_size(mesh->num_faces, dtype, &need))) return rc;
  if (scratch_bytes < need) return fail(GMR_EWORKSPACE, "scratch too small");
  if (!gm || !gc || !gcol || !gp || !gcv || !topo) return fail(GMR_EINVAL, "null pointer argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == GMR_F64) return convert_backward_t<double>(mesh, rescale, gm, gc, gcol, gp, gcv, topo, scratch, st);
  return convert_backward_t<float>(mesh, rescale, gm, gc, gcol, gp, gcv, topo, scratch, st);
}

// ---- export and evaluation metrics ------------------------

int gmr_export_gaussians(const double* means, const double* cov3d, const double* colors, const double* opacities,
                         int64_t n, float* records, void* stream) {
  if (n < 0) return fail(GMR_EINVAL, "negative count");
  if (n == 0) return GMR_OK;
  if (!means || !cov3d || !colors || !opacities || !records) return fail(GMR_EINVAL, "null pointer argument");
  pdl_launch(export_records, dim3(grid_for((uint64_t)n, 128)), dim3(128), 0, (cudaStream_t)stream, means, cov3d, colors, opacities, n,
                                                                               records);
  GMR_LAUNCHED();
  return GMR_OK;
}

namespace {
int nn_chunks(int64_t n, int64_t m) {
  const int64_t qblocks = (n + kNnThreads * kNnQ - 1) / (kNnThreads * kNnQ);
  int64_t c = (4 * 148 + qblocks - 1) / std::max<int64_t>(qblocks, 1);
  c = std::min<int64_t>(c, std::max<int64_t>(1, (m + kNnTile - 1) / kNnTile));
  return (int)std::max<int64_t>(1, std::min<int64_t>(c, 64));
}
size_t nn_bytes(int64_t n, int64_t m) {
  const int c = nn_chunks(n, m);
  return align_up((size_t)c * n * 8) + align_up((size_t)c * n * 4);
}
int nn_run(const double* q, int64_t n, const double* pts, int64_t m, const double* qn, const double* pn,
           double* d2, double* cosv, int32_t* idx, void* scratch, cudaStream_t st) {
  const int c = nn_chunks(n, m);
  const int64_t chunk = (m + c - 1) / c;
  double* bd = (double*)scratch;
  int32_t* bi = (int32_t*)((char*)scratch + align_up((size_t)c * n * 8));
  dim3 grid((unsigned)((n + kNnThreads * kNnQ - 1) / (kNnThreads * kNnQ)), (unsigned)c);
  pdl_launch(nn_partial, dim3(grid), dim3(kNnThreads), 0, st, q, n, pts, m, chunk, bd, bi);
  GMR_LAUNCHED();
  pdl_launch(nn_merge, dim3(grid_for((uint64_t)n, 256)), dim3(256), 0, st, bd, bi, n, c, qn, pn, d2, cosv, idx);
  GMR_LAUNCHED();
  return GMR_OK;
}
constexpr int kSumBlocks = 148;
}  // namespace

int gmr_nearest_scratch_size(int64_t n, int64_t m, size_t* bytes) {
  if (!bytes || n < 0 || m < 1) return fail(GMR_EINVAL, "bad sizes");
  *bytes = nn_bytes(n, m);
  return GMR_OK;
}

int gmr_nearest(const double* queries, int64_t n, const double* points, int64_t m, double* d2, int32_t* index,
                void* scratch, size_t scratch_bytes, void* stream) {
  if (n < 0 || m < 1) return fail(GMR_EINVAL, "need n >= 0 queries and m >= 1 points");
  if (n == 0) return GMR_OK;
  if (!queries || !points || !d2 || !scratch) return fail(GMR_EINVAL, "null pointer argument");
  if (m >= 0x7fffffff) return fail(GMR_EINVAL, "too many points");
  if (scratch_bytes < nn_bytes(n, m)) return fail(GMR_EWORKSPACE, "scratch too small");
  return nn_run(queries, n, points, m, nullptr, nullptr, d2, nullptr, index, scratch, (cudaStream_t)stream);
}

int gmr_chamfer_scratch_size(int64_t na, int64_t nb, size_t* bytes) {
  if (!bytes || na < 1 || nb < 1) return fail(GMR_EINVAL, "bad sizes");
  const int64_t mx = std::max(na, nb);
  *bytes = std::max(nn_bytes(na, nb), nn_bytes(nb, na)) + 2 * align_up((size_t)mx * 8) + align_up(kSumBlocks * 8);
  return GMR_OK;
}

int gmr_chamfer_nc(const double* pts_a, const double* nrm_a, int64_t na, const double* pts_b, const double* nrm_b,
                   int64_t nb, double* out4, void* scratch, size_t scratch_bytes, void* stream) {
  if (na < 1 || nb < 1) return fail(GMR_EINVAL, "need at least one sample on each side");
  if (!pts_a || !pts_b || !out4 || !scratch) return fail(GMR_EINVAL, "null pointer argument");
  if (na >= 0x7fffffff || nb >= 0x7fffffff) return fail(GMR_EINVAL, "too many samples");
  size_t need;
  gmr_chamfer_scratch_size(na, nb, &need);
  if (scratch_bytes < need) return fail(GMR_EWORKSPACE, "scratch too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t mx = std::max(na, nb);
  char* base = (char*)scratch;
  const size_t nnb = std::max(nn_bytes(na, nb), nn_bytes(nb, na));
  double* d2 = (double*)(base + nnb);
  double* cs = (double*)(base + nnb + align_up((size_t)mx * 8));
  double* part = (double*)(base + nnb + 2 * align_up((size_t)mx * 8));
  const bool normals = nrm_a && nrm_b;
  // a -> b: out[0] = mean d^2, out[2] = mean |cos|; b -> a: out[1], out[3]
  for (int dir = 0; dir < 2; ++dir) {
    const double* q = dir ? pts_b : pts_a;
    const double* p = dir ? pts_a : pts_b;
    const int64_t n = dir ? nb : na, m = dir ? na : nb;
    int rc = nn_run(q, n, p, m, normals ? (dir ? nrm_b : nrm_a) : nullptr, normals ? (dir ? nrm_a : nrm_b) : nullptr,
                    d2, normals ? cs : nullptr, nullptr, scratch, st);
    if (rc) return rc;
    pdl_launch(block_sums, dim3(kSumBlocks), dim3(256), 0, st, d2, n, part);
    GMR_LAUNCHED();
    pdl_launch(final_sum, dim3(1), dim3(32), 0, st, part, kSumBlocks, 1.0 / (double)n, out4 + dir);
    GMR_LAUNCHED();
    if (normals) {
      pdl_launch(block_sums, dim3(kSumBlocks), dim3(256), 0, st, cs, n, part);
      GMR_LAUNCHED();
      pdl_launch(final_sum, dim3(1), dim3(32), 0, st, part, kSumBlocks, 1.0 / (double)n, out4 + 2 + dir);
      GMR_LAUNCHED();
    }
  }
  return GMR_OK;
}

int gmr_surface_prepare_size(int64_t F, size_t* bytes) {
  if (!bytes || F < 1 || F > kSurfaceMaxFaces) return fail(GMR_EINVAL, "need 1..%lld facets", (long long)kSurfaceMaxFaces);
  *bytes = 4 * align_up(F * 8) + align_up(F * 24) + align_up(F * 12) + align_up(64) + align_up(kPwMaxLeaves * 16);
  return GMR_OK;
}

namespace {
struct SurfaceLayout {
  double *area, *cdf, *total, *nrm;
  int32_t* fsorted;
  int64_t* leaf_off;
  double* leaf_sum;
};
SurfaceLayout surface_layout(void* prep, int64_t F) {
  char* b = (char*)prep;
  SurfaceLayout L;
  L.area = (double*)b; b += align_up(F * 8);
  L.cdf = (double*)b; b += align_up(F * 8);
  L.nrm = (double*)b; b += align_up(F * 24);
  L.fsorted = (int32_t*)b; b += align_up(F * 12);
  L.total = (double*)b; b += align_up(64);
  L.leaf_off = (int64_t*)b; b += align_up(kPwMaxLeaves * 8);
  L.leaf_sum = (double*)b;
  return L;
}
}  // namespace

int gmr_surface_prepare(const double* positions, const int32_t* faces, int64_t V, int64_t F, void* prep,
                        size_t prep_bytes, double* total_out, void* stream) {
  size_t need;
  int rc = gmr_surface_prepare_size(F, &need);
  if (rc) return rc;
  if (!positions || !faces || !prep || V < 1) return fail(GMR_EINVAL, "null or empty argument");
  if (prep_bytes < need) return fail(GMR_EWORKSPACE, "prepared buffer too small");
  cudaStream_t st = (cudaStream_t)stream;
  SurfaceLayout L = surface_layout(prep, F);
  pdl_launch(surface_faces, dim3(grid_for((uint64_t)F, 256)), dim3(256), 0, st, positions, faces, F, L.area, L.nrm, L.fsorted);
  GMR_LAUNCHED();
  pdl_launch(pairwise_total, dim3(1), dim3(kPwThreads), 0, st, L.area, F, L.leaf_off, L.leaf_sum, L.total);
  GMR_LAUNCHED();
  pdl_launch(cumsum_seq, dim3(1), dim3(32), 0, st, L.area, F, L.cdf);
  GMR_LAUNCHED();
  pdl_launch(cdf_divide, dim3(grid_for((uint64_t)F, 256)), dim3(256), 0, st, L.cdf, F, L.total);
  GMR_LAUNCHED();
  if (total_out) GMR_CUDA(cudaMemcpyAsync(total_out, L.total, 8, cudaMemcpyDeviceToDevice, st));
  return GMR_OK;
}

int gmr_surface_sample(const double* positions, int64_t F, const void* prep, const double* uniforms, int64_t n,
                       double* points, double* normals, void* stream) {
  if (F < 1 || F > kSurfaceMaxFaces || n < 0) return fail(GMR_EINVAL, "bad sizes");
  if (n == 0) return GMR_OK;
  if (!positions || !prep || !uniforms || !points || !normals) return fail(GMR_EINVAL, "null pointer argument");
  SurfaceLayout L = surface_layout((void*)prep, F);
  pdl_launch(surface_points, dim3(grid_for((uint64_t)n, 256)), dim3(256), 0, (cudaStream_t)stream, positions, L.fsorted, L.nrm, L.cdf, F,
                                                                               uniforms, n, points, normals);
  GMR_LAUNCHED();
  return GMR_OK;
}

int gmr_image_metrics_scratch_size(int32_t B, int32_t H, int32_t W, int32_t C, size_t* bytes) {
  if (!bytes || B < 1 || H < 1 || W < 1 || C < 1) return fail(GMR_EINVAL, "bad sizes");
  const size_t px = (size_t)B * H * W;
  *bytes = align_up(px * C * 8) + align_up(px * 5 * 8) + align_up(px * 8) + align_up(kSsimWin * 8);
  return GMR_OK;
}

int gmr_image_metrics(const double* a, const double* b, int32_t B, int32_t H, int32_t W, int32_t C, double* mse,
                      double* ssim, void* scratch, size_t scratch_bytes, void* stream) {
  if (B < 1 || H < 1 || W < 1 || C < 1) return fail(GMR_EINVAL, "bad image shape");
  if (!a || !b || !mse || !scratch) return fail(GMR_EINVAL, "null pointer argument");
  if (ssim && (H < kSsimWin || W < kSsimWin))
    return fail(GMR_EINVAL, "images must be at least %d pixels on each side", kSsimWin);
  size_t need;
  gmr_image_metrics_scratch_size(B, H, W, C, &need);
  if (scratch_bytes < need) return fail(GMR_EWORKSPACE, "scratch too small");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t px = (size_t)B * H * W;
  char* base = (char*)scratch;
  double* sq = (double*)base;
  double* tmp = (double*)(base + align_up(px * C * 8));
  double* smap = (double*)(base + align_up(px * C * 8) + align_up(px * 5 * 8));
  double* kern = (double*)(base + align_up(px * C * 8) + align_up(px * 5 * 8) + align_up(px * 8));
  // PSNR: per-image mean squared error (metrics.py:96)
  pdl_launch(sq_diff, dim3(grid_for(px * C, 256)), dim3(256), 0, st, a, b, (int64_t)(px * C), sq);
  GMR_LAUNCHED();
  pdl_launch(image_sums, dim3(B), dim3(256), 0, st, sq, (int64_t)H * W * C, 1.0 / ((double)H * W * C), mse, 0);
  GMR_LAUNCHED();
  if (!ssim) return GMR_OK;
  // Gaussian window (metrics.py:102-106) in float64, k / k.sum() with the
  // sum in numpy's pairwise order for 11 terms (8 lanes, then the tail)
  static const struct Window {
    double k[kSsimWin];
    Window() {
      for (int i = 0; i < kSsimWin; ++i) {
        const double x = (double)(i - kSsimHalf);
        k[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
      }
      double s = ((k[0] + k[1]) + (k[2] + k[3])) + ((k[4] + k[5]) + (k[6] + k[7]));
      for (int i = 8; i < kSsimWin; ++i) s += k[i];
      for (int i = 0; i < kSsimWin; ++i) k[i] /= s;
    }
  } window;
  GMR_CUDA(cudaMemcpyAsync(kern, window.k, sizeof(window.k), cudaMemcpyHostToDevice, st));
  const double c1 = (0.01 * 1.0) * (0.01 * 1.0), c2 = (0.03 * 1.0) * (0.03 * 1.0);
  const double inner = (double)(H - 2 * kSsimHalf) * (double)(W - 2 * kSsimHalf);
  for (int ch = 0; ch < C; ++ch) {
    pdl_launch(ssim_axis0, dim3(grid_for(px, 256)), dim3(256), 0, st, a, b, B, H, W, C, ch, kern, tmp);
    GMR_LAUNCHED();
    pdl_launch(ssim_axis1, dim3(grid_for(px, 256)), dim3(256), 0, st, tmp, B, H, W, kern, c1, c2, smap);
    GMR_LAUNCHED();
    pdl_launch(image_sums, dim3(B), dim3(256), 0, st, smap, (int64_t)H * W, 1.0 / (inner * C), ssim, ch > 0);
    GMR_LAUNCHED();
  }
  return GMR_OK;
}

}  // extern "C"
