/*
 * gmr.h — C ABI of the B200-native Gaussian Mesh Renderer hot path.
 *
 * Replaces the reference's numpy render path (meshsplat, pure Python; see
 * SURVEY.md §8b).  Every entry point is stream-ordered on a caller-supplied
 * cudaStream_t (passed as void*), takes plain device pointers, never
 * allocates and never frees: the caller owns every buffer, including the
 * workspace, whose size the *_workspace_size functions report.
 *
 *   reference entry point (file:line)               replaced by
 *   render.py:441-450  render_mesh                   gmr_render_forward  (+ gmr_status)
 *   render.py:453-467  render_backward               gmr_render_backward (+ gmr_topology_build)
 *   render.py:272-291  rasterize                     gmr_rasterize_forward
 *   render.py:294-361  rasterize_backward            gmr_rasterize_backward
 *   render.py:103-145  project_cloud                 fused into gmr_render_forward (K1); gmr_project
 *   render.py:364-402  project_cloud_backward        fused into gmr_render_backward (K5); gmr_project_backward
 *   convert.py:313-368 convert_mesh (embed route)    gmr_convert
 *   convert.py:371-437 convert_backward              gmr_convert_backward
 *   losses.py:151-162  total_loss view loop          B views per gmr_render_* call
 *   losses.py:43-73    color_loss, silhouette_loss   gmr_render_forward_loss (fused)
 *   losses.py:76-123, optim.py:29-135, :271-295      gmr_fit_step (regularisers + Adam)
 *   losses.py:76-123   edge_length / laplacian loss  gmr_mesh_regularizers
 *   losses.py:43-73    color_loss, silhouette_loss   gmr_image_loss (stand-alone)
 *   dataset.py:118-164 make_views (render + _save_png) gmr_render_images_u8
 *   convert.py:497-532 export_gaussians              gmr_export_gaussians
 *   metrics.py:40-86   chamfer / normal consistency  gmr_chamfer_nc, gmr_nearest
 *   metrics.py:89-172  psnr, ssim, image_metrics     gmr_image_metrics
 *
 * Scalars: every floating-point buffer is either float32 (GMR_F32, the fast
 * path; `fit`'s default dtype, reference optim.py:161) or float64
 * (GMR_F64, the parity path; render_mesh's default dtype, render.py:442).
 * Indices are int32.  Errors: functions return GMR_OK (0) or a negative
 * code; gmr_last_error() returns a thread-local message.
 */
#ifndef GMR_H_
#define GMR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GMR_OK = 0,
  GMR_EINVAL = -1,      /* bad argument (shape, null pointer, dtype)          */
  GMR_ENONFINITE = -2,  /* a kept splat has a non-finite parameter            */
  GMR_EWORKSPACE = -3,  /* workspace too small for the declared sizes         */
  GMR_ECUDA = -4,       /* a CUDA runtime call failed                         */
  GMR_ECAPACITY = -5    /* tile entries exceeded entry_capacity (see status)  */
};

enum { GMR_F32 = 0, GMR_F64 = 1 };

#define GMR_MAX_VIEWS_PER_CALL 4096

/* Pinhole camera (reference camera.py:15-58): p_cam = R p_world + t,
 * pixel centres at integer coordinates.  Host memory, always float64. */
typedef struct {
  double R[9];   /* row-major world->camera rotation */
  double t[3];
  double fx, fy, cx, cy;
  double near_plane, far_plane;
} GmrCamera;

/* Device-resident mesh (reference mesh.py:46-130). positions/colors are
 * V*3 scalars of the call's dtype; faces are F*3 int32. */
typedef struct {
  const void* positions;
  const void* colors;
  const int32_t* faces;
  int64_t num_vertices;
  int64_t num_faces;
} GmrMesh;

/* Raster settings shared by a batch of views. */
typedef struct {
  int32_t width, height;   /* all views of one call share W x H           */
  double background[3];    /* constant background colour (render.py:288) */
  int32_t dtype;           /* GMR_F32 or GMR_F64                          */
  int32_t rescale;         /* convert.py:313 rescale flag (default 1)     */
  int32_t flags;           /* GMR_FLAG_* below                            */
} GmrRaster;

/* GmrRaster.flags: keep each item's (radius, depth) for gmr_copy_splats. */
#define GMR_FLAG_DEBUG_AUX 1
/* GmrRaster.flags: emit every tile of each splat's rectangle, exactly the
 * reference's _RasterPlan lists (render.py:214-226).  By default a splat of
 * at most 32 tiles skips the tiles its padded alpha >= 1/255 ellipse cannot
 * reach (entries whose blend coverage would be empty): images and gradients
 * are bit-identical either way, the tile lists are then a subsequence of the
 * reference's. */
#define GMR_FLAG_FULL_TILE_LISTS 2
/* GmrRaster.flags: order each (view, tile) list by depth after the tile sort
 * (one CTA per tile list, in shared memory up to 2048 entries) instead of
 * sorting all B*F splats by depth before emission.  The lists are identical
 * either way ((tile, depth, source), render.py:227); per-tile ordering is
 * faster when every list is short and slower when a few lists hold most of
 * the entries (a distant mesh).  Byte 60 of the workspace (the device
 * status) holds the longest list of the last forward, so a caller can pick
 * the flag from the previous call. */
#define GMR_FLAG_TILE_DEPTH_SORT 4

/* Result of a forward pass, read back by gmr_status (synchronises). */
typedef struct {
  int64_t entries;          /* tile entries E summed over the views         */
  int64_t entry_capacity;   /* capacity the forward was planned with        */
  int64_t kept;             /* splats that survived depth+screen culling    */
  int32_t overflow;         /* 1: entries > capacity; outputs not written   */
  int32_t nonfinite_field;  /* -1, or 0..5 = mean2d,cov2d,conic,depth,color,opacity */
  int64_t nonfinite_item;   /* first offending item (view*F + face) or -1   */
} GmrStatus;

const char* gmr_last_error(void);
const char* gmr_version(void);

/* Per-stage device timers (CUDA events on the launching stream; calling
 * thread only).  Stages: 0 convert+project, 1 depth sort, 2 count scan +
 * entry emission, 3 tile sort + ranges, 4 blend forward, 5 blend backward,
 * 6 face backward (projection + conversion), 7 vertex gather.
 * gmr_timing_read waits for the recorded events and returns the number of
 * stages; ms / launches may be null. */
void gmr_timing_enable(int32_t on);
/* Number of kernels this thread has launched through the library. */
int64_t gmr_launch_count(void);
int gmr_timing_read(double* ms, int64_t* launches, int32_t n, int32_t reset);

/* ---- mesh path: B views in one call --------------------------------- */

/* Bytes of workspace for F faces, B views of W x H, and up to
 * entry_capacity tile entries (summed over views). */
int gmr_render_workspace_size(int64_t num_faces, int32_t num_views, int32_t width,
                              int32_t height, int64_t entry_capacity, int32_t dtype,
                              size_t* bytes);

/* Forward: rgb [B,H,W,3], alpha [B,H,W] (dtype).  The workspace carries the
 * per-view splat records, sorted tile entries, tile ranges and final
 * transmittance to gmr_render_backward and must not be touched between the
 * two calls. */
int gmr_render_forward(const GmrMesh* mesh, const GmrCamera* cameras, int32_t num_views,
                       const GmrRaster* raster, void* rgb, void* alpha, void* workspace,
                       size_t workspace_bytes, int64_t entry_capacity, void* stream);

/* Forward with the image losses fused into the blend epilogue (reference
 * losses.py:43-73 and the w/n scaling of total_loss, :158-160): for target
 * images target_rgb [B,H,W,3] / target_mask [B,H,W] (dtype) it also writes
 * g_rgb = d(w_c/n * sum_v MSE_v)/d rgb and g_alpha likewise for the clamped
 * BCE (scale_rgb = w_c/n, scale_alpha = w_s/n), and loss_sums (device, 2
 * doubles) = (sum of squared colour errors, sum of BCE terms) over all
 * pixels of all views -- divide by 3HW and HW for the per-view means. */
/* gmr_render_forward with an early status: right after binning has counted
 * the tile entries (before sorting and blending), the 64-byte status (the
 * layout gmr_status reads: entries, kept, first non-finite item per field,
 * overflow flag) is copied to `status_host` (pinned host memory, may be
 * null) and `status_event` (a cudaEvent_t, may be null) is recorded.  A host
 * that waits on the event can validate the call (capacity, non-finite input)
 * while the forward is still blending, and enqueue follow-up work without
 * draining the stream.  On overflow the remaining stages stay within the
 * workspace and their outputs are invalid. */
int gmr_render_forward_ex(const GmrMesh* mesh, const GmrCamera* cameras, int32_t num_views,
                          const GmrRaster* raster, void* rgb, void* alpha, void* workspace,
                          size_t workspace_bytes, int64_t entry_capacity, void* status_host,
                          void* status_event, void* stream);

int gmr_render_forward_loss(const GmrMesh* mesh, const GmrCamera* cameras, int32_t num_views,
                            const GmrRaster* raster, const void* target_rgb,
                            const void* target_mask, double scale_rgb, double scale_alpha,
                            void* rgb, void* alpha, void* g_rgb, void* g_alpha,
                            double* loss_sums, void* workspace, size_t workspace_bytes,
                            int64_t entry_capacity, void* stream);

/* Forward only, 8-bit images: the render of gmr_render_forward quantised in
 * the blend epilogue exactly as the reference's dataset writer does before
 * PNG encoding (dataset.py:59-61: np.round(np.clip(float64(x), 0, 1) * 255),
 * round half to even).  rgb8 [B,H,W,3] and alpha8 [B,H,W] are device uint8.
 * Same workspace and entry-capacity contract as gmr_render_forward. */
int gmr_render_images_u8(const GmrMesh* mesh, const GmrCamera* cameras, int32_t num_views,
                         const GmrRaster* raster, uint8_t* rgb8, uint8_t* alpha8, void* workspace,
                         size_t workspace_bytes, int64_t entry_capacity, void* stream);

/* ---- device-resident optimisation step (reference optim.py / losses.py) -- */

typedef struct {
  double* positions;        /* [V,3] float64 parameters, updated in place     */
  double* colors;           /* [V,3]                                         */
  float* positions_f32;     /* float32 render copies refreshed by the step   */
  float* colors_f32;        /*   (may be null)                               */
  double* m_pos;            /* VectorAdam state: [V,3] and [V]               */
  double* v_pos;
  double* m_col;            /* ScalarAdam state: [V,3] and [V,3]             */
  double* v_col;
  int64_t* step_counts;     /* [2] accepted steps (positions, colours)        */
  int32_t* flags;           /* [2] scratch, zero before the first step        */
} GmrFitState;

/* Static mesh graph: unique undirected edges [E,2] (lexsorted, smaller index
 * first, mesh.py:96-106), the vertex -> (edge, endpoint) CSR in np.add.at
 * order (slot = 2 edge + endpoint, all endpoint-1 slots before endpoint-0
 * ones, losses.py:95-96) and the sorted neighbour CSR (mesh.py:114-126). */
typedef struct {
  const int32_t* edges;
  int64_t num_edges;
  const int32_t* ve_ptr;
  const int32_t* ve_slot;
  const int32_t* adj_ptr;
  const int32_t* adj;
} GmrMeshGraph;

int gmr_fit_scratch_size(int64_t num_vertices, int64_t num_edges, size_t* bytes);

/* One optimisation step (optim.py:271-295): total gradient = image terms
 * (grad_img_*, float32, from gmr_render_backward) + w_edge * edge-length +
 * w_lap * Laplacian gradients; VectorAdam on positions, ScalarAdam + [0,1]
 * clip on colours (a step with a non-finite gradient is rejected, as in the
 * reference); history_row (device, 5 doubles) = (total, color, silhouette,
 * edge, laplacian) with color = img_loss_sums[0] * inv_nc and silhouette =
 * img_loss_sums[1] * inv_na (the loss sums of gmr_render_forward_loss). */
int gmr_fit_step(const GmrFitState* state, const GmrMeshGraph* graph, int64_t num_vertices,
                 const float* grad_img_pos, const float* grad_img_col,
                 const double* img_loss_sums, double inv_nc, double inv_na, double w_color,
                 double w_sil, double w_edge, double w_lap, double lr_pos, double lr_col,
                 double beta1, double beta2, double eps, int32_t optimize_colors,
                 double* history_row, void* scratch, size_t scratch_bytes, void* stream);

/* The mesh regularisers of total_loss on their own (losses.py:76-123):
 * values (device, 2 doubles) = (edge-length loss, Laplacian loss) of the
 * float64 positions [V,3]; grad_edge / grad_laplacian (device [V,3]
 * doubles, either may be null) their gradients, accumulated in the
 * reference's np.add.at order over the static graph.  Scratch size:
 * gmr_fit_scratch_size. */
int gmr_mesh_regularizers(const double* positions, const GmrMeshGraph* graph, int64_t num_vertices,
                          double* values, double* grad_edge, double* grad_laplacian, void* scratch,
                          size_t scratch_bytes, void* stream);

/* The image losses of the drop-in color_loss / silhouette_loss
 * (losses.py:43-73) over n float64 elements: kind 0 = mean squared error of
 * x against target, grad = 2 (x - target) / n; kind 1 = binary cross-entropy
 * of alpha x against mask target with the reference's 1e-6 clamp and
 * clamp-gated grad.  value (device, 1 double) = the mean. */
int gmr_image_loss_scratch_size(int64_t n, size_t* bytes);
int gmr_image_loss(int32_t kind, const double* x, const double* target, int64_t n, double* grad,
                   double* value, void* scratch, size_t scratch_bytes, void* stream);

/* Synchronise `stream` and read the status of the last forward that used
 * `workspace`.  Returns GMR_ECAPACITY / GMR_ENONFINITE as appropriate. */
int gmr_status(const void* workspace, GmrStatus* status, void* stream);

/* Static face->vertex scatter plan (CSR in the reference's np.add.at order,
 * convert.py:427-436).  Built once per topology. */
int gmr_topology_size(int64_t num_faces, int64_t num_vertices, size_t* bytes);
int gmr_topology_build(const int32_t* faces, int64_t num_faces, int64_t num_vertices,
                       void* topology, size_t topology_bytes, void* stream);

/* Backward of sum(g_rgb*rgb) + sum(g_alpha*alpha) over all B views:
 * grad_positions / grad_colors [V,3] (dtype) are OVERWRITTEN with the sum
 * over views (reference losses.py:160-162 semantics when the caller
 * pre-scales g by w/n).  `rgb` is the forward's output.  After a forward
 * that overflowed its entry capacity (GmrStatus.overflow) the gradients are
 * written as zeros and nothing outside the workspace is read. */
int gmr_render_backward(const GmrMesh* mesh, const GmrCamera* cameras, int32_t num_views,
                        const GmrRaster* raster, const void* rgb, const void* grad_rgb,
                        const void* grad_alpha, void* grad_positions, void* grad_colors,
                        const void* topology, void* workspace, size_t workspace_bytes,
                        int64_t entry_capacity, void* stream);

/* ---- projection stage (project_cloud / project_cloud_backward) --------- */

/* project_cloud (render.py:103-145) for one camera: K Gaussians (means
 * [K,3], cov3d [K,3,3], dtype) -> per Gaussian t_cam [K,3] and depth [K]
 * always; for Gaussians inside the depth window also mean2d [K,2], cov2d
 * [K,2,2] (+0.3 px^2 dilation), conic [K,3] and radius [K]; kept [K] = 1
 * where the Gaussian passes the depth window and the 3-sigma screen box
 * (the caller compacts the kept ones in cloud order, as the reference's
 * SplatBatch). */
int gmr_project(const void* means, const void* cov3d, int64_t K, const GmrCamera* camera, int32_t width,
                int32_t height, int32_t dtype, void* mean2d, void* cov2d, void* conic, void* depth, void* radius,
                void* t_cam, uint8_t* kept, void* stream);
/* project_cloud_backward (render.py:364-402): for K kept Gaussians (t_cam
 * [K,3] of the forward, cov3d [K,3,3]) and upstream g_mean2d [K,2], g_cov2d
 * [K,2,2] (general, not necessarily symmetric) -> g_mean3d [K,3], g_cov3d
 * [K,3,3]. */
int gmr_project_backward(const void* t_cam, const void* cov3d, int64_t K, const GmrCamera* camera, int32_t dtype,
                         const void* g_mean2d, const void* g_cov2d, void* g_mean3d, void* g_cov3d, void* stream);

/* ---- splat path (rasterize / rasterize_backward stage functions) ------ */

/* K splats: mean2d [K,2], cov2d [K,2,2], depth [K], color [K,3],
 * opacity [K] (dtype), already in tie-break (source) order. */
typedef struct {
  const void* mean2d;
  const void* cov2d;
  const void* depth;
  const void* color;
  const void* opacity;
  int64_t count;
} GmrSplats;

int gmr_raster_workspace_size(int64_t num_splats, int32_t width, int32_t height,
                              int64_t entry_capacity, int32_t dtype, size_t* bytes);
int gmr_rasterize_forward(const GmrSplats* splats, const GmrRaster* raster, void* rgb,
                          void* alpha, void* workspace, size_t workspace_bytes,
                          int64_t entry_capacity, void* stream);
/* Outputs g_mean2d [K,2], g_cov2d [K,2,2], g_color [K,3], g_opacity [K]. */
int gmr_rasterize_backward(const GmrSplats* splats, const GmrRaster* raster, const void* rgb,
                           const void* grad_rgb, const void* grad_alpha, void* g_mean2d,
                           void* g_cov2d, void* g_color, void* g_opacity, void* workspace,
                           size_t workspace_bytes, int64_t entry_capacity, void* stream);

/* Inspection (bit-exact binning checks).  `items_per_view` is F (mesh
 * path, mesh_path=1) or K (splat path, views=1); sizes as in the forward.
 * gmr_copy_entries: the sorted tile entries (item = view*F + face, or splat
 * index; `entries` from gmr_status) and the (views*T + 1) tile bounds.
 * gmr_copy_splats: per item, the screen record [8] (mean_x, mean_y,
 * conic a, b, c, ext_x, ext_y, radius; dtype), tile rect (uint2:
 * tx0|ty0<<16, tx1|ty1<<16), tile count (uint32, 0 = culled) and, when
 * the forward ran with GMR_FLAG_DEBUG_AUX, aux [2] = (radius, depth). */
int gmr_copy_entries(const void* workspace, int64_t items_per_view, int32_t views,
                     const GmrRaster* raster, int64_t entry_capacity, int32_t mesh_path,
                     uint32_t* entry_items, uint32_t* bounds, void* stream);
int gmr_copy_splats(const void* workspace, int64_t items_per_view, int32_t views,
                    const GmrRaster* raster, int64_t entry_capacity, int32_t mesh_path,
                    void* records, void* rects, uint32_t* counts, void* aux, void* stream);

/* ---- single-stage entry points ----------------------------------------- */

/* convert_mesh embed route: means [F,3], cov3d [F,3,3], colors [F,3]. */
int gmr_convert(const GmrMesh* mesh, int32_t rescale, int32_t dtype, void* means, void* cov3d,
                void* colors, uint8_t* degenerate, void* stream);
/* convert_backward: vertex grads [V,3] from facet grads (overwrites). */
int gmr_convert_backward(const GmrMesh* mesh, int32_t rescale, int32_t dtype,
                         const void* grad_means, const void* grad_cov3d,
                         const void* grad_colors, void* grad_positions, void* grad_colors_v,
                         const void* topology, void* scratch, size_t scratch_bytes, void* stream);
int gmr_convert_scratch_size(int64_t num_faces, int32_t dtype, size_t* bytes);

/* gmr_fit_step with every per-iteration input on the device, so that one
 * captured CUDA graph per view replays the whole iteration: at
 * it = *iteration (device int64), the learning rates are lr_schedule[2 it]
 * (positions) and [2 it + 1] (colours), the losses go to history[5 it ..],
 * the render's 64-byte status (render_status, may be null) is copied to
 * statuses[64 it ..], and *iteration is incremented last.  A step whose
 * render status shows an entry overflow or a non-finite splat is rejected
 * (no parameter or moment changes; the host re-runs with more capacity). */
int gmr_fit_step_scheduled(const GmrFitState* state, const GmrMeshGraph* graph, int64_t num_vertices,
                           const float* grad_img_pos, const float* grad_img_col,
                           const double* img_loss_sums, double inv_nc, double inv_na, double w_color,
                           double w_silhouette, double w_edge, double w_laplacian,
                           const double* lr_schedule, int64_t* iteration, double beta1, double beta2,
                           double eps, int32_t optimize_colors, double* history,
                           const void* render_status, void* statuses, void* scratch,
                           size_t scratch_bytes, void* stream);

/* ---- export and evaluation (all float64 inputs) ------- */

/* export_gaussians (convert.py:497-532): per Gaussian, the 14 float32 fields
 * of the splat-viewer PLY record (x y z, f_dc_0..2, opacity logit, log
 * scale_0..2, rot_0..3 = unit quaternion w x y z with w >= 0), from means
 * [n,3], cov3d [n,3,3] (lower triangle read, as eigh does), colors [n,3],
 * opacities [n].  records [n,14] on the device; the caller writes the header.
 * Eigenvectors of repeated eigenvalues are not unique, so rot/scale match the
 * reference as a factorisation (R diag(s^2) R^T = cov3d), not bit for bit. */
int gmr_export_gaussians(const double* means, const double* cov3d, const double* colors,
                         const double* opacities, int64_t n, float* records, void* stream);

/* sample_surface (mesh.py:560-622) in two steps.  gmr_surface_prepare: per
 * facet area / unit normal (placeholder (0,0,1) below area 1e-12) / sorted
 * corner indices, the total area as numpy's pairwise sum and the CDF as the
 * sequential cumsum / total -- all with numpy's float64 rounding -- into
 * `prep` (device); total_out (device, may be null) gets the total area.
 * gmr_surface_sample: for n uniform triples u (device [n,3], the reference's
 * Philox stream), facet = searchsorted(cdf, u0, 'left') clipped to F-1,
 * (u1, u2) folded when u1 + u2 > 1, point = a + b1 (b - a) + b2 (c - a) over
 * the sorted corners, normal = the facet normal. */
int gmr_surface_prepare_size(int64_t num_faces, size_t* bytes);
int gmr_surface_prepare(const double* positions, const int32_t* faces, int64_t num_vertices,
                        int64_t num_faces, void* prep, size_t prep_bytes, double* total_out, void* stream);
int gmr_surface_sample(const double* positions, int64_t num_faces, const void* prep,
                       const double* uniforms, int64_t n, double* points, double* normals, void* stream);

/* cKDTree(points).query(queries) by exact float64 brute force:
 * d2[i] = (distance to the nearest point)^2 computed as cKDTree returns it
 * (sqrt of ((dx^2 + dy^2) + dz^2), then squared), index[i] its point index
 * (ties: lowest index).  index may be null. */
int gmr_nearest_scratch_size(int64_t n_queries, int64_t n_points, size_t* bytes);
int gmr_nearest(const double* queries, int64_t n_queries, const double* points, int64_t n_points,
                double* d2, int32_t* index, void* scratch, size_t scratch_bytes, void* stream);

/* One Chamfer / normal-consistency pass (metrics.py:40-46, 69-77) between
 * sample sets a and b: out4 (device) = (mean d2 a->b, mean d2 b->a,
 * mean |n_a . n_nn(a)|, mean |n_b . n_nn(b)|).  Normals may be null (then
 * out4[2..3] are not written). */
int gmr_chamfer_scratch_size(int64_t n_a, int64_t n_b, size_t* bytes);
int gmr_chamfer_nc(const double* points_a, const double* normals_a, int64_t n_a,
                   const double* points_b, const double* normals_b, int64_t n_b, double* out4,
                   void* scratch, size_t scratch_bytes, void* stream);

/* PSNR / SSIM inputs (metrics.py:89-160) for B image pairs [B,H,W,C]:
 * mse[b] = mean squared difference (PSNR = min(10 log10(1/mse), 99) on the
 * host), ssim[b] = channel-averaged single-scale SSIM (11-tap Gaussian,
 * sigma 1.5, reflect borders, interior mean).  ssim may be null. */
int gmr_image_metrics_scratch_size(int32_t B, int32_t H, int32_t W, int32_t C, size_t* bytes);
int gmr_image_metrics(const double* a, const double* b, int32_t B, int32_t H, int32_t W, int32_t C,
                      double* mse, double* ssim, void* scratch, size_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GMR_H_ */
