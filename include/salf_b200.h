/*
 * salf_b200.h -- C ABI of the B200-native SaLF render path (libsalf_b200.so).
 *
 * Every entry point replaces one function of the reference's Python render
 * API (paths relative to /root/reference/pkg/src/salf); the Python mirror in
 * paper_2507_18713_b200/ binds them through ctypes.
 *
 * Conventions
 *   - all array arguments are caller-owned DEVICE pointers (one device per
 *     call, the current CUDA device); no hidden allocation: scratch comes from
 *     a caller-provided workspace sized by the matching *_workspace_bytes();
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *     calls are stream-ordered and re-entrant across streams;
 *   - return 0 on success or a SALF_E* code; salf_last_error() returns a
 *     thread-local message.  EINVAL maps to the reference's ValueError with
 *     the same text, ENOTERM to its RuntimeError (octree.py:251-252).
 */
#ifndef SALF_B200_H
#define SALF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SALF_OK 0
#define SALF_EINVAL 1     /* contract violation -> ValueError            */
#define SALF_ENOTERM 2    /* marcher did not terminate -> RuntimeError   */
#define SALF_ECUDA 3      /* CUDA runtime error -> RuntimeError          */
#define SALF_EWORKSPACE 4 /* workspace too small; see *_workspace_bytes  */

#define SALF_PINHOLE 0
#define SALF_FISHEYE 1
#define SALF_EQUIRECT 2

#define SALF_DENSITY_SDF 0
#define SALF_DENSITY_RAW 1

#define SALF_PRM_STRIDE 28 /* floats per voxel: w_s[4] w_c[9] w_sh[12] pad[3] */
#define SALF_SAVED_STRIDE 8 /* doubles per pixel/ray kept for the backward     */

/* Device view of a flat voxel list (reference render_raster.py:44-60,
 * scene.py:82-223).  geo = (cx, cy, cz, edge) f64 with centres computed as
 * aabb_min + (ijk + 0.5) * edge; aux = (a = exp(log_a), 1 / exp(log_b),
 * 2 / edge, 0) f64; prm = f32 fields (exact for salf.v1 scenes, whose params
 * are f32 on disk). */
typedef struct {
  int64_t n;
  const double *geo;
  const double *aux;
  const float *prm;
  const double *rot;  /* M x 9 voxel rotation matrices (flattened actors), or NULL */
  int32_t density_mode;
  int32_t pad;
} salf_scene_t;

/* CameraModel (reference sensors.py:45-74); rot = quat_to_matrix(q), row-major. */
typedef struct {
  int32_t kind, width, height, pad;
  double fx, fy, cx, cy;
  double k[4];
  double position[3];
  double rot[9];
  double readout_duration;
  double linear_velocity[3];
  double angular_velocity[3];
  double t0;
} salf_camera_t;

/* LidarModel (reference sensors.py:77-98); beam elevations are a device array. */
typedef struct {
  int32_t n_beams, steps;
  double azimuth_start, azimuth_end, scan_period;
  double position[3];
  double rot[9];
  double linear_velocity[3];
  double angular_velocity[3];
  double t0;
} salf_lidar_t;

/* Linear octree (reference octree.py:34-44): node word = id_or_offset with
 * the leaf flag folded in: word >= 0 -> internal node, children at word;
 * word == -1 -> empty; word <= -2 -> leaf of voxel (-word - 2). */
typedef struct {
  int64_t n_nodes;
  const int32_t *nodes;
  double root_min[3];
  double root_edge;
  int32_t max_depth;
  int32_t jump_levels;  /* K of the jump table below (0: none)              */
  const void *jump;     /* optional, salf_octree_jump_build: descents start at depth K */
} salf_octree_t;

typedef struct {
  double background[3];
  double near;           /* NEAR_PLANE 0.05 (render_raster.py:30)      */
  double stop_threshold; /* STOP_THRESHOLD 0.99 (render_ray.py:31)    */
  int32_t tile;          /* TILE_SIZE 16 (render_raster.py:29)         */
  int32_t exact_color;   /* 1: color in fp64 (parity mode); 0: fp32    */
} salf_raster_opts_t;

const char *salf_last_error(void);
int salf_device_sm_count(void);

/* ---- rasterizer (reference render_raster.py) ------------------------- */

/* project_voxels (render_raster.py:97-129) + the per-voxel half of
 * cull_and_bin (:143-176): rect (M x 4: umin, vmin, umax, vmax; NaN if
 * culled), z_center, culled, the reference tile span `span_ref` and the
 * tightened render span `span_fit` (M x 4 int32: tx0, ty0, tx1, ty1; empty
 * when tx0 > tx1), 64-bit orderable depth keys, and `vrange` (M x 2 int32:
 * the conservative footprint's pixel rows, then columns, each lo | hi << 16,
 * widened by one pixel; lo > hi when empty) that the composite uses to skip
 * entries a warp's 8 x 4 pixel block cannot hit.  Any output may be NULL.  (The composite and
 * backward also take an optional `tile_order`: the launch order of the
 * tiles, e.g. by list length descending; NULL = row-major.) */
int salf_project_voxels(const salf_scene_t *scene, const salf_camera_t *cam, double near,
                        int32_t tile, double *rect, double *z_center, uint8_t *culled,
                        int32_t *span_ref, int32_t *span_fit, uint64_t *zkey, int32_t *vrange,
                        void *stream);

/* Workspace for salf_raster_bin given M voxels and an instance capacity. */
size_t salf_raster_bin_workspace_bytes(int64_t n_voxels, int64_t capacity, int32_t n_tiles);

/* cull_and_bin (render_raster.py:143-182): CSR of depth-sorted per-tile voxel
 * lists.  mode 0 = reference lists (straddlers in every tile; bit-exact
 * export), mode 1 = render lists (tightened spans; per-tile subsequence of
 * mode 0 that drops only voxels no pixel of the tile can hit).
 * Writes offsets[n_tiles + 1] (int64), entries[capacity] (int32) and
 * counts[2] (int64, DEVICE memory): counts[0] = visible voxels, counts[1] =
 * instances.  Stream-ordered, no host synchronisation (hand-written radix sort,
 * see salf_sort.cuh).  When counts[1] > capacity the frame's lists are
 * incomplete: the caller checks counts[1] after the stream reaches it and
 * re-bins with capacity >= counts[1]. */
int salf_raster_bin(const salf_scene_t *scene, const salf_camera_t *cam, double near,
                    int32_t tile, int32_t mode, const uint64_t *zkey, const int32_t *span,
                    const uint8_t *visible_hint, void *workspace, size_t workspace_bytes,
                    int64_t capacity, int64_t *offsets, int32_t *entries,
                    int64_t *counts, void *stream);

/* The binning's stable LSD radix sort (replaces np.lexsort at
 * render_raster.py:177), exported for tests and callers that sort their own
 * keys: (keys_in, vals_in)[0, n) -> (keys_out, vals_out) by key bits
 * [begin_bit, end_bit), higher key bits zero, ties in input order.  key_bytes
 * 4 or 8; n = min(*n_dev, n_max) read on the device (n_dev NULL: n_max);
 * n_max < 2^30.  Inputs are not modified.  Device pointers, stream-ordered. */
size_t salf_sort_pairs_workspace_bytes(int64_t n_max, int32_t key_bytes, int32_t begin_bit, int32_t end_bit);
int salf_sort_pairs(const void *keys_in, const int32_t *vals_in, void *keys_out, int32_t *vals_out,
                    int32_t key_bytes, const int64_t *n_dev, int64_t n_max, int32_t begin_bit, int32_t end_bit,
                    void *workspace, size_t workspace_bytes, void *stream);

/* Sort (u64 key, int32 value) pairs that are unique as pairs into (key, value)
 * order -- for input in ascending value order the permutation of the stable
 * sort above, which is how the binning's depth rank (render_raster.py:177,
 * z[vox] ties broken by voxel index) uses it.  Splitter bucket sort: five
 * launches, workspace independent of n; n_max < 2^32.  Device pointers,
 * stream-ordered, inputs not modified. */
size_t salf_sort_pairs_unique_workspace_bytes(void);
int salf_sort_pairs_unique(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out, int32_t *vals_out,
                           const int64_t *n_dev, int64_t n_max, void *workspace, size_t workspace_bytes,
                           void *stream);

/* rasterize (render_raster.py:201-301) over prebuilt render bins.
 * out_rgb (H*W*3), out_opacity, out_depth f32; saved (H*W*8 f64, nullable):
 * acc_rgb[3], acc_w, acc_wt, T_final, n_stop (entries examined), n_included
 * -- kept for the backward (and the work statistics of the ALU roofline). */
int salf_raster_composite(const salf_scene_t *scene, const salf_camera_t *cam,
                          const salf_raster_opts_t *opts, const int64_t *offsets,
                          const int32_t *entries, float *out_rgb, float *out_opacity,
                          float *out_depth, double *saved, const int32_t *vrange,
                          const int32_t *tile_order, uint32_t *hitbits, void *stream);

/* Words of the hit-word array (nullable `hitbits` of salf_raster_composite /
 * salf_raster_backward, uint32): bit b of word w of pixel slot p of tile t says
 * list position 32w + b of the tile is an included hit of that pixel -- the
 * reference's hit and inclusion decisions (render_raster.py:241, :267) as the
 * certified forward (or its fp64 redo) took them.  The backward then visits
 * only those pairs and re-derives each chord in fp64.  Default mode only. */
size_t salf_raster_hitbits_words(int64_t capacity, int32_t n_tiles);

/* Raster backward (no reference function: defined as backward_records,
 * backward.py:35-101, applied to the raster pairs -- see DESIGN.md).
 * d_rgb (H*W*3) and d_depth (H*W) f64; grad (M x 27 f64, accumulated).
 * d_depth may be NULL (no depth loss): a colour-only kernel runs, with the
 * values zero depth seeds would give. */
int salf_raster_backward(const salf_scene_t *scene, const salf_camera_t *cam,
                         const salf_raster_opts_t *opts, const int64_t *offsets,
                         const int32_t *entries, const double *saved, const double *d_rgb,
                         const double *d_depth, double *grad, const int32_t *vrange,
                         const int32_t *tile_order, const uint32_t *hitbits, void *stream);

/* Launch order for the tile kernels (a scheduling choice only, results do
 * not depend on it): tiles by list length, longest first, ties in tile
 * order (lengths saturate at 65535).  order: n_tiles int32; workspace of
 * salf_raster_tile_order_workspace_bytes(n_tiles) bytes. */
size_t salf_raster_tile_order_workspace_bytes(int32_t n_tiles);
int salf_raster_tile_order(const int64_t *offsets, int32_t n_tiles, int32_t *order, void *workspace,
                           size_t workspace_bytes, void *stream);

/* Deterministic variant of salf_raster_backward (SPEC.md:531, :541 ordered
 * reductions; SURVEY §7 hard part 5): one fixed-order 27-row per (tile,
 * entry) instance into the workspace, instances stable-sorted by voxel, each
 * voxel's rows summed sequentially in fp64 and added to grad -- bitwise
 * identical across runs.  n_instances = length of `entries`; workspace of
 * salf_raster_backward_det_workspace_bytes(n_instances, M) bytes. */
size_t salf_raster_backward_det_workspace_bytes(int64_t n_instances, int64_t n_voxels);
int salf_raster_backward_deterministic(const salf_scene_t *scene, const salf_camera_t *cam,
                                       const salf_raster_opts_t *opts, const int64_t *offsets,
                                       const int32_t *entries, int64_t n_instances, const double *saved,
                                       const double *d_rgb, const double *d_depth, double *grad,
                                       const int32_t *vrange, const int32_t *tile_order,
                                       const uint32_t *hitbits, void *workspace, size_t workspace_bytes,
                                       void *stream);

/* Deterministic variant of salf_ray_backward: each included segment's
 * 27-row goes to slot row_start[ray] + k (row_start: (n + 1) exclusive scan
 * of the forward's per-ray segment counts, saved[:, 6]), then the ordered
 * per-voxel reduction of salf_raster_backward_deterministic.  Bitwise
 * identical across runs.  Workspace: salf_ray_backward_det_workspace_bytes(n_slots, M). */
size_t salf_ray_backward_det_workspace_bytes(int64_t n_slots, int64_t n_voxels);
int salf_ray_backward_deterministic(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                                    const double *origins, const double *dirs, const uint8_t *valid,
                                    const salf_raster_opts_t *opts, const double *saved, const double *d_rgb,
                                    const double *d_depth, double *grad, const int64_t *row_start, int64_t n_slots,
                                    void *workspace, size_t workspace_bytes, void *stream);

/* ---- sensors (reference sensors.py) ----------------------------------- */

/* gen_camera_rays + apply_rolling_shutter (sensors.py:129-190):
 * origins/dirs (N x 3 f64), t_stamps (N f64), valid (N u8), N = W*H. */
int salf_camera_rays(const salf_camera_t *cam, double *origins, double *dirs,
                     double *t_stamps, uint8_t *valid, void *stream);
/* The same as a whole RayBatch in one launch: plus keys (N x 2 i64: row,
 * col; sensors.py:157-160), nullable. */
int salf_camera_batch(const salf_camera_t *cam, double *origins, double *dirs, double *t_stamps,
                      uint8_t *valid, int64_t *keys, void *stream);

/* gen_lidar_rays (sensors.py:193-232), beam-major. */
int salf_lidar_rays(const salf_lidar_t *lidar, const double *beam_elevations, double *origins,
                    double *dirs, double *t_stamps, void *stream);
/* The same as a whole RayBatch in one launch: plus keys (N x 2 i64: beam,
 * step; sensors.py:228-231) and valid (N u8, all 1); keys / valid nullable. */
int salf_lidar_batch(const salf_lidar_t *lidar, const double *beam_elevations, double *origins,
                     double *dirs, double *t_stamps, int64_t *keys, uint8_t *valid, void *stream);

/* ---- octree (reference octree.py) -------------------------------------- */

/* build_octree (octree.py:54-125) on the host: level (u8), ijk (int32 x3)
 * host arrays.  Node layout identical to the reference DFS.  Call with
 * nodes == NULL to get the node count in *n_nodes first. */
int salf_octree_build_host(int64_t n, const uint8_t *level, const int32_t *ijk,
                           int32_t root_depth, int32_t *nodes, int64_t capacity,
                           int64_t *n_nodes, int32_t *max_depth);

/* build_octree on the device, same layout as the host
 * build.  Step 1: every voxel v (depth D = root_depth + level) writes the
 * packed preorder keys of its D ancestors at keys[base[v] ..] (base =
 * exclusive scan of D) and of itself at self_key[v].  The caller sorts and
 * uniques the ancestor keys (internal nodes in reference DFS order).
 * Step 2: nodes (1 + 8 n_internal words, pre-filled with -1) get every
 * internal node's child-block word and every voxel's leaf word; *contained
 * is set when a voxel sits at an internal node's depth (reference error
 * "stored voxel contains another stored voxel"). */
int salf_octree_ancestor_keys(int64_t n, const uint8_t *level, const int32_t *ijk, int32_t root_depth,
                              const int64_t *base, uint64_t *keys, uint64_t *self_key, void *stream);
int salf_octree_fill(int64_t n, int64_t n_internal, const uint64_t *internal, const uint64_t *self_key,
                     int32_t *nodes, int32_t *contained, void *stream);

/* Jump table for the octree descent (a B200-side acceleration structure,
 * no reference counterpart): for each of the 8^K cells of the depth-K grid
 * the node word the reference's descent reaches after K levels (INT32_MIN if
 * the path ends above depth K), then per axis the 2^K corners after K levels
 * accumulated in the reference's order (octree.py:152-163).  A query starts
 * there and continues level by level, so results are bit-identical.
 * salf_octree_jump_bytes(K) bytes of device memory; K <= 8. */
size_t salf_octree_jump_bytes(int32_t levels);
int salf_octree_jump_build(const salf_octree_t *tree, int32_t levels, void *jump, void *stream);

/* query_batch (octree.py:136-166): flag (i8), vid (i64), corner (x3), edge. */
int salf_octree_query(const salf_octree_t *tree, int64_t n, const double *p, int8_t *flag,
                      int64_t *vid, double *corner, double *edge, int32_t *out_of_root,
                      void *stream);

/* march_batch (octree.py:276-295): per-ray segment counts, then the hit
 * list in per-ray march order.  counts[n]; if seg_vid != NULL the caller
 * passes starts (exclusive scan of counts) and the segments are written. */
int salf_march(const salf_octree_t *tree, int64_t n, const double *origins, const double *dirs,
               const double *t_max, const salf_scene_t *scene, double stop_threshold,
               int32_t early_stop, int64_t *counts, const int64_t *starts, int64_t *seg_vid,
               double *seg_t0, double *seg_t1, int32_t *status, void *stream);

/* integrate_rays (render_ray.py:161-239) for a static scene, fused march +
 * shade + composite: out_rgb (N x 3), out_opacity, out_depth (f32);
 * saved (N x 8 f64, nullable) as for the rasterizer; status (N int32):
 * 0 ok, 1 round cap hit (the reference would raise RuntimeError). */
int salf_ray_forward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                     const double *origins, const double *dirs, const uint8_t *valid,
                     const salf_raster_opts_t *opts, float *out_rgb, float *out_opacity,
                     float *out_depth, double *saved, int32_t *status, void *stream);

/* render_lidar_ranges (render_ray.py:297-306) for a LiDAR batch: the fused
 * march/shade/composite without colour (the reference computes and discards
 * it), out_depth / out_opacity (N f32), saved (N x 8 f64, nullable), status.
 * Optional intensity / ray-drop extension (not in the
 * reference): feat (M x 8 f32) alpha-blended with the colour
 * weights into out_feat (N x 8, nullable), then a linear head (2 x 13 f32:
 * 8 feature weights, depth weight, 3 view-dir weights, bias) and a sigmoid ->
 * out_head (N x 2: intensity, drop probability).  feat == NULL: depth only.
 * feat_acc64 (N x 8 f64, nullable): the blended feature as fp64 totals of the
 * exact per-segment products -- what salf_lidar_backward takes as Facc. */
int salf_lidar_forward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                       const double *origins, const double *dirs, const salf_raster_opts_t *opts,
                       const float *feat, const float *head, float *out_depth, float *out_opacity,
                       float *out_feat, float *out_head, double *feat_acc64, double *saved, int32_t *status,
                       void *stream);

/* Backward of salf_lidar_forward: depth seeds d_depth (N f64) plus, for the
 * intensity / ray-drop extension, dF = dL/d(blended feature) (N x 8 f64)
 * with the forward's feat_acc64 as Facc (N x 8 f64): field-parameter
 * gradients into grad (M x 27) and feature gradients into feat_grad (M x 8).
 * feat == NULL: depth-only backward. */
int salf_lidar_backward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                        const double *origins, const double *dirs, const salf_raster_opts_t *opts,
                        const double *saved, const double *d_depth, const float *feat, const double *dF,
                        const double *Facc, double *grad, double *feat_grad, void *stream);

/* ---- dynamic actors (reference render_ray.py:161-239, next row of SURVEY §8f) --
 * Actor segments are marched with salf_march in each actor's canonical frame,
 * then shaded into 24-double records (t0, t1, t_mid, delta, x[3], s, e, sigma,
 * alpha, 1-alpha, c[3], a, 1/b, dir[3], owner, global voxel id, pad[2]). */
/* Rays into an actor's canonical frame + the actor-box test, on the device
 * (render_ray.py:180-190; octree.py:175-194): pose_idx[n] (int64, nullable =
 * row 0) selects a row of poses (P x 12 f64: translation[3], row-major
 * rotation[9]) -- the host evaluates Actor.pose_at once per DISTINCT timestamp
 * of the batch; o_actor / d_actor (n x 3 f64) and hit[n] (uint8) out.
 * half_extents: HOST pointer to 3 doubles. */
int salf_actor_rays(int64_t n, const double *origins, const double *dirs, const int64_t *pose_idx,
                    const double *poses, const double *half_extents, double *o_actor, double *d_actor,
                    uint8_t *hit, void *stream);

int salf_shade_segments(const salf_scene_t *scene, int64_t n, const double *seg_origin,
                        const double *seg_dir, const int64_t *seg_vid, const double *seg_t0,
                        const double *seg_t1, int32_t owner, int64_t vid_offset, int32_t exact_color,
                        double *records, void *stream);

/* integrate_rays with live actors: the static march (no early stop) merged per
 * ray with the actor records of CSR ex_start[n + 1] / ex_rec, sorted by
 * (t0, owner, vid) -- the reference's lexsort order. */
int salf_ray_forward_merge(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                           const double *origins, const double *dirs, const uint8_t *valid,
                           const salf_raster_opts_t *opts, const int64_t *ex_start, const double *ex_rec,
                           float *out_rgb, float *out_opacity, float *out_depth, double *saved,
                           int32_t *status, void *stream);

/* Its backward: static gradients into grad (M x 27), actor gradients into
 * ex_grad (sum of actor voxel counts x 27, by global voxel id). */
int salf_ray_backward_merge(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                            const double *origins, const double *dirs, const uint8_t *valid,
                            const salf_raster_opts_t *opts, const int64_t *ex_start, const double *ex_rec,
                            const double *saved, const double *d_rgb, const double *d_depth, double *grad,
                            double *ex_grad, void *stream);

/* backward_records (backward.py:35-101) for the ray path, re-marching each
 * ray: d_rgb (N x 3), d_depth (N) f64; grad (M x 27 f64, accumulated).
 * d_rgb may be NULL (depth-only seeds, e.g. LiDAR): a kernel without the
 * colour terms runs, with the values zero colour seeds would give. */
int salf_ray_backward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                      const double *origins, const double *dirs, const uint8_t *valid,
                      const salf_raster_opts_t *opts, const double *saved, const double *d_rgb,
                      const double *d_depth, double *grad, void *stream);

/* ---- rest of the training step ---------------------
 * Parameter block `params`: (M, 27) f64 rows w_s[4] w_c[9] w_sh[12] log_a
 * log_b, the gradient buffer's layout. */

/* adam_step (optim.py:48-62): one update of n = M*27 values; step = t >= 1. */
int salf_adam_step(int64_t n, double *params, const double *grad, double *m, double *v, double lr,
                   double beta1, double beta2, double eps, int64_t step, void *stream);

/* Refresh the device scene's prm (f32) and aux (a, 1/b) from the block. */
int salf_scene_refresh(const double *params, int64_t n_voxels, float *prm, double *aux, void *stream);

/* loss_eikonal (losses.py:49-60) over voxel indices idx; adds gradients into
 * grad and sum |.| into *loss_sum (device). */
int salf_loss_eikonal(const double *params, int64_t n_idx, const int64_t *idx, double *grad,
                      double *loss_sum, void *stream);

/* Centre opacity over the voxel edge (loss_empty's ranking key, losses.py:216-228). */
int salf_center_alpha(const double *params, const double *geo, int32_t density_mode, int64_t n_idx,
                      const int64_t *idx, double *alpha, void *stream);

/* loss_empty gradient (losses.py:230-249) for the k lowest-opacity outer voxels sel. */
int salf_loss_empty_grad(const double *params, const double *geo, int32_t density_mode, int64_t k,
                         const int64_t *sel, double *grad, void *stream);

/* loss_opacity_lidar (losses.py:188-226) for n points located in leaves vid. */
int salf_loss_opacity_lidar(const double *params, const double *geo, int32_t density_mode, int64_t n,
                            const double *points, const int64_t *vid, double *grad, double *loss_sum,
                            void *stream);

/* loss_smooth (losses.py:95-185) over deduplicated face pairs (fine voxel,
 * same-or-coarser neighbour, axis, sign): adds gradients into grad and
 * (sum |dSDF|, sum |dColour|) into loss_sums[2] (means use 4n and 12n). */
int salf_loss_smooth(const double *params, const double *geo, int64_t n_pairs, const int64_t *fine,
                     const int64_t *coarse, const int32_t *axis, const double *sign, double *grad,
                     double *loss_sums, void *stream);

/* ---- secondary-ray effects (reference render_ray.py:310-489) ---------- */

enum { SALF_SPHERE_MIRROR = 0, SALF_SPHERE_GLASS = 1, SALF_SPHERE_OPAQUE = 2 };

/* InjectedSphere (render_ray.py:313-330). */
typedef struct {
  double center[3];
  double radius;
  double ior;
  double albedo[3];
  int32_t material, pad;
} salf_sphere_t;

/* One wave of trace_effects (render_ray.py:360-489) after the wave's rays
 * were rendered through the volume (vol_rgb n x 3 f32, vol_saved n x 8 f64
 * from salf_ray_forward): sphere hits, volume-vs-sphere decision, sun
 * shadows, accumulation into out (n_pixels x 3 f64, atomic adds at pix),
 * and the next wave in slots 2i / 2i+1 (next_flag marks the used slots;
 * capacity 2n).  spheres: device array; sun_dir: 3 host doubles (unit). */
int salf_effects_wave(int64_t n, const double *origins, const double *dirs, const double *t_stamps,
                      const double *weight, const int32_t *budget, const int64_t *pix,
                      const float *vol_rgb, const double *vol_saved, int32_t n_spheres,
                      const salf_sphere_t *spheres, const double *sun_dir, double *out,
                      double *next_origins, double *next_dirs, double *next_t_stamps, double *next_weight,
                      int32_t *next_budget, int64_t *next_pix, uint8_t *next_flag, void *stream);

/* L1 loss seed and value (losses.py:22-31): d_out[i] = sign(pred[i] - gt[i]) * scale
 * where selected (mask[i / group] != 0; mask NULL selects all), else 0;
 * *loss_sum += sum of |pred - gt| over the selection (f64 accumulation).
 * pred: n f32; gt: n f32 or f64 (gt_f64). */
int salf_l1_seed(int64_t n, const float *pred, const void *gt, int32_t gt_f64, const uint8_t *mask,
                 int32_t group, double scale, double *d_out, double *loss_sum, void *stream);

/* ---- densify / prune (reference densify.py:39-94, optim.py:35-40) ------- */

/* Centre opacity and the prune / eligible flags of every voxel
 * (densify.py:39-46, :62-70): flags bit 0 = prune (opacity < prune_opacity),
 * bit 1 = eligible for splitting (kept and level < max_levels - 1).
 * params: (n x 27) f64 parameter block; geo: (n x 4) f64 (edge at [3]);
 * opacity (n f64) may be NULL. */
int salf_densify_flags(int64_t n, const double *params, const double *geo, const uint8_t *level,
                       int32_t density_mode, double prune_opacity, int32_t max_levels, uint8_t *flags,
                       double *opacity, void *stream);

/* grad_acc[i] += ||dL/dW_c[i]||_2 over the (n x 27) gradient block (trainer.py:193). */
int salf_grad_norm_acc(int64_t n, const double *grad, double *acc, void *stream);

/* The densified set (densify.py:72-91): rows [0, n_keep) gathered from
 * keep_idx, then 8 children per split_idx entry (level + 1, 2 ijk + offset,
 * offsets x fastest) inheriting the parameters; Adam moments m/v (optional,
 * NULL to skip) carried for kept rows and zeroed for children (optim.py:35-40). */
int salf_densify_apply(int64_t n_keep, const int64_t *keep_idx, int64_t n_split, const int64_t *split_idx,
                       const uint8_t *level, const int32_t *ijk, const double *params, const double *m,
                       const double *v, uint8_t *level_out, int32_t *ijk_out, double *params_out,
                       double *m_out, double *v_out, void *stream);

/* Device scene arrays from (level, ijk, params) (scene.py:186-194): geo
 * (n x 4 f64: centre, edge), aux (n x 4 f64: exp(log_a), 1/exp(log_b),
 * 2/edge, 0), prm (n x SALF_PRM_STRIDE f32). aabb_min: 3 host doubles. */
int salf_voxel_geometry(int64_t n, const uint8_t *level, const int32_t *ijk, const double *aabb_min,
                        double base_edge, const double *params, double *geo, double *aux, float *prm,
                        void *stream);

/* salf.v1 voxel records (container.py:27-35; 121-byte little-endian records,
 * device copy of voxels.bin, 16-byte aligned) decoded straight into the
 * device layout: level (u8), ijk (i32 x3), params (n x 27 f64), geo, aux,
 * prm as salf_voxel_geometry; *bad |= 1 << f for non-finite values in field
 * f (0 w_s, 1 w_c, 2 w_sh, 3 log_a, 4 log_b; container.py:56-59). */
int salf_decode_records(int64_t n, const uint8_t *records, const double *aabb_min, double base_edge,
                        uint8_t *level, int32_t *ijk, double *params, double *geo, double *aux, float *prm,
                        int32_t *bad, void *stream);

/* FP64 peak probe (benchmark utility): grid x 256 threads x 64*iters DFMA. */
int salf_fp64_peak(double *scratch, int32_t grid, int32_t iters, void *stream);

/* FP32 peak probe (benchmark utility): grid x 256 threads x 64*iters FFMA. */
int salf_fp32_peak(float *scratch, int32_t grid, int32_t iters, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SALF_B200_H */
