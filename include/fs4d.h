/*
 * fs4d.h — C ABI of libfs4d.so, the sm_100a implementation of the FE-4DGS
 * per-frame render path (HexPlane+MLP deformation, tile rasterizer, and their
 * analytic backward passes).
 *
 * The reference (`featsplat`, /root/reference/pkg/src/featsplat) is pure
 * Python/NumPy and has no FFI; its "plugin boundary" is a set of Python
 * functions.  Every entry point below replaces one of them and cites it:
 *
 *   fs4d_deform_fwd   <- deformation.deform_with_cache   deformation.py:105-136
 *                        (hexplane.query_with_cache       hexplane.py:118-142,
 *                         numerics.mlp_forward            numerics.py:56-75)
 *   fs4d_deform_bwd   <- deformation.deform_backward     deformation.py:139-183
 *                        (hexplane.query_backward         hexplane.py:145-187,
 *                         numerics.mlp_backward           numerics.py:78-105)
 *   fs4d_render_fwd   <- rasterizer.render               rasterizer.py:264-303
 *                        (project :117-185, bin_tiles :188-207,
 *                         _tile_alphas :215-234, _composite_weights :244-261)
 *   fs4d_render_bwd   <- rasterizer.render_backward      rasterizer.py:320-452
 *                        (gaussians.covariance_backward   gaussians.py:203-218)
 *   fs4d_render_export_projected / fs4d_render_export_tiles
 *                     <- rasterizer.project / bin_tiles results (ProjectedGaussians,
 *                        per-tile lists) read back from a forward record.
 *
 * and the callers either side of the path:
 *   fs4d_l1_loss_grad / fs4d_photometric_loss_grad / fs4d_l1
 *                     <- training._photometric_terms/_grads training.py:300-338,
 *                        semantic.feature_loss(_backward) semantic.py:171-181
 *   fs4d_adam_step    <- numerics.adam_step numerics.py:137-159 (per array,
 *                        training.py:431-442), all arrays in one launch
 *   fs4d_tv_loss_grad <- hexplane.tv_loss / tv_backward hexplane.py:190-222
 *   fs4d_resize_bilinear(_backward) <- semantic.resize_bilinear(_backward) semantic.py:82-123
 *   fs4d_decode_features(_backward) / fs4d_decoder_feature_loss
 *                     <- semantic.decode_features_with_cache / _backward semantic.py:145-168
 *   fs4d_grad_stats_add / fs4d_density_classify / fs4d_density_apply / fs4d_reset_opacity
 *                     <- gaussians.ViewspaceGradStats.add, densify_and_prune,
 *                        prune_only, reset_opacity gaussians.py:309-425
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; all float data is fp32,
 *    row-major in the reference's logical layout ([K,3] positions, [K,4]
 *    (w,x,y,z) rotations, [H,W,C] images, [Ra,Rb,C] planes, [out,in] weights).
 *  - Every call is stream-ordered, allocation-free and never synchronises the
 *    device.  Host-detectable errors (bad configuration, skewed intrinsics,
 *    record/snapshot mismatch, undersized workspace) are returned directly.
 *    Device-detected errors (non-finite parameters, degenerate quaternions,
 *    pair-buffer overflow) are written to the caller's device status block
 *    (FS4D_STATUS_WORDS int32) and read by the host when it chooses to.
 *  - Error codes mirror featsplat/errors.py:4-35 and the CLI exit codes.
 */
#ifndef FS4D_H_
#define FS4D_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS4D_ABI_VERSION 1

/* status / return codes (errors.py:4-35) */
#define FS4D_OK 0
#define FS4D_ERR_CONFIG 1        /* ConfigurationError                    */
#define FS4D_ERR_DATA 2          /* DataError (e.g. skewed intrinsics)    */
#define FS4D_ERR_NUMERIC 3       /* NumericalError (non-finite inputs)    */
#define FS4D_ERR_CONTRACT 4      /* ContractViolation (stale record)      */
#define FS4D_ERR_CAPACITY 5      /* pair buffer too small: grow + retry   */
#define FS4D_ERR_DEGENERATE 6    /* DegenerateRotationError (|q|<1e-12)   */
#define FS4D_ERR_CUDA 7          /* CUDA launch failure                   */

/* device status block layout (int32 words) */
#define FS4D_STATUS_WORDS 32
#define FS4D_ST_CODE 0           /* first device error code (atomicCAS)       */
#define FS4D_ST_BAD_FIELDS 1     /* bitmask of cloud fields with non-finite   */
#define FS4D_ST_N_VISIBLE 2      /* kept Gaussians after culls (M)            */
#define FS4D_ST_PAIRS_LO 3       /* total (tile, Gaussian) pairs, low word    */
#define FS4D_ST_PAIRS_HI 4       /*                              high word    */
#define FS4D_ST_BAD_INDEX 8      /* 8 words: first bad index per field        */
#define FS4D_ST_DEGEN_INDEX 16   /* first degenerate-quaternion index         */

/* cloud field ids (order of rasterizer.py:120-127 finite checks) */
#define FS4D_FIELD_POSITIONS 0
#define FS4D_FIELD_ROTATIONS 1
#define FS4D_FIELD_LOG_SCALES 2
#define FS4D_FIELD_OPACITY 3
#define FS4D_FIELD_COLORS 4
#define FS4D_FIELD_FEATURES 5
#define FS4D_FIELD_SH 6

#define FS4D_MAX_LEVELS 8
#define FS4D_MAX_TRUNK 16
#define FS4D_N_BRANCHES 4        /* position, rotation, scale, opacity (deformation.py:19) */

/* GaussianCloud (gaussians.py:39-94) as SoA device arrays.  sh_rest is the
 * build's SH extension ([K, (L+1)^2-1, 3], degree-0 term is colors_raw);
 * NULL when sh_degree == 0. */
typedef struct Fs4dCloud {
  int64_t K;
  int32_t D;          /* feature channels N */
  int32_t sh_degree;  /* 0..3 */
  float* positions;       /* [K,3] */
  float* rotations;       /* [K,4] raw (w,x,y,z) */
  float* log_scales;      /* [K,3] */
  float* opacity_logits;  /* [K]   */
  float* colors_raw;      /* [K,3] */
  float* sh_rest;         /* [K,(L+1)^2-1,3] or NULL */
  float* features;        /* [K,D] */
} Fs4dCloud;

/* CameraFrame intrinsics/extrinsics (gaussians.py:97-133) in float64. */
typedef struct Fs4dCamera {
  int32_t height, width;
  double K[9];   /* 3x3 row-major */
  double T[16];  /* 4x4 world->camera, row-major */
} Fs4dCamera;

/* RasterConfig (rasterizer.py:26-35). */
typedef struct Fs4dRasterConfig {
  int32_t tile;            /* only 16 is implemented on device */
  int32_t with_features;
  double z_near, lowpass, alpha_cap, alpha_skip, stop_transmittance;
  double background[3];
} Fs4dRasterConfig;

/* Sizes a render record (workspace) is laid out for; passed unchanged to the
 * forward and the backward call (the record's snapshot_len/height/width
 * contract, rasterizer.py:330-331). */
typedef struct Fs4dRecordInfo {
  int64_t K;
  int32_t height, width, D, sh_degree, tile, pad_;
  int64_t pair_capacity;
} Fs4dRecordInfo;

/* RenderOutput images (rasterizer.py:95-100), all device, row-major. */
typedef struct Fs4dImages {
  float* color;      /* [H,W,3] */
  float* depth;      /* [H,W]   */
  float* feature;    /* [H,W,D] (D = 0 when with_features == 0) */
  float* alpha;      /* [H,W]   */
  int32_t* n_contrib;/* [H,W] live contributor count (RenderOutput.pixel_record), may be NULL */
} Fs4dImages;

/* Upstream image gradients for render_backward; NULL == zeros. */
typedef struct Fs4dImageGrads {
  const float* d_color;   /* [H,W,3] */
  const float* d_depth;   /* [H,W]   */
  const float* d_feature; /* [H,W,D] */
  const float* d_alpha;   /* [H,W]   */
} Fs4dImageGrads;

/* ProjectedGaussians export (rasterizer.py:38-61), depth-sorted, M rows. */
typedef struct Fs4dProjected {
  float* mean2d;        /* [K,2]   */
  float* cov2d;         /* [K,3]   (a, b, c) of the symmetric 2x2 */
  float* conic;         /* [K,3]   */
  float* view_depth;    /* [K]     */
  float* radius;        /* [K]     */
  float* color;         /* [K,3]   */
  float* opacity;       /* [K]     */
  int32_t* source_index;/* [K]     */
  int32_t* tiles_touched;/*[K]     */
} Fs4dProjected;

/* HexPlaneField (hexplane.py:49-92). planes[l][p] is [res[l][p][0], res[l][p][1], channels]. */
typedef struct Fs4dHexPlane {
  int32_t levels, channels;
  int32_t res[FS4D_MAX_LEVELS][6][2];
  float* planes[FS4D_MAX_LEVELS][6];
  double aabb[6];  /* lo xyz, hi xyz */
  /* Optional order in which the plane gathers / scatters visit the K
   * Gaussians (a permutation of [0, K), e.g. fs4d_locality_order), or NULL
   * for index order.  Every Gaussian's latent is computed independently, so
   * any permutation gives identical results (the backward's float atomics
   * are unordered either way); a spatially coherent one turns most corner-
   * row fetches into L1 hits. */
  const int32_t* order;
} Fs4dHexPlane;

/* LinearLayer (numerics.py:17-41): y = act(x W^T + b), W [out,in]. */
typedef struct Fs4dLinear {
  float* weight;
  float* bias;
  int32_t in_dim, out_dim, relu;
} Fs4dLinear;

/* DeformationNet (deformation.py:32-73).  Branch order: position, rotation,
 * scale, opacity.  The same struct carries gradient buffers in deform_bwd. */
typedef struct Fs4dDeformNet {
  int32_t latent_dim, width, depth, feature_dim;
  int32_t enable_grid, enable_feature_update;
  Fs4dLinear trunk[FS4D_MAX_TRUNK];
  Fs4dLinear ext[FS4D_N_BRANCHES][2];
  Fs4dLinear head[FS4D_N_BRANCHES];
  Fs4dLinear feat[2];
} Fs4dDeformNet;

/* ---- library info ---- */
int fs4d_abi_version(void);
const char* fs4d_last_error(void);          /* thread-local message of the last failing call */
const char* fs4d_build_info(void);

/* Initialise a device status block (FS4D_STATUS_WORDS int32) before a call:
 * zero codes/counters, INT32_MAX in the first-index slots. */
int fs4d_status_reset(int32_t* status, void* stream);

/* Fold the status block `src` of a finished call into the accumulating block
 * `dst`, stream-ordered (no host sync): the first error code and its words
 * win, repeated capacity overflows keep the largest pair count.  With
 * gate_adam != 0 an error in src also sets dst[FS4D_ST_ADAM_BAD_SEG] =
 * FS4D_ADAM_GATED so that a following fs4d_adam_step with status = dst
 * touches nothing -- a training step whose render failed (pair-buffer
 * overflow, non-finite snapshot) never updates the parameters.  No reference
 * counterpart (the reference raises synchronously, rasterizer.py:120-131). */
#define FS4D_ADAM_GATED (-1)
int fs4d_status_merge(const int32_t* src, int32_t* dst, int32_t gate_adam, void* stream);

/* ---- optional per-stage timing ----
 * When enabled, every entry point brackets its stages with CUDA events
 * recorded on the launching stream; collect() waits on them, returns the
 * summed milliseconds and call counts per stage, and resets.  Disabled by
 * default (no events are recorded). */
#define FS4D_STAGE_DEFORM_FWD 0   /* weight pack + k_deform_fwd           */
#define FS4D_STAGE_PREPROCESS 1   /* k_preprocess (projection, fp64)      */
#define FS4D_STAGE_DEPTH_SORT 2   /* radix depth sort + tie fix-up        */
#define FS4D_STAGE_BINNING 3      /* count, scan, emit, tile sort, ranges */
#define FS4D_STAGE_BLEND 4        /* k_blend                              */
#define FS4D_STAGE_BLEND_BWD 5    /* k_blend_bwd                          */
#define FS4D_STAGE_PREPROCESS_BWD 6
#define FS4D_STAGE_DEFORM_BWD 7
#define FS4D_STAGE_DEFORM_GATHER 8 /* HexPlane latent gather (inside DEFORM_FWD) */
#define FS4D_STAGE_DEFORM_MLP 9    /* tcgen05 MLP + delta apply (inside DEFORM_FWD) */
#define FS4D_N_STAGES 10
int fs4d_profile_enable(int on);
int fs4d_profile_collect(double* ms_total, int64_t* calls, int32_t n_stages);

/* Spatially coherent visiting order of a cloud for Fs4dHexPlane.order:
 * Gaussians sorted by the 30-bit Morton code of their position normalised
 * by aabb (lo xyz, hi xyz) and clipped to it, ties by index (stable radix
 * sort).  A model-load-time permutation: it never changes results, only
 * cache locality, so it may be reused while positions drift. */
size_t fs4d_locality_order_workspace_bytes(int64_t K);
int fs4d_locality_order(const float* positions, int64_t K, const double* aabb, int32_t* order,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ---- deformation ---- */
/* Bytes of device scratch the deform calls need (packed weights + per-CTA
 * weight-gradient partials for the backward). */
size_t fs4d_deform_workspace_bytes(const Fs4dDeformNet* net, int64_t K);

/* Bytes of the activation cache deform_with_cache keeps for deform_backward
 * (deformation.py:105-136 returns it as `cache`): per 128 Gaussians the
 * tensor-core operand images of latent, hidden, e1, e2 and F_feat's hidden
 * layer.  0 when the net shape is outside the tensor-core backward (the
 * backward then recomputes the forward and needs no cache). */
size_t fs4d_deform_cache_bytes(const Fs4dDeformNet* net, const Fs4dHexPlane* field, int64_t K);

/* deform / deform_with_cache: writes snapshot->{positions, rotations,
 * log_scales, opacity_logits, features}; colors_raw / sh_rest are aliased by
 * the caller (deformation.py:131), as are features when
 * enable_feature_update == 0.  cache == NULL is `deform` (no cache); a cache
 * of fs4d_deform_cache_bytes() bytes is `deform_with_cache`. */
int fs4d_deform_fwd(const Fs4dCloud* cloud, const Fs4dHexPlane* field,
                    const Fs4dDeformNet* net, double t, Fs4dCloud* snapshot,
                    void* cache, size_t cache_bytes,
                    void* workspace, size_t workspace_bytes,
                    int32_t* status, void* stream);

/* deform_backward: snapshot_grads carries dL/d{positions, rotations,
 * log_scales, opacity_logits, features} of the snapshot.  Writes cloud_grads
 * (positions incl. the grid term, others pass through), net_grads (weight /
 * bias pointers of the struct, zeroed and accumulated) and plane_grads
 * (shapes of field->planes, zeroed and accumulated; ignored when
 * enable_grid == 0).  `cache` is the deform_with_cache cache of the same
 * (cloud, t) -- a mismatch raises FS4D_ERR_CONTRACT in the status block -- or
 * NULL, in which case the forward is recomputed (deformation.py:139 takes the
 * cache; the recompute path serves callers that kept none). */
int fs4d_deform_bwd(const Fs4dCloud* cloud, const Fs4dHexPlane* field,
                    const Fs4dDeformNet* net, double t,
                    const void* cache, size_t cache_bytes,
                    const Fs4dCloud* snapshot_grads, Fs4dCloud* cloud_grads,
                    Fs4dDeformNet* net_grads, Fs4dHexPlane* plane_grads,
                    int32_t accumulate,
                    void* workspace, size_t workspace_bytes,
                    int32_t* status, void* stream);
/* Deterministic variant (fixed-order reductions): the
 * HexPlane plane gradients accumulate in int64 fixed point -- one scale per
 * plane, 2^(62 - ceil(log2 B)) with B = K * C * max|d latent| * the product of
 * the other five planes' max |value| (a bound on the plane's total L1 mass),
 * computed on device -- so integer adds make the scatter order irrelevant
 * and the result bitwise reproducible (rounding unit ~B * 2^-62).  Every other
 * output of the tensor-core backward is already produced in a fixed order.
 * Needs the cached tensor-core path (width 64, depth 1, levels * channels =
 * 64, feature_dim <= 16); det_workspace of
 * fs4d_deform_bwd_det_workspace_bytes bytes. */
int fs4d_deform_bwd_deterministic(const Fs4dCloud* cloud, const Fs4dHexPlane* field, const Fs4dDeformNet* net,
                                  double t, const void* cache, size_t cache_bytes,
                                  const Fs4dCloud* snapshot_grads, Fs4dCloud* cloud_grads,
                                  Fs4dDeformNet* net_grads, Fs4dHexPlane* plane_grads, int32_t accumulate,
                                  void* workspace, size_t workspace_bytes, void* det_workspace,
                                  size_t det_workspace_bytes, int32_t* status, void* stream);
size_t fs4d_deform_bwd_det_workspace_bytes(const Fs4dDeformNet* net, const Fs4dHexPlane* field);
/* fs4d_deform_bwd (det_workspace NULL) or fs4d_deform_bwd_deterministic
 * (det_workspace non-NULL) that also records `passthrough_event` (a
 * cudaEvent_t, may be NULL) on `stream` as soon as every cloud gradient
 * except positions is written -- the pass-through rows of
 * deformation.py:172-181 -- so a data-parallel caller can all-reduce those
 * rows while the MLP and HexPlane backward still run (the gradient exchange
 * of training.py:459-539 across ranks). */
int fs4d_deform_bwd_split(const Fs4dCloud* cloud, const Fs4dHexPlane* field, const Fs4dDeformNet* net,
                          double t, const void* cache, size_t cache_bytes,
                          const Fs4dCloud* snapshot_grads, Fs4dCloud* cloud_grads,
                          Fs4dDeformNet* net_grads, Fs4dHexPlane* plane_grads, int32_t accumulate,
                          void* workspace, size_t workspace_bytes, void* det_workspace,
                          size_t det_workspace_bytes, void* passthrough_event, int32_t* status,
                          void* stream);
/* accumulate != 0 adds into every output instead of overwriting it (gradient
 * accumulation over the (view, t) pairs of a training step).  Non-NULL
 * cloud_grads fields other than positions receive the pass-through snapshot
 * gradients (deformation.py:178-181; colours/SH bypass the deformation,
 * training.py:518). */

/* Fused L1 photometric + feature loss and its upstream gradients
 * (training.py:302-338 with an all-ones mask, semantic.py:171-181 at render
 * resolution): dC = w_rgb*sign(C-Ct)/(3HW), dF = w_feat*sign(F-Ft)/(HW); the
 * weighted loss is atomically added to *loss (device double). */
int fs4d_l1_loss_grad(const float* color, const float* color_target, const float* feature,
                      const float* feature_target, int32_t height, int32_t width, int32_t D,
                      double w_rgb, double w_feat, float* d_color, float* d_feature, double* loss,
                      void* stream);

/* ---- training-step glue ---- */

/* Masked photometric L1 (training.py:300-338 _photometric_terms /
 * _photometric_grads): rgb = sum|C-I|[mask]/n_rgb with n_rgb = 3*count(mask);
 * depth = sum|D-Dt|[dmask]/n_d with dmask = mask & (alpha >= 0.5);
 * dC = lambda_rgb*sign(C-I)*mask/n_rgb, dD = lambda_depth*sign(D-Dt)*dmask/n_d
 * (zero when the count is zero).  mask (uint8 [H,W]) may be NULL (all ones);
 * depth/depth_target/alpha/d_depth may be NULL (no depth term).  terms[4]
 * (device double, may be NULL) receives {rgb, depth, n_rgb, n_d}; *loss (may
 * be NULL) += lambda_rgb*rgb + lambda_depth*depth.  workspace:
 * fs4d_photometric_workspace_bytes(H, W). */
size_t fs4d_photometric_workspace_bytes(int32_t height, int32_t width);
int fs4d_photometric_loss_grad(const float* color, const float* image, const uint8_t* mask,
                               const float* depth, const float* depth_target, const float* alpha,
                               int32_t height, int32_t width, double lambda_rgb, double lambda_depth,
                               float* d_color, float* d_depth, double* terms, double* loss,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Generic L1 (semantic.py:171-181 feature_loss / feature_loss_backward):
 * *loss += scale * sum|pred - target|; grad = scale * sign(pred - target)
 * (either output may be NULL).  feature_loss is scale = 1/(H*W). */
int fs4d_l1(const float* pred, const float* target, int64_t n, double scale, float* grad,
            double* loss, void* stream);

/* dst[i] (+)= srcs[0][i] + ... + srcs[n_src-1][i] in that order, one pass
 * (accumulate != 0 adds to dst): the training step's per-lane gradient
 * buffers summed before the all-reduce.  srcs is a host array of up to 8
 * device pointers.  No reference counterpart (the reference has one lane). */
int fs4d_sum_buffers(float* dst, const float* const* srcs, int32_t n_src, int64_t n, int32_t accumulate,
                     void* stream);

/* HexPlane query on its own (hexplane.query / query_with_cache,
 * hexplane.py:113-142): latent [K, levels * channels] (level-major, the
 * reference's concat order) of positions [K, 3] at time t (clipped to
 * [0, 1]); coordinates and cells in fp64 as in deformation.  1..4 levels. */
int fs4d_hexplane_query(const Fs4dHexPlane* field, const float* positions, int64_t K, double t, float* latent,
                        void* stream);
/* hexplane.query_backward (hexplane.py:145-187): plane_grads (same shapes as
 * field; written, or added with accumulate != 0) receive d latent / d plane
 * for the upstream d_latent [K, levels * channels]; d_positions [K, 3] (written
 * or added) the position gradient, zero on every axis whose coordinate was
 * clamped (outside the aabb, hexplane.py:186). */
int fs4d_hexplane_query_backward(const Fs4dHexPlane* field, const float* positions, int64_t K, double t,
                                 const float* d_latent, Fs4dHexPlane* plane_grads, float* d_positions,
                                 int32_t accumulate, void* stream);

/* One dense layer of numerics.mlp_forward / mlp_backward (numerics.py:56-105)
 * for any shape (API helper; the deformation MLP itself runs fused on the
 * tensor cores inside fs4d_deform_*): pre = x W^T + b, y = ReLU(pre) or pre,
 * x [batch, in], W [out, in] (layer->relu selects the activation).  The
 * backward writes dx = g W (dx may be NULL), dW = g^T x, db = sum_b g with
 * g = dy * (pre > 0) for ReLU layers; dW / db are written, or added with
 * accumulate != 0, and reduced over the batch in a fixed order
 * (deterministic). */
int fs4d_linear_forward(const float* x, int64_t batch, const Fs4dLinear* layer, float* pre, float* y, void* stream);
size_t fs4d_linear_backward_workspace_bytes(int64_t batch, int32_t in_dim, int32_t out_dim);
int fs4d_linear_backward(const float* x, const float* pre, int64_t batch, const Fs4dLinear* layer, const float* dy,
                         float* dx, float* d_weight, float* d_bias, int32_t accumulate, void* workspace,
                         size_t workspace_bytes, void* stream);

/* rasterizer._tile_alphas (rasterizer.py:215-234) replayed from a render
 * record: for the G Gaussians source_index[G] and the pixels
 * [x0, x0+nx) x [y0, y0+ny) (row-major P = nx*ny), alpha / g2d / a_raw
 * [G, P] exactly as the record's blend evaluated them (same footprint,
 * q-skip, cap and skip decisions). */
int fs4d_render_tile_alphas(const Fs4dRecordInfo* info, const void* workspace, size_t workspace_bytes,
                            const Fs4dRasterConfig* cfg, const int32_t* source_index, int64_t G, int32_t x0,
                            int32_t y0, int32_t nx, int32_t ny, float* alpha, float* g2d, float* a_raw, void* stream);
/* rasterizer._composite_weights (rasterizer.py:244-261) of alpha [G, P]:
 * t_exc, contrib (0/1 bytes), w [G, P] and t_final [P], front to back in
 * fp32 with the blend's multiplication order. */
int fs4d_composite_weights(const float* alpha, int64_t G, int64_t P, double stop, float* t_exc, uint8_t* contrib,
                           float* w, float* t_final, void* stream);

/* Adam over a flat parameter buffer (numerics.py:119-159 AdamState /
 * adam_step, applied per parameter array as training.py:431-442 does).
 * Every segment is one reference parameter array: [offset, offset+count) of
 * params/grads/m/v, its learning rate (lr_at_step of its schedule,
 * numerics.py:189-199, computed by the host) and eps (training.py:46-47).
 * step_counts[i] (device int32) is segment i's AdamState.step_count; it is
 * incremented by the call.  A non-finite gradient anywhere aborts the whole
 * step before any parameter or moment is touched (numerics.py:149-153):
 * status[FS4D_ST_ADAM_BAD_SEG] gets the first bad segment,
 * status[FS4D_ST_ADAM_BAD_COUNT] the number of non-finite entries, and the
 * status code FS4D_ERR_NUMERIC. */
#define FS4D_MAX_ADAM_SEGMENTS 128
#define FS4D_ST_ADAM_BAD_SEG 17
#define FS4D_ST_ADAM_BAD_COUNT 18
typedef struct Fs4dAdamSegment {
  int64_t offset, count;
  double lr, eps, beta1, beta2;
} Fs4dAdamSegment;
int fs4d_adam_step(float* params, const float* grads, float* m, float* v, int32_t* step_counts,
                   const Fs4dAdamSegment* segments /* host array */, int32_t n_segments,
                   int32_t* status, void* stream);
/* Same, stepping only the segments with active[i] != 0 (host array; NULL =
 * all): the reference steps only the arrays present in its gradient dict
 * (training.py:513-515 drops `features` without feature supervision,
 * :519-529 adds grid.* only with the HexPlane enabled, :531 decoder.* only
 * with the feature loss), so an inactive array keeps its parameters,
 * moments and step count. */
int fs4d_adam_step_masked(float* params, const float* grads, float* m, float* v, int32_t* step_counts,
                          const Fs4dAdamSegment* segments /* host array */, const int32_t* active /* host */,
                          int32_t n_segments, int32_t* status, void* stream);

/* HexPlane total-variation regulariser (hexplane.py:190-222): with tv = sum
 * over planes of mean squared axis-adjacent differences, *loss (may be NULL)
 * += scale * tv and grads (same shapes as field, may be NULL) receive
 * d(scale * tv)/d(plane), overwritten or (accumulate != 0) added -- so the
 * TV term folds into the plane-gradient segment of the flat buffer before
 * the all-reduce, in one pass over the planes. */
int fs4d_tv_loss_grad(const Fs4dHexPlane* field, Fs4dHexPlane* grads, double scale,
                      int32_t accumulate, double* loss, void* stream);

/* Corner-aligned bilinear resize of [hi,wi,C] to [ho,wo,C]
 * (semantic.py:82-102) and its adjoint (semantic.py:105-123, computed as a
 * deterministic two-pass gather instead of np.add.at).  The adjoint needs
 * fs4d_resize_workspace_bytes(ho, wi, C) of scratch. */
int fs4d_resize_bilinear(const float* in, int32_t hi, int32_t wi, int32_t C, float* out, int32_t ho,
                         int32_t wo, void* stream);
size_t fs4d_resize_workspace_bytes(int32_t ho, int32_t wi, int32_t C);
int fs4d_resize_bilinear_backward(const float* d_out, int32_t ho, int32_t wo, int32_t C, float* d_in,
                                  int32_t hi, int32_t wi, void* workspace, size_t workspace_bytes,
                                  void* stream);

/* PointwiseDecoder (semantic.py:126-168): out[ho,wo,Ct] = resize(rendered
 * [hi,wi,N]) @ W^T + b with W [Ct,N]; `resized` [ho,wo,N] (the cache) may be
 * NULL.  Backward: d_weight [Ct,N], d_bias [Ct], d_rendered [hi,wi,N] from
 * d_out and the cache; partial sums are reduced in a fixed order (bitwise
 * deterministic).  The fused loss variant computes the decoder output, the
 * feature L1 against `teacher` (semantic.py:171-181, scaled by lambda) and
 * the whole backward in one pass without writing the decoded map:
 *   *loss += lambda * sum|dec - teacher| / (ho*wo). */
size_t fs4d_decoder_workspace_bytes(int32_t hi, int32_t wi, int32_t N, int32_t ho, int32_t wo, int32_t Ct);
int fs4d_decode_features(const float* rendered, int32_t hi, int32_t wi, int32_t N, const float* weight,
                         const float* bias, int32_t Ct, int32_t ho, int32_t wo, float* out, float* resized,
                         void* stream);
int fs4d_decode_features_backward(const float* d_out, const float* resized, const float* weight, int32_t hi,
                                  int32_t wi, int32_t N, int32_t Ct, int32_t ho, int32_t wo,
                                  float* d_rendered, float* d_weight, float* d_bias, int32_t accumulate,
                                  void* workspace, size_t workspace_bytes, void* stream);
int fs4d_decoder_feature_loss(const float* rendered, int32_t hi, int32_t wi, int32_t N, const float* weight,
                              const float* bias, int32_t Ct, const float* teacher, int32_t ho, int32_t wo,
                              double lambda, float* d_rendered, float* d_weight, float* d_bias,
                              int32_t accumulate, double* loss, void* workspace, size_t workspace_bytes,
                              void* stream);

/* ---- adaptive density control (gaussians.py:309-425) ---- */
/* DensityControlConfig (gaussians.py:330-334) plus the scene extent. */
typedef struct Fs4dDensityConfig {
  double grad_threshold, percent_dense, prune_opacity, split_factor, extent;
} Fs4dDensityConfig;

/* ViewspaceGradStats.add (gaussians.py:319-321): accum[idx[i]] += norms[i],
 * count[idx[i]] += 1 for i < n (n = min(n, *n_dev) when n_dev != NULL; the
 * indices of one render_backward are distinct).  indices NULL: norms is the
 * dense per-Gaussian form of fs4d_render_bwd ([K], negative = culled, skipped).
 * accum / count are float64. */
int fs4d_grad_stats_add(double* accum, double* count, const int32_t* indices, const float* norms, int64_t n,
                        const int32_t* n_dev, void* stream);

/* densify_and_prune (gaussians.py:349-405) / prune_only (gaussians.py:408-417)
 * as stream compaction.  Step 1 classifies every row in fp64 and builds the
 * reference's output row order ([kept | clones | split children set 0 | set
 * 1]); counts (device int32[4]) = {n_keep, n_clone, n_split, n_out}.  The
 * caller reads the counts, draws the split samples exactly as the reference
 * does (rng.standard_normal((n_split, 3)) twice -> float64 [2, n_split, 3]) and
 * runs step 2, which writes the new cloud (out->K >= n_out rows), the grad
 * stats (zeroed for densify, compacted for prune_only) and any per-row extra
 * arrays (Adam moments: copied for kept rows, zero for new rows,
 * gaussians.py:336-346).  capacity bounds n_out (CAPACITY status if above). */
size_t fs4d_density_workspace_bytes(int64_t K, int64_t capacity);
int fs4d_density_classify(const Fs4dCloud* cloud, const double* accum, const double* count,
                          const Fs4dDensityConfig* cfg, int32_t prune_only, int64_t capacity, int32_t* counts,
                          void* workspace, size_t workspace_bytes, int32_t* status, void* stream);
int fs4d_density_apply(const Fs4dCloud* cloud, const double* split_normals, const Fs4dDensityConfig* cfg,
                       int64_t capacity, int32_t n_keep, int32_t n_clone, int32_t n_split, Fs4dCloud* out,
                       const double* stats_accum_in, const double* stats_count_in, double* stats_accum_out,
                       double* stats_count_out, int32_t stats_reset, int32_t n_extra,
                       const float* const* extra_in /* host array of device pointers */,
                       float* const* extra_out, const int32_t* extra_width /* host */,
                       void* workspace, size_t workspace_bytes, int32_t* status, void* stream);

/* reset_opacity (gaussians.py:420-425): logit(min(sigmoid(x), cap)) in place. */
int fs4d_reset_opacity(float* opacity_logits, int64_t K, double cap, void* stream);

/* ---- rasterizer ---- */
size_t fs4d_render_workspace_bytes(const Fs4dRecordInfo* info);

/* render: project -> depth sort -> tile binning -> per-tile blend.  The
 * workspace becomes the RasterRecord replayed by fs4d_render_bwd. */
int fs4d_render_fwd(const Fs4dCloud* snapshot, const Fs4dCamera* cam,
                    const Fs4dRasterConfig* cfg, const Fs4dRecordInfo* info,
                    void* workspace, size_t workspace_bytes,
                    Fs4dImages* out, int32_t* status, void* stream);

/* render_backward: grads->{positions, rotations, log_scales, opacity_logits,
 * colors_raw, sh_rest, features} are fully written (zeros for culled rows).
 * viewspace_index / viewspace_norm get the first M entries (depth order).
 * With viewspace_index NULL the depth order is not materialised (no global
 * sort), rows are visited in source order, and a non-NULL viewspace_norm is
 * written densely per Gaussian ([K], -1 for culled rows). */
int fs4d_render_bwd(const Fs4dCloud* snapshot, const Fs4dCamera* cam,
                    const Fs4dRasterConfig* cfg, const Fs4dRecordInfo* info,
                    void* workspace, size_t workspace_bytes,
                    const Fs4dImageGrads* upstream, Fs4dCloud* grads,
                    int32_t* viewspace_index, float* viewspace_norm,
                    int32_t* status, void* stream);

/* Deterministic variant of fs4d_render_bwd: the blend backward writes one
 * partial per (tile pair, row-split CTA) -- the CTA's warps added in a fixed
 * order in shared memory -- and a gather sums each Gaussian's partials over
 * its tiles in row-major order, instead of float atomics: gradients are
 * bitwise reproducible run to run.  D <= 16 feature
 * channels; det_workspace of fs4d_render_bwd_det_workspace_bytes bytes. */
int fs4d_render_bwd_deterministic(const Fs4dCloud* snapshot, const Fs4dCamera* cam, const Fs4dRasterConfig* cfg,
                                  const Fs4dRecordInfo* info, void* workspace, size_t workspace_bytes,
                                  const Fs4dImageGrads* upstream, Fs4dCloud* grads, int32_t* viewspace_index,
                                  float* viewspace_norm, void* det_workspace, size_t det_workspace_bytes,
                                  int32_t* status, void* stream);
size_t fs4d_render_bwd_det_workspace_bytes(const Fs4dRecordInfo* info);

/* Read back a forward record: depth-sorted ProjectedGaussians (first M rows). */
int fs4d_render_export_projected(const Fs4dRecordInfo* info, const void* workspace,
                                 size_t workspace_bytes, Fs4dProjected* out,
                                 void* stream);

/* Read back tile lists: tile_ranges [n_tiles,2] (start,end) into pair_values
 * [pairs] (depth rank of the Gaussian, i.e. row of the ProjectedGaussians). */
int fs4d_render_export_tiles(const Fs4dRecordInfo* info, const void* workspace,
                             size_t workspace_bytes, int32_t* tile_ranges,
                             int32_t* pair_rows, int64_t max_pairs, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FS4D_H_ */
