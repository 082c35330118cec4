// extern "C" surface of libfs4d.so (declared in include/fs4d.h).
#include <stdio.h>
#include <string.h>

#include <vector>

#include "render_common.cuh"

namespace fs4d {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS4D_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return FS4D_OK;
}

// ---------------------------------------------------------------------------
// stage profiler: pairs of CUDA events per stage invocation
// ---------------------------------------------------------------------------
struct ProfRec {
  int stage;
  cudaEvent_t a, b;
};
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof_done;
static ProfRec g_prof_open[FS4D_N_STAGES];
static std::vector<cudaEvent_t> g_prof_pool;

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void profile_mark(int stage, bool begin, cudaStream_t s) {
  if (!g_prof_on || stage < 0 || stage >= FS4D_N_STAGES) return;
  if (begin) {
    g_prof_open[stage].stage = stage;
    g_prof_open[stage].a = prof_event();
    cudaEventRecord(g_prof_open[stage].a, s);
  } else {
    g_prof_open[stage].b = prof_event();
    cudaEventRecord(g_prof_open[stage].b, s);
    g_prof_done.push_back(g_prof_open[stage]);
  }
}

// defined in the kernel translation units
int render_forward(const Fs4dCloud&, const Fs4dCamera&, const Fs4dRasterConfig&, const RenderLayout&, void*,
                   Fs4dImages&, int32_t*, cudaStream_t);
int render_backward(const Fs4dCloud&, const Fs4dCamera&, const Fs4dRasterConfig&, const RenderLayout&, void*,
                    const Fs4dImageGrads&, Fs4dCloud&, int32_t*, float*, void*, size_t, cudaStream_t);
size_t render_bwd_det_bytes(const RenderLayout&);
int render_export_projected(const RenderLayout&, void*, Fs4dProjected&, cudaStream_t);
int render_export_tiles(const RenderLayout&, void*, int32_t*, int32_t*, int64_t, cudaStream_t);
size_t deform_workspace_bytes(const Fs4dDeformNet& net, int64_t K, int* nparts_out);
size_t deform_cache_bytes(const Fs4dDeformNet& net, const Fs4dHexPlane& field, int64_t K);
int deform_forward(const Fs4dCloud&, const Fs4dHexPlane&, const Fs4dDeformNet&, double, Fs4dCloud&, void*, size_t,
                   void*, size_t, cudaStream_t);
int deform_backward(const Fs4dCloud&, const Fs4dHexPlane&, const Fs4dDeformNet&, double, const void*, size_t,
                    const Fs4dCloud&, Fs4dCloud&, Fs4dDeformNet&, Fs4dHexPlane*, int, void*, size_t, int32_t*, void*,
                    size_t, cudaStream_t, cudaEvent_t = nullptr);
size_t deform_backward_det_bytes(const Fs4dDeformNet&, const Fs4dHexPlane&);
int l1_loss_grad(const float*, const float*, const float*, const float*, int, int, int, double, double, float*, float*,
                 double*, cudaStream_t);

size_t photometric_workspace_bytes(int, int);
int photometric_loss_grad(const float*, const float*, const uint8_t*, const float*, const float*, const float*, int,
                          int, double, double, float*, float*, double*, double*, void*, cudaStream_t);
int l1(const float*, const float*, int64_t, double, float*, double*, cudaStream_t);
int adam_step(float*, const float*, float*, float*, int32_t*, const Fs4dAdamSegment*, int, const int32_t*, int32_t*,
              cudaStream_t);
int hexplane_query(const Fs4dHexPlane&, const float*, int64_t, double, float*, cudaStream_t);
int sum_buffers(float*, const float* const*, int, int64_t, int, cudaStream_t);
size_t linear_backward_workspace_bytes(int64_t, int, int);
int linear_forward(const float*, int64_t, const Fs4dLinear&, float*, float*, cudaStream_t);
int linear_backward(const float*, const float*, int64_t, const Fs4dLinear&, const float*, float*, float*, float*, int,
                    void*, cudaStream_t);
int render_tile_alphas(const RenderLayout&, void*, const int32_t*, int64_t, int, int, int, int, float, float, float*,
                       float*, float*, cudaStream_t);
int composite_weights(const float*, int64_t, int64_t, float, float*, uint8_t*, float*, float*, cudaStream_t);
int hexplane_query_backward(const Fs4dHexPlane&, const float*, int64_t, double, const float*, Fs4dHexPlane&, float*, int,
                            cudaStream_t);
int tv_loss_grad(const Fs4dHexPlane&, Fs4dHexPlane*, double, int, double*, cudaStream_t);
int resize_bilinear(const float*, int, int, int, float*, int, int, cudaStream_t);
size_t resize_workspace_bytes(int, int, int);
int resize_bilinear_backward(const float*, int, int, int, float*, int, int, float*, cudaStream_t);
size_t decoder_workspace_bytes(int, int, int, int, int, int);
int decode_features(const float*, int, int, int, const float*, const float*, int, int, int, float*, float*,
                    cudaStream_t);
int decode_features_backward(const float*, const float*, const float*, int, int, int, int, int, int, float*, float*,
                             float*, int, void*, size_t, cudaStream_t);
int decoder_feature_loss(const float*, int, int, int, const float*, const float*, int, const float*, int, int, double,
                         float*, float*, float*, int, double*, void*, size_t, cudaStream_t);

size_t density_workspace_bytes(int64_t, int64_t);
int stats_add(double*, double*, const int32_t*, const float*, int64_t, const int32_t*, cudaStream_t);
int density_classify(const Fs4dCloud&, const double*, const double*, const Fs4dDensityConfig&, int, int64_t,
                     int32_t*, void*, size_t, int32_t*, cudaStream_t);
int density_apply(const Fs4dCloud&, const double*, const Fs4dDensityConfig&, int64_t, int32_t, int32_t, int32_t,
                  Fs4dCloud&, const double*, const double*, double*, double*, int, int, const float* const*,
                  float* const*, const int32_t*, void*, size_t, int32_t*, cudaStream_t);
int reset_opacity(float*, int64_t, double, cudaStream_t);

size_t locality_order_workspace_bytes(int64_t);
int locality_order(const float*, int64_t, const double*, int32_t*, void*, size_t, cudaStream_t);

static int check_cloud(const Fs4dCloud* c, bool need_colors) {
  if (!c) return fail(FS4D_ERR_CONFIG, "null cloud");
  if (c->K < 0 || c->K > 0x7FFFFFFF) return fail(FS4D_ERR_CONFIG, "cloud size out of range");
  if (c->D < 0) return fail(FS4D_ERR_CONFIG, "negative feature dimension");
  if (c->sh_degree < 0 || c->sh_degree > 3) return fail(FS4D_ERR_CONFIG, "sh_degree must be in [0, 3]");
  if (c->K > 0) {
    if (!c->positions || !c->rotations || !c->log_scales || !c->opacity_logits)
      return fail(FS4D_ERR_CONFIG, "cloud pointer missing");
    if (need_colors && !c->colors_raw) return fail(FS4D_ERR_CONFIG, "cloud colors missing");
    if (c->D > 0 && !c->features) return fail(FS4D_ERR_CONFIG, "cloud features missing");
    if (c->sh_degree > 0 && !c->sh_rest) return fail(FS4D_ERR_CONFIG, "sh_rest missing for sh_degree > 0");
  }
  return FS4D_OK;
}

static int check_camera(const Fs4dCamera* cam) {
  if (!cam) return fail(FS4D_ERR_CONFIG, "null camera");
  if (cam->height <= 0 || cam->width <= 0) return fail(FS4D_ERR_DATA, "image size must be positive");
  if (!(cam->K[0] > 0) || !(cam->K[4] > 0)) return fail(FS4D_ERR_DATA, "intrinsics must have positive focal lengths");
  // rasterizer.py:128-130
  if (cam->K[1] > 1e-9 || cam->K[1] < -1e-9) return fail(FS4D_ERR_DATA, "intrinsics with skew are not supported");
  return FS4D_OK;
}

static int check_record(const Fs4dRecordInfo* info, const Fs4dCloud* snap, const Fs4dCamera* cam,
                        const Fs4dRasterConfig* cfg, size_t ws_bytes, const void* ws) {
  if (!info || !cfg) return fail(FS4D_ERR_CONFIG, "null record info / config");
  if (cfg->tile != kTile) return fail(FS4D_ERR_CONFIG, "only tile = 16 is implemented on device");
  if (info->pair_capacity < 0) return fail(FS4D_ERR_CONFIG, "negative pair capacity");
  if (info->pair_capacity > 0x7FFFFFFFll) return fail(FS4D_ERR_CONFIG, "pair capacity above 2^31");
  // rasterizer.py:330-331 (stale record)
  if (snap && info->K != snap->K) return fail(FS4D_ERR_CONTRACT, "record does not match this snapshot/frame");
  if (cam && (info->height != cam->height || info->width != cam->width))
    return fail(FS4D_ERR_CONTRACT, "record does not match this snapshot/frame");
  if (snap && info->D != snap->D) return fail(FS4D_ERR_CONTRACT, "record feature dimension mismatch");
  RenderLayout L = make_layout(*info);
  if (!ws || ws_bytes < L.total) return fail(FS4D_ERR_CONFIG, "render workspace too small");
  return FS4D_OK;
}

__global__ void k_status_reset(int32_t* st) {
  int i = threadIdx.x;
  if (i < FS4D_STATUS_WORDS)
    st[i] = (i >= FS4D_ST_BAD_INDEX && i <= FS4D_ST_ADAM_BAD_SEG) ? 0x7FFFFFFF : 0;
}

// One thread: fold a finished call's status block into an accumulating one
// (stream-ordered after the call, so no host sync).  The first error wins;
// repeated capacity overflows keep the largest pair count; gate_adam makes
// a later fs4d_adam_step on `dst` a no-op.
__global__ void k_status_merge(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int gate_adam) {
  const int code = src[FS4D_ST_CODE];
  if (code == FS4D_OK) return;
  if (dst[FS4D_ST_CODE] == FS4D_OK) {
    for (int i = 0; i < FS4D_ST_ADAM_BAD_SEG; ++i) dst[i] = src[i];
  } else if (code == FS4D_ERR_CAPACITY && dst[FS4D_ST_CODE] == FS4D_ERR_CAPACITY) {
    const unsigned long long a = ((unsigned long long)(unsigned)src[FS4D_ST_PAIRS_HI] << 32) |
                                 (unsigned)src[FS4D_ST_PAIRS_LO];
    const unsigned long long b = ((unsigned long long)(unsigned)dst[FS4D_ST_PAIRS_HI] << 32) |
                                 (unsigned)dst[FS4D_ST_PAIRS_LO];
    if (a > b) {
      dst[FS4D_ST_PAIRS_LO] = src[FS4D_ST_PAIRS_LO];
      dst[FS4D_ST_PAIRS_HI] = src[FS4D_ST_PAIRS_HI];
    }
  }
  if (gate_adam) dst[FS4D_ST_ADAM_BAD_SEG] = FS4D_ADAM_GATED;
}

}  // namespace fs4d

using namespace fs4d;

extern "C" {

int fs4d_abi_version(void) { return FS4D_ABI_VERSION; }

const char* fs4d_last_error(void) { return g_last_error.c_str(); }

#ifndef FS4D_SOURCE_HASH
#define FS4D_SOURCE_HASH "unknown"
#endif
const char* fs4d_build_info(void) {
  static char buf[256];
  snprintf(buf, sizeof(buf), "libfs4d abi=%d arch=sm_100a cuda=%d.%d src=%s", FS4D_ABI_VERSION, CUDART_VERSION / 1000,
           (CUDART_VERSION % 1000) / 10, FS4D_SOURCE_HASH);
  return buf;
}

int fs4d_profile_enable(int on) {
  g_prof_on = on != 0;
  return FS4D_OK;
}

int fs4d_profile_collect(double* ms_total, int64_t* calls, int32_t n_stages) {
  for (int i = 0; i < n_stages; ++i) {
    if (ms_total) ms_total[i] = 0.0;
    if (calls) calls[i] = 0;
  }
  for (const ProfRec& r : g_prof_done) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (r.stage < n_stages) {
      if (ms_total) ms_total[r.stage] += ms;
      if (calls) calls[r.stage] += 1;
    }
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_done.clear();
  return check_launch("profile_collect");
}

int fs4d_status_reset(int32_t* status, void* stream) {
  if (!status) return fail(FS4D_ERR_CONFIG, "null status block");
  k_status_reset<<<1, FS4D_STATUS_WORDS, 0, (cudaStream_t)stream>>>(status);
  return check_launch("status_reset");
}

int fs4d_status_merge(const int32_t* src, int32_t* dst, int32_t gate_adam, void* stream) {
  if (!src || !dst) return fail(FS4D_ERR_CONFIG, "null status block");
  k_status_merge<<<1, 1, 0, (cudaStream_t)stream>>>(src, dst, gate_adam);
  return check_launch("status_merge");
}

size_t fs4d_deform_workspace_bytes(const Fs4dDeformNet* net, int64_t K) {
  if (!net) return 0;
  return deform_workspace_bytes(*net, K, nullptr);
}

size_t fs4d_deform_cache_bytes(const Fs4dDeformNet* net, const Fs4dHexPlane* field, int64_t K) {
  if (!net || !field || K < 0) return 0;
  return deform_cache_bytes(*net, *field, K);
}

int fs4d_deform_fwd(const Fs4dCloud* cloud, const Fs4dHexPlane* field, const Fs4dDeformNet* net, double t,
                    Fs4dCloud* snapshot, void* cache, size_t cache_bytes, void* workspace, size_t workspace_bytes,
                    int32_t* status, void* stream) {
  (void)status;
  int rc = check_cloud(cloud, false);
  if (rc) return rc;
  if (!field || !net || !snapshot) return fail(FS4D_ERR_CONFIG, "null deform argument");
  if (snapshot->K != cloud->K) return fail(FS4D_ERR_CONFIG, "snapshot size mismatch");
  return deform_forward(*cloud, *field, *net, t, *snapshot, cache, cache_bytes, workspace, workspace_bytes,
                        (cudaStream_t)stream);
}

int fs4d_deform_bwd(const Fs4dCloud* cloud, const Fs4dHexPlane* field, const Fs4dDeformNet* net, double t,
                    const void* cache, size_t cache_bytes, const Fs4dCloud* snapshot_grads, Fs4dCloud* cloud_grads,
                    Fs4dDeformNet* net_grads, Fs4dHexPlane* plane_grads, int32_t accumulate, void* workspace,
                    size_t workspace_bytes, int32_t* status, void* stream) {
  int rc = check_cloud(cloud, false);
  if (rc) return rc;
  if (!field || !net || !snapshot_grads || !cloud_grads || !net_grads)
    return fail(FS4D_ERR_CONFIG, "null deform_bwd argument");
  if (snapshot_grads->K != cloud->K || cloud_grads->K != cloud->K)
    return fail(FS4D_ERR_CONTRACT, "gradient rows do not match the cloud");
  return deform_backward(*cloud, *field, *net, t, cache, cache_bytes, *snapshot_grads, *cloud_grads, *net_grads,
                         plane_grads, accumulate, workspace, workspace_bytes, status, nullptr, 0,
                         (cudaStream_t)stream);
}

int fs4d_deform_bwd_deterministic(const Fs4dCloud* cloud, const Fs4dHexPlane* field, const Fs4dDeformNet* net, double t,
                    const void* cache, size_t cache_bytes, const Fs4dCloud* snapshot_grads, Fs4dCloud* cloud_grads,
                    Fs4dDeformNet* net_grads, Fs4dHexPlane* plane_grads, int32_t accumulate, void* workspace,
                    size_t workspace_bytes, void* det_workspace, size_t det_workspace_bytes,
                                   int32_t* status, void* stream) {
  if (!det_workspace) return fail(FS4D_ERR_CONFIG, "null deterministic workspace");
  int rc = check_cloud(cloud, false);
  if (rc) return rc;
  if (!field || !net || !snapshot_grads || !cloud_grads || !net_grads)
    return fail(FS4D_ERR_CONFIG, "null deform_bwd argument");
  if (snapshot_grads->K != cloud->K || cloud_grads->K != cloud->K)
    return fail(FS4D_ERR_CONTRACT, "gradient rows do not match the cloud");
  return deform_backward(*cloud, *field, *net, t, cache, cache_bytes, *snapshot_grads, *cloud_grads, *net_grads,
                         plane_grads, accumulate, workspace, workspace_bytes, status, det_workspace,
                         det_workspace_bytes, (cudaStream_t)stream);
}

int fs4d_deform_bwd_split(const Fs4dCloud* cloud, const Fs4dHexPlane* field, const Fs4dDeformNet* net, double t,
                          const void* cache, size_t cache_bytes, const Fs4dCloud* snapshot_grads,
                          Fs4dCloud* cloud_grads, Fs4dDeformNet* net_grads, Fs4dHexPlane* plane_grads,
                          int32_t accumulate, void* workspace, size_t workspace_bytes, void* det_workspace,
                          size_t det_workspace_bytes, void* passthrough_event, int32_t* status, void* stream) {
  int rc = check_cloud(cloud, false);
  if (rc) return rc;
  if (!field || !net || !snapshot_grads || !cloud_grads || !net_grads)
    return fail(FS4D_ERR_CONFIG, "null deform_bwd argument");
  if (snapshot_grads->K != cloud->K || cloud_grads->K != cloud->K)
    return fail(FS4D_ERR_CONTRACT, "gradient rows do not match the cloud");
  return deform_backward(*cloud, *field, *net, t, cache, cache_bytes, *snapshot_grads, *cloud_grads, *net_grads,
                         plane_grads, accumulate, workspace, workspace_bytes, status, det_workspace,
                         det_workspace ? det_workspace_bytes : 0, (cudaStream_t)stream,
                         (cudaEvent_t)passthrough_event);
}

size_t fs4d_deform_bwd_det_workspace_bytes(const Fs4dDeformNet* net, const Fs4dHexPlane* field) {
  if (!net || !field) return 0;
  return deform_backward_det_bytes(*net, *field);
}

int fs4d_sum_buffers(float* dst, const float* const* srcs, int32_t n_src, int64_t n, int32_t accumulate,
                     void* stream) {
  if (!dst || n < 0 || n_src < 0 || (n_src > 0 && !srcs)) return fail(FS4D_ERR_CONFIG, "bad sum_buffers arguments");
  for (int j = 0; j < n_src; ++j)
    if (!srcs[j]) return fail(FS4D_ERR_CONFIG, "null sum_buffers source");
  return sum_buffers(dst, srcs, n_src, n, accumulate, (cudaStream_t)stream);
}

int fs4d_hexplane_query(const Fs4dHexPlane* field, const float* positions, int64_t K, double t, float* latent,
                        void* stream) {
  if (!field || K < 0 || (K > 0 && (!positions || !latent))) return fail(FS4D_ERR_CONFIG, "bad hexplane_query arguments");
  return hexplane_query(*field, positions, K, t, latent, (cudaStream_t)stream);
}

int fs4d_hexplane_query_backward(const Fs4dHexPlane* field, const float* positions, int64_t K, double t,
                                 const float* d_latent, Fs4dHexPlane* plane_grads, float* d_positions,
                                 int32_t accumulate, void* stream) {
  if (!field || !plane_grads || K < 0 || (K > 0 && (!positions || !d_latent || !d_positions)))
    return fail(FS4D_ERR_CONFIG, "bad hexplane_query_backward arguments");
  return hexplane_query_backward(*field, positions, K, t, d_latent, *plane_grads, d_positions, accumulate,
                                 (cudaStream_t)stream);
}

int fs4d_l1_loss_grad(const float* color, const float* color_target, const float* feature,
                      const float* feature_target, int32_t height, int32_t width, int32_t D, double w_rgb,
                      double w_feat, float* d_color, float* d_feature, double* loss, void* stream) {
  if (!color || !color_target || !d_color || height <= 0 || width <= 0 || D < 0)
    return fail(FS4D_ERR_CONFIG, "bad l1 loss arguments");
  if (D > 0 && (!feature || !feature_target || !d_feature)) return fail(FS4D_ERR_CONFIG, "feature buffers missing");
  return l1_loss_grad(color, color_target, feature, feature_target, height, width, D, w_rgb, w_feat, d_color,
                      d_feature, loss, (cudaStream_t)stream);
}

size_t fs4d_photometric_workspace_bytes(int32_t height, int32_t width) {
  return photometric_workspace_bytes(height, width);
}

int fs4d_photometric_loss_grad(const float* color, const float* image, const uint8_t* mask, const float* depth,
                               const float* depth_target, const float* alpha, int32_t height, int32_t width,
                               double lambda_rgb, double lambda_depth, float* d_color, float* d_depth, double* terms,
                               double* loss, void* workspace, size_t workspace_bytes, void* stream) {
  if (!color || !image || !d_color || height <= 0 || width <= 0)
    return fail(FS4D_ERR_CONFIG, "bad photometric loss arguments");
  const bool with_depth = depth != nullptr;
  if (with_depth && (!depth_target || !alpha || !d_depth))
    return fail(FS4D_ERR_CONFIG, "depth term needs depth, depth_target, alpha and d_depth");
  if (!workspace || workspace_bytes < photometric_workspace_bytes(height, width))
    return fail(FS4D_ERR_CONFIG, "photometric workspace too small");
  return photometric_loss_grad(color, image, mask, depth, depth_target, alpha, height, width, lambda_rgb,
                               lambda_depth, d_color, with_depth ? d_depth : nullptr, terms, loss, workspace,
                               (cudaStream_t)stream);
}

int fs4d_l1(const float* pred, const float* target, int64_t n, double scale, float* grad, double* loss,
            void* stream) {
  if (n < 0 || (n > 0 && (!pred || !target))) return fail(FS4D_ERR_CONFIG, "bad l1 arguments");
  return l1(pred, target, n, scale, grad, loss, (cudaStream_t)stream);
}

int fs4d_adam_step_masked(float* params, const float* grads, float* m, float* v, int32_t* step_counts,
                          const Fs4dAdamSegment* segments, const int32_t* active, int32_t n_segments,
                          int32_t* status, void* stream) {
  if (n_segments < 0 || n_segments > FS4D_MAX_ADAM_SEGMENTS)
    return fail(FS4D_ERR_CONFIG, "adam segment count out of range");
  if (n_segments == 0) return FS4D_OK;
  if (!params || !grads || !m || !v || !step_counts || !segments || !status)
    return fail(FS4D_ERR_CONFIG, "null adam argument");
  for (int i = 0; i < n_segments; ++i) {
    if (active && !active[i]) continue;
    const Fs4dAdamSegment& g = segments[i];
    // numerics.py:143-144: a non-positive learning rate is a configuration error
    if (!(g.lr > 0.0)) return fail(FS4D_ERR_CONFIG, "learning rate must be positive, got " + std::to_string(g.lr));
    if (g.offset < 0 || g.count < 0) return fail(FS4D_ERR_CONFIG, "bad adam segment bounds");
    if (!(g.beta1 >= 0.0 && g.beta1 < 1.0) || !(g.beta2 >= 0.0 && g.beta2 < 1.0) || !(g.eps >= 0.0))
      return fail(FS4D_ERR_CONFIG, "bad adam hyper-parameters");
  }
  return adam_step(params, grads, m, v, step_counts, segments, n_segments, active, status, (cudaStream_t)stream);
}

int fs4d_adam_step(float* params, const float* grads, float* m, float* v, int32_t* step_counts,
                   const Fs4dAdamSegment* segments, int32_t n_segments, int32_t* status, void* stream) {
  return fs4d_adam_step_masked(params, grads, m, v, step_counts, segments, nullptr, n_segments, status, stream);
}

static int check_field(const Fs4dHexPlane* f) {
  if (!f) return fail(FS4D_ERR_CONFIG, "null field");
  if (f->levels < 0 || f->levels > FS4D_MAX_LEVELS || f->channels <= 0)
    return fail(FS4D_ERR_CONFIG, "bad field levels / channels");
  for (int l = 0; l < f->levels; ++l)
    for (int q = 0; q < 6; ++q)
      if (!f->planes[l][q] || f->res[l][q][0] < 1 || f->res[l][q][1] < 1)
        return fail(FS4D_ERR_CONFIG, "bad plane pointer / resolution");
  return FS4D_OK;
}

int fs4d_tv_loss_grad(const Fs4dHexPlane* field, Fs4dHexPlane* grads, double scale, int32_t accumulate, double* loss,
                      void* stream) {
  if (int rc = check_field(field)) return rc;
  if (grads) {
    if (grads->levels != field->levels) return fail(FS4D_ERR_CONFIG, "gradient field level mismatch");
    for (int l = 0; l < field->levels; ++l)
      for (int q = 0; q < 6; ++q)
        if (!grads->planes[l][q]) return fail(FS4D_ERR_CONFIG, "null plane gradient");
  }
  return tv_loss_grad(*field, grads, scale, accumulate, loss, (cudaStream_t)stream);
}

int fs4d_resize_bilinear(const float* in, int32_t hi, int32_t wi, int32_t C, float* out, int32_t ho, int32_t wo,
                         void* stream) {
  if (hi <= 0 || wi <= 0 || C <= 0 || ho <= 0 || wo <= 0 || !in || !out)
    return fail(FS4D_ERR_CONFIG, "bad resize arguments");
  return resize_bilinear(in, hi, wi, C, out, ho, wo, (cudaStream_t)stream);
}

size_t fs4d_resize_workspace_bytes(int32_t ho, int32_t wi, int32_t C) { return resize_workspace_bytes(ho, wi, C); }

int fs4d_resize_bilinear_backward(const float* d_out, int32_t ho, int32_t wo, int32_t C, float* d_in, int32_t hi,
                                  int32_t wi, void* workspace, size_t workspace_bytes, void* stream) {
  if (hi <= 0 || wi <= 0 || C <= 0 || ho <= 0 || wo <= 0 || !d_out || !d_in)
    return fail(FS4D_ERR_CONFIG, "bad resize arguments");
  if (!workspace || workspace_bytes < resize_workspace_bytes(ho, wi, C))
    return fail(FS4D_ERR_CONFIG, "resize workspace too small");
  return resize_bilinear_backward(d_out, ho, wo, C, d_in, hi, wi, (float*)workspace, (cudaStream_t)stream);
}

size_t fs4d_decoder_workspace_bytes(int32_t hi, int32_t wi, int32_t N, int32_t ho, int32_t wo, int32_t Ct) {
  return decoder_workspace_bytes(hi, wi, N, ho, wo, Ct);
}

int fs4d_decode_features(const float* rendered, int32_t hi, int32_t wi, int32_t N, const float* weight,
                         const float* bias, int32_t Ct, int32_t ho, int32_t wo, float* out, float* resized,
                         void* stream) {
  if (!rendered || !weight || !bias || !out) return fail(FS4D_ERR_CONFIG, "null decoder argument");
  return decode_features(rendered, hi, wi, N, weight, bias, Ct, ho, wo, out, resized, (cudaStream_t)stream);
}

int fs4d_decode_features_backward(const float* d_out, const float* resized, const float* weight, int32_t hi,
                                  int32_t wi, int32_t N, int32_t Ct, int32_t ho, int32_t wo, float* d_rendered,
                                  float* d_weight, float* d_bias, int32_t accumulate, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (!d_out || !resized || !weight || !d_rendered || !d_weight || !d_bias)
    return fail(FS4D_ERR_CONFIG, "null decoder backward argument");
  return decode_features_backward(d_out, resized, weight, hi, wi, N, Ct, ho, wo, d_rendered, d_weight, d_bias,
                                  accumulate, workspace, workspace_bytes, (cudaStream_t)stream);
}

int fs4d_decoder_feature_loss(const float* rendered, int32_t hi, int32_t wi, int32_t N, const float* weight,
                              const float* bias, int32_t Ct, const float* teacher, int32_t ho, int32_t wo,
                              double lambda, float* d_rendered, float* d_weight, float* d_bias, int32_t accumulate,
                              double* loss, void* workspace, size_t workspace_bytes, void* stream) {
  if (!rendered || !weight || !bias || !teacher || !d_rendered || !d_weight || !d_bias)
    return fail(FS4D_ERR_CONFIG, "null decoder loss argument");
  return decoder_feature_loss(rendered, hi, wi, N, weight, bias, Ct, teacher, ho, wo, lambda, d_rendered, d_weight,
                              d_bias, accumulate, loss, workspace, workspace_bytes, (cudaStream_t)stream);
}

int fs4d_grad_stats_add(double* accum, double* count, const int32_t* indices, const float* norms, int64_t n,
                        const int32_t* n_dev, void* stream) {
  if (n < 0 || (n > 0 && (!accum || !count || !norms))) return fail(FS4D_ERR_CONFIG, "bad stats arguments");
  return stats_add(accum, count, indices, norms, n, n_dev, (cudaStream_t)stream);
}

size_t fs4d_density_workspace_bytes(int64_t K, int64_t capacity) {
  if (K < 0 || capacity < 0) return 0;
  return density_workspace_bytes(K, capacity);
}

static int check_density_cfg(const Fs4dDensityConfig* cfg) {
  if (!cfg) return fail(FS4D_ERR_CONFIG, "null density config");
  if (!(cfg->split_factor > 0.0) || !(cfg->extent >= 0.0)) return fail(FS4D_ERR_CONFIG, "bad density config");
  return FS4D_OK;
}

int fs4d_density_classify(const Fs4dCloud* cloud, const double* accum, const double* count,
                          const Fs4dDensityConfig* cfg, int32_t prune_only, int64_t capacity, int32_t* counts,
                          void* workspace, size_t workspace_bytes, int32_t* status, void* stream) {
  if (int rc = check_cloud(cloud, true)) return rc;
  if (int rc = check_density_cfg(cfg)) return rc;
  if (cloud->K > 0 && (!accum || !count) && !prune_only) return fail(FS4D_ERR_CONFIG, "grad stats missing");
  if (capacity > 0x7FFFFFFFll) return fail(FS4D_ERR_CONFIG, "density capacity above 2^31");
  if (!status) return fail(FS4D_ERR_CONFIG, "null status block");
  return density_classify(*cloud, accum, count, *cfg, prune_only, capacity, counts, workspace, workspace_bytes,
                          status, (cudaStream_t)stream);
}

int fs4d_density_apply(const Fs4dCloud* cloud, const double* split_normals, const Fs4dDensityConfig* cfg,
                       int64_t capacity, int32_t n_keep, int32_t n_clone, int32_t n_split, Fs4dCloud* out,
                       const double* stats_accum_in, const double* stats_count_in, double* stats_accum_out,
                       double* stats_count_out, int32_t stats_reset, int32_t n_extra, const float* const* extra_in,
                       float* const* extra_out, const int32_t* extra_width, void* workspace, size_t workspace_bytes,
                       int32_t* status, void* stream) {
  if (int rc = check_cloud(cloud, true)) return rc;
  if (int rc = check_cloud(out, true)) return rc;
  if (int rc = check_density_cfg(cfg)) return rc;
  if (out->D != cloud->D || out->sh_degree != cloud->sh_degree) return fail(FS4D_ERR_CONFIG, "output cloud shape");
  if (n_keep < 0 || n_clone < 0 || n_split < 0) return fail(FS4D_ERR_CONFIG, "negative density counts");
  if (stats_accum_out && (!stats_count_out || (!stats_reset && (!stats_accum_in || !stats_count_in))))
    return fail(FS4D_ERR_CONFIG, "grad stats arrays missing");
  if (n_extra > 0 && (!extra_in || !extra_out || !extra_width)) return fail(FS4D_ERR_CONFIG, "extra arrays missing");
  return density_apply(*cloud, split_normals, *cfg, capacity, n_keep, n_clone, n_split, *out, stats_accum_in,
                       stats_count_in, stats_accum_out, stats_count_out, stats_reset, n_extra, extra_in, extra_out,
                       extra_width, workspace, workspace_bytes, status, (cudaStream_t)stream);
}

int fs4d_reset_opacity(float* opacity_logits, int64_t K, double cap, void* stream) {
  if (!(cap > 0.0 && cap < 1.0)) return fail(FS4D_ERR_CONFIG, "opacity cap must lie in (0, 1)");
  if (K < 0 || (K > 0 && !opacity_logits)) return fail(FS4D_ERR_CONFIG, "bad reset_opacity arguments");
  return reset_opacity(opacity_logits, K, cap, (cudaStream_t)stream);
}

size_t fs4d_locality_order_workspace_bytes(int64_t K) { return K < 0 ? 0 : locality_order_workspace_bytes(K); }

int fs4d_locality_order(const float* positions, int64_t K, const double* aabb, int32_t* order, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (K < 0 || K > 0x7FFFFFFF || !aabb || (K > 0 && (!positions || !order)))
    return fail(FS4D_ERR_CONFIG, "bad locality order arguments");
  return locality_order(positions, K, aabb, order, workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t fs4d_render_workspace_bytes(const Fs4dRecordInfo* info) {
  if (!info) return 0;
  return make_layout(*info).total;
}

int fs4d_render_fwd(const Fs4dCloud* snapshot, const Fs4dCamera* cam, const Fs4dRasterConfig* cfg,
                    const Fs4dRecordInfo* info, void* workspace, size_t workspace_bytes, Fs4dImages* out,
                    int32_t* status, void* stream) {
  int rc = check_cloud(snapshot, true);
  if (rc) return rc;
  if ((rc = check_camera(cam))) return rc;
  if ((rc = check_record(info, snapshot, cam, cfg, workspace_bytes, workspace))) return rc;
  if (!out || !out->color || !out->depth || !out->alpha) return fail(FS4D_ERR_CONFIG, "null output image");
  if (cfg->with_features && snapshot->D > 0 && !out->feature) return fail(FS4D_ERR_CONFIG, "null feature image");
  RenderLayout L = make_layout(*info);
  return render_forward(*snapshot, *cam, *cfg, L, workspace, *out, status, (cudaStream_t)stream);
}

int fs4d_render_bwd(const Fs4dCloud* snapshot, const Fs4dCamera* cam, const Fs4dRasterConfig* cfg,
                    const Fs4dRecordInfo* info, void* workspace, size_t workspace_bytes,
                    const Fs4dImageGrads* upstream, Fs4dCloud* grads, int32_t* viewspace_index,
                    float* viewspace_norm, int32_t* status, void* stream) {
  (void)status;
  int rc = check_cloud(snapshot, true);
  if (rc) return rc;
  if ((rc = check_camera(cam))) return rc;
  if ((rc = check_record(info, snapshot, cam, cfg, workspace_bytes, workspace))) return rc;
  if (!upstream || !grads) return fail(FS4D_ERR_CONFIG, "null backward argument");
  if (viewspace_index && !viewspace_norm) return fail(FS4D_ERR_CONFIG, "viewspace_index without viewspace_norm");
  if (grads->K != snapshot->K || grads->D != snapshot->D || grads->sh_degree != snapshot->sh_degree)
    return fail(FS4D_ERR_CONFIG, "gradient buffers do not match the snapshot");
  if (cfg->with_features && snapshot->D > 64)
    return fail(FS4D_ERR_CONFIG, "render backward supports at most 64 feature channels");
  RenderLayout L = make_layout(*info);
  return render_backward(*snapshot, *cam, *cfg, L, workspace, *upstream, *grads, viewspace_index, viewspace_norm,
                         nullptr, 0, (cudaStream_t)stream);
}

int fs4d_render_bwd_deterministic(const Fs4dCloud* snapshot, const Fs4dCamera* cam, const Fs4dRasterConfig* cfg,
                    const Fs4dRecordInfo* info, void* workspace, size_t workspace_bytes,
                    const Fs4dImageGrads* upstream, Fs4dCloud* grads, int32_t* viewspace_index,
                    float* viewspace_norm, void* det_workspace, size_t det_workspace_bytes,
                                   int32_t* status, void* stream) {
  (void)status;
  int rc = check_cloud(snapshot, true);
  if (rc) return rc;
  if ((rc = check_camera(cam))) return rc;
  if ((rc = check_record(info, snapshot, cam, cfg, workspace_bytes, workspace))) return rc;
  if (!upstream || !grads) return fail(FS4D_ERR_CONFIG, "null backward argument");
  if (viewspace_index && !viewspace_norm) return fail(FS4D_ERR_CONFIG, "viewspace_index without viewspace_norm");
  if (grads->K != snapshot->K || grads->D != snapshot->D || grads->sh_degree != snapshot->sh_degree)
    return fail(FS4D_ERR_CONFIG, "gradient buffers do not match the snapshot");
  if (cfg->with_features && snapshot->D > 64)
    return fail(FS4D_ERR_CONFIG, "render backward supports at most 64 feature channels");
  RenderLayout L = make_layout(*info);
  if (!det_workspace) return fail(FS4D_ERR_CONFIG, "null deterministic workspace");
  return render_backward(*snapshot, *cam, *cfg, L, workspace, *upstream, *grads, viewspace_index, viewspace_norm,
                         det_workspace, det_workspace_bytes, (cudaStream_t)stream);
}

size_t fs4d_render_bwd_det_workspace_bytes(const Fs4dRecordInfo* info) {
  if (!info) return 0;
  return render_bwd_det_bytes(make_layout(*info));
}


int fs4d_render_export_projected(const Fs4dRecordInfo* info, const void* workspace, size_t workspace_bytes,
                                 Fs4dProjected* out, void* stream) {
  if (!info || !out) return fail(FS4D_ERR_CONFIG, "null export argument");
  RenderLayout L = make_layout(*info);
  if (!workspace || workspace_bytes < L.total) return fail(FS4D_ERR_CONFIG, "render workspace too small");
  return render_export_projected(L, const_cast<void*>(workspace), *out, (cudaStream_t)stream);
}

static int check_linear(const Fs4dLinear* L) {
  if (!L || !L->weight || !L->bias || L->in_dim <= 0 || L->out_dim <= 0)
    return fail(FS4D_ERR_CONFIG, "bad linear layer");
  return FS4D_OK;
}

int fs4d_linear_forward(const float* x, int64_t batch, const Fs4dLinear* layer, float* pre, float* y, void* stream) {
  int rc = check_linear(layer);
  if (rc) return rc;
  if (batch < 0 || (batch > 0 && (!x || !pre || !y))) return fail(FS4D_ERR_CONFIG, "bad linear_forward arguments");
  return linear_forward(x, batch, *layer, pre, y, (cudaStream_t)stream);
}

size_t fs4d_linear_backward_workspace_bytes(int64_t batch, int32_t in_dim, int32_t out_dim) {
  if (batch < 0 || in_dim <= 0 || out_dim <= 0) return 0;
  return linear_backward_workspace_bytes(batch, in_dim, out_dim);
}

int fs4d_linear_backward(const float* x, const float* pre, int64_t batch, const Fs4dLinear* layer, const float* dy,
                         float* dx, float* d_weight, float* d_bias, int32_t accumulate, void* workspace,
                         size_t workspace_bytes, void* stream) {
  int rc = check_linear(layer);
  if (rc) return rc;
  if (batch < 0 || !d_weight || !d_bias || (batch > 0 && (!x || !pre || !dy)))
    return fail(FS4D_ERR_CONFIG, "bad linear_backward arguments");
  if (!workspace || workspace_bytes < linear_backward_workspace_bytes(batch, layer->in_dim, layer->out_dim))
    return fail(FS4D_ERR_CONFIG, "linear_backward workspace too small");
  return linear_backward(x, pre, batch, *layer, dy, dx, d_weight, d_bias, accumulate, workspace, (cudaStream_t)stream);
}

int fs4d_render_tile_alphas(const Fs4dRecordInfo* info, const void* workspace, size_t workspace_bytes,
                            const Fs4dRasterConfig* cfg, const int32_t* source_index, int64_t G, int32_t x0,
                            int32_t y0, int32_t nx, int32_t ny, float* alpha, float* g2d, float* a_raw, void* stream) {
  if (!info || !cfg) return fail(FS4D_ERR_CONFIG, "null tile_alphas argument");
  RenderLayout L = make_layout(*info);
  if (!workspace || workspace_bytes < L.total) return fail(FS4D_ERR_CONFIG, "render workspace too small");
  if (G < 0 || nx < 0 || ny < 0 || (G > 0 && (!source_index || !alpha || !g2d || !a_raw)))
    return fail(FS4D_ERR_CONFIG, "bad tile_alphas arguments");
  if (x0 < 0 || y0 < 0 || x0 + nx > L.W || y0 + ny > L.H) return fail(FS4D_ERR_CONFIG, "tile outside the image");
  return render_tile_alphas(L, const_cast<void*>(workspace), source_index, G, x0, y0, nx, ny, (float)cfg->alpha_cap,
                            (float)cfg->alpha_skip, alpha, g2d, a_raw, (cudaStream_t)stream);
}

int fs4d_composite_weights(const float* alpha, int64_t G, int64_t P, double stop, float* t_exc, uint8_t* contrib,
                           float* w, float* t_final, void* stream) {
  if (G < 0 || P < 0 || (P > 0 && !t_final) || (G * P > 0 && (!alpha || !t_exc || !contrib || !w)))
    return fail(FS4D_ERR_CONFIG, "bad composite_weights arguments");
  return composite_weights(alpha, G, P, (float)stop, t_exc, contrib, w, t_final, (cudaStream_t)stream);
}

int fs4d_render_export_tiles(const Fs4dRecordInfo* info, const void* workspace, size_t workspace_bytes,
                             int32_t* tile_ranges, int32_t* pair_rows, int64_t max_pairs, void* stream) {
  if (!info) return fail(FS4D_ERR_CONFIG, "null export argument");
  RenderLayout L = make_layout(*info);
  if (!workspace || workspace_bytes < L.total) return fail(FS4D_ERR_CONFIG, "render workspace too small");
  return render_export_tiles(L, const_cast<void*>(workspace), tile_ranges, pair_rows, max_pairs, (cudaStream_t)stream);
}

}  // extern "C"
