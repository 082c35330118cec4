// Deformation network on device: HexPlane query + MLP stacks + raw-space deltas.
//
// Reference: deformation.deform_with_cache / deform_backward
// (deformation.py:105-183), hexplane.query_with_cache / query_backward
// (hexplane.py:84-187), numerics.mlp_forward / mlp_backward (numerics.py:56-105).
//
// Layout: a persistent CTA walks tiles of TG Gaussians.  Per tile:
//   1. HexPlane gather, one warp per Gaussian, lane = channel: every corner
//      fetch is one coalesced 128 B read of a channel-last plane row
//      (planes are L2-resident: 9.7 MB at the headline config);
//   2. the MLP stacks run as small [TG x in] x [in x out] products on
//      shared-memory activation tiles (channel-major [dim][TG]); weights are
//      pre-transposed/padded once per call into a packed blob so each k-step
//      is one broadcast float4 weight load + one activation load + 4 FMA;
//   3. deltas are added in raw parameter space (deformation.py:126-133).
// The backward pass recomputes the forward tile, back-propagates through the
// stacks, accumulates weight gradients into CTA-private partial buffers
// (reduced by a final kernel — deterministic, no atomics on weights), and
// scatters plane gradients with coalesced red.global.add per corner.
#include "common.cuh"
#include <stdlib.h>
#include <string.h>

namespace fs4d {

constexpr int kMaxLayers = FS4D_MAX_TRUNK + 4 * 2 + 4 + 2;
constexpr int kDefThreads = 256;

struct LayerDesc {
  int in, out, out_pad, relu;
  int64_t off_w, off_b;  // into the packed blob: Wt [in][out_pad], b [out_pad]
  const float* w;        // original [out,in]
  const float* b;
};

struct NetDesc {
  int L, width, half, depth, D, enable_grid, enable_feat;
  int n_layers;
  // layer indices
  int trunk0, ext0 /* ext[b][k] = ext0 + 2*b + k */, head0, feat0;
  LayerDesc layers[kMaxLayers];
  int64_t packed_floats;
  int max_dim;
};

struct FieldDesc {
  int levels, C;
  int res[FS4D_MAX_LEVELS][6][2];
  const float* planes[FS4D_MAX_LEVELS][6];
  float* gplanes[FS4D_MAX_LEVELS][6];
  double lo[3], span[3];
};

__constant__ int c_plane_axes[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};  // hexplane.py:16

__host__ __device__ inline int round4(int x) { return (x + 3) / 4 * 4; }
static inline size_t align_up_sz(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// host: describe / pack the net
// ---------------------------------------------------------------------------
static int build_net_desc(const Fs4dDeformNet& n, NetDesc& d) {
  if (n.depth < 1 || n.depth > FS4D_MAX_TRUNK) return fail(FS4D_ERR_CONFIG, "deformation depth out of range");
  if (n.width <= 0 || (n.width & 1)) return fail(FS4D_ERR_CONFIG, "deformation width must be even");
  d.L = n.latent_dim;
  d.width = n.width;
  d.half = n.width / 2;
  d.depth = n.depth;
  d.D = n.feature_dim;
  d.enable_grid = n.enable_grid;
  d.enable_feat = n.enable_feature_update;
  int k = 0;
  int64_t off = 0;
  int maxd = d.L;
  auto add = [&](const Fs4dLinear& l, int in, int out, int relu) -> int {
    LayerDesc& L = d.layers[k];
    L.in = in;
    L.out = out;
    L.out_pad = round4(out);
    L.relu = relu;
    L.w = l.weight;
    L.b = l.bias;
    L.off_w = off;
    off += (int64_t)in * L.out_pad;
    L.off_b = off;
    off += L.out_pad;
    if (L.out_pad > maxd) maxd = L.out_pad;
    return k++;
  };
  d.trunk0 = 0;
  for (int i = 0; i < n.depth; ++i) add(n.trunk[i], i == 0 ? d.L : d.width, d.width, 1);
  d.ext0 = k;
  for (int b = 0; b < FS4D_N_BRANCHES; ++b) {
    add(n.ext[b][0], d.width, d.half, 1);
    add(n.ext[b][1], d.half, d.half, 1);
  }
  d.head0 = k;
  const int hd[4] = {3, 4, 3, 1};  // deformation.py:20
  for (int b = 0; b < FS4D_N_BRANCHES; ++b) add(n.head[b], d.half, hd[b], 0);
  d.feat0 = k;
  add(n.feat[0], 4 * d.half, d.half, 1);
  add(n.feat[1], d.half, d.D, 0);
  d.n_layers = k;
  d.packed_floats = off;
  d.max_dim = maxd;
  // validate shapes against the struct
  for (int i = 0; i < n.depth; ++i)
    if (n.trunk[i].in_dim != d.layers[i].in || n.trunk[i].out_dim != d.layers[i].out)
      return fail(FS4D_ERR_CONFIG, "trunk layer shape mismatch");
  for (int b = 0; b < 4; ++b) {
    if (n.ext[b][0].in_dim != d.width || n.ext[b][0].out_dim != d.half || n.ext[b][1].in_dim != d.half ||
        n.ext[b][1].out_dim != d.half || n.head[b].in_dim != d.half || n.head[b].out_dim != hd[b])
      return fail(FS4D_ERR_CONFIG, "branch layer shape mismatch");
  }
  if (n.feat[0].in_dim != 4 * d.half || n.feat[0].out_dim != d.half || n.feat[1].in_dim != d.half ||
      n.feat[1].out_dim != d.D)
    return fail(FS4D_ERR_CONFIG, "feature MLP shape mismatch");
  return FS4D_OK;
}

struct PackArgs {
  LayerDesc layers[kMaxLayers];
  int n_layers;
  float* blob;
};

__global__ void k_pack_weights(PackArgs a) {
  const LayerDesc& L = a.layers[blockIdx.y];
  const int64_t n = (int64_t)L.in * L.out_pad + L.out_pad;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < (int64_t)L.in * L.out_pad) {
      int i = (int)(e / L.out_pad), o = (int)(e % L.out_pad);
      a.blob[L.off_w + e] = o < L.out ? L.w[(int64_t)o * L.in + i] : 0.f;
    } else {
      int o = (int)(e - (int64_t)L.in * L.out_pad);
      a.blob[L.off_b + o] = o < L.out ? L.b[o] : 0.f;
    }
  }
}

// ---------------------------------------------------------------------------
// device building blocks
// ---------------------------------------------------------------------------
struct DefArgs {
  int64_t K;
  int TG;
  double t;  // clipped time
  const float* pos;
  const float* rot;
  const float* ls;
  const float* op;
  const float* feat;
  float* o_pos;
  float* o_rot;
  float* o_ls;
  float* o_op;
  float* o_feat;
  // backward
  const float* g_pos;
  const float* g_rot;
  const float* g_ls;
  const float* g_op;
  const float* g_feat;
  float* cg_pos;
  int accumulate;
  float* wpart;  // [gridDim.x][packed_floats] per-CTA weight-gradient partials
  NetDesc net;
  FieldDesc field;
  const float* blob;
};

// y[o][g] = act(b[o] + sum_i W[o][i] x[i][g]) for o < out_pad (padding rows are 0)
__device__ __forceinline__ void dense_fwd(const LayerDesc& L, const float* __restrict__ blob, const float* x, float* y,
                                          int TG) {
  const float* Wt = blob + L.off_w;
  const float* bias = blob + L.off_b;
  const int nob = L.out_pad >> 2;
  for (int idx = threadIdx.x; idx < nob * TG; idx += blockDim.x) {
    const int g = idx % TG, o = (idx / TG) * 4;
    float4 acc = __ldg(reinterpret_cast<const float4*>(bias + o));
    const float* xg = x + g;
    const float* w = Wt + o;
#pragma unroll 4
    for (int i = 0; i < L.in; ++i) {
      const float xv = xg[i * TG];
      const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (int64_t)i * L.out_pad));
      acc.x = fmaf(wv.x, xv, acc.x);
      acc.y = fmaf(wv.y, xv, acc.y);
      acc.z = fmaf(wv.z, xv, acc.z);
      acc.w = fmaf(wv.w, xv, acc.w);
    }
    if (L.relu) {
      acc.x = fmaxf(acc.x, 0.f);
      acc.y = fmaxf(acc.y, 0.f);
      acc.z = fmaxf(acc.z, 0.f);
      acc.w = fmaxf(acc.w, 0.f);
    }
    y[(o + 0) * TG + g] = acc.x;
    y[(o + 1) * TG + g] = acc.y;
    y[(o + 2) * TG + g] = acc.z;
    y[(o + 3) * TG + g] = acc.w;
  }
}

// gx[i][g] (+)= sum_o W[o][i] gy[o][g]   (W^T gy; gy padding rows must be 0)
__device__ __forceinline__ void dense_bwd_x(const LayerDesc& L, const float* __restrict__ blob, const float* gy,
                                            float* gx, int TG, bool accumulate) {
  // one thread = one Gaussian x 4 input channels: 4 independent FMA chains fed
  // by a warp-uniform float4 of the original [out,in] weight row
  if ((L.in & 3) == 0) {
    const int nib = L.in >> 2;
    for (int idx = threadIdx.x; idx < nib * TG; idx += blockDim.x) {
      const int g = idx % TG, i0 = (idx / TG) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (accumulate) acc = make_float4(gx[i0 * TG + g], gx[(i0 + 1) * TG + g], gx[(i0 + 2) * TG + g], gx[(i0 + 3) * TG + g]);
      const float* w = L.w + i0;
      for (int o = 0; o < L.out; ++o) {
        const float gv = gy[o * TG + g];
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (int64_t)o * L.in));
        acc.x = fmaf(wv.x, gv, acc.x);
        acc.y = fmaf(wv.y, gv, acc.y);
        acc.z = fmaf(wv.z, gv, acc.z);
        acc.w = fmaf(wv.w, gv, acc.w);
      }
      gx[i0 * TG + g] = acc.x;
      gx[(i0 + 1) * TG + g] = acc.y;
      gx[(i0 + 2) * TG + g] = acc.z;
      gx[(i0 + 3) * TG + g] = acc.w;
    }
    return;
  }
  const float* Wt = blob + L.off_w;
  for (int idx = threadIdx.x; idx < L.in * TG; idx += blockDim.x) {
    const int g = idx % TG, i = idx / TG;
    const float* w = Wt + (int64_t)i * L.out_pad;
    float acc = accumulate ? gx[i * TG + g] : 0.f;
    for (int o = 0; o < L.out_pad; o += 4) {
      const float4 wv = __ldg(reinterpret_cast<const float4*>(w + o));
      acc = fmaf(wv.x, gy[(o + 0) * TG + g], acc);
      acc = fmaf(wv.y, gy[(o + 1) * TG + g], acc);
      acc = fmaf(wv.z, gy[(o + 2) * TG + g], acc);
      acc = fmaf(wv.w, gy[(o + 3) * TG + g], acc);
    }
    gx[i * TG + g] = acc;
  }
}

// part[Wt][i][o] += sum_g gy[o][g] x[i][g] ; part[b][o] += sum_g gy[o][g]  (ng valid rows)
__device__ __forceinline__ void dense_bwd_w(const LayerDesc& L, float* __restrict__ part, const float* gy,
                                            const float* x, int TG, int ng) {
  float* Wt = part + L.off_w;
  float* bias = part + L.off_b;
  // 4 (out) x 4 (in) register tile per thread: 16 independent accumulators,
  // 8 shared loads per 16 FMA (gy padding rows are zero, x rows >= in masked)
  const int nob = L.out_pad >> 2, nib = (L.in + 3) >> 2;
  for (int idx = threadIdx.x; idx < nob * nib; idx += blockDim.x) {
    const int o0 = (idx % nob) * 4, i0 = (idx / nob) * 4;
    float acc[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[q][r] = 0.f;
    const bool full_i = i0 + 4 <= L.in;
    for (int g = 0; g < ng; ++g) {
      float gv[4], xv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) gv[q] = gy[(o0 + q) * TG + g];
#pragma unroll
      for (int r = 0; r < 4; ++r) xv[r] = (full_i || i0 + r < L.in) ? x[(i0 + r) * TG + g] : 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[q][r] = fmaf(gv[q], xv[r], acc[q][r]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (o0 + q < L.out && i0 + r < L.in) Wt[(int64_t)(i0 + r) * L.out_pad + o0 + q] += acc[q][r];
  }
  for (int o = threadIdx.x; o < L.out; o += blockDim.x) {
    const float* gyo = gy + o * TG;
    float acc = 0.f;
    for (int g = 0; g < ng; ++g) acc += gyo[g];
    bias[o] += acc;
  }
}

// normalized coordinates (hexplane.py:84-92).  Evaluated in fp64 so the cell
// choice (floor) and the strict `inside` test match the float64 reference; the
// interpolation itself runs in fp32.
__device__ __forceinline__ void norm_coords(const FieldDesc& f, const float* p, double t, double c[4],
                                            bool inside[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double raw = ((double)p[k] - f.lo[k]) / f.span[k];
    inside[k] = raw > 0.0 && raw < 1.0;
    c[k] = fmin(fmax(raw, 0.0), 1.0);
  }
  c[3] = t;
}

struct Bilin {
  int64_t base;  // (i0 * Rb + j0) * C
  int rowstride; // Rb * C
  float fa, fb;
};

// hexplane.py:95-110
__device__ __forceinline__ Bilin bilinear_cell(int ra, int rb, int C, double ca, double cb) {
  const double u = ca * (double)(ra - 1), v = cb * (double)(rb - 1);
  int i0 = (int)floor(u), j0 = (int)floor(v);
  i0 = min(max(i0, 0), ra - 2);
  j0 = min(max(j0, 0), rb - 2);
  Bilin b;
  b.base = ((int64_t)i0 * rb + j0) * C;
  b.rowstride = rb * C;
  b.fa = (float)(u - (double)i0);
  b.fb = (float)(v - (double)j0);
  return b;
}

// Gather the latent of Gaussian g (one warp, lanes over channels) into lat[dim][TG].
__device__ __forceinline__ void hexplane_gather(const FieldDesc& f, const double c[4], float* lat, int g, int TG,
                                                int lane) {
  const int C = f.C;
  for (int l = 0; l < f.levels; ++l) {
    Bilin bl[6];
#pragma unroll
    for (int p = 0; p < 6; ++p)
      bl[p] = bilinear_cell(f.res[l][p][0], f.res[l][p][1], C, c[c_plane_axes[p][0]], c[c_plane_axes[p][1]]);
    for (int ch = lane; ch < C; ch += 32) {
      float prod = 1.f;
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const float* pl = f.planes[l][p] + bl[p].base + ch;
        const float p00 = __ldg(pl), p01 = __ldg(pl + C);
        const float p10 = __ldg(pl + bl[p].rowstride), p11 = __ldg(pl + bl[p].rowstride + C);
        const float fa = bl[p].fa, fb = bl[p].fb;
        const float v = (1.f - fa) * (1.f - fb) * p00 + fa * (1.f - fb) * p10 + (1.f - fa) * fb * p01 + fa * fb * p11;
        prod *= v;
      }
      lat[(l * C + ch) * TG + g] = prod;
    }
  }
}

// shared-memory plan (floats), channel-major [dim][TG]
struct SmemPlan {
  int lat, ping, pong, e1, cat, delta, ff, dz;  // forward
  int trunk_outs;  // backward: depth x width
  int e1s;         // backward: 4 x half
  int g_a, g_b, g_cat, g_ff, g_delta, g_dz;  // backward gradient buffers
  int total;
};

__host__ __device__ inline SmemPlan make_plan(const NetDesc& n, int TG, bool backward) {
  SmemPlan s;
  int o = 0;
  const int md = n.max_dim > n.width ? n.max_dim : n.width;
  const int hp = round4(n.half);
  const int Dp = round4(n.D > 0 ? n.D : 1);
  s.lat = o; o += round4(n.L > 0 ? n.L : 1) * TG;
  s.ping = o; o += md * TG;
  s.pong = o; o += md * TG;
  s.e1 = o; o += hp * TG;
  s.cat = o; o += 4 * hp * TG;
  s.delta = o; o += 12 * TG;
  s.ff = o; o += hp * TG;
  s.dz = o; o += Dp * TG;
  s.trunk_outs = s.e1s = s.g_a = s.g_b = s.g_cat = s.g_ff = s.g_delta = s.g_dz = 0;
  if (backward) {
    s.trunk_outs = o; o += n.depth * round4(n.width) * TG;
    s.e1s = o; o += 4 * hp * TG;
    s.g_a = o; o += md * TG;
    s.g_b = o; o += md * TG;
    s.g_cat = o; o += 4 * hp * TG;
    s.g_ff = o; o += hp * TG;
    s.g_delta = o; o += 12 * TG;
    s.g_dz = o; o += Dp * TG;
  }
  s.total = o;
  return s;
}

// Forward MLP for one tile with the latent already in lat.  When `store` is set
// (backward recompute) every trunk output and branch e1 is kept.
__device__ void mlp_tile_fwd(const DefArgs& a, const SmemPlan& sp, float* sm, int TG, bool store) {
  const NetDesc& n = a.net;
  const float* in = sm + sp.lat;
  for (int l = 0; l < n.depth; ++l) {
    float* out = store ? sm + sp.trunk_outs + l * round4(n.width) * TG : sm + ((l & 1) ? sp.pong : sp.ping);
    dense_fwd(n.layers[n.trunk0 + l], a.blob, in, out, TG);
    __syncthreads();
    in = out;
  }
  const float* hidden = in;
  const int hp = round4(n.half);
  for (int b = 0; b < 4; ++b) {
    float* e1 = store ? sm + sp.e1s + b * hp * TG : sm + sp.e1;
    dense_fwd(n.layers[n.ext0 + 2 * b], a.blob, hidden, e1, TG);
    __syncthreads();
    // e2 goes straight into its slot of the F_feat concat (deformation.py:119-120)
    dense_fwd(n.layers[n.ext0 + 2 * b + 1], a.blob, e1, sm + sp.cat + b * n.half * TG, TG);
    __syncthreads();
  }
  const int hoff[4] = {0, 3, 7, 10};
  for (int b = 0; b < 4; ++b) {
    // heads write 4-padded rows; stage through pong then copy the live rows
    dense_fwd(n.layers[n.head0 + b], a.blob, sm + sp.cat + b * n.half * TG, sm + sp.pong, TG);
    __syncthreads();
    const int d = n.layers[n.head0 + b].out;
    for (int idx = threadIdx.x; idx < d * TG; idx += blockDim.x) sm[sp.delta + (hoff[b] + idx / TG) * TG + idx % TG] = sm[sp.pong + idx];
    __syncthreads();
  }
  if (n.enable_feat) {
    dense_fwd(n.layers[n.feat0], a.blob, sm + sp.cat, sm + sp.ff, TG);
    __syncthreads();
    dense_fwd(n.layers[n.feat0 + 1], a.blob, sm + sp.ff, sm + sp.dz, TG);
    __syncthreads();
  }
}

__device__ void latent_tile(const DefArgs& a, const SmemPlan& sp, float* sm, int64_t g0, int ng, int TG) {
  const NetDesc& n = a.net;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* lat = sm + sp.lat;
  if (!n.enable_grid) {
    for (int idx = threadIdx.x; idx < n.L * TG; idx += blockDim.x) lat[idx] = 0.f;
    return;
  }
  for (int g = warp; g < TG; g += nw) {
    if (g < ng) {
      double c[4];
      bool inside[3];
      norm_coords(a.field, a.pos + 3 * (g0 + g), a.t, c, inside);
      hexplane_gather(a.field, c, lat, g, TG, lane);
    } else {
      for (int ch = lane; ch < n.L; ch += 32) lat[ch * TG + g] = 0.f;
    }
  }
}

__global__ void __launch_bounds__(kDefThreads) k_deform_fwd(DefArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int TG = a.TG;
  const SmemPlan sp = make_plan(a.net, TG, false);
  const NetDesc& n = a.net;
  const int64_t ntiles = ceil_div(a.K, TG);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t g0 = tile * TG;
    const int ng = (int)(a.K - g0 < TG ? a.K - g0 : TG);
    latent_tile(a, sp, sm, g0, ng, TG);
    __syncthreads();
    mlp_tile_fwd(a, sp, sm, TG, false);
    // raw-space deltas (deformation.py:126-133)
    for (int idx = threadIdx.x; idx < 11 * TG; idx += blockDim.x) {
      const int comp = idx / TG, g = idx % TG;
      if (g >= ng) continue;
      const int64_t k = g0 + g;
      const float dv = sm[sp.delta + comp * TG + g];
      if (comp < 3) a.o_pos[3 * k + comp] = a.pos[3 * k + comp] + dv;
      else if (comp < 7) a.o_rot[4 * k + comp - 3] = a.rot[4 * k + comp - 3] + dv;
      else if (comp < 10) a.o_ls[3 * k + comp - 7] = a.ls[3 * k + comp - 7] + dv;
      else a.o_op[k] = a.op[k] + dv;
    }
    if (n.enable_feat) {
      for (int idx = threadIdx.x; idx < n.D * TG; idx += blockDim.x) {
        const int g = idx / n.D, c = idx % n.D;  // coalesced over the [K,D] output
        if (g >= ng) continue;
        const int64_t k = g0 + g;
        a.o_feat[(int64_t)n.D * k + c] = a.feat[(int64_t)n.D * k + c] + sm[sp.dz + c * TG + g];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
// Reduce v[0..31] over the warp; afterwards lane L holds the warp sum of v[L].
__device__ __forceinline__ float warp_transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < n / 2; ++k) {
      float send = upper ? v[k] : v[k + n / 2];
      float keep = upper ? v[k + n / 2] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// hexplane.py:145-187 for one Gaussian (one warp): plane scatter + dpos.
__device__ void hexplane_backward_one(const DefArgs& a, const float* glat, int g, int TG, int64_t k, int lane) {
  const FieldDesc& f = a.field;
  const int C = f.C;
  double c[4];
  bool inside[3];
  norm_coords(f, a.pos + 3 * k, a.t, c, inside);
  float dco[4] = {0.f, 0.f, 0.f, 0.f};
  for (int l = 0; l < f.levels; ++l) {
    Bilin bl[6];
#pragma unroll
    for (int p = 0; p < 6; ++p)
      bl[p] = bilinear_cell(f.res[l][p][0], f.res[l][p][1], C, c[c_plane_axes[p][0]], c[c_plane_axes[p][1]]);
    float red[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) red[r] = 0.f;
    for (int ch = lane; ch < C; ch += 32) {
      float s[6], p00[6], p01[6], p10[6], p11[6];
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const float* pl = f.planes[l][p] + bl[p].base + ch;
        p00[p] = __ldg(pl);
        p01[p] = __ldg(pl + C);
        p10[p] = __ldg(pl + bl[p].rowstride);
        p11[p] = __ldg(pl + bl[p].rowstride + C);
        const float fa = bl[p].fa, fb = bl[p].fb;
        s[p] = (1.f - fa) * (1.f - fb) * p00[p] + fa * (1.f - fb) * p10[p] + (1.f - fa) * fb * p01[p] + fa * fb * p11[p];
      }
      // product of the other five via prefix/suffix (hexplane.py:131-139)
      float pre[6], suf[6];
      pre[0] = 1.f;
#pragma unroll
      for (int p = 1; p < 6; ++p) pre[p] = pre[p - 1] * s[p - 1];
      suf[5] = 1.f;
#pragma unroll
      for (int p = 4; p >= 0; --p) suf[p] = suf[p + 1] * s[p + 1];
      const float up = glat[(l * C + ch) * TG + g];
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const float coef = up * pre[p] * suf[p];
        const float fa = bl[p].fa, fb = bl[p].fb;
        float* gp = f.gplanes[l][p] + bl[p].base + ch;
        if (coef != 0.f) {
          red_add(gp, coef * (1.f - fa) * (1.f - fb));
          red_add(gp + bl[p].rowstride, coef * fa * (1.f - fb));
          red_add(gp + C, coef * (1.f - fa) * fb);
          red_add(gp + bl[p].rowstride + C, coef * fa * fb);
        }
        const float dfa = (1.f - fb) * (p10[p] - p00[p]) + fb * (p11[p] - p01[p]);
        const float dfb = (1.f - fa) * (p01[p] - p00[p]) + fa * (p11[p] - p10[p]);
        red[2 * p] += coef * dfa;
        red[2 * p + 1] += coef * dfb;
      }
    }
    warp_transpose_reduce32(red, lane);
    // lane 2p holds sum(coef*dfa) of plane p, lane 2p+1 sum(coef*dfb)
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const float sa = __shfl_sync(0xffffffffu, red[0], 2 * p);
      const float sb = __shfl_sync(0xffffffffu, red[0], 2 * p + 1);
      dco[c_plane_axes[p][0]] += sa * (float)(f.res[l][p][0] - 1);
      dco[c_plane_axes[p][1]] += sb * (float)(f.res[l][p][1] - 1);
    }
  }
  if (lane < 3) {
    const float d = inside[lane] ? (float)((double)dco[lane] / f.span[lane]) : 0.f;
    a.cg_pos[3 * k + lane] = (a.accumulate ? a.cg_pos[3 * k + lane] : 0.f) + a.g_pos[3 * k + lane] + d;
  }
}

__global__ void __launch_bounds__(kDefThreads) k_deform_bwd(DefArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int TG = a.TG;
  const SmemPlan sp = make_plan(a.net, TG, true);
  const NetDesc& n = a.net;
  const int hp = round4(n.half);
  const int wp = round4(n.width);
  float* part = a.wpart + (int64_t)blockIdx.x * n.packed_floats;
  const int64_t ntiles = ceil_div(a.K, TG);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t g0 = tile * TG;
    const int ng = (int)(a.K - g0 < TG ? a.K - g0 : TG);
    latent_tile(a, sp, sm, g0, ng, TG);
    __syncthreads();
    mlp_tile_fwd(a, sp, sm, TG, true);

    // upstream gradients (rows >= ng are zero so padded Gaussians add nothing)
    const int hoff[5] = {0, 3, 7, 10, 11};
    for (int idx = threadIdx.x; idx < 12 * TG; idx += blockDim.x) {
      const int comp = idx / TG, g = idx % TG;
      float v = 0.f;
      if (g < ng && comp < 11) {
        const int64_t k = g0 + g;
        if (comp < 3) v = a.g_pos[3 * k + comp];
        else if (comp < 7) v = a.g_rot[4 * k + comp - 3];
        else if (comp < 10) v = a.g_ls[3 * k + comp - 7];
        else v = a.g_op[k];
      }
      sm[sp.g_delta + idx] = v;
    }
    const int Dp = round4(n.D > 0 ? n.D : 1);
    for (int idx = threadIdx.x; idx < Dp * TG; idx += blockDim.x) {
      const int c = idx / TG, g = idx % TG;
      sm[sp.g_dz + idx] = (g < ng && c < n.D && n.enable_feat) ? a.g_feat[(int64_t)n.D * (g0 + g) + c] : 0.f;
    }
    for (int idx = threadIdx.x; idx < 4 * hp * TG; idx += blockDim.x) sm[sp.g_cat + idx] = 0.f;
    __syncthreads();

    // F_feat (deformation.py:157-161)
    if (n.enable_feat) {
      const LayerDesc& L1 = n.layers[n.feat0 + 1];
      dense_bwd_w(L1, part, sm + sp.g_dz, sm + sp.ff, TG, ng);
      dense_bwd_x(L1, a.blob, sm + sp.g_dz, sm + sp.g_ff, TG, false);
      __syncthreads();
      for (int idx = threadIdx.x; idx < n.half * TG; idx += blockDim.x)
        if (sm[sp.ff + idx] <= 0.f) sm[sp.g_ff + idx] = 0.f;
      for (int idx = n.half * TG + threadIdx.x; idx < hp * TG; idx += blockDim.x) sm[sp.g_ff + idx] = 0.f;
      __syncthreads();
      const LayerDesc& L0 = n.layers[n.feat0];
      dense_bwd_w(L0, part, sm + sp.g_ff, sm + sp.cat, TG, ng);
      dense_bwd_x(L0, a.blob, sm + sp.g_ff, sm + sp.g_cat, TG, false);
      __syncthreads();
    }
    // branches (deformation.py:168-177); g_a accumulates d_hidden
    for (int idx = threadIdx.x; idx < wp * TG; idx += blockDim.x) sm[sp.g_a + idx] = 0.f;
    __syncthreads();
    const float* hidden = sm + sp.trunk_outs + (n.depth - 1) * wp * TG;
    for (int b = 0; b < 4; ++b) {
      const LayerDesc& LH = n.layers[n.head0 + b];
      // head grads: stage the branch's 4-padded delta grad in g_b
      for (int idx = threadIdx.x; idx < LH.out_pad * TG; idx += blockDim.x) {
        const int r = idx / TG, g = idx % TG;
        sm[sp.g_b + idx] = r < LH.out ? sm[sp.g_delta + (hoff[b] + r) * TG + g] : 0.f;
      }
      __syncthreads();
      float* e2 = sm + sp.cat + b * n.half * TG;
      float* ge2 = sm + sp.g_cat + b * n.half * TG;  // holds d_joint slice; add head contribution
      dense_bwd_w(LH, part, sm + sp.g_b, e2, TG, ng);
      dense_bwd_x(LH, a.blob, sm + sp.g_b, ge2, TG, true);
      __syncthreads();
      for (int idx = threadIdx.x; idx < n.half * TG; idx += blockDim.x)
        if (e2[idx] <= 0.f) ge2[idx] = 0.f;
      // copy to a 4-padded buffer for the next dense_bwd_x
      for (int idx = threadIdx.x; idx < hp * TG; idx += blockDim.x)
        sm[sp.g_b + idx] = idx < n.half * TG ? ge2[idx] : 0.f;
      __syncthreads();
      const LayerDesc& LE1 = n.layers[n.ext0 + 2 * b + 1];
      const float* e1 = sm + sp.e1s + b * hp * TG;
      dense_bwd_w(LE1, part, sm + sp.g_b, e1, TG, ng);
      dense_bwd_x(LE1, a.blob, sm + sp.g_b, sm + sp.g_ff, TG, false);
      __syncthreads();
      for (int idx = threadIdx.x; idx < hp * TG; idx += blockDim.x) {
        float v = idx < n.half * TG ? sm[sp.g_ff + idx] : 0.f;
        if (idx < n.half * TG && e1[idx] <= 0.f) v = 0.f;
        sm[sp.g_ff + idx] = v;
      }
      __syncthreads();
      const LayerDesc& LE0 = n.layers[n.ext0 + 2 * b];
      dense_bwd_w(LE0, part, sm + sp.g_ff, hidden, TG, ng);
      dense_bwd_x(LE0, a.blob, sm + sp.g_ff, sm + sp.g_a, TG, true);
      __syncthreads();
    }
    // trunk (deformation.py:178-179), g_a = d_hidden
    float* gcur = sm + sp.g_a;
    float* gnext = sm + sp.g_b;
    for (int l = n.depth - 1; l >= 0; --l) {
      const float* out = sm + sp.trunk_outs + l * wp * TG;
      const LayerDesc& LT = n.layers[n.trunk0 + l];
      for (int idx = threadIdx.x; idx < wp * TG; idx += blockDim.x) {
        float v = idx < n.width * TG ? gcur[idx] : 0.f;
        if (idx < n.width * TG && out[idx] <= 0.f) v = 0.f;
        gcur[idx] = v;
      }
      __syncthreads();
      const float* xin = l == 0 ? sm + sp.lat : sm + sp.trunk_outs + (l - 1) * wp * TG;
      dense_bwd_w(LT, part, gcur, xin, TG, ng);
      dense_bwd_x(LT, a.blob, gcur, gnext, TG, false);
      __syncthreads();
      float* tmp = gcur;
      gcur = gnext;
      gnext = tmp;
    }
    // gcur = d_latent [L][TG] -> plane scatter + position gradient
    if (n.enable_grid) {
      for (int g = warp; g < ng; g += nw) hexplane_backward_one(a, gcur, g, TG, g0 + g, lane);
    } else {
      for (int idx = threadIdx.x; idx < 3 * ng; idx += blockDim.x)
        a.cg_pos[3 * g0 + idx] = (a.accumulate ? a.cg_pos[3 * g0 + idx] : 0.f) + a.g_pos[3 * g0 + idx];
    }
    __syncthreads();
  }
}

// sum CTA partials into the [out,in] weight / [out] bias gradient buffers
struct ReduceArgs {
  LayerDesc layers[kMaxLayers];
  float* gw[kMaxLayers];
  float* gb[kMaxLayers];
  int n_layers;
  int nparts;
  int accumulate;
  int64_t packed_floats;
  const float* wpart;
};

__global__ void k_reduce_wgrads(ReduceArgs a) {
  const LayerDesc& L = a.layers[blockIdx.y];
  const int64_t nw = (int64_t)L.in * L.out;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nw + L.out; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t src;
    float* dst;
    if (e < nw) {
      const int o = (int)(e / L.in), i = (int)(e % L.in);
      src = L.off_w + (int64_t)i * L.out_pad + o;
      dst = a.gw[blockIdx.y] + e;
    } else {
      const int o = (int)(e - nw);
      src = L.off_b + o;
      dst = a.gb[blockIdx.y] + o;
    }
    float s = 0.f;
    for (int p = 0; p < a.nparts; ++p) s += a.wpart[(int64_t)p * a.packed_floats + src];
    *dst = a.accumulate ? *dst + s : s;
  }
}

// cloud gradients that pass straight through the deformation
// (deformation.py:178-181: rotations, log-scales, opacity logits, features;
// colours and SH bypass it, training.py:518)
struct PassArgs {
  const float* src[6];
  float* dst[6];
  int64_t n[6];
  int64_t block_start[7];  // blocks of kPassChunk elements per field, prefix sums
  int accumulate;
};
constexpr int kPassChunk = 256 * 16;  // elements per block (16 per thread)

// Pass-through cloud gradients (deformation.py:178-181; colours / SH bypass
// the deformation, training.py:518): every field's elements split into
// equal chunks of one flat block index space, float4 accesses when aligned.
__global__ void __launch_bounds__(256) k_grad_passthrough(PassArgs a) {
  int f = 0;
  while (f < 5 && (int64_t)blockIdx.x >= a.block_start[f + 1]) ++f;
  const int64_t lo = ((int64_t)blockIdx.x - a.block_start[f]) * kPassChunk;
  const int64_t hi = min(lo + kPassChunk, a.n[f]);
  const float* src = a.src[f];
  float* dst = a.dst[f];
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (vec && hi - lo == kPassChunk) {
    const float4* s4 = reinterpret_cast<const float4*>(src + lo);
    float4* d4 = reinterpret_cast<float4*>(dst + lo);
#pragma unroll
    for (int r = 0; r < kPassChunk / 4 / 256; ++r) {
      const int e = r * 256 + threadIdx.x;
      float4 v = __ldg(s4 + e);
      if (a.accumulate) {
        const float4 o = d4[e];
        v = make_float4(o.x + v.x, o.y + v.y, o.z + v.z, o.w + v.w);
      }
      d4[e] = v;
    }
    return;
  }
  for (int64_t e = lo + threadIdx.x; e < hi; e += 256) dst[e] = a.accumulate ? dst[e] + src[e] : src[e];
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
static int build_field_desc(const Fs4dHexPlane& h, const Fs4dDeformNet& n, FieldDesc& f) {
  f.levels = h.levels;
  f.C = h.channels;
  if (n.enable_grid) {
    if (h.levels < 1 || h.levels > FS4D_MAX_LEVELS) return fail(FS4D_ERR_CONFIG, "hexplane levels out of range");
    if (h.levels * h.channels != n.latent_dim) return fail(FS4D_ERR_CONFIG, "latent_dim != levels * channels");
  }
  for (int l = 0; l < FS4D_MAX_LEVELS; ++l)
    for (int p = 0; p < 6; ++p) {
      f.res[l][p][0] = h.res[l][p][0];
      f.res[l][p][1] = h.res[l][p][1];
      f.planes[l][p] = h.planes[l][p];
      f.gplanes[l][p] = nullptr;
      if (l < h.levels && n.enable_grid && (h.res[l][p][0] < 2 || h.res[l][p][1] < 2))
        return fail(FS4D_ERR_CONFIG, "plane resolutions must be >= 2");
    }
  for (int k = 0; k < 3; ++k) {
    f.lo[k] = h.aabb[k];
    f.span[k] = h.aabb[3 + k] - h.aabb[k];
    if (n.enable_grid && !(h.aabb[3 + k] > h.aabb[k])) return fail(FS4D_ERR_CONFIG, "aabb must have hi > lo");
  }
  return FS4D_OK;
}

static int pick_tg(const NetDesc& n, bool backward, size_t* smem_bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (max_optin <= 0) max_optin = 227 * 1024;
  // odd tile sizes make the [dim][TG] column reads bank-conflict free
  for (int tg = 63; tg >= 7; tg = (tg - 1) / 2) {
    SmemPlan sp = make_plan(n, tg, backward);
    size_t b = (size_t)sp.total * 4;
    // forward: keep two CTAs per SM when possible
    if (b <= (size_t)max_optin && (backward || tg <= 7 || b * 2 <= (size_t)max_optin)) {
      *smem_bytes = b;
      return tg;
    }
  }
  SmemPlan sp = make_plan(n, 7, backward);
  *smem_bytes = (size_t)sp.total * 4;
  return *smem_bytes <= (size_t)max_optin ? 7 : 0;
}

static size_t blob_bytes(const NetDesc& d) { return align_up_sz((size_t)d.packed_floats * 4, 256); }

bool tc_path_ok(const Fs4dDeformNet& n, const Fs4dHexPlane& f);
size_t tc_workspace_bytes(const Fs4dDeformNet& n, int64_t K);
int deform_forward_tc(const Fs4dCloud& cloud, const Fs4dHexPlane& field, const Fs4dDeformNet& net, double t,
                      Fs4dCloud& snap, void* ws, uint8_t* cache, cudaStream_t s);
bool tc_bwd_ok(const Fs4dDeformNet& n, const Fs4dHexPlane& f);
size_t tc_cache_bytes(const Fs4dDeformNet& n, const Fs4dHexPlane& f, int64_t K);
int deform_backward_tc(const Fs4dCloud& cloud, const Fs4dHexPlane& field, const Fs4dDeformNet& net, double t,
                       const uint8_t* cache, const Fs4dCloud& sg, Fs4dCloud& cg, Fs4dDeformNet& ng,
                       Fs4dHexPlane* pg, int accumulate, void* ws, int32_t* status, void* det_ws, size_t det_bytes,
                       cudaStream_t s);
size_t deform_bwd_det_bytes(const Fs4dHexPlane& f);

static bool tc_enabled() { return !getenv("FS4D_NO_TC"); }

// activation cache of deform_with_cache: 0 when the tensor-core backward does
// not cover this net (the backward then recomputes the forward itself)
size_t deform_cache_bytes(const Fs4dDeformNet& net, const Fs4dHexPlane& field, int64_t K) {
  return tc_enabled() ? tc_cache_bytes(net, field, K) : 0;
}

size_t deform_workspace_bytes(const Fs4dDeformNet& net, int64_t K, int* nparts_out) {
  NetDesc d;
  if (build_net_desc(net, d) != FS4D_OK) return 0;
  int nparts = kNumSMs * 2;
  if (nparts_out) *nparts_out = nparts;
  (void)K;
  const size_t generic = blob_bytes(d) + (size_t)nparts * d.packed_floats * 4 + 256;
  const size_t tc = tc_workspace_bytes(net, K);
  return generic > tc ? generic : tc;
}


static int pack_net(const NetDesc& d, float* blob, cudaStream_t s) {
  PackArgs pa;
  for (int i = 0; i < d.n_layers; ++i) pa.layers[i] = d.layers[i];
  pa.n_layers = d.n_layers;
  pa.blob = blob;
  dim3 grid(8, d.n_layers);
  k_pack_weights<<<grid, 256, 0, s>>>(pa);
  return FS4D_OK;
}

static int fill_args(const Fs4dCloud& cloud, const Fs4dHexPlane& field, const Fs4dDeformNet& net, double t,
                     void* ws, size_t ws_bytes, bool backward, DefArgs& a, size_t* smem) {
  int rc = build_net_desc(net, a.net);
  if (rc) return rc;
  rc = build_field_desc(field, net, a.field);
  if (rc) return rc;
  if (net.enable_feature_update && cloud.D != net.feature_dim)
    return fail(FS4D_ERR_CONFIG, "cloud feature dim does not match the deformation net");
  const size_t need = deform_workspace_bytes(net, cloud.K, nullptr);
  if (!ws || ws_bytes < need) return fail(FS4D_ERR_CONFIG, "deform workspace too small");
  a.K = cloud.K;
  a.t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);  // hexplane.py:90
  a.pos = cloud.positions;
  a.rot = cloud.rotations;
  a.ls = cloud.log_scales;
  a.op = cloud.opacity_logits;
  a.feat = cloud.features;
  a.blob = (const float*)ws;
  a.wpart = (float*)((char*)ws + blob_bytes(a.net));
  a.TG = pick_tg(a.net, backward, smem);
  if (a.TG <= 0) return fail(FS4D_ERR_CONFIG, "deformation net too wide for shared memory");
  return FS4D_OK;
}

int deform_forward(const Fs4dCloud& cloud, const Fs4dHexPlane& field, const Fs4dDeformNet& net, double t,
                   Fs4dCloud& snap, void* cache, size_t cache_bytes, void* ws, size_t ws_bytes, cudaStream_t s) {
  DefArgs a;
  memset(&a, 0, sizeof(a));
  size_t smem = 0;
  int rc = fill_args(cloud, field, net, t, ws, ws_bytes, false, a, &smem);
  if (rc) return rc;
  if (cloud.K == 0) return FS4D_OK;
  a.o_pos = snap.positions;
  a.o_rot = snap.rotations;
  a.o_ls = snap.log_scales;
  a.o_op = snap.opacity_logits;
  a.o_feat = snap.features;
  StageTimer st(FS4D_STAGE_DEFORM_FWD, s);
  const size_t cneed = deform_cache_bytes(net, field, cloud.K);
  if (cache && cneed && cache_bytes < cneed) return fail(FS4D_ERR_CONFIG, "deform cache too small");
  if (tc_path_ok(net, field) && tc_enabled())
    return deform_forward_tc(cloud, field, net, t, snap, ws, cneed ? (uint8_t*)cache : nullptr, s);
  pack_net(a.net, (float*)ws, s);
  cudaFuncSetAttribute(k_deform_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = ceil_div(cloud.K, a.TG);
  const int grid = (int)(ntiles < kNumSMs * 2 ? ntiles : kNumSMs * 2);
  k_deform_fwd<<<grid, kDefThreads, smem, s>>>(a);
  return check_launch("deform_fwd");
}

size_t deform_backward_det_bytes(const Fs4dDeformNet& net, const Fs4dHexPlane& field) {
  if (!tc_enabled() || !tc_bwd_ok(net, field)) return 0;
  return deform_bwd_det_bytes(field);
}

int deform_backward(const Fs4dCloud& cloud, const Fs4dHexPlane& field, const Fs4dDeformNet& net, double t,
                    const void* cache, size_t cache_bytes, const Fs4dCloud& sg, Fs4dCloud& cg, Fs4dDeformNet& ng,
                    Fs4dHexPlane* pg, int accumulate, void* ws, size_t ws_bytes, int32_t* status, void* det_ws,
                    size_t det_bytes, cudaStream_t s, cudaEvent_t pass_done) {
  DefArgs a;
  memset(&a, 0, sizeof(a));
  size_t smem = 0;
  int rc = fill_args(cloud, field, net, t, ws, ws_bytes, true, a, &smem);
  if (rc) return rc;
  a.g_pos = sg.positions;
  a.g_rot = sg.rotations;
  a.g_ls = sg.log_scales;
  a.g_op = sg.opacity_logits;
  a.g_feat = sg.features;
  a.cg_pos = cg.positions;
  a.accumulate = accumulate;
  if (net.enable_grid) {
    if (!pg) return fail(FS4D_ERR_CONFIG, "plane gradient buffers required when the grid is enabled");
    for (int l = 0; l < field.levels; ++l)
      for (int p = 0; p < 6; ++p) {
        a.field.gplanes[l][p] = pg->planes[l][p];
        if (!accumulate)
          cudaMemsetAsync(pg->planes[l][p], 0,
                          (size_t)field.res[l][p][0] * field.res[l][p][1] * field.channels * 4, s);
      }
  }
  StageTimer st(FS4D_STAGE_DEFORM_BWD, s);
  {
    const int n_sh = (sg.sh_degree + 1) * (sg.sh_degree + 1) - 1;
    PassArgs pa;
    const float* srcs[6] = {sg.rotations, sg.log_scales, sg.opacity_logits, sg.colors_raw, sg.sh_rest, sg.features};
    float* dsts[6] = {cg.rotations, cg.log_scales, cg.opacity_logits, cg.colors_raw, cg.sh_rest, cg.features};
    const int64_t ns[6] = {cloud.K * 4, cloud.K * 3, cloud.K, cloud.K * 3, cloud.K * n_sh * 3, cloud.K * cloud.D};
    int64_t blocks = 0;
    for (int f = 0; f < 6; ++f) {
      const bool on = ns[f] > 0 && srcs[f] && dsts[f];
      pa.src[f] = on ? srcs[f] : nullptr;
      pa.dst[f] = on ? dsts[f] : nullptr;
      pa.n[f] = on ? ns[f] : 0;
      pa.block_start[f] = blocks;
      blocks += ceil_div(pa.n[f], kPassChunk);
    }
    pa.block_start[6] = blocks;
    pa.accumulate = accumulate;
    if (blocks > 0) k_grad_passthrough<<<(unsigned)blocks, 256, 0, s>>>(pa);
    // every cloud gradient except positions is final here: a caller can start
    // reducing those rows (all-reduce bucket) while the MLP / HexPlane
    // backward below runs
    if (pass_done) cudaEventRecord(pass_done, s);
  }
  const size_t cneed = deform_cache_bytes(net, field, cloud.K);
  if (det_ws && !(cache && cneed))
    return fail(FS4D_ERR_CONFIG,
                "the deterministic deform backward needs the tensor-core path with its forward cache "
                "(width 64, depth 1, levels * channels = 64, feature_dim <= 16)");
  if (cache && cneed) {
    if (cache_bytes < cneed) return fail(FS4D_ERR_CONFIG, "deform cache too small");
    return deform_backward_tc(cloud, field, net, t, (const uint8_t*)cache, sg, cg, ng, pg, accumulate, ws, status,
                              det_ws, det_bytes, s);
  }
  const int64_t ntiles = ceil_div(cloud.K, a.TG);
  const int grid = (int)(ntiles < kNumSMs * 2 ? (ntiles > 0 ? ntiles : 1) : kNumSMs * 2);
  cudaMemsetAsync(a.wpart, 0, (size_t)grid * a.net.packed_floats * 4, s);
  pack_net(a.net, (float*)ws, s);
  if (cloud.K > 0) {
    cudaFuncSetAttribute(k_deform_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_deform_bwd<<<grid, kDefThreads, smem, s>>>(a);
  }
  ReduceArgs ra;
  memset(&ra, 0, sizeof(ra));
  const NetDesc& d = a.net;
  Fs4dLinear* gl[kMaxLayers];
  int k = 0;
  for (int i = 0; i < d.depth; ++i) gl[k++] = &ng.trunk[i];
  for (int b = 0; b < 4; ++b) {
    gl[k++] = &ng.ext[b][0];
    gl[k++] = &ng.ext[b][1];
  }
  for (int b = 0; b < 4; ++b) gl[k++] = &ng.head[b];
  gl[k++] = &ng.feat[0];
  gl[k++] = &ng.feat[1];
  for (int i = 0; i < d.n_layers; ++i) {
    ra.layers[i] = d.layers[i];
    ra.gw[i] = gl[i]->weight;
    ra.gb[i] = gl[i]->bias;
    if (!ra.gw[i] || !ra.gb[i]) return fail(FS4D_ERR_CONFIG, "missing net gradient buffer");
  }
  ra.n_layers = d.n_layers;
  ra.nparts = grid;
  ra.accumulate = accumulate;
  ra.packed_floats = d.packed_floats;
  ra.wpart = a.wpart;
  dim3 rg(16, d.n_layers);
  k_reduce_wgrads<<<rg, 256, 0, s>>>(ra);
  return check_launch("deform_bwd");
}

}  // namespace fs4d
