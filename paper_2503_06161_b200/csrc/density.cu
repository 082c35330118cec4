// Adaptive density control as device stream compaction:
//   * view-space gradient statistics (gaussians.py:309-327, ViewspaceGradStats)
//   * densify_and_prune (gaussians.py:349-405): clone small / split large
//     high-gradient Gaussians, prune transparent ones
//   * prune_only (gaussians.py:408-417) and reset_opacity (gaussians.py:420-425)
//
// The reference rebuilds the cloud as [kept rows (original order) | clones
// (index order) | split children, first sample set | second sample set]; the
// device does the same with three exclusive scans and one row-gather pass, so
// the result is row-for-row the reference's.  Every decision is taken in fp64
// (same thresholds as the float64 reference).  Split offsets need
// rng.standard_normal((n_split, 3)) twice, drawn by the caller from the
// reference's own generator so the random stream is the reference's.
#include <math.h>

#include <algorithm>

#include "scan_sort.cuh"

namespace fs4d {

namespace {
constexpr int kT = 256;

__device__ __forceinline__ double sigmoid_dd(double x) {  // gaussians.py:25-31
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}
}  // namespace

// ViewspaceGradStats.add (gaussians.py:319-321): the indices of one render
// are distinct, so plain read-modify-writes are race-free and deterministic.
__global__ void __launch_bounds__(kT) k_stats_add(double* __restrict__ accum, double* __restrict__ count,
                                                  const int32_t* __restrict__ idx, const float* __restrict__ norms,
                                                  int64_t n, const int32_t* __restrict__ n_dev) {
  const int64_t m = n_dev ? min((int64_t)*n_dev, n) : n;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kT) {
    if (!idx && norms[i] < 0.f) continue;  // dense form: culled Gaussian
    const int64_t g = idx ? (int64_t)idx[i] : i;
    accum[g] += (double)norms[i];
    count[g] += 1.0;
  }
}

// flags per row: bit0 keep, bit1 clone, bit2 split (parent survives as two
// children), bit3 prune.  Scan inputs are the three u32 indicator arrays.
__global__ void __launch_bounds__(kT) k_density_classify(Fs4dCloud c, const double* __restrict__ accum,
                                                         const double* __restrict__ count, Fs4dDensityConfig cfg,
                                                         int prune_only, uint32_t* __restrict__ keep,
                                                         uint32_t* __restrict__ clone, uint32_t* __restrict__ split) {
  const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (i >= c.K) return;
  const double opac = sigmoid_dd((double)c.opacity_logits[i]);
  const bool prune = opac < cfg.prune_opacity;  // gaussians.py:369
  if (prune_only) {                              // gaussians.py:410
    keep[i] = !prune;
    clone[i] = 0;
    split[i] = 0;
    return;
  }
  const double avg = accum[i] / fmax(count[i], 1.0);  // averages(), gaussians.py:323-324
  const bool high = avg >= cfg.grad_threshold;
  double ms = exp((double)c.log_scales[3 * i]);
  ms = fmax(ms, exp((double)c.log_scales[3 * i + 1]));
  ms = fmax(ms, exp((double)c.log_scales[3 * i + 2]));
  const bool small = ms <= cfg.percent_dense * cfg.extent;
  const bool sp = high && !small;
  keep[i] = !(prune || sp);
  clone[i] = high && small && !prune;
  split[i] = sp && !prune;
}

struct DensityMap {
  const uint32_t *keep, *clone, *split;
  const uint64_t *keep_off, *clone_off, *split_off, *totals;  // totals: n_keep, n_clone, n_split
  int32_t* src;   // [cap] source row
  int32_t* aux;   // [cap] -1 keep / clone; split: sample set * n_split + sample row
};

__global__ void __launch_bounds__(kT) k_density_map(DensityMap m, int64_t K, int64_t cap, int32_t* counts,
                                                    int32_t* status) {
  const uint64_t nk = m.totals[0], nc = m.totals[1], ns = m.totals[2];
  const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (i == 0 && counts) {
    counts[0] = (int32_t)nk;
    counts[1] = (int32_t)nc;
    counts[2] = (int32_t)ns;
    counts[3] = (int32_t)(nk + nc + 2 * ns);
  }
  if ((int64_t)(nk + nc + 2 * ns) > cap) {
    if (i == 0) raise_status(status, FS4D_ERR_CAPACITY);
    return;
  }
  if (i >= K) return;
  if (m.keep[i]) {
    const uint64_t d = m.keep_off[i];
    m.src[d] = (int32_t)i;
    m.aux[d] = -1;
  }
  if (m.clone[i]) {
    const uint64_t d = nk + m.clone_off[i];
    m.src[d] = (int32_t)i;
    m.aux[d] = -1;
  }
  if (m.split[i]) {
    const uint64_t s = m.split_off[i], d = nk + nc + s;
    m.src[d] = (int32_t)i;
    m.aux[d] = (int32_t)s;
    m.src[d + ns] = (int32_t)i;
    m.aux[d + ns] = (int32_t)(ns + s);
  }
}

struct DensityGather {
  Fs4dCloud in, out;
  const int32_t *src, *aux;
  const double* normals;  // [2, n_split, 3] standard normals (host rng)
  double log_split;       // log(split_factor)
  int n_rows;             // rows [0, n_rows) of the output
  int n_new_from;         // first row that is new (clone / split): Adam moments are zero there
  // extra per-row arrays compacted with the same map (Adam moments, ...):
  // rows < n_new_from copy src, rows >= n_new_from are zero
  const double *st_acc_in, *st_cnt_in;  // ViewspaceGradStats in (prune_only compacts them)
  double *st_acc_out, *st_cnt_out;      // out; zeroed when st_reset (densify_and_prune)
  int st_reset;
  int n_extra;
  const float* extra_in[32];
  float* extra_out[32];
  int extra_width[32];
  int32_t* status;
};

__global__ void __launch_bounds__(kT) k_density_gather(const __grid_constant__ DensityGather g) {
  const int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (r >= g.n_rows) return;
  const int64_t s = g.src[r];
  const int aux = g.aux[r];
  const Fs4dCloud& a = g.in;
  const Fs4dCloud& b = g.out;
  double pos[3] = {a.positions[3 * s], a.positions[3 * s + 1], a.positions[3 * s + 2]};
  double ls[3] = {a.log_scales[3 * s], a.log_scales[3 * s + 1], a.log_scales[3 * s + 2]};
  if (aux >= 0) {  // split child (gaussians.py:380-392)
    const double q0 = a.rotations[4 * s], q1 = a.rotations[4 * s + 1], q2 = a.rotations[4 * s + 2],
                 q3 = a.rotations[4 * s + 3];
    const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    if (qn < 1e-12) {  // normalize_quats raises (gaussians.py:174-178)
      atomicMin(&g.status[FS4D_ST_DEGEN_INDEX], (int32_t)s);
      raise_status(g.status, FS4D_ERR_DEGENERATE);
    }
    const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
    const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                            {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                            {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    const double* zs = g.normals + 3 * (int64_t)aux;
    const double smp[3] = {zs[0] * exp(ls[0]), zs[1] * exp(ls[1]), zs[2] * exp(ls[2])};
#pragma unroll
    for (int k = 0; k < 3; ++k) pos[k] += R[k][0] * smp[0] + R[k][1] * smp[1] + R[k][2] * smp[2];
#pragma unroll
    for (int k = 0; k < 3; ++k) ls[k] -= g.log_split;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    b.positions[3 * r + k] = (float)pos[k];
    b.log_scales[3 * r + k] = (float)ls[k];
    b.colors_raw[3 * r + k] = a.colors_raw[3 * s + k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) b.rotations[4 * r + k] = a.rotations[4 * s + k];
  b.opacity_logits[r] = a.opacity_logits[s];
  for (int k = 0; k < a.D; ++k) b.features[(int64_t)a.D * r + k] = a.features[(int64_t)a.D * s + k];
  if (a.sh_degree > 0) {
    const int n = ((a.sh_degree + 1) * (a.sh_degree + 1) - 1) * 3;
    for (int k = 0; k < n; ++k) b.sh_rest[(int64_t)n * r + k] = a.sh_rest[(int64_t)n * s + k];
  }
  if (g.st_acc_out) {  // gaussians.py:397-398 (reset) / 414-415 (compacted)
    g.st_acc_out[r] = g.st_reset ? 0.0 : g.st_acc_in[s];
    g.st_cnt_out[r] = g.st_reset ? 0.0 : g.st_cnt_in[s];
  }
  const bool fresh = r >= g.n_new_from;  // _remap_adam pads zeros (gaussians.py:336-346)
  for (int e = 0; e < g.n_extra; ++e) {
    const int wd = g.extra_width[e];
    for (int k = 0; k < wd; ++k)
      g.extra_out[e][(int64_t)wd * r + k] = fresh ? 0.f : g.extra_in[e][(int64_t)wd * s + k];
  }
}

// reset_opacity (gaussians.py:420-425): logit(min(sigmoid(x), cap)) in fp64
__global__ void __launch_bounds__(kT) k_reset_opacity(float* __restrict__ ol, int64_t K, double cap) {
  const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (i >= K) return;
  const double p = fmin(sigmoid_dd((double)ol[i]), cap);
  ol[i] = (float)(log(p) - log1p(-p));
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct DensityLayout {
  size_t keep, clone, split, keep_off, clone_off, split_off, totals, src, aux, scratch, total;
};

static DensityLayout density_layout(int64_t K, int64_t cap) {
  DensityLayout L;
  size_t o = 0;
  auto take = [&](size_t b) {
    const size_t at = o;
    o += (b + 255) / 256 * 256;
    return at;
  };
  L.keep = take(4 * (size_t)K);
  L.clone = take(4 * (size_t)K);
  L.split = take(4 * (size_t)K);
  L.keep_off = take(8 * (size_t)K);
  L.clone_off = take(8 * (size_t)K);
  L.split_off = take(8 * (size_t)K);
  L.totals = take(8 * 4);
  L.src = take(4 * (size_t)cap);
  L.aux = take(4 * (size_t)cap);
  L.scratch = take(scan_scratch_bytes(K));
  L.total = o;
  return L;
}

size_t density_workspace_bytes(int64_t K, int64_t cap) { return density_layout(K, cap).total; }

int stats_add(double* accum, double* count, const int32_t* idx, const float* norms, int64_t n, const int32_t* n_dev,
              cudaStream_t s) {
  if (n <= 0) return FS4D_OK;
  k_stats_add<<<(unsigned)std::min<int64_t>(ceil_div(n, kT), kNumSMs * 8), kT, 0, s>>>(accum, count, idx, norms, n,
                                                                                      n_dev);
  return check_launch("stats_add");
}

int density_classify(const Fs4dCloud& c, const double* accum, const double* count, const Fs4dDensityConfig& cfg,
                     int prune_only, int64_t cap, int32_t* counts, void* ws, size_t ws_bytes, int32_t* status,
                     cudaStream_t s) {
  const int64_t K = c.K;
  const DensityLayout L = density_layout(K, cap);
  if (!ws || ws_bytes < L.total) return fail(FS4D_ERR_CONFIG, "density workspace too small");
  char* b = (char*)ws;
  uint32_t *keep = (uint32_t*)(b + L.keep), *clone = (uint32_t*)(b + L.clone), *split = (uint32_t*)(b + L.split);
  uint64_t* totals = (uint64_t*)(b + L.totals);
  if (K > 0) {
    k_density_classify<<<(unsigned)ceil_div(K, kT), kT, 0, s>>>(c, accum, count, cfg, prune_only, keep, clone, split);
    exclusive_scan_u32_to_u64(keep, (uint64_t*)(b + L.keep_off), K, nullptr, totals + 0, b + L.scratch, s);
    exclusive_scan_u32_to_u64(clone, (uint64_t*)(b + L.clone_off), K, nullptr, totals + 1, b + L.scratch, s);
    exclusive_scan_u32_to_u64(split, (uint64_t*)(b + L.split_off), K, nullptr, totals + 2, b + L.scratch, s);
  } else {
    cudaMemsetAsync(totals, 0, 8 * 3, s);
  }
  DensityMap m{keep, clone, split, (const uint64_t*)(b + L.keep_off), (const uint64_t*)(b + L.clone_off),
               (const uint64_t*)(b + L.split_off), totals, (int32_t*)(b + L.src), (int32_t*)(b + L.aux)};
  k_density_map<<<(unsigned)std::max<int64_t>(1, ceil_div(K, kT)), kT, 0, s>>>(m, K, cap, counts, status);
  return check_launch("density_classify");
}

int density_apply(const Fs4dCloud& in, const double* normals, const Fs4dDensityConfig& cfg, int64_t cap,
                  int32_t n_keep, int32_t n_clone, int32_t n_split, Fs4dCloud& out, const double* st_acc_in,
                  const double* st_cnt_in, double* st_acc_out, double* st_cnt_out, int st_reset, int n_extra,
                  const float* const* extra_in, float* const* extra_out, const int32_t* extra_width, void* ws,
                  size_t ws_bytes, int32_t* status, cudaStream_t s) {
  const DensityLayout L = density_layout(in.K, cap);
  if (!ws || ws_bytes < L.total) return fail(FS4D_ERR_CONFIG, "density workspace too small");
  if (n_extra < 0 || n_extra > 32) return fail(FS4D_ERR_CONFIG, "at most 32 extra per-row arrays");
  const int64_t n_rows = (int64_t)n_keep + n_clone + 2 * (int64_t)n_split;
  if (n_rows > cap || out.K < n_rows) return fail(FS4D_ERR_CAPACITY, "density output capacity too small");
  if (n_split > 0 && !normals) return fail(FS4D_ERR_CONFIG, "split samples missing");
  DensityGather g;
  g.in = in;
  g.out = out;
  char* b = (char*)ws;
  g.src = (const int32_t*)(b + L.src);
  g.aux = (const int32_t*)(b + L.aux);
  g.normals = normals;
  g.log_split = log(cfg.split_factor);
  g.n_rows = (int)n_rows;
  g.n_new_from = n_keep;
  g.st_acc_in = st_acc_in;
  g.st_cnt_in = st_cnt_in;
  g.st_acc_out = st_acc_out;
  g.st_cnt_out = st_cnt_out;
  g.st_reset = st_reset;
  g.n_extra = n_extra;
  for (int e = 0; e < n_extra; ++e) {
    g.extra_in[e] = extra_in[e];
    g.extra_out[e] = extra_out[e];
    g.extra_width[e] = extra_width[e];
  }
  g.status = status;
  if (n_rows > 0) k_density_gather<<<(unsigned)ceil_div(n_rows, kT), kT, 0, s>>>(g);
  return check_launch("density_apply");
}

int reset_opacity(float* ol, int64_t K, double cap, cudaStream_t s) {
  if (K > 0) k_reset_opacity<<<(unsigned)ceil_div(K, kT), kT, 0, s>>>(ol, K, cap);
  return check_launch("reset_opacity");
}

}  // namespace fs4d
