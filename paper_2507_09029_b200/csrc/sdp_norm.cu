// Channels-last GroupNorm (+ optional fused ReLU) over contiguous, possibly
// ragged channel groups -- the active-channel GroupNorm of a compact
// width-wise subnetwork (ops.py:140-204: statistics over each group's live
// channels only), and plain GroupNorm when the groups are equal.
//
// Layout: x, y, dy, dx are bf16 [B, HW, C] (PyTorch channels_last), group g
// covers channels [gs[g], gs[g+1]).  A thread-block cluster of 8 CTAs per
// (sample, group), each over 1/8 of the pixels, reducing the group sums
// through distributed shared memory:
//   k_gn_fwd  mean, then centred variance (fp32, two passes) over the
//             group's HW x Cg elements, then
//             y = act((x - mean) * rstd * gamma[c] + beta[c])
//   k_gn_bwd  with dz = dy * [y > 0] (ReLU) and xhat recomputed:
//             s1 = sum dz*gamma, s2 = sum dz*gamma*xhat over the group;
//             dx = rstd * (dz*gamma - s1/n - xhat * s2/n);
//             dgamma[c] = sum dz*xhat, dbeta[c] = sum dz through per-CTA
//             partial rows and an ordered fold (deterministic: no atomics)
// Each CTA reads its part of the slab two or three times; the later reads
// hit L1/L2.
#include "sdp_common.cuh"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace sdp {

constexpr int kGnThreads = 256;
constexpr int kGnMaxC = 1024;  // channels per group handled by the shared partials
constexpr int kGnU = 8;        // pixels per thread per round in the backward (loads in flight)

template <int NT>
__device__ __forceinline__ void block_sum2(float& a, float& b) {
  __shared__ float sa[NT / 32], sb[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sa[warp] = a;
    sb[warp] = b;
  }
  __syncthreads();
  a = lane < NT / 32 ? sa[lane] : 0.f;
  b = lane < NT / 32 ? sb[lane] : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
}

// A cluster of up to kGnCluster CTAs per (sample, group), each over a contiguous
// range of pixels of the group's slab; the group statistics are reduced
// across the cluster through distributed shared memory.  Element e of a CTA's
// range -> (pixel, channel): e = pixel * cg + k.
constexpr int kGnCluster = 8;

// CTAs per (sample, group): enough that each has >= 2048 elements of work,
// a power of two <= kGnPartsCap (small late-layer slabs: fewer CTAs, fewer
// cluster barriers).  Same-box A/B of graphed ResNet-18 steps (batch 64, 2
// groups): cap 8 / 4 / 2 / 1 -> C2 9.5 / 9.1 / 9.3 / 10.1 ms, DP 12.6 / 12.0
// / 12.2 / 13.5 ms GPU time; 8-CTA clusters of the 32x32 layers ran in two
// waves of co-scheduled clusters.
constexpr int kGnPartsCap = 4;

static int gn_parts(int hw, int max_cg) {
  const int64_t slab = static_cast<int64_t>(hw) * max_cg;
  int parts = 1;
  while (parts < kGnPartsCap && slab / (2 * parts) >= 2048) parts *= 2;
  return parts;
}

template <typename Kernel, typename... Args>
static cudaError_t launch_clustered(Kernel k, unsigned grid, int parts, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGnThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = parts;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

__device__ __forceinline__ void cluster_sum2(cg::cluster_group& cl, float2* s_part, float& a, float& b) {
  // a, b: this CTA's block-reduced partials (valid in every thread)
  if (threadIdx.x == 0) *s_part = make_float2(a, b);
  cl.sync();
  float ta = 0.f, tb = 0.f;
  const int nb = static_cast<int>(cl.num_blocks());
  for (int r = 0; r < nb; ++r) {
    const float2 v = *cl.map_shared_rank(s_part, r);
    ta += v.x;
    tb += v.y;
  }
  cl.sync();  // every CTA has read every partial before any is overwritten
  a = ta;
  b = tb;
}

// 8 channels per 16-B vector when the group's channel range and the row
// pitch are 8-aligned (every equal-group layer); otherwise one channel per
// element.  The slab walk is (pixel, channel-vector) with the vector index
// fixed per thread when the CTA width is a multiple of the vectors per pixel.
struct Bf8 {
  float v[8];
};

__device__ __forceinline__ Bf8 ld8(const __nv_bfloat16* p) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  Bf8 r;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    r.v[2 * k] = f.x;
    r.v[2 * k + 1] = f.y;
  }
  return r;
}

__device__ __forceinline__ void st8(__nv_bfloat16* p, const float* v) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// gamma / beta in fp32 or bf16 (the parameter's own dtype: no cast kernels)
struct Affine {
  const void* p;
  bool bf16;
  __device__ __forceinline__ float operator[](int i) const {
    return bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]) : static_cast<const float*>(p)[i];
  }
};

struct GnSlab {
  int b, g, c0, cg, p0, p1;
  int64_t base;  // element (p0, c0) of sample b
};

__device__ __forceinline__ GnSlab gn_slab(int bg, int part, int parts, int hw, int c, const int32_t* gs,
                                          int groups) {
  GnSlab t;
  t.b = bg / groups;
  t.g = bg % groups;
  t.c0 = gs[t.g];
  t.cg = gs[t.g + 1] - t.c0;
  const int per = (hw + parts - 1) / parts;
  t.p0 = min(hw, part * per);
  t.p1 = min(hw, t.p0 + per);
  t.base = (static_cast<int64_t>(t.b) * hw + t.p0) * c + t.c0;
  return t;
}

template <bool RELU, bool VEC>
__global__ void __launch_bounds__(kGnThreads, 4)
k_gn_fwd(const __nv_bfloat16* __restrict__ x, int hw, int c, const int32_t* __restrict__ gs, int groups,
         const Affine gamma, const Affine beta, float eps,
         __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ float2 s_part;
  const int parts = static_cast<int>(cl.num_blocks());
  const int bg = blockIdx.x / parts, part = static_cast<int>(cl.block_rank());
  const GnSlab t = gn_slab(bg, part, parts, hw, c, gs, groups);
  const float n_all = static_cast<float>(hw) * t.cg;
  constexpr bool vec = VEC;  // host-checked: every group start, C and the pointers 8-aligned
  const int cv = vec ? t.cg / 8 : t.cg;                // vectors (or channels) per pixel
  const int nv = (t.p1 - t.p0) * cv;
  // one pass: sums of (x - K) and (x - K)^2 around the group's first element
  // K (every CTA reads the same K), so the variance does not cancel
  const float K = __bfloat162float(x[static_cast<int64_t>(t.b) * hw * c + t.c0]);
  // UF items per thread per round, all loads issued before the arithmetic
  constexpr int UF = vec ? 4 : 8;
  float s0 = 0.f, sq = 0.f;
  for (int q0 = threadIdx.x; q0 < nv; q0 += UF * kGnThreads) {
    if (vec) {
      Bf8 r[UF];
#pragma unroll
      for (int u = 0; u < UF; ++u) {
        const int q = q0 + u * kGnThreads;
        const int pix = q / cv, kv = q - pix * cv;
        if (q < nv) r[u] = ld8(x + t.base + static_cast<int64_t>(pix) * c + kv * 8);
      }
#pragma unroll
      for (int u = 0; u < UF; ++u)
        if (q0 + u * kGnThreads < nv) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float d = r[u].v[k] - K;
            s0 += d;
            sq += d * d;
          }
        }
    } else {
      float v[UF];
#pragma unroll
      for (int u = 0; u < UF; ++u) {
        const int q = q0 + u * kGnThreads;
        const int pix = q / cv, kv = q - pix * cv;
        v[u] = q < nv ? __bfloat162float(x[t.base + static_cast<int64_t>(pix) * c + kv]) - K : 0.f;
      }
#pragma unroll
      for (int u = 0; u < UF; ++u) {
        s0 += v[u];
        sq += v[u] * v[u];
      }
    }
  }
  block_sum2<kGnThreads>(s0, sq);
  cluster_sum2(cl, &s_part, s0, sq);
  const float md = s0 / n_all;
  const float mean = K + md;
  const float rstd = rsqrtf(fmaxf(sq / n_all - md * md, 0.f) + eps);
  if (part == 0 && threadIdx.x == 0) {
    mean_out[bg] = mean;
    rstd_out[bg] = rstd;
  }
  for (int q = threadIdx.x; q < nv; q += kGnThreads) {
    const int pix = q / cv, kv = q - pix * cv;
    const int64_t i = t.base + static_cast<int64_t>(pix) * c + (vec ? kv * 8 : kv);
    if (vec) {
      const Bf8 r = ld8(x + i);
      float o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int ch = t.c0 + kv * 8 + k;
        o[k] = (r.v[k] - mean) * rstd * gamma[ch] + beta[ch];
        if (RELU) o[k] = fmaxf(o[k], 0.f);
      }
      st8(y + i, o);
    } else {
      float v = (__bfloat162float(x[i]) - mean) * rstd * gamma[t.c0 + kv] + beta[t.c0 + kv];
      if (RELU) v = fmaxf(v, 0.f);
      y[i] = __float2bfloat16_rn(v);
    }
  }
}

// Backward, deterministic end to end (no floating-point atomics):
//   k_gn_bwd       one CTA per (sample, group, part) as in the forward.  The
//                  thread -> (channel, pixel phase) map is fixed: cw = min(cg,
//                  256) channels per pass, pstep = 256 / cw phases per
//                  channel, so each thread keeps its channel's dgamma / dbeta
//                  partial in registers; the CTA folds the phases of a channel
//                  in ascending order and writes ONE partial row
//                  part[(b * parts + part) * C + c] for its group's channels.
//   k_gn_bwd_fold  sums the batch * parts partial rows of every channel in a
//                  fixed order and writes dgamma / dbeta in the affine dtype.
// Every partial-row entry is written by exactly one CTA, so the workspace
// needs no zeroing and calls need no counters.
template <bool RELU>
__global__ void __launch_bounds__(kGnThreads, 4)
k_gn_bwd(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ y,
         const __nv_bfloat16* __restrict__ dy, int hw, int c, const int32_t* __restrict__ gs, int groups,
         const Affine gamma, const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
         __nv_bfloat16* __restrict__ dx, float* __restrict__ part_g, float* __restrict__ part_b) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ float s_pg[kGnMaxC], s_pb[kGnMaxC];
  __shared__ float2 s_part;
  const int parts = static_cast<int>(cl.num_blocks());
  const int bg = blockIdx.x / parts, part = static_cast<int>(cl.block_rank());
  const GnSlab t = gn_slab(bg, part, parts, hw, c, gs, groups);
  const float mean = mean_in[bg], rstd = rstd_in[bg];
  const int npix = t.p1 - t.p0;
  const int cw = min(t.cg, kGnThreads);       // channels per pass
  const int pstep = kGnThreads / cw;          // pixel phases per channel
  const int ph = threadIdx.x / cw;            // this thread's phase (>= pstep: idle)
  const bool on = ph < pstep;
  const int kv0 = threadIdx.x - ph * cw;
  // pass 1: the group sums s1 = sum dz*gamma, s2 = sum dz*gamma*xhat and the
  // per-channel partials, kGnU pixels per round with all their loads in flight
  float s1 = 0.f, s2 = 0.f;
  if (on) {
    for (int kv = kv0; kv < t.cg; kv += cw) {
      const float gch = gamma[t.c0 + kv];
      const __nv_bfloat16* xb = x + t.base + kv;
      const __nv_bfloat16* yb = y + t.base + kv;
      const __nv_bfloat16* db = dy + t.base + kv;
      float pgs = 0.f, pbs = 0.f;
      for (int p0 = ph; p0 < npix; p0 += kGnU * pstep) {
        float vx[kGnU], vd[kGnU], vy[kGnU];
#pragma unroll
        for (int u = 0; u < kGnU; ++u) {
          const int pix = p0 + u * pstep;
          const int64_t o = static_cast<int64_t>(pix < npix ? pix : 0) * c;
          vx[u] = __bfloat162float(xb[o]);
          vd[u] = pix < npix ? __bfloat162float(db[o]) : 0.f;
          vy[u] = RELU ? __bfloat162float(yb[o]) : 1.f;
        }
#pragma unroll
        for (int u = 0; u < kGnU; ++u) {
          const float dz = RELU && !(vy[u] > 0.f) ? 0.f : vd[u];
          const float xh = (vx[u] - mean) * rstd;
          s1 += dz * gch;
          s2 += dz * gch * xh;
          pgs += dz * xh;
          pbs += dz;
        }
      }
      s_pg[ph * t.cg + kv] = pgs;
      s_pb[ph * t.cg + kv] = pbs;
    }
  }
  block_sum2<kGnThreads>(s1, s2);  // (its barriers also publish s_pg / s_pb)
  const float inv_n = 1.f / (static_cast<float>(hw) * t.cg);
  cluster_sum2(cl, &s_part, s1, s2);
  s1 *= inv_n;
  s2 *= inv_n;
  // this CTA's partial row: channel k = phases 0, 1, ... in order
  const int64_t row = static_cast<int64_t>(t.b * parts + part) * c + t.c0;
  for (int k = threadIdx.x; k < t.cg; k += kGnThreads) {
    float a = 0.f, b = 0.f;
    for (int r = 0; r < pstep; ++r) {
      a += s_pg[r * t.cg + k];
      b += s_pb[r * t.cg + k];
    }
    part_g[row + k] = a;
    part_b[row + k] = b;
  }
  // pass 2: dx (the slab re-read hits L1/L2)
  if (on) {
    for (int kv = kv0; kv < t.cg; kv += cw) {
      const float gch = gamma[t.c0 + kv];
      const __nv_bfloat16* xb = x + t.base + kv;
      const __nv_bfloat16* yb = y + t.base + kv;
      const __nv_bfloat16* db = dy + t.base + kv;
      __nv_bfloat16* dxb = dx + t.base + kv;
      for (int p0 = ph; p0 < npix; p0 += kGnU * pstep) {
        float vx[kGnU], vd[kGnU], vy[kGnU];
#pragma unroll
        for (int u = 0; u < kGnU; ++u) {
          const int pix = p0 + u * pstep;
          const int64_t o = static_cast<int64_t>(pix < npix ? pix : 0) * c;
          vx[u] = __bfloat162float(xb[o]);
          vd[u] = __bfloat162float(db[o]);
          vy[u] = RELU ? __bfloat162float(yb[o]) : 1.f;
        }
#pragma unroll
        for (int u = 0; u < kGnU; ++u) {
          const int pix = p0 + u * pstep;
          const float dz = RELU && !(vy[u] > 0.f) ? 0.f : vd[u];
          const float xh = (vx[u] - mean) * rstd;
          if (pix < npix) dxb[static_cast<int64_t>(pix) * c] = __float2bfloat16_rn(rstd * (dz * gch - s1 - xh * s2));
        }
      }
    }
  }
}

// 32 channels per CTA; warp w sums partial rows w, w + 8, ... in ascending
// order (loads batched), then the 8 warp sums fold in warp order.
constexpr int kGnFoldWarps = 8;
__global__ void __launch_bounds__(32 * kGnFoldWarps)
k_gn_bwd_fold(const float* __restrict__ part_g, const float* __restrict__ part_b, int rows, int c,
              void* __restrict__ dgamma, void* __restrict__ dbeta, bool bf16) {
  __shared__ float s_g[kGnFoldWarps][32], s_b[kGnFoldWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  float a = 0.f, b = 0.f;
  if (col < c) {
    constexpr int U = 4;
    for (int r0 = warp; r0 < rows; r0 += U * kGnFoldWarps) {
      float va[U], vb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u * kGnFoldWarps;
        va[u] = r < rows ? part_g[static_cast<int64_t>(r) * c + col] : 0.f;
        vb[u] = r < rows ? part_b[static_cast<int64_t>(r) * c + col] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a += va[u];
        b += vb[u];
      }
    }
  }
  s_g[warp][lane] = a;
  s_b[warp][lane] = b;
  __syncthreads();
  if (warp == 0 && col < c) {
    float ta = 0.f, tb = 0.f;
#pragma unroll
    for (int w = 0; w < kGnFoldWarps; ++w) {
      ta += s_g[w][lane];
      tb += s_b[w][lane];
    }
    if (bf16) {
      static_cast<__nv_bfloat16*>(dgamma)[col] = __float2bfloat16_rn(ta);
      static_cast<__nv_bfloat16*>(dbeta)[col] = __float2bfloat16_rn(tb);
    } else {
      static_cast<float*>(dgamma)[col] = ta;
      static_cast<float*>(dbeta)[col] = tb;
    }
  }
}

static int check_groups(int b, int hw, int c, int groups) {
  if (b < 0 || hw < 1 || c < 1 || groups < 1) return set_error(SDP_ERR_USAGE, "bad group-norm shape");
  return SDP_OK;
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_group_norm_fwd(const void* x_bf16, int batch, int hw, int channels, const int32_t* group_starts,
                       int groups, int max_group_channels, const void* gamma, const void* beta, float eps,
                       int flags, void* y_bf16, float* mean, float* rstd, void* stream) {
  const bool relu = flags & SDP_GN_RELU;
  const Affine ga{gamma, (flags & SDP_GN_AFFINE_BF16) != 0}, be{beta, (flags & SDP_GN_AFFINE_BF16) != 0};
  if (int rc = check_groups(batch, hw, channels, groups)) return rc;
  if (max_group_channels > kGnMaxC) return set_error(SDP_ERR_USAGE, "a group of more than %d channels", kGnMaxC);
  if (batch == 0) return SDP_OK;
  const int parts = gn_parts(hw, max_group_channels);
  const unsigned grid = static_cast<unsigned>(batch) * groups * parts;
  cudaStream_t s = as_stream(stream);
  auto xb = static_cast<const __nv_bfloat16*>(x_bf16);
  auto yb = static_cast<__nv_bfloat16*>(y_bf16);
  const bool vec = (flags & SDP_GN_GROUPS_ALIGNED8) && (channels % 8) == 0 &&
                   ((reinterpret_cast<uintptr_t>(x_bf16) | reinterpret_cast<uintptr_t>(y_bf16)) & 15) == 0;
#define SDP_GN_FWD(R, V)                                                                                \
  SDP_CUDA_CHECK(launch_clustered(k_gn_fwd<R, V>, grid, parts, s, xb, hw, channels, group_starts, groups, \
                                  ga, be, eps, yb, mean, rstd))
  if (relu) {
    if (vec) SDP_GN_FWD(true, true); else SDP_GN_FWD(true, false);
  } else {
    if (vec) SDP_GN_FWD(false, true); else SDP_GN_FWD(false, false);
  }
#undef SDP_GN_FWD
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_group_norm_bwd_scratch(int batch, int hw, int channels, int max_group_channels, long long* floats) {
  if (!floats) return set_error(SDP_ERR_USAGE, "null output");
  if (batch < 0 || hw < 1 || channels < 1 || max_group_channels < 1)
    return set_error(SDP_ERR_USAGE, "bad group-norm shape");
  *floats = 2ll * batch * gn_parts(hw, max_group_channels) * channels;
  return SDP_OK;
}

int sdp_group_norm_bwd(const void* x_bf16, const void* y_bf16, const void* dy_bf16, int batch, int hw,
                       int channels, const int32_t* group_starts, int groups, int max_group_channels,
                       const void* gamma, const float* mean, const float* rstd, int flags, void* dx_bf16,
                       void* dgamma, void* dbeta, float* scratch, long long scratch_floats, void* stream) {
  const bool relu = flags & SDP_GN_RELU;
  const bool bf16 = (flags & SDP_GN_AFFINE_BF16) != 0;
  const Affine ga{gamma, bf16};
  if (int rc = check_groups(batch, hw, channels, groups)) return rc;
  if (max_group_channels > kGnMaxC) return set_error(SDP_ERR_USAGE, "a group of more than %d channels", kGnMaxC);
  if (batch == 0) return set_error(SDP_ERR_USAGE, "group-norm backward needs batch > 0");
  if (!dgamma || !dbeta || !scratch) return set_error(SDP_ERR_USAGE, "null device pointer");
  const int parts = gn_parts(hw, max_group_channels);
  const int64_t rows = static_cast<int64_t>(batch) * parts;
  if (scratch_floats < 2 * rows * channels)
    return set_error(SDP_ERR_USAGE, "group-norm backward scratch holds %lld floats, needs %lld", scratch_floats,
                     static_cast<long long>(2 * rows * channels));
  const unsigned grid = static_cast<unsigned>(batch) * groups * parts;
  cudaStream_t s = as_stream(stream);
  auto xb = static_cast<const __nv_bfloat16*>(x_bf16);
  auto yb = static_cast<const __nv_bfloat16*>(y_bf16);
  auto db = static_cast<const __nv_bfloat16*>(dy_bf16);
  auto dxb = static_cast<__nv_bfloat16*>(dx_bf16);
  float* pg = scratch;
  float* pb = scratch + rows * channels;
  if (relu)
    SDP_CUDA_CHECK(launch_clustered(k_gn_bwd<true>, grid, parts, s, xb, yb, db, hw, channels, group_starts, groups,
                                    ga, mean, rstd, dxb, pg, pb));
  else
    SDP_CUDA_CHECK(launch_clustered(k_gn_bwd<false>, grid, parts, s, xb, yb, db, hw, channels, group_starts, groups,
                                    ga, mean, rstd, dxb, pg, pb));
  SDP_LAUNCH_CHECK();
  k_gn_bwd_fold<<<(channels + 31) / 32, 32 * kGnFoldWarps, 0, s>>>(pg, pb, static_cast<int>(rows), channels, dgamma,
                                                                  dbeta, bf16);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
