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
//             dgamma[c] += sum dz*xhat, dbeta[c] += sum dz (fp32 atomics from
//             per-CTA shared-memory partials)
// Each CTA reads its part of the slab two or three times; the later reads
// hit L1/L2.
#include "sdp_common.cuh"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace sdp {

constexpr int kGnThreads = 256;
constexpr int kGnMaxC = 1024;  // channels per group handled by the shared partials

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

// A cluster of kGnCluster CTAs per (sample, group), each over a contiguous
// range of pixels of the group's slab; the group statistics are reduced
// across the cluster through distributed shared memory.  Element e of a CTA's
// range -> (pixel, channel): e = pixel * cg + k.
constexpr int kGnCluster = 8;

__device__ __forceinline__ float cluster_sum(cg::cluster_group& cl, float* s_part, float v) {
  // v: this CTA's block-reduced partial (valid in every thread)
  if (threadIdx.x == 0) *s_part = v;
  cl.sync();
  float t = 0.f;
#pragma unroll
  for (int r = 0; r < kGnCluster; ++r) t += *cl.map_shared_rank(s_part, r);
  cl.sync();  // every CTA has read every partial before any is overwritten
  return t;
}

template <bool RELU>
__global__ void __cluster_dims__(kGnCluster, 1, 1) __launch_bounds__(kGnThreads)
k_gn_fwd(const __nv_bfloat16* __restrict__ x, int hw, int c, const int32_t* __restrict__ gs, int groups,
         const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
         __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ float s_part;
  const int bg = blockIdx.x / kGnCluster, part = static_cast<int>(cl.block_rank());
  const int b = bg / groups, g = bg % groups;
  const int c0 = gs[g], cg_ = gs[g + 1] - c0;
  const int per = (hw + kGnCluster - 1) / kGnCluster;
  const int p0 = min(hw, part * per), p1 = min(hw, p0 + per);
  const int64_t base = (static_cast<int64_t>(b) * hw + p0) * c + c0;
  const int n = (p1 - p0) * cg_;
  const float n_all = static_cast<float>(hw) * cg_;
  // two passes (the second hits L1/L2): mean, then the centred sum of squares
  float s0 = 0.f, unused = 0.f;
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const int pix = e / cg_, k = e - pix * cg_;
    s0 += __bfloat162float(x[base + static_cast<int64_t>(pix) * c + k]);
  }
  block_sum2<kGnThreads>(s0, unused);
  const float mean = cluster_sum(cl, &s_part, s0) / n_all;
  float sq = 0.f;
  unused = 0.f;
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const int pix = e / cg_, k = e - pix * cg_;
    const float d = __bfloat162float(x[base + static_cast<int64_t>(pix) * c + k]) - mean;
    sq += d * d;
  }
  block_sum2<kGnThreads>(sq, unused);
  const float rstd = rsqrtf(cluster_sum(cl, &s_part, sq) / n_all + eps);
  if (part == 0 && threadIdx.x == 0) {
    mean_out[bg] = mean;
    rstd_out[bg] = rstd;
  }
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const int pix = e / cg_, k = e - pix * cg_;
    const int64_t i = base + static_cast<int64_t>(pix) * c + k;
    float v = (__bfloat162float(x[i]) - mean) * rstd * gamma[c0 + k] + beta[c0 + k];
    if (RELU) v = fmaxf(v, 0.f);
    y[i] = __float2bfloat16_rn(v);
  }
}

template <bool RELU>
__global__ void __cluster_dims__(kGnCluster, 1, 1) __launch_bounds__(kGnThreads)
k_gn_bwd(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ y,
         const __nv_bfloat16* __restrict__ dy, int hw, int c, const int32_t* __restrict__ gs, int groups,
         const float* __restrict__ gamma, const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
         __nv_bfloat16* __restrict__ dx, float* __restrict__ dgamma, float* __restrict__ dbeta) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ float s_dg[kGnMaxC], s_db[kGnMaxC];
  __shared__ float s_part;
  const int bg = blockIdx.x / kGnCluster, part = static_cast<int>(cl.block_rank());
  const int b = bg / groups, g = bg % groups;
  const int c0 = gs[g], cg_ = gs[g + 1] - c0;
  const int per = (hw + kGnCluster - 1) / kGnCluster;
  const int p0 = min(hw, part * per), p1 = min(hw, p0 + per);
  const int64_t base = (static_cast<int64_t>(b) * hw + p0) * c + c0;
  const int n = (p1 - p0) * cg_;
  const float mean = mean_in[bg], rstd = rstd_in[bg];
  for (int k = threadIdx.x; k < cg_; k += kGnThreads) {
    s_dg[k] = 0.f;
    s_db[k] = 0.f;
  }
  __syncthreads();
  // a thread's channel is fixed when the group width divides the CTA width
  // (every equal-group layer): per-channel partials stay in registers
  const bool fixed = (kGnThreads % cg_) == 0;
  float s1 = 0.f, s2 = 0.f, pg = 0.f, pb = 0.f;
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const int pix = e / cg_, k = e - pix * cg_;
    const int64_t i = base + static_cast<int64_t>(pix) * c + k;
    float dz = __bfloat162float(dy[i]);
    if (RELU && !(__bfloat162float(y[i]) > 0.f)) dz = 0.f;
    const float xh = (__bfloat162float(x[i]) - mean) * rstd;
    const float dzg = dz * gamma[c0 + k];
    s1 += dzg;
    s2 += dzg * xh;
    if (fixed) {
      pg += dz * xh;
      pb += dz;
    } else {
      atomicAdd(&s_dg[k], dz * xh);
      atomicAdd(&s_db[k], dz);
    }
  }
  if (fixed && threadIdx.x < n) {
    const int k = threadIdx.x % cg_;
    atomicAdd(&s_dg[k], pg);
    atomicAdd(&s_db[k], pb);
  }
  block_sum2<kGnThreads>(s1, s2);
  const float inv_n = 1.f / (static_cast<float>(hw) * cg_);
  s1 = cluster_sum(cl, &s_part, s1) * inv_n;
  s2 = cluster_sum(cl, &s_part, s2) * inv_n;
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const int pix = e / cg_, k = e - pix * cg_;
    const int64_t i = base + static_cast<int64_t>(pix) * c + k;
    float dz = __bfloat162float(dy[i]);
    if (RELU && !(__bfloat162float(y[i]) > 0.f)) dz = 0.f;
    const float xh = (__bfloat162float(x[i]) - mean) * rstd;
    dx[i] = __float2bfloat16_rn(rstd * (dz * gamma[c0 + k] - s1 - xh * s2));
  }
  __syncthreads();
  for (int k = threadIdx.x; k < cg_; k += kGnThreads) {
    atomicAdd(&dgamma[c0 + k], s_dg[k]);
    atomicAdd(&dbeta[c0 + k], s_db[k]);
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
                       int groups, int max_group_channels, const float* gamma, const float* beta, float eps,
                       int relu, void* y_bf16, float* mean, float* rstd, void* stream) {
  if (int rc = check_groups(batch, hw, channels, groups)) return rc;
  if (max_group_channels > kGnMaxC) return set_error(SDP_ERR_USAGE, "a group of more than %d channels", kGnMaxC);
  if (batch == 0) return SDP_OK;
  const unsigned grid = static_cast<unsigned>(batch) * groups * kGnCluster;
  cudaStream_t s = as_stream(stream);
  auto xb = static_cast<const __nv_bfloat16*>(x_bf16);
  auto yb = static_cast<__nv_bfloat16*>(y_bf16);
  if (relu)
    k_gn_fwd<true><<<grid, kGnThreads, 0, s>>>(xb, hw, channels, group_starts, groups, gamma, beta, eps, yb, mean, rstd);
  else
    k_gn_fwd<false><<<grid, kGnThreads, 0, s>>>(xb, hw, channels, group_starts, groups, gamma, beta, eps, yb, mean, rstd);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_group_norm_bwd(const void* x_bf16, const void* y_bf16, const void* dy_bf16, int batch, int hw,
                       int channels, const int32_t* group_starts, int groups, int max_group_channels,
                       const float* gamma, const float* mean, const float* rstd, int relu, void* dx_bf16,
                       float* dgamma, float* dbeta, void* stream) {
  if (int rc = check_groups(batch, hw, channels, groups)) return rc;
  if (max_group_channels > kGnMaxC) return set_error(SDP_ERR_USAGE, "a group of more than %d channels", kGnMaxC);
  if (batch == 0) return SDP_OK;
  const unsigned grid = static_cast<unsigned>(batch) * groups * kGnCluster;
  cudaStream_t s = as_stream(stream);
  auto xb = static_cast<const __nv_bfloat16*>(x_bf16);
  auto yb = static_cast<const __nv_bfloat16*>(y_bf16);
  auto db = static_cast<const __nv_bfloat16*>(dy_bf16);
  auto dxb = static_cast<__nv_bfloat16*>(dx_bf16);
  if (relu)
    k_gn_bwd<true><<<grid, kGnThreads, 0, s>>>(xb, yb, db, hw, channels, group_starts, groups, gamma, mean, rstd,
                                              dxb, dgamma, dbeta);
  else
    k_gn_bwd<false><<<grid, kGnThreads, 0, s>>>(xb, yb, db, hw, channels, group_starts, groups, gamma, mean, rstd,
                                               dxb, dgamma, dbeta);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
