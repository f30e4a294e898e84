// Row LayerNorm on bf16 activations (GPT-2 blocks of the C4 training step,
// train._layer_norm): y = (x - mean) * rstd * gamma + beta over the last dim.
//
// Layout: x, y, dy, dx bf16 [rows, cols] row-major, cols = 256 * V (V = 1..8:
// one warp per row, each lane V 16-B vectors of 8 bf16); gamma / beta bf16
// [cols]; mean / rstd fp32 [rows] saved for the backward.
//   k_ln_fwd       the row stays in registers: mean, then the centred
//                  variance (two passes over registers, fp32), one write.
//   k_ln_bwd       xhat recomputed from the saved statistics;
//                  dx = rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat));
//                  every lane keeps its columns' dgamma / dbeta partial sums
//                  in registers over the rows its warp visits, the CTA folds
//                  its warps (a fixed tree through shared memory) and writes
//                  one partial row.
//   k_ln_bwd_fold  sums the per-CTA partial rows in a fixed order
//                  (deterministic, no atomics) and writes bf16 dgamma / dbeta.
// HBM bytes per element: fwd 2 read + 2 write; bwd 4 read (x, dy) + 2 write.
#include "sdp_common.cuh"

namespace sdp {

constexpr int kLnThreads = 256;
constexpr int kLnWarps = kLnThreads / 32;
constexpr int kLnMaxV = 8;  // cols <= 2048

__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {  // streamed once: no L1 allocation
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
  return u;
}

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

__device__ __forceinline__ float warp_sum(float a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// column of lane l's vector k: 256 * k + 8 * l (+ 0..7)
template <int V>
__global__ void __launch_bounds__(kLnThreads) k_ln_fwd(const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                        const __nv_bfloat16* __restrict__ gamma,
                                                        const __nv_bfloat16* __restrict__ beta, float eps,
                                                        __nv_bfloat16* __restrict__ y, float* __restrict__ mean,
                                                        float* __restrict__ rstd,
                                                        const __nv_bfloat16* __restrict__ x2,
                                                        __nv_bfloat16* __restrict__ sum_out) {
  constexpr int cols = 256 * V;
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kLnWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  float v[V][8];
#pragma unroll
  for (int k = 0; k < V; ++k) unpack8(ld_nc_v4(xr + 32 * k + lane), v[k]);
  if (x2) {  // fused residual add: s = bf16(x + x2) is both an output and the normalised row
    const uint4* x2r = reinterpret_cast<const uint4*>(x2 + row * cols);
    uint4* sr = reinterpret_cast<uint4*>(sum_out + row * cols);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float w[8];
      unpack8(ld_nc_v4(x2r + 32 * k + lane), w);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[k][i] += w[i];
      const uint4 packed = pack8(v[k]);
      sr[32 * k + lane] = packed;
      unpack8(packed, v[k]);  // the rounded sum, as an unfused bf16 add would hand over
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[k][i];
  const float mu = warp_sum(s) * (1.f / cols);
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float c = v[k][i] - mu;
      q += c * c;
    }
  const float r = rsqrtf(warp_sum(q) * (1.f / cols) + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    float g[8], b[8], o[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(gamma) + 32 * k + lane), g);
    unpack8(__ldg(reinterpret_cast<const uint4*>(beta) + 32 * k + lane), b);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = (v[k][i] - mu) * r * g[i] + b[i];
    yr[32 * k + lane] = pack8(o);
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = r;
  }
}

template <int V>
__global__ void __launch_bounds__(kLnThreads, (V <= 3 ? 2 : 1)) k_ln_bwd(const __nv_bfloat16* __restrict__ dy,
                                                        const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                        const __nv_bfloat16* __restrict__ gamma,
                                                        const float* __restrict__ mean,
                                                        const float* __restrict__ rstd,
                                                        __nv_bfloat16* __restrict__ dx, float* __restrict__ part,
                                                        const __nv_bfloat16* __restrict__ dres) {
  constexpr int cols = 256 * V;
  __shared__ float s_dg[kLnWarps / 2][cols];
  __shared__ float s_db[kLnWarps / 2][cols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // dgamma / dbeta partials in registers; gamma re-read per row (L1 hits) so
  // that two CTAs fit per SM (128 registers)
  const uint4* gv = reinterpret_cast<const uint4*>(gamma);
  float dg[V][8], db[V][8];
#pragma unroll
  for (int k = 0; k < V; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) dg[k][i] = db[k][i] = 0.f;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * kLnWarps + warp; row < rows;
       row += static_cast<int64_t>(gridDim.x) * kLnWarps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * cols);
    float xh[V][8], d[V][8];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      unpack8(ld_nc_v4(xr + 32 * k + lane), xh[k]);
      unpack8(ld_nc_v4(dyr + 32 * k + lane), d[k]);
    }
    const float mu = __ldg(mean + row), r = __ldg(rstd + row);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float g[8];
      unpack8(__ldg(gv + 32 * k + lane), g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        xh[k][i] = (xh[k][i] - mu) * r;
        dg[k][i] += d[k][i] * xh[k][i];
        db[k][i] += d[k][i];
        d[k][i] *= g[i];  // dy * gamma from here on
        s1 += d[k][i];
        s2 += d[k][i] * xh[k][i];
      }
    }
    s1 = warp_sum(s1) * (1.f / cols);
    s2 = warp_sum(s2) * (1.f / cols);
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
    const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + row * cols) : nullptr;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = r * (d[k][i] - s1 - xh[k][i] * s2);
      if (rr) {  // fused gradient accumulation of the residual branch
        float e[8];
        unpack8(ld_nc_v4(rr + 32 * k + lane), e);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] += e[i];
      }
      dxr[32 * k + lane] = pack8(o);
    }
  }
  // fold the 8 warps' partials as a fixed tree (4+4, 2+2, 1+1: deterministic,
  // three barriers), then warp 0 writes the CTA's partial row
#pragma unroll
  for (int half = kLnWarps / 2; half >= 1; half >>= 1) {
    if (warp >= half && warp < 2 * half) {
#pragma unroll
      for (int k = 0; k < V; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          s_dg[warp - half][256 * k + 8 * lane + i] = dg[k][i];
          s_db[warp - half][256 * k + 8 * lane + i] = db[k][i];
        }
    }
    __syncthreads();
    if (warp < half) {
#pragma unroll
      for (int k = 0; k < V; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          dg[k][i] += s_dg[warp][256 * k + 8 * lane + i];
          db[k][i] += s_db[warp][256 * k + 8 * lane + i];
        }
    }
    __syncthreads();
  }
  if (warp == 0) {
    float4* out = reinterpret_cast<float4*>(part + static_cast<int64_t>(blockIdx.x) * 2 * cols);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int c4 = (256 * k + 8 * lane) / 4;
      out[c4] = make_float4(dg[k][0], dg[k][1], dg[k][2], dg[k][3]);
      out[c4 + 1] = make_float4(dg[k][4], dg[k][5], dg[k][6], dg[k][7]);
      out[cols / 4 + c4] = make_float4(db[k][0], db[k][1], db[k][2], db[k][3]);
      out[cols / 4 + c4 + 1] = make_float4(db[k][4], db[k][5], db[k][6], db[k][7]);
    }
  }
}

// 32 columns per CTA; each of the 32 warps sums every 32nd partial row (in
// order, loads batched), then the 32 slices are folded in warp order:
// deterministic
constexpr int kFoldWarps = 32;

__global__ void __launch_bounds__(32 * kFoldWarps) k_ln_bwd_fold(const float* __restrict__ part, int parts, int cols,
                                                                 __nv_bfloat16* __restrict__ dgamma,
                                                                 __nv_bfloat16* __restrict__ dbeta) {
  __shared__ float sa[kFoldWarps][33], sb[kFoldWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float a = 0.f, b = 0.f;
  if (c < cols) {
#pragma unroll 4
    for (int p = warp; p < parts; p += kFoldWarps) {
      a += part[static_cast<int64_t>(p) * 2 * cols + c];
      b += part[static_cast<int64_t>(p) * 2 * cols + cols + c];
    }
  }
  sa[warp][lane] = a;
  sb[warp][lane] = b;
  __syncthreads();
  if (warp == 0 && c < cols) {
    for (int w = 1; w < kFoldWarps; ++w) {
      a += sa[w][lane];
      b += sb[w][lane];
    }
    dgamma[c] = __float2bfloat16_rn(a);
    dbeta[c] = __float2bfloat16_rn(b);
  }
}

static int ln_check(int64_t rows, int cols, const void* a, const void* b) {
  if (rows < 0) return set_error(SDP_ERR_USAGE, "negative row count");
  if (cols <= 0 || cols % 256 != 0 || cols / 256 > kLnMaxV)
    return set_error(SDP_ERR_USAGE, "layer norm width %d: a multiple of 256 up to %d", cols, 256 * kLnMaxV);
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) != 0)
    return set_error(SDP_ERR_USAGE, "layer norm buffers must be 16-B aligned");
  return SDP_OK;
}

}  // namespace sdp

using namespace sdp;

extern "C" {

static int ln_fwd(const void* x_bf16, const void* x2_bf16, void* sum_bf16, int64_t rows, int cols,
                  const void* gamma_bf16, const void* beta_bf16, float eps, void* y_bf16, float* mean, float* rstd,
                  void* stream) {
  if (int rc = ln_check(rows, cols, x_bf16, y_bf16)) return rc;
  if (int rc = ln_check(rows, cols, gamma_bf16, beta_bf16)) return rc;
  if (x2_bf16 || sum_bf16) {
    if (!x2_bf16 || !sum_bf16) return set_error(SDP_ERR_USAGE, "fused add needs both the addend and the sum buffer");
    if (int rc = ln_check(rows, cols, x2_bf16, sum_bf16)) return rc;
  }
  if (rows == 0) return SDP_OK;
  auto x2b = static_cast<const __nv_bfloat16*>(x2_bf16);
  auto sb = static_cast<__nv_bfloat16*>(sum_bf16);
  const unsigned grid = static_cast<unsigned>((rows + kLnWarps - 1) / kLnWarps);
  cudaStream_t s = as_stream(stream);
  auto xb = static_cast<const __nv_bfloat16*>(x_bf16);
  auto gb = static_cast<const __nv_bfloat16*>(gamma_bf16);
  auto bb = static_cast<const __nv_bfloat16*>(beta_bf16);
  auto yb = static_cast<__nv_bfloat16*>(y_bf16);
  switch (cols / 256) {
#define SDP_LN_FWD(V) \
  case V: k_ln_fwd<V><<<grid, kLnThreads, 0, s>>>(xb, rows, gb, bb, eps, yb, mean, rstd, x2b, sb); break;
    SDP_LN_FWD(1) SDP_LN_FWD(2) SDP_LN_FWD(3) SDP_LN_FWD(4) SDP_LN_FWD(5) SDP_LN_FWD(6) SDP_LN_FWD(7) SDP_LN_FWD(8)
#undef SDP_LN_FWD
  }
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_layer_norm_fwd(const void* x_bf16, int64_t rows, int cols, const void* gamma_bf16,
                       const void* beta_bf16, float eps, void* y_bf16, float* mean, float* rstd, void* stream) {
  return ln_fwd(x_bf16, nullptr, nullptr, rows, cols, gamma_bf16, beta_bf16, eps, y_bf16, mean, rstd, stream);
}

int sdp_add_layer_norm_fwd(const void* a_bf16, const void* b_bf16, int64_t rows, int cols, const void* gamma_bf16,
                           const void* beta_bf16, float eps, void* sum_bf16, void* y_bf16, float* mean, float* rstd,
                           void* stream) {
  return ln_fwd(a_bf16, b_bf16, sum_bf16, rows, cols, gamma_bf16, beta_bf16, eps, y_bf16, mean, rstd, stream);
}

int sdp_layer_norm_bwd_parts(int64_t rows, int cols) {
  // one CTA per resident slot (the partial-sum registers limit occupancy)
  int sms = 148, dev = 0, per_sm = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  switch (cols / 256) {
    case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ln_bwd<1>, kLnThreads, 0); break;
    case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ln_bwd<2>, kLnThreads, 0); break;
    case 3: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ln_bwd<3>, kLnThreads, 0); break;
    default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ln_bwd<4>, kLnThreads, 0); break;
  }
  cudaGetLastError();
  const int64_t need = (rows + kLnWarps - 1) / kLnWarps;
  const int64_t slots = static_cast<int64_t>(sms) * (per_sm > 0 ? per_sm : 1);
  return static_cast<int>(need < slots ? (need > 0 ? need : 1) : slots);
}

static int ln_bwd(const void* dy_bf16, const void* x_bf16, const void* dres_bf16, int64_t rows, int cols,
                  const void* gamma_bf16, const float* mean, const float* rstd, void* dx_bf16, void* dgamma_bf16,
                  void* dbeta_bf16, float* scratch, int parts, void* stream) {
  if (dres_bf16)
    if (int rc = ln_check(rows, cols, dres_bf16, dres_bf16)) return rc;
  auto rb = static_cast<const __nv_bfloat16*>(dres_bf16);
  if (int rc = ln_check(rows, cols, x_bf16, dy_bf16)) return rc;
  if (int rc = ln_check(rows, cols, dx_bf16, gamma_bf16)) return rc;
  if (parts <= 0) return set_error(SDP_ERR_USAGE, "layer norm backward needs parts > 0");
  cudaStream_t s = as_stream(stream);
  auto db = static_cast<const __nv_bfloat16*>(dy_bf16);
  auto xb = static_cast<const __nv_bfloat16*>(x_bf16);
  auto gb = static_cast<const __nv_bfloat16*>(gamma_bf16);
  auto dxb = static_cast<__nv_bfloat16*>(dx_bf16);
  if (rows > 0) {
    switch (cols / 256) {
#define SDP_LN_BWD(V) \
  case V: k_ln_bwd<V><<<parts, kLnThreads, 0, s>>>(db, xb, rows, gb, mean, rstd, dxb, scratch, rb); break;
      SDP_LN_BWD(1) SDP_LN_BWD(2) SDP_LN_BWD(3) SDP_LN_BWD(4)
#undef SDP_LN_BWD
      default:
        return set_error(SDP_ERR_USAGE, "layer norm backward width %d: up to 1024", cols);
    }
    SDP_LAUNCH_CHECK();
  } else {
    SDP_CUDA_CHECK(cudaMemsetAsync(scratch, 0, sizeof(float) * 2 * cols * parts, s));
  }
  k_ln_bwd_fold<<<(cols + 31) / 32, 32 * kFoldWarps, 0, s>>>(scratch, parts, cols, static_cast<__nv_bfloat16*>(dgamma_bf16),
                                                   static_cast<__nv_bfloat16*>(dbeta_bf16));
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_layer_norm_bwd(const void* dy_bf16, const void* x_bf16, int64_t rows, int cols, const void* gamma_bf16,
                       const float* mean, const float* rstd, void* dx_bf16, void* dgamma_bf16, void* dbeta_bf16,
                       float* scratch, int parts, void* stream) {
  return ln_bwd(dy_bf16, x_bf16, nullptr, rows, cols, gamma_bf16, mean, rstd, dx_bf16, dgamma_bf16, dbeta_bf16,
                scratch, parts, stream);
}

int sdp_layer_norm_bwd_res(const void* dy_bf16, const void* x_bf16, const void* dres_bf16, int64_t rows, int cols,
                           const void* gamma_bf16, const float* mean, const float* rstd, void* dx_bf16,
                           void* dgamma_bf16, void* dbeta_bf16, float* scratch, int parts, void* stream) {
  return ln_bwd(dy_bf16, x_bf16, dres_bf16, rows, cols, gamma_bf16, mean, rstd, dx_bf16, dgamma_bf16, dbeta_bf16,
                scratch, parts, stream);
}

}  // extern "C"
