// Row-wise cross-entropy over bf16 logits for the chunked, fused LM head of
// the C4 training step (train._LinearCrossEntropy): the [rows, V] logits of a
// chunk are read once per pass and never widened to fp32 in memory.
//
//   k_ce_fwd  one CTA per row: online max / sum-exp over the row (fp32) ->
//             lse[r] and the row's loss lse - logit[target]
//   k_ce_bwd  dlogits = bf16((exp(logit - lse) - [j == target]) * g / n),
//             16-B vectors, g read from device memory (graph-capturable)
#include "sdp_common.cuh"

namespace sdp {

constexpr int kCeThreads = 256;

__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
  m = mm;
}

__device__ __forceinline__ void accum8(float& m, float& s, const uint4& u) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  float x[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    x[2 * k] = f.x;
    x[2 * k + 1] = f.y;
  }
  float cm = x[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) cm = fmaxf(cm, x[k]);
  float cs = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) cs += __expf(x[k] - cm);
  online_merge(m, s, cm, cs);
}

// One CTA per row.  Rows of an odd vocabulary (GPT-2: 50257) start at any
// 2-B offset: a scalar head up to the first 16-B boundary, 16-B vectors, a
// scalar tail.
__global__ void __launch_bounds__(kCeThreads)
k_ce_fwd(const __nv_bfloat16* __restrict__ logits, int vocab, const int64_t* __restrict__ targets,
         float* __restrict__ lse, float* __restrict__ loss_rows) {
  const int64_t r = blockIdx.x;
  const __nv_bfloat16* row = logits + r * static_cast<int64_t>(vocab);
  float m = -INFINITY, s = 0.f;
  const int head = min(vocab, static_cast<int>(((16 - (reinterpret_cast<uintptr_t>(row) & 15)) & 15) / 2));
  const int nv = (vocab - head) / 8;
  const int tail0 = head + nv * 8;
  for (int j = threadIdx.x; j < head; j += kCeThreads) online_merge(m, s, __bfloat162float(row[j]), 1.f);
  const uint4* rv = reinterpret_cast<const uint4*>(row + head);
  int q = threadIdx.x;
  for (; q + kCeThreads < nv; q += 2 * kCeThreads) {  // two 16-B loads in flight
    const uint4 u0 = __ldg(rv + q), u1 = __ldg(rv + q + kCeThreads);
    accum8(m, s, u0);
    accum8(m, s, u1);
  }
  for (; q < nv; q += kCeThreads) accum8(m, s, __ldg(rv + q));
  for (int j = tail0 + threadIdx.x; j < vocab; j += kCeThreads) online_merge(m, s, __bfloat162float(row[j]), 1.f);
  // warp then CTA merge of (max, sum)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    online_merge(m, s, m2, s2);
  }
  __shared__ float sm[kCeThreads / 32], ss[kCeThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < kCeThreads / 32 ? sm[lane] : -INFINITY;
    s = lane < kCeThreads / 32 ? ss[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
      online_merge(m, s, m2, s2);
    }
    if (lane == 0) {
      const float l = m + __logf(s);
      lse[r] = l;
      loss_rows[r] = l - __bfloat162float(row[targets[r]]);
    }
  }
}

// Flat over the chunk (rows x vocab contiguous, 16-B aligned base): 8 logits
// per 16-B vector; a vector crosses at most one row boundary (vocab >= 8).
__global__ void __launch_bounds__(kCeThreads)
k_ce_bwd(const __nv_bfloat16* __restrict__ logits, int64_t rows, int vocab,
         const int64_t* __restrict__ targets, const float* __restrict__ lse,
         const float* __restrict__ grad_out, float inv_n, __nv_bfloat16* __restrict__ dlogits) {
  const float g = *grad_out * inv_n;
  const int64_t n = rows * vocab;
  const int64_t nv = n / 8;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nv;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i0 = q * 8;
    const int64_t r0 = i0 / vocab;
    const int64_t bound = (r0 + 1) * vocab;
    const float l0 = lse[r0];
    const int64_t t0 = r0 * vocab + targets[r0];
    const bool cross = i0 + 8 > bound;
    const float l1 = cross ? lse[r0 + 1] : l0;
    const int64_t t1 = cross ? bound + targets[r0 + 1] : t0;
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(logits) + q);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      const int64_t ia = i0 + 2 * k, ib = ia + 1;
      float a = __expf(f.x - (ia < bound ? l0 : l1));
      float b = __expf(f.y - (ib < bound ? l0 : l1));
      if (ia == (ia < bound ? t0 : t1)) a -= 1.f;
      if (ib == (ib < bound ? t0 : t1)) b -= 1.f;
      oh[k] = __floats2bfloat162_rn(a * g, b * g);
    }
    reinterpret_cast<uint4*>(dlogits)[q] = o;
  }
  for (int64_t i = nv * 8 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / vocab;
    float a = __expf(__bfloat162float(logits[i]) - lse[r]);
    if (i - r * vocab == targets[r]) a -= 1.f;
    dlogits[i] = __float2bfloat16_rn(a * g);
  }
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_ce_rows_fwd(const void* logits_bf16, int64_t rows, int vocab, const int64_t* targets, float* lse,
                    float* loss_rows, void* stream) {
  if (rows < 0 || vocab < 1) return set_error(SDP_ERR_USAGE, "bad cross-entropy shape");
  if (rows == 0) return SDP_OK;
  if (!logits_bf16 || !targets || !lse || !loss_rows) return set_error(SDP_ERR_USAGE, "null device pointer");
  if (rows > 0x7fffffff) return set_error(SDP_ERR_USAGE, "too many rows");
  k_ce_fwd<<<static_cast<unsigned>(rows), kCeThreads, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(logits_bf16), vocab, targets, lse, loss_rows);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_ce_rows_bwd(const void* logits_bf16, int64_t rows, int vocab, const int64_t* targets,
                    const float* lse, const float* grad_out, float inv_n, void* dlogits_bf16, void* stream) {
  if (rows < 0 || vocab < 1) return set_error(SDP_ERR_USAGE, "bad cross-entropy shape");
  if (rows == 0) return SDP_OK;
  if (!logits_bf16 || !targets || !lse || !grad_out || !dlogits_bf16)
    return set_error(SDP_ERR_USAGE, "null device pointer");
  if ((reinterpret_cast<uintptr_t>(logits_bf16) | reinterpret_cast<uintptr_t>(dlogits_bf16)) % 16)
    return set_error(SDP_ERR_USAGE, "cross-entropy logits must be 16-byte aligned");
  if (vocab < 8) return set_error(SDP_ERR_USAGE, "vocabulary below 8 entries");
  const int64_t work = rows * vocab / 8 + 1;
  const int grid = static_cast<int>(std::min<int64_t>((work + kCeThreads - 1) / kCeThreads,
                                                      static_cast<int64_t>(sm_count()) * 8));
  k_ce_bwd<<<grid, kCeThreads, 0, as_stream(stream)>>>(static_cast<const __nv_bfloat16*>(logits_bf16), rows,
                                                     vocab, targets, lse, grad_out, inv_n,
                                                     static_cast<__nv_bfloat16*>(dlogits_bf16));
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
