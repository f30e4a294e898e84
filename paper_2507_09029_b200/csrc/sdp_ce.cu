// Row-wise cross-entropy over bf16 logits for the chunked, fused LM head of
// the C4 training step (train._LinearCrossEntropy): the [rows, V] logits of a
// chunk are read once per pass and never widened to fp32 in memory.
//
//   k_ce_fwd  one CTA per row: online max / sum-exp over the row (fp32) ->
//             lse[r] and the row's loss lse - logit[target]
//   k_ce_bwd  dlogits = bf16((exp(logit - lse) - [j == target]) * g / n),
//             one CTA per row, 16-B vectors, g read from device memory
//             (graph-capturable)
// Rows have a pitch >= vocab so the head GEMMs see a 64-aligned leading
// dimension (GPT-2's 50257 would force cuBLAS onto align-1 mma.sync kernels).
#include "sdp_common.cuh"

namespace sdp {

constexpr int kCeThreads = 256;

__device__ __forceinline__ uint4 ld_stream_v4(const uint4* p) {  // read once: no L1 allocation
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
  return u;
}

__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
  m = mm;
}

// Per-thread running (max, sum-exp): a vector whose max does not exceed the
// running max adds its 8 exponentials directly; a rescale (one more exp) only
// when the max grows -- ~8 exponentials per 8 logits (MUFU-bound otherwise).
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
  if (cm > m) {
    s = (m == -INFINITY) ? 0.f : s * __expf(m - cm);
    m = cm;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) s += __expf(x[k] - m);
}

// One CTA of 128 threads per row: 16 CTAs per SM keep a whole 2048-row
// chunk resident at once (no wave tail; measured 50 -> ? us vs 256-thread
// CTAs), four 16-B loads in flight per thread.  Rows of an odd vocabulary
// (GPT-2: 50257) start at any 2-B offset: a scalar head up to the first 16-B
// boundary, 16-B vectors, a scalar tail.
constexpr int kCeFwdThreads = 128;

__global__ void __launch_bounds__(kCeFwdThreads)
k_ce_fwd(const __nv_bfloat16* __restrict__ logits, int64_t rows, int vocab, int64_t pitch,
         const int64_t* __restrict__ targets, float* __restrict__ lse, float* __restrict__ loss_rows) {
  constexpr int NT = kCeFwdThreads;
  const int64_t r = blockIdx.x;
  const __nv_bfloat16* row = logits + r * pitch;
  float m = -INFINITY, s = 0.f;
  const int head = min(vocab, static_cast<int>(((16 - (reinterpret_cast<uintptr_t>(row) & 15)) & 15) / 2));
  const int nv = (vocab - head) / 8;
  const int tail0 = head + nv * 8;
  for (int j = threadIdx.x; j < head; j += NT) online_merge(m, s, __bfloat162float(row[j]), 1.f);
  const uint4* rv = reinterpret_cast<const uint4*>(row + head);
  int q = threadIdx.x;
  for (; q + 3 * NT < nv; q += 4 * NT) {  // four 16-B loads in flight
    const uint4 u0 = ld_stream_v4(rv + q), u1 = ld_stream_v4(rv + q + NT);
    const uint4 u2 = ld_stream_v4(rv + q + 2 * NT), u3 = ld_stream_v4(rv + q + 3 * NT);
    accum8(m, s, u0);
    accum8(m, s, u1);
    accum8(m, s, u2);
    accum8(m, s, u3);
  }
  for (; q < nv; q += NT) accum8(m, s, ld_stream_v4(rv + q));
  for (int j = tail0 + threadIdx.x; j < vocab; j += NT) online_merge(m, s, __bfloat162float(row[j]), 1.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    online_merge(m, s, m2, s2);
  }
  __shared__ float sm[NT / 32], ss[NT / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    m = sm[0];
    s = ss[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) online_merge(m, s, sm[w], ss[w]);
    const float l = m + __logf(s);
    lse[r] = l;
    loss_rows[r] = l - __bfloat162float(row[targets[r]]);
  }
}

// Rows of `pitch` elements (pitch >= vocab; columns [vocab, pitch) are the
// padding of a GEMM-friendly leading dimension and get dlogits = 0).  With
// pitch % 8 == 0 and a 16-B aligned base every 16-B vector stays in one row;
// otherwise the flat scalar loop covers every element.
__global__ void __launch_bounds__(kCeThreads)
k_ce_bwd(const __nv_bfloat16* __restrict__ logits, int64_t rows, int vocab, int64_t pitch,
         const int64_t* __restrict__ targets, const float* __restrict__ lse,
         const float* __restrict__ grad_out, float inv_n, __nv_bfloat16* __restrict__ dlogits) {
  const float g = *grad_out * inv_n;
  if (pitch % 8 == 0) {  // CTAs walk rows; lse / target read once per row
    const int vpr = static_cast<int>(pitch / 8);
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
      const float l = lse[r];
      const int t = static_cast<int>(targets[r]);
      const uint4* src = reinterpret_cast<const uint4*>(logits + r * pitch);
      uint4* dst = reinterpret_cast<uint4*>(dlogits + r * pitch);
#pragma unroll 2
      for (int q = threadIdx.x; q < vpr; q += kCeThreads) {
        const uint4 u = ld_stream_v4(src + q);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
        const int j0 = q * 8;
        uint4 o;
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h[k]);
          const int ja = j0 + 2 * k, jb = ja + 1;
          float a = ja < vocab ? __expf(f.x - l) : 0.f;
          float b = jb < vocab ? __expf(f.y - l) : 0.f;
          if (ja == t) a -= 1.f;
          if (jb == t) b -= 1.f;
          oh[k] = __floats2bfloat162_rn(a * g, b * g);
        }
        dst[q] = o;
      }
    }
    return;
  }
  const int64_t n = rows * pitch;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / pitch;
    const int64_t j = i - r * pitch;
    float a = j < vocab ? __expf(__bfloat162float(logits[i]) - lse[r]) : 0.f;
    if (j == targets[r]) a -= 1.f;
    dlogits[i] = __float2bfloat16_rn(a * g);
  }
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_ce_rows_fwd(const void* logits_bf16, int64_t rows, int vocab, int64_t pitch, const int64_t* targets,
                    float* lse, float* loss_rows, void* stream) {
  if (rows < 0 || vocab < 1 || pitch < vocab) return set_error(SDP_ERR_USAGE, "bad cross-entropy shape");
  if (rows == 0) return SDP_OK;
  if (!logits_bf16 || !targets || !lse || !loss_rows) return set_error(SDP_ERR_USAGE, "null device pointer");
  if (rows > 0x7fffffff) return set_error(SDP_ERR_USAGE, "too many rows");
  k_ce_fwd<<<static_cast<unsigned>(rows), kCeFwdThreads, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(logits_bf16), rows, vocab, pitch, targets, lse, loss_rows);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_ce_rows_bwd(const void* logits_bf16, int64_t rows, int vocab, int64_t pitch, const int64_t* targets,
                    const float* lse, const float* grad_out, float inv_n, void* dlogits_bf16, void* stream) {
  if (rows < 0 || vocab < 1 || pitch < vocab) return set_error(SDP_ERR_USAGE, "bad cross-entropy shape");
  if (rows == 0) return SDP_OK;
  if (!logits_bf16 || !targets || !lse || !grad_out || !dlogits_bf16)
    return set_error(SDP_ERR_USAGE, "null device pointer");
  if ((reinterpret_cast<uintptr_t>(logits_bf16) | reinterpret_cast<uintptr_t>(dlogits_bf16)) % 16)
    return set_error(SDP_ERR_USAGE, "cross-entropy logits must be 16-byte aligned");
  const int grid = static_cast<int>(
      pitch % 8 == 0 ? std::min<int64_t>(rows, 0x7fffffff)
                     : std::min<int64_t>((rows * pitch + kCeThreads - 1) / kCeThreads,
                                         static_cast<int64_t>(sm_count()) * 8));
  k_ce_bwd<<<grid, kCeThreads, 0, as_stream(stream)>>>(static_cast<const __nv_bfloat16*>(logits_bf16), rows,
                                                     vocab, pitch, targets, lse, grad_out, inv_n,
                                                     static_cast<__nv_bfloat16*>(dlogits_bf16));
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
