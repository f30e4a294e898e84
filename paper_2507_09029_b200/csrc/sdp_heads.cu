// Attention-head gradient merge for the GPT-2 blocks of the C4 training step
// (train._SplitHeads): dq, dk, dv [b, nh, t, hd] with any (batch, head, seq)
// strides and contiguous head rows (the SDPA backward returns them either
// [b, nh, t, hd]- or [b, t, nh, hd]-major) -> one [b, t, 3, nh, hd] buffer,
// i.e. the [b*t, 3e] gradient of the fused qkv projection.  One thread per
// 16-B output vector: stores are fully coalesced, loads move whole head rows.
// HBM bytes: 2 B read + 2 B written per element.
#include "sdp_common.cuh"

namespace sdp {

__global__ void __launch_bounds__(256) k_merge_heads(const uint4* __restrict__ q, const uint4* __restrict__ k,
                                                     const uint4* __restrict__ v, int64_t b, int64_t t, int nh,
                                                     int hdv, int64_t sb, int64_t sh, int64_t st,
                                                     uint4* __restrict__ out) {
  const int64_t total = b * t * 3 * nh * hdv;
  for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int dv = static_cast<int>(o % hdv);
    int64_t rest = o / hdv;
    const int h = static_cast<int>(rest % nh);
    rest /= nh;
    const int i = static_cast<int>(rest % 3);
    rest /= 3;  // = bi * t + ti
    const int64_t ti = rest % t, bi = rest / t;
    const uint4* src = i == 0 ? q : (i == 1 ? k : v);
    out[o] = __ldcs(src + bi * sb + h * sh + ti * st + dv);
  }
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_merge_heads(const void* dq, const void* dk, const void* dv, int64_t batch, int64_t seq, int heads,
                    int head_dim, int elem_bytes, int64_t stride_batch, int64_t stride_head, int64_t stride_seq,
                    void* out, void* stream) {
  if (batch < 0 || seq < 0 || heads <= 0 || head_dim <= 0 || (elem_bytes != 2 && elem_bytes != 4))
    return set_error(SDP_ERR_USAGE, "bad head-merge shape");
  if ((static_cast<int64_t>(head_dim) * elem_bytes) % 16 != 0)
    return set_error(SDP_ERR_USAGE, "head rows must be a multiple of 16 bytes");
  if (((reinterpret_cast<uintptr_t>(dq) | reinterpret_cast<uintptr_t>(dk) | reinterpret_cast<uintptr_t>(dv) |
        reinterpret_cast<uintptr_t>(out)) & 15) != 0)
    return set_error(SDP_ERR_USAGE, "head-merge buffers must be 16-B aligned");
  const int hdv = static_cast<int>(static_cast<int64_t>(head_dim) * elem_bytes / 16);
  const int64_t per_vec = 16 / elem_bytes;
  if (stride_batch % per_vec || stride_head % per_vec || stride_seq % per_vec)
    return set_error(SDP_ERR_USAGE, "head-merge strides must keep 16-B vectors aligned");
  const int64_t total = batch * seq * 3 * heads * hdv;
  if (total == 0) return SDP_OK;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(sm_count()) * 16));
  k_merge_heads<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint4*>(dq), static_cast<const uint4*>(dk),
                                                     static_cast<const uint4*>(dv), batch, seq, heads, hdv,
                                                     stride_batch / per_vec, stride_head / per_vec,
                                                     stride_seq / per_vec, static_cast<uint4*>(out));
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"

// Column sums of a bf16 [rows, cols] matrix -> bf16 [cols] (fp32 accumulation):
// the bias gradients of the GPT-2 projections (train._Linear).  Stage 1: CTA
// (column block of 256, row part) -- 32 lanes x 16-B column vectors, 8 row
// lanes -- folds its rows into an fp32 partial row; stage 2 sums the parts in
// order (deterministic).  HBM: 2 B read per element.
namespace sdp {

constexpr int kCsParts = 64;

__global__ void __launch_bounds__(256) k_colsum_part(const uint4* __restrict__ x, int64_t rows, int nvec,
                                                     float* __restrict__ part) {
  __shared__ float s[8][32 * 8 + 1];
  const int lane = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int v = blockIdx.x * 32 + lane;
  const int64_t per = (rows + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = blockIdx.y * per, r1 = r0 + per < rows ? r0 + per : rows;
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
  if (v < nvec) {
    int64_t r = r0 + rl;
    for (; r + 24 < r1; r += 32) {
      uint4 u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) u[j] = __ldcs(x + (r + 8 * j) * nvec + v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[j]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h[k]);
          acc[2 * k] += f.x;
          acc[2 * k + 1] += f.y;
        }
      }
    }
    for (; r < r1; r += 8) {
      const uint4 u = __ldcs(x + r * nvec + v);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) s[rl][lane * 8 + k] = acc[k];
  __syncthreads();
  const int cols = nvec * 8;
  const int c = blockIdx.x * 256 + threadIdx.x;  // one column per thread
  if (c < cols) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += s[j][threadIdx.x];
    part[static_cast<int64_t>(blockIdx.y) * cols + c] = t;
  }
}

__global__ void k_colsum_fold(const float* __restrict__ part, int parts, int cols, __nv_bfloat16* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float t = 0.f;
#pragma unroll 8
  for (int p = 0; p < parts; ++p) t += part[static_cast<int64_t>(p) * cols + c];
  out[c] = __float2bfloat16_rn(t);
}

}  // namespace sdp

extern "C" {

int sdp_col_sum_parts(void) { return sdp::kCsParts; }

int sdp_col_sum_bf16(const void* x_bf16, int64_t rows, int cols, void* out_bf16, float* scratch, void* stream) {
  using namespace sdp;
  if (rows < 0 || cols <= 0 || cols % 8) return set_error(SDP_ERR_USAGE, "column sum: cols must be a positive multiple of 8");
  if (((reinterpret_cast<uintptr_t>(x_bf16)) & 15) != 0) return set_error(SDP_ERR_USAGE, "column sum input must be 16-B aligned");
  if (!out_bf16 || !scratch) return set_error(SDP_ERR_USAGE, "null device pointer");
  cudaStream_t s = as_stream(stream);
  const int nvec = cols / 8;
  const int parts = rows >= kCsParts * 8 ? kCsParts : 1;
  if (rows > 0) {
    k_colsum_part<<<dim3((nvec + 31) / 32, parts), 256, 0, s>>>(static_cast<const uint4*>(x_bf16), rows, nvec, scratch);
  } else {
    SDP_CUDA_CHECK(cudaMemsetAsync(scratch, 0, sizeof(float) * cols * parts, s));
  }
  k_colsum_fold<<<(cols + 255) / 256, 256, 0, s>>>(scratch, parts, cols, static_cast<__nv_bfloat16*>(out_bf16));
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
