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
