// Convolution-weight gradients from channels-last (OHWI) bf16 into the fp32
// replica's reference (OIHW) layout, for all of a worker's live conv weights
// in ONE launch (train.SubnetTrainer._store_grads).  cuDNN's NHWC kernels
// return channels-last weight gradients; a per-weight strided copy + cast
// cost ~5 us per weight, 20 per ResNet-18 worker step.
//
// One CTA per (weight, output channel): the [K, I] block (K = kh*kw) is read
// contiguously into shared memory, then written transposed as [I, K], also
// contiguously.  HBM bytes per element: 2 read + 4 written.
#include "sdp_common.cuh"

namespace sdp {

constexpr int kCgThreads = 256;
constexpr int kCgMaxBlock = 8192;  // K * I per output channel

__global__ void __launch_bounds__(kCgThreads) k_conv_grad_oihw(const sdp_conv_grad_desc* __restrict__ descs,
                                                               const __nv_bfloat16* __restrict__ src,
                                                               float* __restrict__ dst) {
  __shared__ float buf[kCgMaxBlock];
  const sdp_conv_grad_desc d = descs[blockIdx.y];
  const int o = blockIdx.x;
  if (o >= d.out_channels) return;
  const int ki = d.in_channels * d.kernel_elems;
  const __nv_bfloat16* s = src + d.offset + static_cast<int64_t>(o) * ki;
  for (int j = threadIdx.x; j < ki; j += kCgThreads) buf[j] = __bfloat162float(s[j]);  // j = k * I + i
  __syncthreads();
  float* t = dst + d.offset + static_cast<int64_t>(o) * ki;
  const int kk = d.kernel_elems, ii = d.in_channels;
  for (int j = threadIdx.x; j < ki; j += kCgThreads) {  // j = i * K + k
    const int i = j / kk, k = j - i * kk;
    t[j] = buf[k * ii + i];
  }
}

// The forward direction for the training copy: bf16 OIHW weights -> bf16
// OHWI (channels-last) for all of a worker's conv weights in one launch.
__global__ void __launch_bounds__(kCgThreads) k_conv_w_ohwi(const sdp_conv_grad_desc* __restrict__ descs,
                                                            const __nv_bfloat16* __restrict__ src,
                                                            __nv_bfloat16* __restrict__ dst) {
  __shared__ __nv_bfloat16 buf[kCgMaxBlock];
  const sdp_conv_grad_desc d = descs[blockIdx.y];
  const int o = blockIdx.x;
  if (o >= d.out_channels) return;
  const int ki = d.in_channels * d.kernel_elems;
  const __nv_bfloat16* s = src + d.offset + static_cast<int64_t>(o) * ki;
  for (int j = threadIdx.x; j < ki; j += kCgThreads) buf[j] = s[j];  // j = i * K + k
  __syncthreads();
  __nv_bfloat16* t = dst + d.offset + static_cast<int64_t>(o) * ki;
  const int kk = d.kernel_elems, ii = d.in_channels;
  for (int j = threadIdx.x; j < ki; j += kCgThreads) {  // j = k * I + i
    const int k = j / ii, i = j - k * ii;
    t[j] = buf[i * kk + k];
  }
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_conv_grads_to_oihw(const sdp_conv_grad_desc* descs, int n_desc, int max_out_channels, const void* src_bf16,
                           float* dst, void* stream) {
  if (n_desc < 0 || max_out_channels < 0) return set_error(SDP_ERR_USAGE, "bad conv-gradient table");
  if (n_desc == 0 || max_out_channels == 0) return SDP_OK;
  if (!descs || !src_bf16 || !dst) return set_error(SDP_ERR_USAGE, "null device pointer");
  if (n_desc > 65535) return set_error(SDP_ERR_USAGE, "at most 65535 conv weights per call");
  k_conv_grad_oihw<<<dim3(static_cast<unsigned>(max_out_channels), static_cast<unsigned>(n_desc)), kCgThreads, 0,
                     as_stream(stream)>>>(descs, static_cast<const __nv_bfloat16*>(src_bf16), dst);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_conv_grad_max_block(void) { return kCgMaxBlock; }

int sdp_conv_weights_to_ohwi(const sdp_conv_grad_desc* descs, int n_desc, int max_out_channels, const void* src_bf16,
                             void* dst_bf16, void* stream) {
  if (n_desc < 0 || max_out_channels < 0) return set_error(SDP_ERR_USAGE, "bad conv-weight table");
  if (n_desc == 0 || max_out_channels == 0) return SDP_OK;
  if (!descs || !src_bf16 || !dst_bf16) return set_error(SDP_ERR_USAGE, "null device pointer");
  if (n_desc > 65535) return set_error(SDP_ERR_USAGE, "at most 65535 conv weights per call");
  k_conv_w_ohwi<<<dim3(static_cast<unsigned>(max_out_channels), static_cast<unsigned>(n_desc)), kCgThreads, 0,
                  as_stream(stream)>>>(descs, static_cast<const __nv_bfloat16*>(src_bf16),
                                       static_cast<__nv_bfloat16*>(dst_bf16));
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
