// Gradient-alignment diagnostic (diagnostics.py:33-78) as a GPU reduction.
//
// restricted_cosine(g_masked, g_unmasked, support) needs, per layer, the dot
// product and both squared norms over the worker's support.  Pass 1: one CTA
// per task (a chunk of one layer's slice) accumulates in float64, reduces with
// warp shuffles + shared memory and writes its 4 partials; pass 2 sums each
// layer's partials in task order -- deterministic, no float atomics.
#include "sdp_common.cuh"

namespace sdp {

constexpr int kDiagThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__global__ void __launch_bounds__(kDiagThreads)
k_restricted_dots(const T* __restrict__ a, const T* __restrict__ b, const uint8_t* __restrict__ support,
                  const sdp_reduce_task* __restrict__ tasks, double* __restrict__ partials) {
  const sdp_reduce_task tk = tasks[blockIdx.x];
  double ab = 0.0, aa = 0.0, bb = 0.0, n = 0.0;
  for (int64_t k = threadIdx.x; k < tk.length; k += kDiagThreads) {
    const int64_t j = tk.offset + k;
    if (support && !support[j]) continue;
    const double x = static_cast<double>(a[j]), y = static_cast<double>(b[j]);
    ab = fma(x, y, ab);
    aa = fma(x, x, aa);
    bb = fma(y, y, bb);
    n += 1.0;
  }
  __shared__ double s[4][kDiagThreads / 32];
  ab = warp_sum(ab);
  aa = warp_sum(aa);
  bb = warp_sum(bb);
  n = warp_sum(n);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s[0][warp] = ab;
    s[1][warp] = aa;
    s[2][warp] = bb;
    s[3][warp] = n;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0.0;
    for (int w = 0; w < kDiagThreads / 32; ++w) t += s[threadIdx.x][w];
    partials[static_cast<int64_t>(blockIdx.x) * 4 + threadIdx.x] = t;
  }
}

__global__ void k_sum_partials(const sdp_reduce_task* __restrict__ tasks, int n_tasks,
                               const double* __restrict__ partials, int n_segments,
                               double* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_segments) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int t = 0; t < n_tasks; ++t)
    if (tasks[t].segment == s)
      for (int k = 0; k < 4; ++k) acc[k] += partials[static_cast<int64_t>(t) * 4 + k];
  for (int k = 0; k < 4; ++k) out[static_cast<int64_t>(s) * 4 + k] = acc[k];
}

}  // namespace sdp

using namespace sdp;

extern "C" int sdp_restricted_dots(int dtype, const void* a, const void* b, const uint8_t* support,
                                   const sdp_reduce_task* tasks, int n_tasks, int n_segments,
                                   double* partials, double* out, void* stream) {
  if (n_tasks < 0 || n_segments < 0) return set_error(SDP_ERR_USAGE, "negative count");
  if (n_segments == 0) return SDP_OK;
  if (!out || (n_tasks > 0 && (!tasks || !partials || !a || !b)))
    return set_error(SDP_ERR_USAGE, "null device pointer");
  cudaStream_t s = as_stream(stream);
  if (n_tasks > 0) {
    if (dtype == SDP_DTYPE_F32)
      k_restricted_dots<float><<<n_tasks, kDiagThreads, 0, s>>>(static_cast<const float*>(a),
          static_cast<const float*>(b), support, tasks, partials);
    else if (dtype == SDP_DTYPE_F64)
      k_restricted_dots<double><<<n_tasks, kDiagThreads, 0, s>>>(static_cast<const double*>(a),
          static_cast<const double*>(b), support, tasks, partials);
    else
      return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
    SDP_LAUNCH_CHECK();
  }
  k_sum_partials<<<(n_segments + 127) / 128, 128, 0, s>>>(tasks, n_tasks, partials, n_segments, out);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}
