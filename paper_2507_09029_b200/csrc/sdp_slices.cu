// Width-wise slice extraction and write-back (models.py:333-382).
//
//   k_masked_extract  theta * mask for one worker (models.py:355), bit-exact
//   k_gather          full -> compact: one CTA per task (a run of compact rows
//                     of one tensor); stores are contiguous over the compact
//                     row, loads follow the row/column index maps
//   k_scatter         compact -> full: one CTA per run of FULL rows; every full
//                     element of a covered row is written once (zero fill) or
//                     accumulated (owner-ordered write-back), stores coalesced
//   k_divide          acc / divisor after owner-ordered accumulation
// Tensors are in canonical [rows, cols, inner] form (include/sdp.h); division
// by `inner` uses a precomputed multiply-high (no integer divide per element).
#include "sdp_common.cuh"

namespace sdp {

constexpr int kSliceThreads = 256;

template <typename T, int MB>
__global__ void k_masked_extract(const T* __restrict__ theta, const typename MaskT<MB>::T* __restrict__ mask,
                                 int64_t total, int worker, T* __restrict__ out) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T m = static_cast<T>((static_cast<uint64_t>(__ldg(mask + j)) >> worker) & 1ull);
    out[j] = theta[j] * m;  // a plain multiply: keeps -0.0 / NaN like numpy
  }
}

__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t mul, uint32_t shr) {
  return mul ? (__umulhi(n, mul) >> shr) : n;
}

template <typename T, bool REVERSE>
__global__ void __launch_bounds__(kSliceThreads)
k_gather(const sdp_slice_desc* __restrict__ descs, const sdp_slice_task* __restrict__ tasks,
         const int32_t* __restrict__ fwd, T* full, T* compact) {
  const sdp_slice_task tk = tasks[blockIdx.x];
  const sdp_slice_desc d = descs[tk.desc];
  const uint32_t row_len = static_cast<uint32_t>(d.ccols) * d.inner;
  // (row, element) pairs of the task flattened over the CTA: independent
  // loads across rows instead of one dependent round trip per row.
  const uint32_t seg = static_cast<uint32_t>(tk.elem_end - tk.elem_begin);
  const uint32_t n_el = static_cast<uint32_t>(tk.row_end - tk.row_begin) * seg;
  const int64_t row_stride = static_cast<int64_t>(d.cols) * d.inner;
#pragma unroll 4
  for (uint32_t idx = threadIdx.x; idx < n_el; idx += kSliceThreads) {
    const uint32_t rr = fast_div(idx, d.rowlen_mul, d.rowlen_shr);  // 0 for single-row tasks
    const uint32_t r = tk.row_begin + rr;
    const uint32_t t = tk.elem_begin + (idx - rr * row_len);
    const int64_t fr = d.row_map >= 0 ? __ldg(fwd + d.row_map + r) : r;
    int64_t src = d.full_offset + fr * row_stride;
    if (d.col_map < 0) {
      src += t;
    } else {
      const uint32_t b = fast_div(t, d.inner_mul, d.inner_shr);
      src += static_cast<int64_t>(__ldg(fwd + d.col_map + b)) * d.inner + (t - b * d.inner);
    }
    const int64_t c = d.compact_offset + static_cast<int64_t>(r) * row_len + t;
    if (REVERSE) full[src] = compact[c];
    else compact[c] = full[src];
  }
}

template <typename T>
__global__ void __launch_bounds__(kSliceThreads)
k_scatter(const sdp_slice_desc* __restrict__ descs, const sdp_slice_task* __restrict__ tasks,
          const int32_t* __restrict__ inv, const T* __restrict__ compact, T* __restrict__ full,
          int flags) {
  const bool zero_fill = (flags & SDP_SCATTER_ZERO_FILL) && !(flags & SDP_SCATTER_ACCUMULATE);
  const bool accumulate = (flags & SDP_SCATTER_ACCUMULATE) != 0;
  const sdp_slice_task tk = tasks[blockIdx.x];
  const sdp_slice_desc d = descs[tk.desc];
  const int64_t crow_len = static_cast<int64_t>(d.ccols) * d.inner;
  const uint32_t row_len = static_cast<uint32_t>(d.cols) * d.inner;
  const uint32_t seg = static_cast<uint32_t>(tk.elem_end - tk.elem_begin);
  const uint32_t n_el = static_cast<uint32_t>(tk.row_end - tk.row_begin) * seg;
#pragma unroll 4
  for (uint32_t idx = threadIdx.x; idx < n_el; idx += kSliceThreads) {
    const uint32_t rr = fast_div(idx, d.rowlen_mul, d.rowlen_shr);  // 0 for single-row tasks
    const uint32_t f = tk.row_begin + rr;
    const uint32_t t = tk.elem_begin + (idx - rr * row_len);
    T* dst = full + d.full_offset + static_cast<int64_t>(f) * row_len + t;
    const int32_t a = d.crows == 0 ? -1 : (d.row_map >= 0 ? __ldg(inv + d.row_map + f) : static_cast<int32_t>(f));
    int64_t src = -1;
    if (a >= 0) {
      if (d.col_map < 0) {
        src = a * crow_len + t;
      } else {
        const uint32_t fb = fast_div(t, d.inner_mul, d.inner_shr);
        const int32_t cb = __ldg(inv + d.col_map + fb);
        if (cb >= 0) src = a * crow_len + static_cast<int64_t>(cb) * d.inner + (t - fb * d.inner);
      }
    }
    if (src >= 0) {
      const T v = compact[d.compact_offset + src];
      *dst = accumulate ? static_cast<T>(*dst + v) : v;
    } else if (zero_fill) {
      *dst = T(0);  // the worker does not hold this element
    }
  }
}

template <typename T>
__global__ void k_divide(const T* __restrict__ acc, const double* __restrict__ divisor, int64_t total,
                         T* __restrict__ out) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[j] = acc[j] / static_cast<T>(divisor[j]);
}

static int grid_for(int64_t n) {
  const int64_t want = (n + kSliceThreads - 1) / kSliceThreads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(sm_count()) * 8)));
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_masked_extract(int dtype, const void* theta, const void* owner_mask, int mask_bytes,
                       int64_t total, int worker, void* out, void* stream) {
  if (!(mask_bytes == 1 || mask_bytes == 2 || mask_bytes == 4 || mask_bytes == 8))
    return set_error(SDP_ERR_CONFIG, "mask_bytes must be 1, 2, 4 or 8");
  if (worker < 0 || worker >= 8 * mask_bytes)
    return set_error(SDP_ERR_CONFIG, "worker id %d outside the mask width", worker);
  if (total <= 0) return SDP_OK;
  const int grid = grid_for(total);
  cudaStream_t s = as_stream(stream);
#define SDP_EXTRACT(TT, MB)                                                                  \
  k_masked_extract<TT, MB><<<grid, kSliceThreads, 0, s>>>(static_cast<const TT*>(theta),    \
      static_cast<const MaskT<MB>::T*>(owner_mask), total, worker, static_cast<TT*>(out))
#define SDP_EXTRACT_T(TT)                  \
  switch (mask_bytes) {                    \
    case 1: SDP_EXTRACT(TT, 1); break;     \
    case 2: SDP_EXTRACT(TT, 2); break;     \
    case 4: SDP_EXTRACT(TT, 4); break;     \
    default: SDP_EXTRACT(TT, 8); break;    \
  }
  if (dtype == SDP_DTYPE_F32) { SDP_EXTRACT_T(float) }
  else if (dtype == SDP_DTYPE_F64) { SDP_EXTRACT_T(double) }
  else return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
#undef SDP_EXTRACT_T
#undef SDP_EXTRACT
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_gather_slices(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                      int n_tasks, const int32_t* fwd_maps, const void* full, void* compact,
                      int flags, void* stream) {
  if (n_tasks < 0) return set_error(SDP_ERR_USAGE, "negative task count");
  if (n_tasks == 0) return SDP_OK;
  if (!descs || !tasks || !full || !compact) return set_error(SDP_ERR_USAGE, "null device pointer");
  cudaStream_t s = as_stream(stream);
  const bool rev = (flags & SDP_GATHER_REVERSE) != 0;
  void* fu = const_cast<void*>(full);
#define SDP_GATHER(TT)                                                                          \
  do {                                                                                          \
    if (rev)                                                                                    \
      k_gather<TT, true><<<n_tasks, kSliceThreads, 0, s>>>(descs, tasks, fwd_maps,              \
                                                           static_cast<TT*>(fu), static_cast<TT*>(compact)); \
    else                                                                                        \
      k_gather<TT, false><<<n_tasks, kSliceThreads, 0, s>>>(descs, tasks, fwd_maps,             \
                                                            static_cast<TT*>(fu), static_cast<TT*>(compact)); \
  } while (0)
  if (dtype == SDP_DTYPE_F32) SDP_GATHER(float);
  else if (dtype == SDP_DTYPE_F64) SDP_GATHER(double);
  else if (dtype == SDP_DTYPE_U8) SDP_GATHER(uint8_t);
  else return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32, SDP_DTYPE_F64 or SDP_DTYPE_U8");
#undef SDP_GATHER
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_scatter_slices(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                       int n_tasks, const int32_t* inv_maps, const void* compact, void* full,
                       int flags, void* stream) {
  if (n_tasks < 0) return set_error(SDP_ERR_USAGE, "negative task count");
  if (n_tasks == 0) return SDP_OK;
  if (!descs || !tasks || !full) return set_error(SDP_ERR_USAGE, "null device pointer");
  cudaStream_t s = as_stream(stream);
  if (dtype == SDP_DTYPE_F32)
    k_scatter<float><<<n_tasks, kSliceThreads, 0, s>>>(descs, tasks, inv_maps, static_cast<const float*>(compact),
                                                       static_cast<float*>(full), flags);
  else if (dtype == SDP_DTYPE_F64)
    k_scatter<double><<<n_tasks, kSliceThreads, 0, s>>>(descs, tasks, inv_maps, static_cast<const double*>(compact),
                                                        static_cast<double*>(full), flags);
  else
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_divide(int dtype, const void* acc, const double* divisor, int64_t total, void* out,
               void* stream) {
  if (total <= 0) return SDP_OK;
  const int grid = grid_for(total);
  cudaStream_t s = as_stream(stream);
  if (dtype == SDP_DTYPE_F32)
    k_divide<float><<<grid, kSliceThreads, 0, s>>>(static_cast<const float*>(acc), divisor, total,
                                                   static_cast<float*>(out));
  else if (dtype == SDP_DTYPE_F64)
    k_divide<double><<<grid, kSliceThreads, 0, s>>>(static_cast<const double*>(acc), divisor, total,
                                                    static_cast<double*>(out));
  else
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
