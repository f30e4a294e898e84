// Width-wise slice extraction and write-back (models.py:333-382).
//
//   k_masked_extract  theta * mask for one worker (models.py:355), bit-exact
//   k_gather          full -> compact sub-tensors (iterates compact elements:
//                     coalesced stores, rows of the source read contiguously)
//   k_scatter         compact -> full with zero fill or accumulate (iterates
//                     full elements through inverse maps: coalesced stores,
//                     every full element written exactly once)
//   k_divide          acc / divisor after owner-ordered accumulation
#include "sdp_common.cuh"

namespace sdp {

constexpr int kSliceThreads = 256;
constexpr int kSliceElems = 4;  // consecutive elements per thread

template <typename T, int MB>
__global__ void k_masked_extract(const T* __restrict__ theta, const typename MaskT<MB>::T* __restrict__ mask,
                                 int64_t total, int worker, T* __restrict__ out) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T m = static_cast<T>((static_cast<uint64_t>(__ldg(mask + j)) >> worker) & 1ull);
    out[j] = theta[j] * m;  // a plain multiply: keeps -0.0 / NaN like numpy
  }
}

__device__ __forceinline__ int find_desc(const sdp_slice_desc* __restrict__ d, int n, int64_t j,
                                         bool by_compact) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    const int64_t off = by_compact ? d[mid].compact_offset : d[mid].full_offset;
    if (off <= j) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int64_t numel(const int64_t* shape, int nd) {
  int64_t n = 1;
  for (int k = 0; k < nd; ++k) n *= shape[k];
  return n;
}

template <typename T>
__global__ void __launch_bounds__(kSliceThreads)
k_gather(const sdp_slice_desc* __restrict__ descs, int n_descs, const int32_t* __restrict__ fwd,
         const T* __restrict__ full, T* __restrict__ compact, int64_t compact_total) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < compact_total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int di = find_desc(descs, n_descs, k, true);
    const sdp_slice_desc& d = descs[di];
    int64_t local = k - d.compact_offset;
    if (local >= numel(d.compact_shape, d.ndim)) continue;  // hole between descriptors
    int64_t src = 0, stride = 1;
    for (int a = d.ndim - 1; a >= 0; --a) {
      const int64_t cs = d.compact_shape[a];
      const int64_t c = local % cs;
      local /= cs;
      const int64_t f = d.map_offset[a] >= 0 ? static_cast<int64_t>(__ldg(fwd + d.map_offset[a] + c)) : c;
      src += f * stride;
      stride *= d.full_shape[a];
    }
    compact[k] = full[d.full_offset + src];
  }
}

template <typename T>
__global__ void __launch_bounds__(kSliceThreads)
k_scatter(const sdp_slice_desc* __restrict__ descs, int n_descs, const int32_t* __restrict__ inv,
          const T* __restrict__ compact, T* __restrict__ full, int64_t lo, int64_t hi, int flags) {
  const bool zero_fill = flags & SDP_SCATTER_ZERO_FILL;
  const bool accumulate = flags & SDP_SCATTER_ACCUMULATE;
  for (int64_t j0 = lo + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * kSliceElems;
       j0 < hi; j0 += static_cast<int64_t>(gridDim.x) * blockDim.x * kSliceElems) {
    int di = find_desc(descs, n_descs, j0, false);
#pragma unroll
    for (int e = 0; e < kSliceElems; ++e) {
      const int64_t j = j0 + e;
      if (j >= hi) break;
      while (di + 1 < n_descs && descs[di + 1].full_offset <= j) ++di;
      const sdp_slice_desc& d = descs[di];
      int64_t local = j - d.full_offset;
      if (local < 0 || local >= numel(d.full_shape, d.ndim)) continue;  // not covered
      int64_t src = 0, stride = 1;
      bool live = true;
      for (int a = d.ndim - 1; a >= 0; --a) {
        const int64_t fs = d.full_shape[a];
        const int64_t f = local % fs;
        local /= fs;
        int64_t c;
        if (d.map_offset[a] >= 0) c = __ldg(inv + d.map_offset[a] + f);
        else c = d.compact_shape[a] > 0 ? f : -1;
        live &= c >= 0;
        src += c * stride;
        stride *= d.compact_shape[a];
      }
      if (live) {
        const T v = compact[d.compact_offset + src];
        full[j] = accumulate ? static_cast<T>(full[j] + v) : v;
      } else if (zero_fill && !accumulate) {
        full[j] = static_cast<T>(0);
      }
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

static int grid_for(int64_t n, int per_thread = 1) {
  const int64_t want = (n + static_cast<int64_t>(kSliceThreads) * per_thread - 1) /
                       (static_cast<int64_t>(kSliceThreads) * per_thread);
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
#define SDP_EXTRACT_T(T)                  \
  switch (mask_bytes) {                   \
    case 1: SDP_EXTRACT(T, 1); break;     \
    case 2: SDP_EXTRACT(T, 2); break;     \
    case 4: SDP_EXTRACT(T, 4); break;     \
    default: SDP_EXTRACT(T, 8); break;    \
  }
  if (dtype == SDP_DTYPE_F32) { SDP_EXTRACT_T(float) }
  else if (dtype == SDP_DTYPE_F64) { SDP_EXTRACT_T(double) }
  else return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
#undef SDP_EXTRACT_T
#undef SDP_EXTRACT
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

static int check_descs(const sdp_slice_desc* d, int n) {
  (void)d;
  if (n < 1) return set_error(SDP_ERR_TOPOLOGY, "no slice descriptors");
  return SDP_OK;
}

int sdp_gather_slices(int dtype, const sdp_slice_desc* descs, int n_descs, const int32_t* fwd_maps,
                      const void* full, void* compact, int64_t compact_total, void* stream) {
  if (check_descs(descs, n_descs)) return SDP_ERR_TOPOLOGY;
  if (compact_total <= 0) return SDP_OK;
  const int grid = grid_for(compact_total);
  cudaStream_t s = as_stream(stream);
  if (dtype == SDP_DTYPE_F32)
    k_gather<float><<<grid, kSliceThreads, 0, s>>>(descs, n_descs, fwd_maps, static_cast<const float*>(full),
                                                   static_cast<float*>(compact), compact_total);
  else if (dtype == SDP_DTYPE_F64)
    k_gather<double><<<grid, kSliceThreads, 0, s>>>(descs, n_descs, fwd_maps, static_cast<const double*>(full),
                                                    static_cast<double*>(compact), compact_total);
  else
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_scatter_slices(int dtype, const sdp_slice_desc* descs, int n_descs, const int32_t* inv_maps,
                       const void* compact, void* full, int64_t full_lo, int64_t full_hi, int flags,
                       void* stream) {
  if (check_descs(descs, n_descs)) return SDP_ERR_TOPOLOGY;
  if (full_hi <= full_lo) return SDP_OK;
  const int grid = grid_for(full_hi - full_lo, kSliceElems);
  cudaStream_t s = as_stream(stream);
  if (dtype == SDP_DTYPE_F32)
    k_scatter<float><<<grid, kSliceThreads, 0, s>>>(descs, n_descs, inv_maps, static_cast<const float*>(compact),
                                                    static_cast<float*>(full), full_lo, full_hi, flags);
  else if (dtype == SDP_DTYPE_F64)
    k_scatter<double><<<grid, kSliceThreads, 0, s>>>(descs, n_descs, inv_maps, static_cast<const double*>(compact),
                                                     static_cast<double*>(full), full_lo, full_hi, flags);
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
