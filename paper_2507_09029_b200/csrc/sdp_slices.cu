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

// theta * mask_w, 16 B of theta per thread per iteration (VE elements, their
// VE mask words read as one aligned word when they fit 8 bytes), scalar tail;
// VEC = false: the scalar loop (unaligned buffers).
template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; };
template <> struct Vec16<double> { using type = double2; };

template <typename T, int MB, bool VEC>
__global__ void k_masked_extract(const T* __restrict__ theta, const typename MaskT<MB>::T* __restrict__ mask,
                                 int64_t total, int worker, T* __restrict__ out) {
  using M = typename MaskT<MB>::T;
  constexpr int VE = 16 / static_cast<int>(sizeof(T));
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int64_t done = 0;
  if constexpr (VEC) {
    using VT = typename Vec16<T>::type;
    const int64_t nvec = total / VE;
    for (int64_t v = tid; v < nvec; v += stride) {
      const VT x = __ldg(reinterpret_cast<const VT*>(theta) + v);
      const T* xe = reinterpret_cast<const T*>(&x);
      uint64_t mw = 0;  // the VE mask words, packed
      if constexpr (MB * VE <= 8) {
        if constexpr (MB * VE == 2) mw = __ldg(reinterpret_cast<const uint16_t*>(mask) + v);
        else if constexpr (MB * VE == 4) mw = __ldg(reinterpret_cast<const uint32_t*>(mask) + v);
        else mw = __ldg(reinterpret_cast<const unsigned long long*>(mask) + v);
      }
      VT y;
      T* ye = reinterpret_cast<T*>(&y);
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        uint64_t m;
        if constexpr (MB * VE <= 8) m = (mw >> (8 * MB * e)) & (MB == 8 ? ~0ull : ((1ull << (8 * MB)) - 1));
        else m = static_cast<uint64_t>(__ldg(mask + v * VE + e));
        ye[e] = xe[e] * static_cast<T>((m >> worker) & 1ull);  // a plain multiply: keeps -0.0 / NaN like numpy
      }
      reinterpret_cast<VT*>(out)[v] = y;
    }
    done = nvec * VE;
  }
  for (int64_t j = done + tid; j < total; j += stride) {
    const T m = static_cast<T>((static_cast<uint64_t>(__ldg(mask + j)) >> worker) & 1ull);
    out[j] = theta[j] * m;
  }
}

__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t mul, uint32_t shr) {
  return mul ? (__umulhi(n, mul) >> shr) : n;
}

// Persistent CTAs (a few per SM) walk the task list interleaved (task
// blockIdx.x + i * gridDim.x).  Per stage, kStage task records and their
// descriptors are loaded in parallel into shared memory: the task -> descriptor
// chain costs one round trip per kStage tasks instead of one per task.
//
// A task is either
//  * tiled (the walked row length >= kSliceThreads): elements
//    [elem_begin, elem_end) of every row in [row_begin, row_end).  A thread
//    owns the row positions tid + k * kSliceThreads; it resolves their column
//    offsets ONCE (the descriptor's expanded column table, col_tab) and reuses
//    them for every row, so a row costs one uniform row-map load plus one load
//    and one store per element -- no per-element division or map chain; or
//  * flat (short rows): whole rows [row_begin, row_end) flattened over the
//    CTA with a multiply-high division per element (small tensors only).
// Data loads of a batch are all issued before its first store.  The
// contiguous side (compact rows for gather, full rows for scatter) is
// accessed at consecutive thread positions (coalesced).  Offsets inside one
// tensor fit in 32 bits (rows * cols * inner < 2^31, checked on the host).
constexpr int kSliceBatch = 6;
template <typename T> constexpr int rows_per_iter() { return sizeof(T) == 8 ? 1 : 2; }
constexpr int kStage = 32;
constexpr int kSliceCtasPerSm = 4;  // <= 64 registers

// Per-launch (full, compact) base pointers of up to SDP_MAX_WORKERS segments
// (workers): a task's `seg` picks its pair, so ONE launch moves every
// worker's slices.  Lives in the kernel parameter space.
struct SegPtrs {
  void* full[SDP_MAX_WORKERS];
  void* compact[SDP_MAX_WORKERS];
  int n;
};

struct SliceStage {
  sdp_slice_task task[kStage];
  sdp_slice_desc desc[kStage];
};

__device__ __forceinline__ int stage_tasks(SliceStage& st, const sdp_slice_desc* __restrict__ descs,
                                           const sdp_slice_task* __restrict__ tasks, int n_tasks,
                                           int first) {
  const int stride = gridDim.x;
  const int n = min(kStage, (n_tasks - first + stride - 1) / stride);
  __syncthreads();  // the previous stage is consumed
  if (threadIdx.x < n) {
    const sdp_slice_task tk = tasks[first + threadIdx.x * stride];
    st.task[threadIdx.x] = tk;
    st.desc[threadIdx.x] = descs[tk.desc];
  }
  __syncthreads();
  return n;
}

template <typename T, bool REVERSE>
__device__ __forceinline__ void gather_tiled(const sdp_slice_task& tk, const sdp_slice_desc& d,
                                             const int32_t* __restrict__ fwd, T* __restrict__ full,
                                             T* __restrict__ compact, uint32_t row_len) {
  constexpr int kRowsPerIter = rows_per_iter<T>();
  const uint32_t row_stride = static_cast<uint32_t>(d.cols) * d.inner;
  T* const fbase = full + d.full_offset;
  T* const cbase = compact + d.compact_offset;
  for (uint32_t eb = tk.elem_begin + threadIdx.x; eb < static_cast<uint32_t>(tk.elem_end);
       eb += kSliceThreads * kSliceBatch) {
    int32_t co[kSliceBatch];  // offset of my element inside the full row, -1 = past the task
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k) {
      const uint32_t t = eb + k * kSliceThreads;
      co[k] = t < static_cast<uint32_t>(tk.elem_end)
                  ? (d.col_tab >= 0 ? __ldg(fwd + d.col_tab + t) : static_cast<int32_t>(t)) : -1;
    }
    for (int r0 = tk.row_begin; r0 < tk.row_end; r0 += kRowsPerIter) {
      T* fr[kRowsPerIter];
      T* cr[kRowsPerIter];
#pragma unroll
      for (int j = 0; j < kRowsPerIter; ++j) {
        const int r = min(r0 + j, tk.row_end - 1);  // a duplicated last row rewrites identical values
        const uint32_t f = d.row_map >= 0 ? __ldg(fwd + d.row_map + r) : static_cast<uint32_t>(r);
        fr[j] = fbase + f * row_stride;
        cr[j] = cbase + static_cast<uint32_t>(r) * row_len + eb;
      }
      T v[kRowsPerIter][kSliceBatch];
#pragma unroll
      for (int j = 0; j < kRowsPerIter; ++j)
#pragma unroll
        for (int k = 0; k < kSliceBatch; ++k)
          if (co[k] >= 0) v[j][k] = REVERSE ? cr[j][k * kSliceThreads] : __ldg(fr[j] + co[k]);
#pragma unroll
      for (int j = 0; j < kRowsPerIter; ++j)
#pragma unroll
        for (int k = 0; k < kSliceBatch; ++k) {
          if (co[k] < 0) continue;
          if (REVERSE) fr[j][co[k]] = v[j][k];
          else cr[j][k * kSliceThreads] = v[j][k];
        }
    }
  }
}

// Row copies (no column map): whole rows move as 16-B vectors -- a gather is
// a typeless copy -- when every row start on both sides is 16-B aligned.
constexpr int kVecPerThread = 2;   // 16-B vectors per thread per row
constexpr int kVecRows = 2;        // rows per iteration: 4 vectors (64 B) in flight per thread

template <typename T>
__device__ __forceinline__ bool rows_vectorizable(const sdp_slice_task& tk, const sdp_slice_desc& d,
                                                  const T* full, const T* compact, uint32_t row_len) {
  constexpr uint32_t VE = 16 / sizeof(T);
  const uint32_t row_stride = static_cast<uint32_t>(d.cols) * d.inner;
  return d.col_tab < 0 && d.col_map < 0 &&
         ((static_cast<uint64_t>(d.full_offset) | static_cast<uint64_t>(d.compact_offset) | row_stride | row_len |
           static_cast<uint32_t>(tk.elem_begin) | static_cast<uint32_t>(tk.elem_end)) % VE) == 0 &&
         (reinterpret_cast<uintptr_t>(full) | reinterpret_cast<uintptr_t>(compact)) % 16 == 0;
}

template <typename T, bool REVERSE>
__device__ __forceinline__ void gather_rows_vec(const sdp_slice_task& tk, const sdp_slice_desc& d,
                                                const int32_t* __restrict__ fwd, T* __restrict__ full,
                                                T* __restrict__ compact, uint32_t row_len) {
  constexpr uint32_t VE = 16 / sizeof(T);
  const uint32_t row_stride = static_cast<uint32_t>(d.cols) * d.inner;
  const uint32_t v0 = tk.elem_begin / VE, v1 = tk.elem_end / VE;
  T* const fbase = full + d.full_offset;
  T* const cbase = compact + d.compact_offset;
  for (uint32_t vb = v0 + threadIdx.x; vb < v1; vb += kSliceThreads * kVecPerThread) {
    for (int r0 = tk.row_begin; r0 < tk.row_end; r0 += kVecRows) {
      uint4* fr[kVecRows];
      uint4* cr[kVecRows];
#pragma unroll
      for (int j = 0; j < kVecRows; ++j) {
        const int r = min(r0 + j, tk.row_end - 1);  // a duplicated last row rewrites identical values
        const uint32_t f = d.row_map >= 0 ? __ldg(fwd + d.row_map + r) : static_cast<uint32_t>(r);
        fr[j] = reinterpret_cast<uint4*>(fbase + f * row_stride);
        cr[j] = reinterpret_cast<uint4*>(cbase + static_cast<uint32_t>(r) * row_len);
      }
      uint4 v[kVecRows][kVecPerThread];
#pragma unroll
      for (int j = 0; j < kVecRows; ++j)
#pragma unroll
        for (int k = 0; k < kVecPerThread; ++k) {
          const uint32_t q = vb + k * kSliceThreads;
          if (q < v1) v[j][k] = REVERSE ? __ldg(cr[j] + q) : __ldg(fr[j] + q);
        }
#pragma unroll
      for (int j = 0; j < kVecRows; ++j)
#pragma unroll
        for (int k = 0; k < kVecPerThread; ++k) {
          const uint32_t q = vb + k * kSliceThreads;
          if (q < v1) {
            if (REVERSE) fr[j][q] = v[j][k];
            else cr[j][q] = v[j][k];
          }
        }
    }
  }
}

template <typename T, bool REVERSE>
__device__ __forceinline__ void gather_flat(const sdp_slice_task& tk, const sdp_slice_desc& d,
                                            const int32_t* __restrict__ fwd, T* __restrict__ full,
                                            T* __restrict__ compact, uint32_t row_len) {
  const uint32_t n_el = static_cast<uint32_t>(tk.row_end - tk.row_begin) * row_len;
  const uint32_t row_stride = static_cast<uint32_t>(d.cols) * d.inner;
  T* const fbase = full + d.full_offset;
  T* const cbase = compact + d.compact_offset + static_cast<int64_t>(tk.row_begin) * row_len;
  for (uint32_t base = threadIdx.x; base < n_el; base += kSliceThreads * kSliceBatch) {
    int32_t src[kSliceBatch];  // element of the full tensor, -1 past the task
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k) {
      const uint32_t idx = base + k * kSliceThreads;
      src[k] = -1;
      if (idx < n_el) {
        const uint32_t rr = fast_div(idx, d.rowlen_mul, d.rowlen_shr);
        const uint32_t r = tk.row_begin + rr;
        const uint32_t t = idx - rr * row_len;
        const uint32_t fr = d.row_map >= 0 ? __ldg(fwd + d.row_map + r) : r;
        uint32_t e = fr * row_stride;
        if (d.col_map < 0) {
          e += t;
        } else {
          const uint32_t b = fast_div(t, d.inner_mul, d.inner_shr);
          e += static_cast<uint32_t>(__ldg(fwd + d.col_map + b)) * d.inner + (t - b * d.inner);
        }
        src[k] = static_cast<int32_t>(e);
      }
    }
    T v[kSliceBatch];
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k)
      if (src[k] >= 0) v[k] = REVERSE ? cbase[base + k * kSliceThreads] : __ldg(fbase + src[k]);
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k) {
      if (src[k] < 0) continue;
      if (REVERSE) fbase[src[k]] = v[k];
      else cbase[base + k * kSliceThreads] = v[k];
    }
  }
}

template <typename T, bool REVERSE>
__global__ void __launch_bounds__(kSliceThreads, kSliceCtasPerSm)
k_gather(const sdp_slice_desc* __restrict__ descs, const sdp_slice_task* __restrict__ tasks, int n_tasks,
         const int32_t* __restrict__ fwd, const __grid_constant__ SegPtrs segs) {
  __shared__ SliceStage st;
  for (int first = blockIdx.x; first < n_tasks; first += kStage * gridDim.x) {
    const int n = stage_tasks(st, descs, tasks, n_tasks, first);
    for (int i = 0; i < n; ++i) {
      const sdp_slice_task& tk = st.task[i];
      const sdp_slice_desc& d = st.desc[i];
      const int sg = segs.n == 1 ? 0 : tk.seg;
      T* const full = static_cast<T*>(segs.full[sg]);
      T* const compact = static_cast<T*>(segs.compact[sg]);
      const uint32_t row_len = static_cast<uint32_t>(d.ccols) * d.inner;
      if (row_len >= kSliceThreads) {
        if (rows_vectorizable<T>(tk, d, full, compact, row_len))
          gather_rows_vec<T, REVERSE>(tk, d, fwd, full, compact, row_len);
        else
          gather_tiled<T, REVERSE>(tk, d, fwd, full, compact, row_len);
      } else {
        gather_flat<T, REVERSE>(tk, d, fwd, full, compact, row_len);
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ void scatter_tiled(const sdp_slice_task& tk, const sdp_slice_desc& d,
                                              const int32_t* __restrict__ inv, const T* __restrict__ compact,
                                              T* __restrict__ full, uint32_t row_len, bool zero_fill,
                                              bool accumulate) {
  constexpr int kRowsPerIter = rows_per_iter<T>();
  const uint32_t crow_len = static_cast<uint32_t>(d.ccols) * d.inner;
  const T* const cbase = compact + d.compact_offset;
  T* const fbase = full + d.full_offset;
  for (uint32_t eb = tk.elem_begin + threadIdx.x; eb < static_cast<uint32_t>(tk.elem_end);
       eb += kSliceThreads * kSliceBatch) {
    int32_t co[kSliceBatch];  // compact column offset, -1 = not held, -2 = past the task
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k) {
      const uint32_t t = eb + k * kSliceThreads;
      co[k] = t < static_cast<uint32_t>(tk.elem_end)
                  ? (d.col_tab >= 0 ? __ldg(inv + d.col_tab + t) : static_cast<int32_t>(t)) : -2;
    }
    for (int r0 = tk.row_begin; r0 < tk.row_end; r0 += kRowsPerIter) {
      T* fr[kRowsPerIter];
      int32_t a[kRowsPerIter];  // compact row, -1 = row not held
#pragma unroll
      for (int j = 0; j < kRowsPerIter; ++j) {
        const int f = min(r0 + j, tk.row_end - 1);  // a duplicated last row rewrites identical values
        a[j] = d.crows == 0 ? -1 : (d.row_map >= 0 ? __ldg(inv + d.row_map + f) : f);
        fr[j] = fbase + static_cast<uint32_t>(f) * row_len + eb;
      }
      T v[kRowsPerIter][kSliceBatch];
      if (accumulate) {
        // the full-side loads go out with the compact ones (one round trip);
        // not idempotent: never apply a duplicated last row twice
        T o[kRowsPerIter][kSliceBatch];
#pragma unroll
        for (int j = 0; j < kRowsPerIter; ++j) {
          const T* crow = cbase + static_cast<uint32_t>(max(a[j], 0)) * crow_len;
          const bool live = r0 + j < tk.row_end && a[j] >= 0;
#pragma unroll
          for (int k = 0; k < kSliceBatch; ++k) {
            v[j][k] = T(0);
            o[j][k] = T(0);
            if (live && co[k] >= 0) {
              v[j][k] = __ldg(crow + co[k]);
              o[j][k] = fr[j][k * kSliceThreads];
            }
          }
        }
#pragma unroll
        for (int j = 0; j < kRowsPerIter; ++j)
#pragma unroll
          for (int k = 0; k < kSliceBatch; ++k) v[j][k] = static_cast<T>(o[j][k] + v[j][k]);
      } else {
#pragma unroll
        for (int j = 0; j < kRowsPerIter; ++j) {
          const T* crow = cbase + static_cast<uint32_t>(max(a[j], 0)) * crow_len;
#pragma unroll
          for (int k = 0; k < kSliceBatch; ++k) {
            v[j][k] = T(0);
            if (a[j] >= 0 && co[k] >= 0) v[j][k] = __ldg(crow + co[k]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kRowsPerIter; ++j) {
        if (accumulate && r0 + j >= tk.row_end) continue;
#pragma unroll
        for (int k = 0; k < kSliceBatch; ++k) {
          const bool held = a[j] >= 0 && co[k] >= 0;
          if (held || (zero_fill && co[k] != -2)) fr[j][k * kSliceThreads] = v[j][k];
        }
      }
    }
  }
}

// Row write-back (no column map) as 16-B vectors: held rows are copied (or
// added elementwise in ACCUMULATE mode), rows the worker does not hold are
// zero-filled in ZERO_FILL mode.
template <typename T>
__device__ __forceinline__ void scatter_rows_vec(const sdp_slice_task& tk, const sdp_slice_desc& d,
                                                 const int32_t* __restrict__ inv, const T* __restrict__ compact,
                                                 T* __restrict__ full, uint32_t row_len, bool zero_fill,
                                                 bool accumulate) {
  constexpr uint32_t VE = 16 / sizeof(T);
  const uint32_t v0 = tk.elem_begin / VE, v1 = tk.elem_end / VE;
  const T* const cbase = compact + d.compact_offset;
  T* const fbase = full + d.full_offset;
  for (uint32_t vb = v0 + threadIdx.x; vb < v1; vb += kSliceThreads * kVecPerThread) {
    for (int r0 = tk.row_begin; r0 < tk.row_end; r0 += kVecRows) {
      uint4* fr[kVecRows];
      const uint4* cr[kVecRows];
      bool held[kVecRows], live[kVecRows];
#pragma unroll
      for (int j = 0; j < kVecRows; ++j) {
        const int f = min(r0 + j, tk.row_end - 1);
        live[j] = r0 + j < tk.row_end;  // never apply a duplicated row twice (accumulate)
        const int32_t a = d.crows == 0 ? -1 : (d.row_map >= 0 ? __ldg(inv + d.row_map + f) : f);
        held[j] = a >= 0;
        fr[j] = reinterpret_cast<uint4*>(fbase + static_cast<uint32_t>(f) * row_len);
        cr[j] = reinterpret_cast<const uint4*>(cbase + static_cast<uint32_t>(max(a, 0)) * row_len);
      }
      uint4 v[kVecRows][kVecPerThread], o[kVecRows][kVecPerThread];
#pragma unroll
      for (int j = 0; j < kVecRows; ++j)
#pragma unroll
        for (int k = 0; k < kVecPerThread; ++k) {
          const uint32_t q = vb + k * kSliceThreads;
          v[j][k] = make_uint4(0, 0, 0, 0);
          if (q < v1 && held[j]) {
            v[j][k] = __ldg(cr[j] + q);
            if (accumulate && live[j]) o[j][k] = fr[j][q];
          }
        }
#pragma unroll
      for (int j = 0; j < kVecRows; ++j)
#pragma unroll
        for (int k = 0; k < kVecPerThread; ++k) {
          const uint32_t q = vb + k * kSliceThreads;
          if (q >= v1 || !live[j]) continue;
          if (accumulate) {
            if (!held[j]) continue;
            T* a = reinterpret_cast<T*>(&o[j][k]);
            const T* b = reinterpret_cast<const T*>(&v[j][k]);
#pragma unroll
            for (uint32_t e = 0; e < VE; ++e) a[e] = static_cast<T>(a[e] + b[e]);
            fr[j][q] = o[j][k];
          } else if (held[j] || zero_fill) {
            fr[j][q] = v[j][k];  // zeros for a row the worker does not hold
          }
        }
    }
  }
}

template <typename T>
__device__ __forceinline__ void scatter_flat(const sdp_slice_task& tk, const sdp_slice_desc& d,
                                             const int32_t* __restrict__ inv, const T* __restrict__ compact,
                                             T* __restrict__ full, uint32_t row_len, bool zero_fill,
                                             bool accumulate) {
  const uint32_t crow_len = static_cast<uint32_t>(d.ccols) * d.inner;
  const uint32_t n_el = static_cast<uint32_t>(tk.row_end - tk.row_begin) * row_len;
  const T* const cbase = compact + d.compact_offset;
  T* const f0 = full + d.full_offset + static_cast<int64_t>(tk.row_begin) * row_len;
  for (uint32_t base = threadIdx.x; base < n_el; base += kSliceThreads * kSliceBatch) {
    int32_t src[kSliceBatch];  // compact element, -1 = not held, -2 = past the task
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k) {
      const uint32_t idx = base + k * kSliceThreads;
      src[k] = -2;
      if (idx < n_el) {
        const uint32_t rr = fast_div(idx, d.rowlen_mul, d.rowlen_shr);
        const uint32_t f = tk.row_begin + rr;
        const uint32_t t = idx - rr * row_len;
        const int32_t a = d.crows == 0 ? -1
                          : (d.row_map >= 0 ? __ldg(inv + d.row_map + f) : static_cast<int32_t>(f));
        int32_t s = -1;
        if (a >= 0) {
          if (d.col_map < 0) {
            s = static_cast<int32_t>(a * crow_len + t);
          } else {
            const uint32_t fb = fast_div(t, d.inner_mul, d.inner_shr);
            const int32_t cb = __ldg(inv + d.col_map + fb);
            if (cb >= 0) s = static_cast<int32_t>(a * crow_len + cb * d.inner + (t - fb * d.inner));
          }
        }
        src[k] = s;
      }
    }
    T v[kSliceBatch];
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k) {
      v[k] = T(0);
      if (src[k] >= 0) v[k] = __ldg(cbase + src[k]);
    }
    if (accumulate) {
#pragma unroll
      for (int k = 0; k < kSliceBatch; ++k)
        if (src[k] >= 0) v[k] = static_cast<T>(f0[base + k * kSliceThreads] + v[k]);
    }
#pragma unroll
    for (int k = 0; k < kSliceBatch; ++k) {
      // zero fill: the worker does not hold this element (v stays 0)
      if (src[k] >= 0 || (src[k] == -1 && zero_fill)) f0[base + k * kSliceThreads] = v[k];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kSliceThreads, kSliceCtasPerSm)
k_scatter(const sdp_slice_desc* __restrict__ descs, const sdp_slice_task* __restrict__ tasks, int n_tasks,
          const int32_t* __restrict__ inv, const __grid_constant__ SegPtrs segs, int flags) {
  __shared__ SliceStage st;
  const bool zero_fill = (flags & SDP_SCATTER_ZERO_FILL) && !(flags & SDP_SCATTER_ACCUMULATE);
  const bool accumulate = (flags & SDP_SCATTER_ACCUMULATE) != 0;
  for (int first = blockIdx.x; first < n_tasks; first += kStage * gridDim.x) {
    const int n = stage_tasks(st, descs, tasks, n_tasks, first);
    for (int i = 0; i < n; ++i) {
      const sdp_slice_task& tk = st.task[i];
      const sdp_slice_desc& d = st.desc[i];
      const int sg = segs.n == 1 ? 0 : tk.seg;
      T* const full = static_cast<T*>(segs.full[sg]);
      const T* const compact = static_cast<const T*>(segs.compact[sg]);
      const uint32_t row_len = static_cast<uint32_t>(d.cols) * d.inner;
      if (row_len >= kSliceThreads) {
        if (rows_vectorizable<T>(tk, d, full, compact, row_len))
          scatter_rows_vec<T>(tk, d, inv, compact, full, row_len, zero_fill, accumulate);
        else
          scatter_tiled<T>(tk, d, inv, compact, full, row_len, zero_fill, accumulate);
      } else {
        scatter_flat<T>(tk, d, inv, compact, full, row_len, zero_fill, accumulate);
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

static int slice_grid(int n_tasks) {
  return std::max(1, std::min(n_tasks, sm_count() * kSliceCtasPerSm));
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
  // 16-B vectors when theta / out are 16-B aligned and the mask words of a
  // vector are aligned to their packed size
  const int esz = dtype == SDP_DTYPE_F64 ? 8 : 4;
  const uintptr_t mal = static_cast<uintptr_t>(mask_bytes) * (16 / esz);
  const bool vec = ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(out)) % 16) == 0 &&
                   reinterpret_cast<uintptr_t>(owner_mask) % (mal < 8 ? mal : 8) == 0;
#define SDP_EXTRACT(TT, MB)                                                                        \
  do {                                                                                             \
    if (vec)                                                                                       \
      k_masked_extract<TT, MB, true><<<grid, kSliceThreads, 0, s>>>(static_cast<const TT*>(theta), \
          static_cast<const MaskT<MB>::T*>(owner_mask), total, worker, static_cast<TT*>(out));     \
    else                                                                                           \
      k_masked_extract<TT, MB, false><<<grid, kSliceThreads, 0, s>>>(static_cast<const TT*>(theta),\
          static_cast<const MaskT<MB>::T*>(owner_mask), total, worker, static_cast<TT*>(out));     \
  } while (0)
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

static int gather_launch(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks, int n_tasks,
                         const int32_t* fwd_maps, const SegPtrs& sp, int flags, void* stream) {
  cudaStream_t s = as_stream(stream);
  const bool rev = (flags & SDP_GATHER_REVERSE) != 0;
  const int grid = slice_grid(n_tasks);
#define SDP_GATHER(TT)                                                                              \
  do {                                                                                              \
    if (rev) k_gather<TT, true><<<grid, kSliceThreads, 0, s>>>(descs, tasks, n_tasks, fwd_maps, sp);  \
    else k_gather<TT, false><<<grid, kSliceThreads, 0, s>>>(descs, tasks, n_tasks, fwd_maps, sp);     \
  } while (0)
  if (dtype == SDP_DTYPE_F32) SDP_GATHER(float);
  else if (dtype == SDP_DTYPE_F64) SDP_GATHER(double);
  else if (dtype == SDP_DTYPE_U8) SDP_GATHER(uint8_t);
  else if (dtype == SDP_DTYPE_U16) SDP_GATHER(uint16_t);
  else return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32, SDP_DTYPE_F64, SDP_DTYPE_U8 or SDP_DTYPE_U16");
#undef SDP_GATHER
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

static int scatter_launch(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks, int n_tasks,
                          const int32_t* inv_maps, const SegPtrs& sp, int flags, void* stream) {
  cudaStream_t s = as_stream(stream);
  const int grid = slice_grid(n_tasks);
  if (dtype == SDP_DTYPE_F32)
    k_scatter<float><<<grid, kSliceThreads, 0, s>>>(descs, tasks, n_tasks, inv_maps, sp, flags);
  else if (dtype == SDP_DTYPE_F64)
    k_scatter<double><<<grid, kSliceThreads, 0, s>>>(descs, tasks, n_tasks, inv_maps, sp, flags);
  else
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

static int segs_from(const sdp_slice_segs* in, SegPtrs& sp, bool need_compact) {
  if (!in) return set_error(SDP_ERR_USAGE, "null segment table");
  if (in->n < 1 || in->n > SDP_MAX_WORKERS)
    return set_error(SDP_ERR_CONFIG, "segment count %d outside [1, %d]", in->n, SDP_MAX_WORKERS);
  sp = SegPtrs{};
  sp.n = in->n;
  for (int k = 0; k < in->n; ++k) {
    if (!in->full[k] || (need_compact && !in->compact[k]))
      return set_error(SDP_ERR_USAGE, "segment %d has a null buffer", k);
    sp.full[k] = const_cast<void*>(in->full[k]);
    sp.compact[k] = const_cast<void*>(in->compact[k]);
  }
  return SDP_OK;
}

int sdp_gather_slices(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                      int n_tasks, const int32_t* fwd_maps, const void* full, void* compact,
                      int flags, void* stream) {
  if (n_tasks < 0) return set_error(SDP_ERR_USAGE, "negative task count");
  if (n_tasks == 0) return SDP_OK;
  if (!descs || !tasks || !full || !compact) return set_error(SDP_ERR_USAGE, "null device pointer");
  SegPtrs sp{};
  sp.n = 1;
  sp.full[0] = const_cast<void*>(full);
  sp.compact[0] = compact;
  return gather_launch(dtype, descs, tasks, n_tasks, fwd_maps, sp, flags, stream);
}

int sdp_gather_slices_multi(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                            int n_tasks, const int32_t* fwd_maps, const sdp_slice_segs* segs, int flags,
                            void* stream) {
  if (n_tasks < 0) return set_error(SDP_ERR_USAGE, "negative task count");
  SegPtrs sp;
  if (int rc = segs_from(segs, sp, true)) return rc;
  if (n_tasks == 0) return SDP_OK;
  if (!descs || !tasks) return set_error(SDP_ERR_USAGE, "null device pointer");
  return gather_launch(dtype, descs, tasks, n_tasks, fwd_maps, sp, flags, stream);
}

int sdp_scatter_slices(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                       int n_tasks, const int32_t* inv_maps, const void* compact, void* full,
                       int flags, void* stream) {
  if (n_tasks < 0) return set_error(SDP_ERR_USAGE, "negative task count");
  if (n_tasks == 0) return SDP_OK;
  if (!descs || !tasks || !full) return set_error(SDP_ERR_USAGE, "null device pointer");
  SegPtrs sp{};
  sp.n = 1;
  sp.full[0] = full;
  sp.compact[0] = const_cast<void*>(compact);
  return scatter_launch(dtype, descs, tasks, n_tasks, inv_maps, sp, flags, stream);
}

int sdp_scatter_slices_multi(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                             int n_tasks, const int32_t* inv_maps, const sdp_slice_segs* segs, int flags,
                             void* stream) {
  if (n_tasks < 0) return set_error(SDP_ERR_USAGE, "negative task count");
  SegPtrs sp;
  if (int rc = segs_from(segs, sp, false)) return rc;
  if (n_tasks == 0) return SDP_OK;
  if (!descs || !tasks) return set_error(SDP_ERR_USAGE, "null device pointer");
  return scatter_launch(dtype, descs, tasks, n_tasks, inv_maps, sp, flags, stream);
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
