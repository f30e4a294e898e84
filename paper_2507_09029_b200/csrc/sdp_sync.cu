// Owner-subset sync: engine.aggregate (engine.py:60-79) as one HBM/NVLink-bound
// kernel.
//
// Work unit = a tile of `tile` consecutive elements of the flat vector.  Each
// CTA owns a CTA-major run of tile descriptors, staged into shared memory by
// one bulk copy (cp.async.bulk + mbarrier, the TMA engine's non-tensor form).
// For each element j with owner set O_j:
//     acc = +0; for w in O_j ascending: acc += replica[w][j]
//     mean = acc / max(|O_j|, 1)                 (IEEE divide)
// and the mean goes to out / out_bf16 and (WRITEBACK) into every owner's replica
// and bf16 shadow.  Uniform tiles (one owner set, the block strategy) run fully
// vectorised 16-B loads with all owners' loads in flight; mixed tiles (neuron
// strategy) read a per-element owner mask and only ever add owners.
//
// Replica pointers may be local (N logical workers co-resident in one HBM) or
// peer-mapped NVLink addresses (one worker per GPU); with world > 1 each rank
// runs only the tiles it leads, bracketed by release/acquire flag barriers.
#include "sdp_common.cuh"

#include <cmath>
#include <type_traits>

namespace sdp {

constexpr int kSyncThreads = 256;
constexpr int kStage = 512;  // descriptors staged per bulk copy (8 KB)
#ifndef SDP_STREAM_CTAS
#define SDP_STREAM_CTAS 4
#endif
constexpr int kStreamCtasPerSm = SDP_STREAM_CTAS;  // resident CTAs of the streaming kernel

template <typename T> struct V;
template <> struct V<float> {
  static constexpr int N = 4;
  struct type { float x[4]; };
  __device__ static __forceinline__ type ld(const float* p) {
    float4 r = ld_stream_f4(reinterpret_cast<const float4*>(p));
    return type{{r.x, r.y, r.z, r.w}};
  }
  __device__ static __forceinline__ type ld_rw(const float* p) {
    float4 r = *reinterpret_cast<const float4*>(p);
    return type{{r.x, r.y, r.z, r.w}};
  }
  __device__ static __forceinline__ void st(float* p, const type& v) {
    st_f4(reinterpret_cast<float4*>(p), make_float4(v.x[0], v.x[1], v.x[2], v.x[3]));
  }
  __device__ static __forceinline__ void st_bf16(__nv_bfloat16* p, const type& v) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x[0], v.x[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn(v.x[2], v.x[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  }
};
template <> struct V<double> {
  static constexpr int N = 2;
  struct type { double x[2]; };
  __device__ static __forceinline__ type ld(const double* p) {
    double2 r = ld_stream_d2(reinterpret_cast<const double2*>(p));
    return type{{r.x, r.y}};
  }
  __device__ static __forceinline__ type ld_rw(const double* p) {
    double2 r = *reinterpret_cast<const double2*>(p);
    return type{{r.x, r.y}};
  }
  __device__ static __forceinline__ void st(double* p, const type& v) {
    st_d2(reinterpret_cast<double2*>(p), make_double2(v.x[0], v.x[1]));
  }
  __device__ static __forceinline__ void st_bf16(__nv_bfloat16* p, const type& v) {
    __nv_bfloat162 a;
    a.x = __double2bfloat16(v.x[0]);
    a.y = __double2bfloat16(v.x[1]);
    *reinterpret_cast<__nv_bfloat162*>(p) = a;
  }
};

__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ __nv_bfloat16 to_bf16(float x) { return __float2bfloat16_rn(x); }
__device__ __forceinline__ __nv_bfloat16 to_bf16(double x) { return __double2bfloat16(x); }
__device__ __forceinline__ bool finite(float x) { return isfinite(x); }
__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

// Kernel parameter block (lives in the constant bank; ~1.3 KB).
struct SyncParams {
  const void* owner_mask;
  const sdp_tile_desc* tiles;
  void* replicas[SDP_MAX_WORKERS];
  void* shadow[SDP_MAX_WORKERS];
  void* out;
  void* out_bf16;
  void* theta;
  void* velocity;
  void* theta_bf16;
  uint32_t* status;
  uint32_t* pads[8];
  double lr, momentum;
  void* second_moment;                                  // Adam v
  double beta1, beta2, omb1, omb2, bias1, bias2, eps;   // Adam scalars
  int64_t total;
  int64_t timeout_cycles;
  const int32_t* slots;                                 // compact storage (or null)
  int64_t slot_stride;
  const sdp_update_desc* updates;                       // LOCAL_UPDATE phase
  const sdp_worker_state* states;
  int32_t updates_per_cta;
  int32_t n_workers, tile, n_tiles, tiles_per_cta, flags, rank, world;
  uint32_t epoch;
  bool has_shadow;
  uint32_t* epoch_ctr;  // device-resident barrier epochs (graph replay), or null
  const int32_t* adam_step;       // device-resident Adam step, or null (then bias1 / bias2)
  const double* adam_bias_table;  // [2 * adam_table_len]: 1 - beta1^t, 1 - beta2^t
  int32_t adam_table_len;
};

// Adam bias corrections: the host scalars, or the device step's table entry.
__device__ __forceinline__ double adam_bias(const SyncParams& p, int k) {
  if (!p.adam_step) return k == 0 ? p.bias1 : p.bias2;
  const int t = min(max(__ldg(p.adam_step), 0), p.adam_table_len - 1);
  return __ldg(p.adam_bias_table + 2 * t + k);
}

// Pairwise per-CTA barrier: CTA b of every rank meets CTA b of every other rank.
// Completion of a launch therefore implies every peer CTA has finished too.
__device__ bool cross_rank_barrier(const SyncParams& p, uint32_t value) {
  bool ok = true;
  __syncthreads();
  if (threadIdx.x < p.world) {
    __threadfence_system();
    const int peer = threadIdx.x;
    st_release_sys(p.pads[peer] + blockIdx.x * p.world + p.rank, value);
    const uint32_t* mine = p.pads[p.rank] + blockIdx.x * p.world + peer;
    const long long t0 = clock64();
    while (static_cast<int32_t>(ld_acquire_sys(mine) - value) < 0) {
      if (clock64() - t0 > p.timeout_cycles) {
        ok = false;
        if (p.status) atomicOr(p.status, SDP_STATUS_BARRIER_TIMEOUT);
        break;
      }
    }
  }
  return __syncthreads_and(ok);
}

__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }

// One optimizer step on one element, every operation rounded exactly where
// numpy rounds it (no FMA contraction):
//   SGD-Nesterov (optim.py:81-84): v = v*mu + g;  th = th - lr*(g + mu*v)
//   Adam (optim.py:101-109): m = b1*m + (1-b1)*g;  v = b2*v + ((1-b2)*g)*g;
//                            th = th - (lr*(m/c1)) / (sqrt(v/c2) + eps)
template <typename T>
__device__ __forceinline__ void optim_step(const SyncParams& p, T g, T& th, T& s1, T& s2) {
  const T lr = static_cast<T>(p.lr);
  if (p.flags & SDP_SYNC_NESTEROV) {
    const T mu = static_cast<T>(p.momentum);
    s1 = add_rn(mul_rn(s1, mu), g);
    th = sub_rn(th, mul_rn(lr, add_rn(g, mul_rn(mu, s1))));
  } else {
    s1 = add_rn(mul_rn(static_cast<T>(p.beta1), s1), mul_rn(static_cast<T>(p.omb1), g));
    s2 = add_rn(mul_rn(static_cast<T>(p.beta2), s2), mul_rn(mul_rn(static_cast<T>(p.omb2), g), g));
    const T mh = div_rn(s1, static_cast<T>(adam_bias(p, 0)));
    const T vh = div_rn(s2, static_cast<T>(adam_bias(p, 1)));
    th = sub_rn(th, div_rn(mul_rn(lr, mh), add_rn(sqrt_rn(vh), static_cast<T>(p.eps))));
  }
}

// The leader's epilogue applies the optimizer to the flat theta only when the
// update is not a separate local phase.
__device__ __forceinline__ bool epilogue_optim(const SyncParams& p) {
  return (p.flags & (SDP_SYNC_NESTEROV | SDP_SYNC_ADAM)) && !(p.flags & SDP_SYNC_LOCAL_UPDATE);
}

template <typename T>
__device__ __forceinline__ void nesterov_elem(const SyncParams& p, int64_t j, T g) {
  T* th = static_cast<T*>(p.theta);
  T* s1 = static_cast<T*>(p.velocity);
  T* s2 = static_cast<T*>(p.second_moment);
  T t = th[j], a = s1[j], b = s2 ? s2[j] : static_cast<T>(0);
  optim_step<T>(p, g, t, a, b);
  s1[j] = a;
  if (s2) s2[j] = b;
  th[j] = t;
  if (p.theta_bf16) static_cast<__nv_bfloat16*>(p.theta_bf16)[j] = to_bf16(t);
}

// Replica / shadow of worker w for tile `tix`: the flat layout (tile tix at
// tix*tile) or the compact owned-tile layout (slot table); null = not stored.
template <typename T, bool CS>
__device__ __forceinline__ T* rep_tile(const SyncParams& p, int w, uint32_t tix) {
  T* base = static_cast<T*>(p.replicas[w]);
  if constexpr (!CS) return base + static_cast<int64_t>(tix) * p.tile;
  const int32_t sl = __ldg(p.slots + static_cast<int64_t>(w) * p.slot_stride + tix);
  return sl < 0 ? nullptr : base + static_cast<int64_t>(sl) * p.tile;
}
template <bool CS>
__device__ __forceinline__ __nv_bfloat16* shadow_tile(const SyncParams& p, int w, uint32_t tix) {
  __nv_bfloat16* base = static_cast<__nv_bfloat16*>(p.shadow[w]);
  if (!base) return nullptr;
  if constexpr (!CS) return base + static_cast<int64_t>(tix) * p.tile;
  const int32_t sl = __ldg(p.slots + static_cast<int64_t>(w) * p.slot_stride + tix);
  return sl < 0 ? nullptr : base + static_cast<int64_t>(sl) * p.tile;
}

// Epilogue for one element (tile tix, flat start s, offset o) with owner set m.
template <typename T, bool CS>
__device__ __forceinline__ void emit_scalar(const SyncParams& p, uint32_t tix, int64_t s, int o, uint64_t m,
                                            T mean) {
  const int64_t j = s + o;
  if (p.out) static_cast<T*>(p.out)[j] = mean;
  if (p.out_bf16) static_cast<__nv_bfloat16*>(p.out_bf16)[j] = to_bf16(mean);
  if (p.flags & SDP_SYNC_WRITEBACK) {
    for (uint64_t b = m; b; b &= b - 1) {
      const int w = __ffsll(static_cast<long long>(b)) - 1;
      rep_tile<T, CS>(p, w, tix)[o] = mean;
      if (p.has_shadow) {
        __nv_bfloat16* sh = shadow_tile<CS>(p, w, tix);
        if (sh) sh[o] = to_bf16(mean);
      }
    }
  }
  if (epilogue_optim(p)) nesterov_elem<T>(p, j, mean);
}

// Scalar path: one element, owner set `m` (partial tiles, unaligned tails).
template <typename T, bool CS>
__device__ __forceinline__ void sync_elem(const SyncParams& p, uint32_t tix, int64_t s, int o, uint64_t m,
                                          uint32_t& st) {
  T acc = static_cast<T>(0);
  for (uint64_t b = m; b; b &= b - 1) {
    const int w = __ffsll(static_cast<long long>(b)) - 1;
    acc = add_rn(acc, rep_tile<const T, CS>(p, w, tix)[o]);
  }
  const int c = __popcll(m);
  const T mean = div_rn(acc, static_cast<T>(c > 0 ? c : 1));
  if (c == 0 && (p.flags & SDP_SYNC_CHECK_UNCOVERED)) {
    for (int w = 0; w < p.n_workers; ++w) {
      const T* g = rep_tile<const T, CS>(p, w, tix);
      if (g && !finite(g[o])) st |= SDP_STATUS_UNCOVERED_LEAK;
    }
  }
  if ((p.flags & SDP_SYNC_CHECK_FINITE) && !finite(mean)) st |= SDP_STATUS_NONFINITE;
  emit_scalar<T, CS>(p, tix, s, o, m, mean);
}

// Epilogue for one vector of VN consecutive elements with a common owner set.
template <typename T, bool CS>
__device__ __forceinline__ void emit_vec(const SyncParams& p, uint32_t tix, int64_t s, int o, uint64_t bits,
                                         const typename V<T>::type& mean) {
  constexpr int VN = V<T>::N;
  const int64_t j = s + o;
  if (p.out) V<T>::st(static_cast<T*>(p.out) + j, mean);
  if (p.out_bf16) V<T>::st_bf16(static_cast<__nv_bfloat16*>(p.out_bf16) + j, mean);
  if (p.flags & SDP_SYNC_WRITEBACK) {
    for (uint64_t b = bits; b; b &= b - 1) {
      const int w = __ffsll(static_cast<long long>(b)) - 1;
      V<T>::st(rep_tile<T, CS>(p, w, tix) + o, mean);
      if (p.has_shadow) {
        __nv_bfloat16* sh = shadow_tile<CS>(p, w, tix);
        if (sh) V<T>::st_bf16(sh + o, mean);
      }
    }
  }
  if (epilogue_optim(p)) {
    T* thp = static_cast<T*>(p.theta) + j;
    T* s1p = static_cast<T*>(p.velocity) + j;
    T* s2p = p.second_moment ? static_cast<T*>(p.second_moment) + j : nullptr;
    typename V<T>::type th = V<T>::ld_rw(thp), s1 = V<T>::ld_rw(s1p), s2 = s1;
    if (s2p) s2 = V<T>::ld_rw(s2p);
#pragma unroll
    for (int e = 0; e < VN; ++e) optim_step<T>(p, mean.x[e], th.x[e], s1.x[e], s2.x[e]);
    V<T>::st(s1p, s1);
    if (s2p) V<T>::st(s2p, s2);
    V<T>::st(thp, th);
    if (p.theta_bf16) V<T>::st_bf16(static_cast<__nv_bfloat16*>(p.theta_bf16) + j, th);
  }
}

// Uniform tile: every element has owner set `bits`.  R vectors per thread per
// round, owners consumed two at a time so 2R 16-B loads are in flight.
template <typename T, int R, bool CS>
__device__ __forceinline__ void sync_uniform_tile(const SyncParams& p, uint32_t tix, int64_t s, uint64_t bits,
                                                  uint32_t& st) {
  constexpr int VN = V<T>::N;
  using Vt = typename V<T>::type;
  const int per_round = R * VN * kSyncThreads;
  const int c = __popcll(bits);
  const T denom = static_cast<T>(c > 0 ? c : 1);
  for (int r0 = 0; r0 < p.tile; r0 += per_round) {
    Vt acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k)
#pragma unroll
      for (int e = 0; e < VN; ++e) acc[k].x[e] = static_cast<T>(0);
    int ov[R];
#pragma unroll
    for (int k = 0; k < R; ++k) ov[k] = r0 + (k * kSyncThreads + threadIdx.x) * VN;
    // Owners in ascending order, K at a time: all K*R 16-B loads of a batch are
    // issued before the first add (K = 2 for R >= 2, 4 for R = 1: fits the
    // 64-register budget of 4 resident CTAs per SM without spills).
    constexpr int K = R >= 2 ? 2 : 4;
    uint64_t b = bits;
    while (b) {
      const T* g[K];
      bool on[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        on[q] = b != 0;
        const int w = on[q] ? __ffsll(static_cast<long long>(b)) - 1 : 0;
        if (on[q]) b &= b - 1;
        g[q] = on[q] ? rep_tile<const T, CS>(p, w, tix) : nullptr;
      }
      Vt a[K][R];
#pragma unroll
      for (int q = 0; q < K; ++q)
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (on[q]) a[q][k] = V<T>::ld(g[q] + ov[k]);
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (on[q]) {
#pragma unroll
          for (int k = 0; k < R; ++k)
#pragma unroll
            for (int e = 0; e < VN; ++e) acc[k].x[e] = add_rn(acc[k].x[e], a[q][k].x[e]);
        }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      Vt mean;
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        mean.x[e] = div_rn(acc[k].x[e], denom);
        if ((p.flags & SDP_SYNC_CHECK_FINITE) && !finite(mean.x[e])) st |= SDP_STATUS_NONFINITE;
      }
      if (c == 0 && (p.flags & SDP_SYNC_CHECK_UNCOVERED)) {
        for (int w = 0; w < p.n_workers; ++w) {
          const T* gw = rep_tile<const T, CS>(p, w, tix);
          if (!gw) continue;
          Vt g = V<T>::ld(gw + ov[k]);
#pragma unroll
          for (int e = 0; e < VN; ++e)
            if (!finite(g.x[e])) st |= SDP_STATUS_UNCOVERED_LEAK;
        }
      }
      emit_vec<T, CS>(p, tix, s, ov[k], bits, mean);
    }
  }
}

// Mixed tile: per-element owner sets from the owner mask (neuron strategy).
// Lane-per-element: a warp covers 32 consecutive elements, each thread EL of
// them at a stride of the CTA width, and the owners some lane of the warp
// needs (a warp-uniform OR of the lanes' masks, within the tile's union) are
// walked in ascending order, KQ at a time with all their loads in flight and
// per-lane predicates -- every load and store is a coalesced, predicated
// access that touches only owned elements, and each element adds exactly its
// own owners in ascending order (GPT-2 width-wise flat `aggregate`: 900 ->
// 796 us, profiles/r2_sync_mixed_variants_v2.jsonl; the R = 4 instantiation,
// whose registers are spoken for, walks the tile's union two at a time).
template <typename T, int MB, int R, bool CS, int KQ>
__device__ __forceinline__ void sync_mixed_tile(const SyncParams& p, uint32_t tix, int64_t s,
                                                uint64_t tile_union, uint32_t& st) {
  constexpr int EL = 4;  // elements per thread per round
  using M = typename MaskT<MB>::T;
  const M* mask = static_cast<const M*>(p.owner_mask) + s;
  const bool wb = (p.flags & SDP_SYNC_WRITEBACK) != 0;
  for (int r0 = 0; r0 < p.tile; r0 += EL * kSyncThreads) {
    int o[EL];
    uint64_t m[EL];
    T acc[EL];
#pragma unroll
    for (int u = 0; u < EL; ++u) {
      o[u] = r0 + u * kSyncThreads + threadIdx.x;
      m[u] = static_cast<uint64_t>(__ldg(mask + o[u]));
      acc[u] = static_cast<T>(0);
    }
    // only the owners some lane of THIS warp needs (warp-uniform; the tile's
    // union is the fallback bound)
    uint64_t b = tile_union;
    if constexpr (KQ > 2) {
      uint64_t lane_any = m[0];
#pragma unroll
      for (int u = 1; u < EL; ++u) lane_any |= m[u];
      const uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(lane_any));
      const uint32_t hi = MB > 4 ? __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(lane_any >> 32)) : 0u;
      b &= (static_cast<uint64_t>(hi) << 32) | lo;
    }
    if constexpr (KQ > 2) {
      while (b) {
        int wq[KQ];
#pragma unroll
        for (int q = 0; q < KQ; ++q) {
          wq[q] = b ? __ffsll(static_cast<long long>(b)) - 1 : 64;
          if (b) b &= b - 1;
        }
        T a[KQ][EL];
#pragma unroll
        for (int q = 0; q < KQ; ++q) {
          if (wq[q] == 64) continue;
          const T* g = rep_tile<const T, CS>(p, wq[q], tix);
#pragma unroll
          for (int u = 0; u < EL; ++u) a[q][u] = ((m[u] >> wq[q]) & 1ull) ? __ldcs(g + o[u]) : static_cast<T>(0);
        }
#pragma unroll
        for (int q = 0; q < KQ; ++q) {
          if (wq[q] == 64) continue;
#pragma unroll
          for (int u = 0; u < EL; ++u)
            if ((m[u] >> wq[q]) & 1ull) acc[u] = add_rn(acc[u], a[q][u]);
        }
      }
    } else {
      while (b) {
        const int w0 = __ffsll(static_cast<long long>(b)) - 1;
        b &= b - 1;
        const bool two = b != 0;
        const int w1 = two ? __ffsll(static_cast<long long>(b)) - 1 : w0;
        if (two) b &= b - 1;
        const T* g0 = rep_tile<const T, CS>(p, w0, tix);
        const T* g1 = rep_tile<const T, CS>(p, w1, tix);
        T a[EL], c[EL];
#pragma unroll
        for (int u = 0; u < EL; ++u) {
          a[u] = ((m[u] >> w0) & 1ull) ? __ldcs(g0 + o[u]) : static_cast<T>(0);
          c[u] = (two && ((m[u] >> w1) & 1ull)) ? __ldcs(g1 + o[u]) : static_cast<T>(0);
        }
#pragma unroll
        for (int u = 0; u < EL; ++u) {
          if ((m[u] >> w0) & 1ull) acc[u] = add_rn(acc[u], a[u]);
          if (two && ((m[u] >> w1) & 1ull)) acc[u] = add_rn(acc[u], c[u]);
        }
      }
    }
    T mean[EL];
#pragma unroll
    for (int u = 0; u < EL; ++u) {
      const int cnt = __popcll(m[u]);
      mean[u] = div_rn(acc[u], static_cast<T>(cnt > 0 ? cnt : 1));
      if ((p.flags & SDP_SYNC_CHECK_FINITE) && !finite(mean[u])) st |= SDP_STATUS_NONFINITE;
      if (cnt == 0 && (p.flags & SDP_SYNC_CHECK_UNCOVERED)) {
        for (int w = 0; w < p.n_workers; ++w) {
          const T* gw = rep_tile<const T, CS>(p, w, tix);
          if (gw && !finite(gw[o[u]])) st |= SDP_STATUS_UNCOVERED_LEAK;
        }
      }
      if (p.out) static_cast<T*>(p.out)[s + o[u]] = mean[u];
      if (p.out_bf16) static_cast<__nv_bfloat16*>(p.out_bf16)[s + o[u]] = to_bf16(mean[u]);
    }
    if (wb) {
      for (uint64_t bb = tile_union; bb; bb &= bb - 1) {
        const int w = __ffsll(static_cast<long long>(bb)) - 1;
        T* rep = rep_tile<T, CS>(p, w, tix);
        __nv_bfloat16* sh = p.has_shadow ? shadow_tile<CS>(p, w, tix) : nullptr;
#pragma unroll
        for (int u = 0; u < EL; ++u)
          if ((m[u] >> w) & 1ull) {
            rep[o[u]] = mean[u];
            if (sh) sh[o[u]] = to_bf16(mean[u]);
          }
      }
    }
    if (epilogue_optim(p)) {
#pragma unroll
      for (int u = 0; u < EL; ++u) nesterov_elem<T>(p, s + o[u], mean[u]);
    }
  }
}

template <typename T, int MB, int R, bool CS>
__device__ __forceinline__ void run_tile(const SyncParams& p, const sdp_tile_desc& d, uint32_t& st) {
  const int len = static_cast<int>(d.len_flags & SDP_TILE_LEN_MASK);
  if (len == 0) return;
  const uint32_t tix = d.tile_index;
  const int64_t s = static_cast<int64_t>(tix) * p.tile;
  const bool uniform = (d.len_flags & SDP_TILE_UNIFORM) != 0;
  if (len == p.tile) {
    if (uniform) sync_uniform_tile<T, R, CS>(p, tix, s, d.owner_bits, st);
    else sync_mixed_tile<T, MB, (R > 2 ? 2 : R), CS, (R > 2 ? 2 : 4)>(p, tix, s, d.owner_bits, st);
  } else {
    const typename MaskT<MB>::T* mask = static_cast<const typename MaskT<MB>::T*>(p.owner_mask);
    for (int e = threadIdx.x; e < len; e += kSyncThreads) {
      const uint64_t m = uniform ? d.owner_bits : static_cast<uint64_t>(mask[s + e]);
      sync_elem<T, CS>(p, tix, s, e, m, st);
    }
  }
}

// Third phase (SDP_SYNC_LOCAL_UPDATE): the optimizer on this rank's local
// workers' stored tiles whose leader ran in this CTA index (on any rank).  The
// gradient is the worker's own replica, which now holds the mean (written by
// the leader, possibly over NVLink, ordered by the exit barrier): read through
// L2 (ld.global.cg), never the non-coherent path.
template <typename T>
__device__ __forceinline__ void local_update(const SyncParams& p, uint32_t& st) {
  constexpr int VN = V<T>::N;
  using Vt = typename V<T>::type;
  const sdp_update_desc* ud = p.updates + static_cast<int64_t>(blockIdx.x) * p.updates_per_cta;
  for (int k = 0; k < p.updates_per_cta; ++k) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(ud + k));
    const int len = static_cast<int>(raw.z);
    if (len == 0) continue;
    const sdp_worker_state& ws = p.states[raw.x];
    const int64_t base = static_cast<int64_t>(raw.y) * p.tile;
    T* th = static_cast<T*>(ws.theta) + base;
    T* s1 = static_cast<T*>(ws.velocity) + base;
    T* s2 = ws.second_moment ? static_cast<T*>(ws.second_moment) + base : nullptr;
    const T* g = static_cast<const T*>(ws.grad) + base;
    __nv_bfloat16* tb = ws.theta_bf16 ? static_cast<__nv_bfloat16*>(ws.theta_bf16) + base : nullptr;
    const int nv = len / VN * VN;
    for (int o = threadIdx.x * VN; o < nv; o += kSyncThreads * VN) {
      Vt gv, tv = V<T>::ld_rw(th + o), v1 = V<T>::ld_rw(s1 + o), v2 = v1;
#pragma unroll
      for (int e = 0; e < VN; ++e) gv.x[e] = ld_cg(g + o + e);
      if (s2) v2 = V<T>::ld_rw(s2 + o);
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        if ((p.flags & SDP_SYNC_CHECK_FINITE) && !finite(gv.x[e])) st |= SDP_STATUS_NONFINITE;
        optim_step<T>(p, gv.x[e], tv.x[e], v1.x[e], v2.x[e]);
      }
      V<T>::st(s1 + o, v1);
      if (s2) V<T>::st(s2 + o, v2);
      V<T>::st(th + o, tv);
      if (tb) V<T>::st_bf16(tb + o, tv);
    }
    for (int o = nv + threadIdx.x; o < len; o += kSyncThreads) {
      const T gg = ld_cg(g + o);
      T t = th[o], a = s1[o], b = s2 ? s2[o] : static_cast<T>(0);
      if ((p.flags & SDP_SYNC_CHECK_FINITE) && !finite(gg)) st |= SDP_STATUS_NONFINITE;
      optim_step<T>(p, gg, t, a, b);
      s1[o] = a;
      if (s2) s2[o] = b;
      th[o] = t;
      if (tb) tb[o] = to_bf16(t);
    }
  }
}

// CS: compact owned-tile storage (slot table); LU: the SDP_SYNC_LOCAL_UPDATE
// phase.  Both are template flags so the plain flat sync keeps its lean,
// spill-free code (a runtime slot-table branch cost it 2% at C4).
template <typename T, int MB, int R, bool CS, bool LU>
__global__ void __launch_bounds__(kSyncThreads, 4)
k_owner_sync(const __grid_constant__ SyncParams p) {
  __shared__ alignas(16) sdp_tile_desc s_desc[kStage];
  __shared__ alignas(8) uint64_t s_bar;
  uint32_t st = 0;
  const uint32_t ep = p.epoch_ctr ? __ldcg(p.epoch_ctr + blockIdx.x) + 1u : p.epoch;
  if (p.world > 1 && !cross_rank_barrier(p, 2u * ep + 1u)) return;

  const int first = blockIdx.x * p.tiles_per_cta;
  const int count = min(p.tiles_per_cta, p.n_tiles - first);
  if (p.tiles_per_cta == 1) {
    // one tile per CTA: a broadcast 16-B load of the descriptor beats the
    // bulk-copy + mbarrier round trip (the CTA has nothing else to overlap)
    if (count == 1) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p.tiles + first));
      sdp_tile_desc d;
      d.owner_bits = (static_cast<uint64_t>(raw.y) << 32) | raw.x;
      d.tile_index = raw.z;
      d.len_flags = raw.w;
      run_tile<T, MB, R, CS>(p, d, st);
    }
  } else {
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int k0 = 0; k0 < count; k0 += kStage) {
      const int nk = min(kStage, count - k0);
      if (threadIdx.x == 0) {
        const uint32_t bytes = static_cast<uint32_t>(nk * sizeof(sdp_tile_desc));
        mbar_arrive_expect_tx(&s_bar, bytes);
        bulk_g2s(s_desc, p.tiles + first + k0, bytes, &s_bar);
      }
      mbar_wait(&s_bar, phase);
      phase ^= 1;
      for (int k = 0; k < nk; ++k) run_tile<T, MB, R, CS>(p, s_desc[k], st);
      __syncthreads();  // s_desc is overwritten by the next stage
    }
  }
  bool ok = true;
  if (p.world > 1) ok = cross_rank_barrier(p, 2u * ep + 2u);
  if constexpr (LU) {
    if (ok) {
      if (p.world == 1) __syncthreads();  // this CTA's own write-back is the only producer
      local_update<T>(p, st);
    }
  }
  if (st && p.status) atomicOr(p.status, st);
  if (p.epoch_ctr && threadIdx.x == 0) p.epoch_ctr[blockIdx.x] = ep;
}

// SDP_SYNC_DIRECT: the latency-bound small-buffer form.  Thread t of CTA b
// owns the VN elements at (b * 256 + t) * VN; it loads their owner masks and
// the same VN elements of ALL N replicas before the first add -- one DRAM
// round trip, where the tiled kernel chains descriptor -> mask -> owners --
// then sums exactly each element's owners in ascending order (non-owners'
// values are loaded but never used) and runs the usual epilogue.  Flat
// replicas only (every worker's buffer spans [0, d)).
template <typename T, int MB, int NW>
__global__ void __launch_bounds__(kSyncThreads)
k_owner_sync_direct(const __grid_constant__ SyncParams p) {
  constexpr int VN = V<T>::N;
  using Vt = typename V<T>::type;
  using M = typename MaskT<MB>::T;
  uint32_t st = 0;
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * kSyncThreads + threadIdx.x) * VN;
  if (j < p.total) {
    const M* mask = static_cast<const M*>(p.owner_mask);
    const int tile = p.tile;
    const uint32_t tix = static_cast<uint32_t>(j / tile);
    const int64_t s = static_cast<int64_t>(tix) * tile;
    const int o = static_cast<int>(j - s);
    if (j + VN <= p.total) {
      uint64_t m[VN];
#pragma unroll
      for (int e = 0; e < VN; ++e) m[e] = static_cast<uint64_t>(__ldg(mask + j + e));
      // every worker's vector, issued before the masks arrive (a filtered
      // form that loaded only the workers a warp's lanes own -- mask first,
      // then data -- measured slower: profiles/r2_direct_ab.jsonl)
      Vt g[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w)
        if (w < p.n_workers) g[w] = V<T>::ld(static_cast<const T*>(p.replicas[w]) + j);
      Vt mean;
      bool same = true;
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        T acc = static_cast<T>(0);
#pragma unroll
        for (int w = 0; w < NW; ++w)
          if (w < p.n_workers && ((m[e] >> w) & 1ull)) acc = add_rn(acc, g[w].x[e]);
        const int c = __popcll(m[e]);
        mean.x[e] = div_rn(acc, static_cast<T>(c > 0 ? c : 1));
        if ((p.flags & SDP_SYNC_CHECK_FINITE) && !finite(mean.x[e])) st |= SDP_STATUS_NONFINITE;
        if (c == 0 && (p.flags & SDP_SYNC_CHECK_UNCOVERED)) {
#pragma unroll
          for (int w = 0; w < NW; ++w)
            if (w < p.n_workers && !finite(g[w].x[e])) st |= SDP_STATUS_UNCOVERED_LEAK;
        }
        same &= m[e] == m[0];
      }
      if (!(p.flags & SDP_SYNC_WRITEBACK) && !epilogue_optim(p)) {
        if (p.out) V<T>::st(static_cast<T*>(p.out) + j, mean);
        if (p.out_bf16) V<T>::st_bf16(static_cast<__nv_bfloat16*>(p.out_bf16) + j, mean);
      } else if (same) {
        emit_vec<T, false>(p, tix, s, o, m[0], mean);
      } else {
#pragma unroll
        for (int e = 0; e < VN; ++e) emit_scalar<T, false>(p, tix, s, o + e, m[e], mean.x[e]);
      }
    } else {  // the vector's tail past d: element by element
      for (int e = 0; j + e < p.total; ++e) {
        const uint64_t m = static_cast<uint64_t>(__ldg(mask + j + e));
        sync_elem<T, false>(p, tix, s, o + e, m, st);
      }
    }
  }
  if (__any_sync(0xffffffffu, st != 0) && st && p.status) atomicOr(p.status, st);
}

// SDP_SYNC_STREAM: the same per-vector sum as k_owner_sync_direct, in a
// grid-stride loop of resident CTAs that reads only what the owners hold:
// a vector's replica loads are issued for the workers some lane of the warp
// owns (a warp-uniform OR of the lanes' masks; a worker's 128-B lines are
// fetched whole anyway, so no owned byte is skipped), and the NEXT vector's
// mask words are requested before this vector's data arrives -- one DRAM
// round trip per iteration with the owned-line traffic of the tiled kernel.
// MEAN: a mean-only launch (no write-back, no optimizer): the epilogue is
// compiled down to the two vector stores.
template <typename T, int MB, int NW, bool MEAN>
__global__ void __launch_bounds__(kSyncThreads, kStreamCtasPerSm)
k_owner_sync_stream(const __grid_constant__ SyncParams p) {
  constexpr int VN = V<T>::N;
  using Vt = typename V<T>::type;
  using W = typename std::conditional<VN == 4, uint32_t, uint16_t>::type;  // VN one-byte masks
  static_assert(MB == 1, "one-byte owner masks");
  uint32_t st = 0;
  const int64_t nvec = p.total / VN;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kSyncThreads;
  const W* mw = reinterpret_cast<const W*>(p.owner_mask);
  const int tile = p.tile;
  int64_t v = static_cast<int64_t>(blockIdx.x) * kSyncThreads + threadIdx.x;
  uint32_t nxt = v < nvec ? static_cast<uint32_t>(__ldg(mw + v)) : 0u;
  for (; v < nvec; v += stride) {
    const uint32_t cur = nxt;
    uint32_t any = 0;
    bool uncov = false;
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      any |= (cur >> (8 * e)) & 0xFFu;
      uncov |= ((cur >> (8 * e)) & 0xFFu) == 0u;
    }
    // the leak check (engine.py:75-78) reads every worker at zero-coverage
    // elements, as the tiled kernel does
    if ((p.flags & SDP_SYNC_CHECK_UNCOVERED) && uncov) any = 0xFFu;
    const uint32_t need = __reduce_or_sync(__activemask(), any);
    const int64_t j = v * VN;
    Vt g[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w)
      if (w < p.n_workers && ((need >> w) & 1u)) g[w] = V<T>::ld(static_cast<const T*>(p.replicas[w]) + j);
    if (v + stride < nvec) nxt = static_cast<uint32_t>(__ldg(mw + v + stride));
    Vt mean;
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      const uint32_t me = (cur >> (8 * e)) & 0xFFu;
      T acc = static_cast<T>(0);
#pragma unroll
      for (int w = 0; w < NW; ++w)
        if ((me >> w) & 1u) acc = add_rn(acc, g[w].x[e]);
      const int c = __popc(me);
      mean.x[e] = div_rn(acc, static_cast<T>(c > 0 ? c : 1));
      if ((p.flags & SDP_SYNC_CHECK_FINITE) && !finite(mean.x[e])) st |= SDP_STATUS_NONFINITE;
      if (c == 0 && (p.flags & SDP_SYNC_CHECK_UNCOVERED)) {
#pragma unroll
        for (int w = 0; w < NW; ++w)
          if (w < p.n_workers && !finite(g[w].x[e])) st |= SDP_STATUS_UNCOVERED_LEAK;
      }
    }
    const uint32_t tix = static_cast<uint32_t>(j / tile);
    const int64_t s = static_cast<int64_t>(tix) * tile;
    const int o = static_cast<int>(j - s);
    bool same = true;
#pragma unroll
    for (int e = 1; e < VN; ++e) same &= ((cur >> (8 * e)) & 0xFFu) == (cur & 0xFFu);
    // mean-only launches (the drop-in `aggregate`): the per-element means go
    // out as whole 16-B vectors whatever the owner sets, and the write-back /
    // optimizer epilogue is compiled out (C3 59 -> 43 us, the c=512 neuron
    // sweep 176 -> 133 us; profiles/r2_stream_mean_ab.jsonl)
    if (MEAN) {
      if (p.out) V<T>::st(static_cast<T*>(p.out) + j, mean);
      if (p.out_bf16) V<T>::st_bf16(static_cast<__nv_bfloat16*>(p.out_bf16) + j, mean);
    } else if (same) {
      emit_vec<T, false>(p, tix, s, o, cur & 0xFFu, mean);
    } else {
#pragma unroll
      for (int e = 0; e < VN; ++e) emit_scalar<T, false>(p, tix, s, o + e, (cur >> (8 * e)) & 0xFFu, mean.x[e]);
    }
  }
  // the last total % VN elements
  const int64_t t0 = nvec * VN;
  if (blockIdx.x == 0 && t0 + threadIdx.x < p.total) {
    const int64_t j = t0 + threadIdx.x;
    const uint32_t tix = static_cast<uint32_t>(j / tile);
    const int64_t s = static_cast<int64_t>(tix) * tile;
    const uint64_t m = static_cast<uint64_t>(__ldg(static_cast<const uint8_t*>(p.owner_mask) + j));
    sync_elem<T, false>(p, tix, s, static_cast<int>(j - s), m, st);
  }
  if (st && p.status) atomicOr(p.status, st);
}

template <typename T>
__global__ void k_nesterov(int64_t total, T* __restrict__ theta, T* __restrict__ vel,
                           const T* __restrict__ grad, double lr, double momentum,
                           __nv_bfloat16* __restrict__ theta_bf16, uint32_t* status) {
  const T mu = static_cast<T>(momentum), lrt = static_cast<T>(lr);
  uint32_t st = 0;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T g = grad[j];
    if (!finite(g)) st = SDP_STATUS_NONFINITE;
    const T v = add_rn(mul_rn(vel[j], mu), g);
    const T t = sub_rn(theta[j], mul_rn(lrt, add_rn(g, mul_rn(mu, v))));
    vel[j] = v;
    theta[j] = t;
    if (theta_bf16) theta_bf16[j] = to_bf16(t);
  }
  if (__any_sync(0xffffffffu, st != 0) && (threadIdx.x & 31) == 0 && status)
    atomicOr(status, SDP_STATUS_NONFINITE);
}

// optim.Adam.update (optim.py:101-109) on a flat vector, numpy's evaluation
// order and rounding (no FMA contraction):
//   m = b1*m + (1-b1)*g;  v = b2*v + ((1-b2)*g)*g;
//   th = th - (lr*(m/c1)) / (sqrt(v/c2) + eps),   c_k = 1 - b_k**t (host)
template <typename T>
__global__ void k_adam(int64_t total, T* __restrict__ theta, T* __restrict__ m, T* __restrict__ v,
                       const T* __restrict__ grad, double lr, double beta1, double beta2, double eps,
                       double bias1, double bias2, __nv_bfloat16* __restrict__ theta_bf16) {
  const T b1 = static_cast<T>(beta1), b2 = static_cast<T>(beta2);
  const T omb1 = static_cast<T>(1.0 - beta1), omb2 = static_cast<T>(1.0 - beta2);
  const T c1 = static_cast<T>(bias1), c2 = static_cast<T>(bias2), lrt = static_cast<T>(lr);
  const T ep = static_cast<T>(eps);
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T g = grad[j];
    const T mm = add_rn(mul_rn(b1, m[j]), mul_rn(omb1, g));
    const T vv = add_rn(mul_rn(b2, v[j]), mul_rn(mul_rn(omb2, g), g));
    const T t = sub_rn(theta[j], div_rn(mul_rn(lrt, div_rn(mm, c1)), add_rn(sqrt_rn(div_rn(vv, c2)), ep)));
    m[j] = mm;
    v[j] = vv;
    theta[j] = t;
    if (theta_bf16) theta_bf16[j] = to_bf16(t);
  }
}

template <typename T>
__global__ void k_check_finite(int64_t total, const T* __restrict__ x, uint32_t* status) {
  bool bad = false;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !finite(__ldcs(x + j));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(status, SDP_STATUS_NONFINITE);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_owner_sync(const sdp_sync_args* a, void* stream) {
  if (!a) return set_error(SDP_ERR_USAGE, "null args");
  if (a->dtype != SDP_DTYPE_F32 && a->dtype != SDP_DTYPE_F64)
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  if (a->n_workers < 1 || a->n_workers > SDP_MAX_WORKERS)
    return set_error(SDP_ERR_CONFIG, "n_workers must lie in [1, %d]", SDP_MAX_WORKERS);
  const int mb = a->mask_bytes;
  if (!(mb == 1 || mb == 2 || mb == 4 || mb == 8) || mb * 8 < a->n_workers)
    return set_error(SDP_ERR_CONFIG, "mask_bytes=%d cannot hold %d workers", mb, a->n_workers);
  if (a->tile < 1024 || a->tile % 1024 || a->tile > (1 << 20))
    return set_error(SDP_ERR_CONFIG, "sync tile must be a multiple of 1024 in [1024, 2^20]");
  if (a->n_tiles < 0 || a->tiles_per_cta < 1) return set_error(SDP_ERR_CONFIG, "bad tile plan");
  if (a->world < 1 || a->world > 8 || a->rank < 0 || a->rank >= a->world)
    return set_error(SDP_ERR_CONFIG, "rank %d / world %d invalid (world <= 8)", a->rank, a->world);
  if (a->n_tiles == 0) return SDP_OK;
  if (!a->tiles || !aligned16(a->tiles)) return set_error(SDP_ERR_USAGE, "tile table must be 16-byte aligned");
  for (int w = 0; w < a->n_workers; ++w) {
    if (!a->replicas[w]) return set_error(SDP_ERR_PROTOCOL, "replica %d is NULL", w);
    if (!aligned16(a->replicas[w]) || (a->shadow_bf16[w] && (reinterpret_cast<uintptr_t>(a->shadow_bf16[w]) & 7u)))
      return set_error(SDP_ERR_USAGE, "replica %d buffers are not 16-byte aligned", w);
  }
  if ((a->out && !aligned16(a->out)) || (a->out_bf16 && (reinterpret_cast<uintptr_t>(a->out_bf16) & 7u)))
    return set_error(SDP_ERR_USAGE, "output buffers are not 16-byte aligned");
  if ((a->flags & SDP_SYNC_NESTEROV) && (a->flags & SDP_SYNC_ADAM))
    return set_error(SDP_ERR_CONFIG, "choose one fused optimizer: Nesterov or Adam");
  const bool local_update = (a->flags & SDP_SYNC_LOCAL_UPDATE) != 0;
  if (local_update) {
    if (!(a->flags & (SDP_SYNC_NESTEROV | SDP_SYNC_ADAM)))
      return set_error(SDP_ERR_CONFIG, "SDP_SYNC_LOCAL_UPDATE needs SDP_SYNC_NESTEROV or SDP_SYNC_ADAM");
    if (a->updates_per_cta < 0 || (a->updates_per_cta > 0 && (!a->updates || !a->states)))
      return set_error(SDP_ERR_USAGE, "local update phase needs its update table and worker states");
    if (a->updates && !aligned16(a->updates)) return set_error(SDP_ERR_USAGE, "update table must be 16-byte aligned");
    if (!a->slots) return set_error(SDP_ERR_USAGE, "SDP_SYNC_LOCAL_UPDATE runs on compact storage: slots is NULL");
  } else if (a->flags & (SDP_SYNC_NESTEROV | SDP_SYNC_ADAM)) {
    if (!a->theta || !a->velocity || !aligned16(a->theta) || !aligned16(a->velocity))
      return set_error(SDP_ERR_USAGE, "fused optimizer needs 16-byte aligned theta and moment buffers");
  }
  if ((a->flags & SDP_SYNC_ADAM) && !local_update) {
    if (!a->second_moment || !aligned16(a->second_moment))
      return set_error(SDP_ERR_USAGE, "fused Adam needs a 16-byte aligned second-moment buffer");
  }
  if (a->flags & SDP_SYNC_ADAM) {
    if (a->adam_step) {
      if (!a->adam_bias_table || a->adam_table_len < 2)
        return set_error(SDP_ERR_USAGE, "a device Adam step needs its bias table (>= 2 entries)");
    } else if (!(a->bias1 > 0.0) || !(a->bias2 > 0.0)) {
      return set_error(SDP_ERR_CONFIG, "Adam bias corrections must be positive (step >= 1)");
    }
  }
  if (a->world > 1) {
    for (int r = 0; r < a->world; ++r)
      if (!a->signal_pads[r]) return set_error(SDP_ERR_USAGE, "signal pad of rank %d missing", r);
  }

  SyncParams p{};
  p.owner_mask = a->owner_mask;
  p.tiles = a->tiles;
  p.has_shadow = false;
  for (int w = 0; w < SDP_MAX_WORKERS; ++w) {
    p.replicas[w] = w < a->n_workers ? a->replicas[w] : nullptr;
    p.shadow[w] = w < a->n_workers ? a->shadow_bf16[w] : nullptr;
    p.has_shadow |= p.shadow[w] != nullptr;
  }
  p.out = a->out;
  p.out_bf16 = a->out_bf16;
  p.theta = a->theta;
  p.velocity = a->velocity;
  p.theta_bf16 = a->theta_bf16;
  p.status = a->status;
  for (int r = 0; r < 8; ++r) p.pads[r] = r < a->world ? a->signal_pads[r] : nullptr;
  p.lr = a->lr;
  p.momentum = a->momentum;
  p.second_moment = (a->flags & SDP_SYNC_ADAM) ? a->second_moment : nullptr;
  p.beta1 = a->beta1;
  p.beta2 = a->beta2;
  p.omb1 = a->one_minus_beta1;
  p.omb2 = a->one_minus_beta2;
  p.bias1 = a->bias1;
  p.bias2 = a->bias2;
  p.adam_step = (a->flags & SDP_SYNC_ADAM) ? a->adam_step : nullptr;
  p.adam_bias_table = a->adam_bias_table;
  p.adam_table_len = a->adam_table_len;
  p.eps = a->eps;
  p.total = a->total;
  p.timeout_cycles = a->timeout_cycles > 0 ? a->timeout_cycles : (int64_t)20000000000ll;
  p.n_workers = a->n_workers;
  p.tile = a->tile;
  p.n_tiles = a->n_tiles;
  p.tiles_per_cta = a->tiles_per_cta;
  p.flags = a->flags;
  p.rank = a->rank;
  p.world = a->world;
  p.epoch = a->epoch;
  p.epoch_ctr = a->world > 1 ? a->epoch_counters : nullptr;
  p.slots = a->slots;
  p.slot_stride = a->slot_stride;
  p.updates = local_update ? a->updates : nullptr;
  p.states = local_update ? a->states : nullptr;
  p.updates_per_cta = local_update ? a->updates_per_cta : 0;
  if (a->slots && a->slot_stride < (a->total + a->tile - 1) / a->tile)
    return set_error(SDP_ERR_USAGE, "slot_stride %lld is below the tile count", (long long)a->slot_stride);

  cudaStream_t s = as_stream(stream);
  if (a->flags & SDP_SYNC_DIRECT) {
    if (a->world != 1 || a->slots || local_update || a->n_workers > 8 || mb != 1 || !a->owner_mask)
      return set_error(SDP_ERR_USAGE, "SDP_SYNC_DIRECT needs world 1, flat replicas, N <= 8 (1-byte owner "
                                      "masks) and the owner mask");
    const int vn = a->dtype == SDP_DTYPE_F32 ? 4 : 2;
    const int64_t per_cta = static_cast<int64_t>(kSyncThreads) * vn;
    const unsigned dgrid = static_cast<unsigned>((a->total + per_cta - 1) / per_cta);
    if (a->flags & SDP_SYNC_STREAM) {
      const unsigned sgrid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(
          (a->total / vn + kSyncThreads - 1) / kSyncThreads, static_cast<int64_t>(sm_count()) * kStreamCtasPerSm)));
      const bool mean_only = !(a->flags & (SDP_SYNC_WRITEBACK | SDP_SYNC_NESTEROV | SDP_SYNC_ADAM));
      if (a->dtype == SDP_DTYPE_F32) {
        if (mean_only) k_owner_sync_stream<float, 1, 8, true><<<sgrid, kSyncThreads, 0, s>>>(p);
        else k_owner_sync_stream<float, 1, 8, false><<<sgrid, kSyncThreads, 0, s>>>(p);
      } else {
        if (mean_only) k_owner_sync_stream<double, 1, 8, true><<<sgrid, kSyncThreads, 0, s>>>(p);
        else k_owner_sync_stream<double, 1, 8, false><<<sgrid, kSyncThreads, 0, s>>>(p);
      }
    } else if (a->dtype == SDP_DTYPE_F32) {
      k_owner_sync_direct<float, 1, 8><<<dgrid, kSyncThreads, 0, s>>>(p);
    } else {
      k_owner_sync_direct<double, 1, 8><<<dgrid, kSyncThreads, 0, s>>>(p);
    }
    SDP_LAUNCH_CHECK();
    return SDP_OK;
  }
  const int grid = a->grid > 0 ? a->grid : (a->n_tiles + a->tiles_per_cta - 1) / a->tiles_per_cta;
  // R vectors of 16 B per thread per round: R = 4 for 4096-element fp32 tiles,
  // smaller tiles (shorter tail on small buffers) run R = 2 or 1.
  const int vn = a->dtype == SDP_DTYPE_F32 ? 4 : 2;
  const int rounds = a->tile / (vn * kSyncThreads);
  const int R = rounds % 4 == 0 ? 4 : (rounds % 2 == 0 ? 2 : 1);
  // the compact / local-update instantiations run at most R = 2 (register budget)
  const bool compact = a->slots != nullptr;
#define SDP_SYNC_LAUNCH(T, MB)                                                              \
  if (local_update) {                                                                       \
    if (R >= 2) k_owner_sync<T, MB, 2, true, true><<<grid, kSyncThreads, 0, s>>>(p);         \
    else k_owner_sync<T, MB, 1, true, true><<<grid, kSyncThreads, 0, s>>>(p);                \
  } else if (compact) {                                                                     \
    if (R >= 2) k_owner_sync<T, MB, 2, true, false><<<grid, kSyncThreads, 0, s>>>(p);        \
    else k_owner_sync<T, MB, 1, true, false><<<grid, kSyncThreads, 0, s>>>(p);               \
  } else {                                                                                  \
    switch (R) {                                                                            \
      case 4: k_owner_sync<T, MB, 4, false, false><<<grid, kSyncThreads, 0, s>>>(p); break;  \
      case 2: k_owner_sync<T, MB, 2, false, false><<<grid, kSyncThreads, 0, s>>>(p); break;  \
      default: k_owner_sync<T, MB, 1, false, false><<<grid, kSyncThreads, 0, s>>>(p); break; \
    }                                                                                       \
  }
  if (a->dtype == SDP_DTYPE_F32) {
    switch (mb) {
      case 1: SDP_SYNC_LAUNCH(float, 1); break;
      case 2: SDP_SYNC_LAUNCH(float, 2); break;
      case 4: SDP_SYNC_LAUNCH(float, 4); break;
      default: SDP_SYNC_LAUNCH(float, 8); break;
    }
  } else {
    switch (mb) {
      case 1: SDP_SYNC_LAUNCH(double, 1); break;
      case 2: SDP_SYNC_LAUNCH(double, 2); break;
      case 4: SDP_SYNC_LAUNCH(double, 4); break;
      default: SDP_SYNC_LAUNCH(double, 8); break;
    }
  }
#undef SDP_SYNC_LAUNCH
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_nesterov_update(int dtype, int64_t total, void* theta, void* velocity, const void* grad,
                        double lr, double momentum, void* theta_bf16, uint32_t* status,
                        void* stream) {
  if (total <= 0) return SDP_OK;
  if (!theta || !velocity || !grad) return set_error(SDP_ERR_USAGE, "null buffer");
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, sm_count() * 8));
  cudaStream_t s = as_stream(stream);
  if (dtype == SDP_DTYPE_F32)
    k_nesterov<float><<<grid, 256, 0, s>>>(total, static_cast<float*>(theta), static_cast<float*>(velocity),
                                           static_cast<const float*>(grad), lr, momentum,
                                           static_cast<__nv_bfloat16*>(theta_bf16), status);
  else if (dtype == SDP_DTYPE_F64)
    k_nesterov<double><<<grid, 256, 0, s>>>(total, static_cast<double*>(theta), static_cast<double*>(velocity),
                                            static_cast<const double*>(grad), lr, momentum,
                                            static_cast<__nv_bfloat16*>(theta_bf16), status);
  else
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_adam_update(int dtype, int64_t total, void* theta, void* m, void* v, const void* grad, double lr,
                    double beta1, double beta2, double eps, int step, void* theta_bf16, void* stream) {
  if (total <= 0) return SDP_OK;
  if (!theta || !m || !v || !grad) return set_error(SDP_ERR_USAGE, "null buffer");
  if (step < 1) return set_error(SDP_ERR_CONFIG, "Adam step must be >= 1 (the reference increments t first)");
  // bias corrections as the reference computes them: 1 - beta**t in double
  const double bias1 = 1.0 - std::pow(beta1, static_cast<double>(step));
  const double bias2 = 1.0 - std::pow(beta2, static_cast<double>(step));
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, sm_count() * 8));
  cudaStream_t s = as_stream(stream);
  auto* tb = static_cast<__nv_bfloat16*>(theta_bf16);
  if (dtype == SDP_DTYPE_F32)
    k_adam<float><<<grid, 256, 0, s>>>(total, static_cast<float*>(theta), static_cast<float*>(m),
                                       static_cast<float*>(v), static_cast<const float*>(grad), lr, beta1, beta2,
                                       eps, bias1, bias2, tb);
  else if (dtype == SDP_DTYPE_F64)
    k_adam<double><<<grid, 256, 0, s>>>(total, static_cast<double*>(theta), static_cast<double*>(m),
                                        static_cast<double*>(v), static_cast<const double*>(grad), lr, beta1,
                                        beta2, eps, bias1, bias2, tb);
  else
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_check_finite(int dtype, int64_t total, const void* x, uint32_t* status, void* stream) {
  if (total <= 0) return SDP_OK;
  if (!x || !status) return set_error(SDP_ERR_USAGE, "null buffer");
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, sm_count() * 8));
  cudaStream_t s = as_stream(stream);
  if (dtype == SDP_DTYPE_F32)
    k_check_finite<float><<<grid, 256, 0, s>>>(total, static_cast<const float*>(x), status);
  else if (dtype == SDP_DTYPE_F64)
    k_check_finite<double><<<grid, 256, 0, s>>>(total, static_cast<const double*>(x), status);
  else
    return set_error(SDP_ERR_CONFIG, "dtype must be SDP_DTYPE_F32 or SDP_DTYPE_F64");
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"
