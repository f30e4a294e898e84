// Shared helpers for libsdp: error state, launch checks, PTX wrappers.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include <algorithm>

#include "../../include/sdp.h"

namespace sdp {

// Per-thread last-error message (sdp_last_error).
int set_error(int code, const char* fmt, ...);

#define SDP_CUDA_CHECK(expr)                                                      \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      cudaGetLastError(); /* consume it: a later launch check must not see it */  \
      return ::sdp::set_error(SDP_ERR_CUDA, "%s failed: %s", #expr,               \
                              cudaGetErrorString(e_));                            \
    }                                                                             \
  } while (0)

#define SDP_LAUNCH_CHECK()                                                        \
  do {                                                                            \
    cudaError_t e_ = cudaGetLastError();                                          \
    if (e_ != cudaSuccess)                                                        \
      return ::sdp::set_error(SDP_ERR_CUDA, "kernel launch failed at %s:%d: %s",  \
                              __FILE__, __LINE__, cudaGetErrorString(e_));        \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// ---- per-element owner mask load (1/2/4/8-byte element types) -------------
template <int B> struct MaskT;
template <> struct MaskT<1> { using T = uint8_t; };
template <> struct MaskT<2> { using T = uint16_t; };
template <> struct MaskT<4> { using T = uint32_t; };
template <> struct MaskT<8> { using T = uint64_t; };

// ---- streaming loads / stores ---------------------------------------------
// Replica reads are touched exactly once per launch: keep them out of L1.
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
// Coherent (L2) loads of data another CTA / GPU wrote during this launch.
__device__ __forceinline__ float ld_cg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
// Peer (NVLink) replicas may be written by the peer between launches, so the
// non-coherent path is only valid within one launch -- which is all we need:
// every launch is bracketed by the cross-GPU barrier.

__device__ __forceinline__ void st_f4(float4* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void st_d2(double2* p, double2 v) {
  asm volatile("st.global.v2.f64 [%0], {%1,%2};"
               :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// ---- mbarrier + bulk copy (TMA engine, non-tensor form) --------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_addr(dst_smem)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" :: "r"(smem_addr(bar)), "r"(phase) : "memory");
}

// ---- system-scope flags for the cross-GPU barrier --------------------------
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace sdp
