// libsdp error state, device queries and CUDA-IPC peer mapping.
#include "sdp_common.cuh"

#include <map>
#include <mutex>
#include <string.h>

namespace sdp {

static thread_local char g_err[1024] = {0};

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n > 0 ? n : 148;
}

// imported peer pointer -> the base cudaIpcOpenMemHandle returned
static std::mutex g_ipc_mu;
static std::map<void*, void*> g_ipc_bases;

typedef int (*cuMemGetAddressRange_fn)(unsigned long long*, size_t*, unsigned long long);

static int alloc_base(const void* ptr, uint64_t* base) {
  static cuMemGetAddressRange_fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f)
      return set_error(SDP_ERR_CUDA, "cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<cuMemGetAddressRange_fn>(f);
  }
  unsigned long long b = 0;
  size_t sz = 0;
  int rc = fn(&b, &sz, reinterpret_cast<unsigned long long>(ptr));
  if (rc != 0) return set_error(SDP_ERR_CUDA, "cuMemGetAddressRange failed (%d)", rc);
  *base = b;
  return SDP_OK;
}

}  // namespace sdp

extern "C" {

int sdp_abi_version(void) { return SDP_ABI_VERSION; }

const char* sdp_last_error(void) { return sdp::g_err; }

int sdp_device_sm_count(int* out) {
  if (!out) return sdp::set_error(SDP_ERR_USAGE, "null out");
  *out = sdp::sm_count();
  return SDP_OK;
}

int sdp_host_ptr_on_device(const void* ptr, int* out) {
  if (!out) return sdp::set_error(SDP_ERR_USAGE, "null out");
  *out = 0;
  if (!ptr) return SDP_OK;
  cudaPointerAttributes at;
  const cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {  // unregistered pageable memory on older drivers
    cudaGetLastError();
    return SDP_OK;
  }
  *out = at.type == cudaMemoryTypeHost && at.devicePointer == ptr ? 1 : 0;
  return SDP_OK;
}

int sdp_ipc_export(const void* ptr, uint8_t* handle_out, uint64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return sdp::set_error(SDP_ERR_USAGE, "null argument");
  uint64_t base = 0;
  int rc = sdp::alloc_base(ptr, &base);
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  SDP_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == SDP_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uint64_t>(ptr) - base;
  return SDP_OK;
}

int sdp_ipc_import(const uint8_t* handle, uint64_t offset, void** ptr_out) {
  if (!handle || !ptr_out) return sdp::set_error(SDP_ERR_USAGE, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  SDP_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  void* p = static_cast<char*>(base) + offset;
  {
    std::lock_guard<std::mutex> g(sdp::g_ipc_mu);
    sdp::g_ipc_bases[p] = base;
  }
  *ptr_out = p;
  return SDP_OK;
}

int sdp_ipc_close(void* ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> g(sdp::g_ipc_mu);
    auto it = sdp::g_ipc_bases.find(ptr);
    if (it == sdp::g_ipc_bases.end())
      return sdp::set_error(SDP_ERR_USAGE, "pointer %p was not imported by sdp_ipc_import", ptr);
    base = it->second;
    sdp::g_ipc_bases.erase(it);
  }
  SDP_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  return SDP_OK;
}

int sdp_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (!bytes) return SDP_OK;
  if (!dst || !src) return sdp::set_error(SDP_ERR_USAGE, "null pointer");
  SDP_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, sdp::as_stream(stream)));
  return SDP_OK;
}

int sdp_enable_peer(int peer) {
  int dev = 0, count = 0;
  SDP_CUDA_CHECK(cudaGetDevice(&dev));
  SDP_CUDA_CHECK(cudaGetDeviceCount(&count));
  if (peer == dev) return SDP_OK;
  if (peer < 0 || peer >= count)
    return sdp::set_error(SDP_ERR_USAGE, "peer device %d outside [0, %d)", peer, count);
  int can = 0;
  SDP_CUDA_CHECK(cudaDeviceCanAccessPeer(&can, dev, peer));
  if (!can) return sdp::set_error(SDP_ERR_CUDA, "device %d cannot access peer %d", dev, peer);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SDP_OK;
  }
  SDP_CUDA_CHECK(e);
  return SDP_OK;
}

}  // extern "C"
