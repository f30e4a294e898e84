// PCIe read-path probe: how fast can SMs pull pinned host memory?
//   (a) 16-B vector loads (what k_owner_sync's zero-copy path does)
//   (b) cp.async.bulk (TMA engine) 8 KB chunks into shared memory
//   (c) cudaMemcpyAsync H2D (copy engine) for reference
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_read_probe tools/pcie_read_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k_vec(const float4* __restrict__ src, size_t n4, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(src + i));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) *out = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CHUNK>
__global__ void k_bulk(const char* __restrict__ src, size_t bytes, float* out) {
  extern __shared__ __align__(128) char buf[];  // 2 x CHUNK
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t nchunks = bytes / CHUNK;
  uint32_t phase[2] = {0, 0};
  float acc = 0.f;
  size_t c = blockIdx.x;
  int slot = 0;
  // prologue: issue the first chunk
  if (threadIdx.x == 0 && c < nchunks) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[0])), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(buf)), "l"(src + c * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[0])) : "memory");
  }
  for (; c < nchunks; c += gridDim.x) {
    const size_t nc = c + gridDim.x;
    if (threadIdx.x == 0 && nc < nchunks) {  // prefetch the next chunk into the other slot
      const int o = slot ^ 1;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[o])), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(buf + o * CHUNK)), "l"(src + nc * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[o])) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 :: "r"(smem_u32(&bar[slot])), "r"(phase[slot]) : "memory");
    phase[slot] ^= 1;
    const float4* v = reinterpret_cast<const float4*>(buf + slot * CHUNK);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) {
      const float4 f = v[i];
      acc += f.x + f.y + f.z + f.w;
    }
    __syncthreads();
    slot ^= 1;
  }
  if (acc == 12345.f) *out = acc;
}

int main() {
  const size_t bytes = 256ull << 20;
  char* h;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  for (size_t i = 0; i < bytes; i += 4096) h[i] = 1;
  char* d;
  cudaMalloc(&d, bytes);
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto report = [&](const char* what, float t) { printf("%-48s %8.3f ms  %6.1f GB/s\n", what, t, bytes / t / 1e6); };
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("copy engine H2D", ms);
    for (int per : {4, 8, 16}) {
      cudaEventRecord(e0);
      k_vec<<<sms * per, 256>>>(reinterpret_cast<const float4*>(h), bytes / 16, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      char name[64];
      snprintf(name, sizeof name, "SM 16-B loads, %d CTAs/SM", per);
      if (rep) report(name, ms);
    }
    cudaFuncSetAttribute(k_bulk<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16384);
    for (int per : {1, 2, 4}) {
      cudaEventRecord(e0);
      k_bulk<8192><<<sms * per, 256, 2 * 8192>>>(h, bytes, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      char name[64];
      snprintf(name, sizeof name, "TMA bulk 8 KB double-buffered, %d CTAs/SM", per);
      if (rep) report(name, ms);
      cudaEventRecord(e0);
      k_bulk<16384><<<sms * per, 256, 2 * 16384>>>(h, bytes, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      snprintf(name, sizeof name, "TMA bulk 16 KB double-buffered, %d CTAs/SM", per);
      if (rep) report(name, ms);
    }
  }
  // (d) concurrent: SM 16-B loads over the first f of the buffer while the copy
  //     engine moves the rest (a hybrid zero-copy + staged sync would do this)
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t j;
  cudaEventCreate(&j);
  for (int rep = 0; rep < 2; ++rep) {
    for (double f : {0.3, 0.4, 0.5, 0.6, 0.7}) {
      const size_t a = ((size_t)(bytes * f) / 4096) * 4096;
      cudaEventRecord(e0, s1);
      cudaStreamWaitEvent(s2, e0, 0);
      k_vec<<<sms * 8, 256, 0, s1>>>(reinterpret_cast<const float4*>(h), a / 16, out);
      cudaMemcpyAsync(d + a, h + a, bytes - a, cudaMemcpyHostToDevice, s2);
      cudaEventRecord(j, s2);
      cudaStreamWaitEvent(s1, j, 0);
      cudaEventRecord(e1, s1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      char name[64];
      snprintf(name, sizeof name, "SM loads %.0f%% || copy engine %.0f%%", 100 * f, 100 * (1 - f));
      if (rep) report(name, ms);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
