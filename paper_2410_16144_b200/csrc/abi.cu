// Misc C-ABI entry points: status strings, version, cached device attributes.
#include <atomic>

#include "common.cuh"

namespace tb {

static std::atomic<int> g_sm_count[64];

int sm_count_cached() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = g_sm_count[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
    v = 148;
  g_sm_count[dev].store(v, std::memory_order_relaxed);
  return v;
}

}  // namespace tb

extern "C" const char *tb_strerror(int status) {
  switch (status) {
    case TB_OK: return "ok";
    case TB_ERR_ARGUMENT: return "invalid argument (size, pointer or format)";
    case TB_ERR_CUDA: return "CUDA runtime error";
    case TB_ERR_UNSUPPORTED: return "shape not supported by this build";
    default: return "unknown status";
  }
}

extern "C" int tb_abi_version(void) { return 4; }

extern "C" int tb_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

extern "C" int tb_stream_synchronize(void *stream) {
  return cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) == cudaSuccess ? TB_OK
                                                                                 : TB_ERR_CUDA;
}
