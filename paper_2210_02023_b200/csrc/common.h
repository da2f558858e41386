// common.h — shared plumbing of the shardplan_b200 C-ABI library: status
// codes (error.hpp:11-49 mapped to ErrorKind+1), thread-local error text,
// CUDA/NCCL checks, and the kernel-launch counter sp_kernel_launches().
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "shardplan_b200.h"

namespace sp {

// Mirrors shardplan::Error (error.hpp:24-45): a kind plus a message. The
// C-ABI boundary converts it to the int status ErrorKind+1.
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) {
  throw Status(code, msg);
}

void set_last_error(const std::string& msg);
void count_launch(uint64_t n = 1);

// Runs f at the C-ABI boundary: 0 on success, ErrorKind+1 on failure.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return SP_OK;
  } catch (const Status& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return SP_ERR_BAD_INPUT;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SP_ERR_BAD_INPUT;
  }
}

inline void cuda_check(cudaError_t e, const char* what, const char* file,
                       int line) {
  if (e != cudaSuccess)
    raise(SP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) +
                           " (" + file + ":" + std::to_string(line) + ")");
}

}  // namespace sp

#define SP_CUDA(x) ::sp::cuda_check((x), #x, __FILE__, __LINE__)
// After every <<<>>> launch: counts it and surfaces launch errors.
#define SP_LAUNCHED()                                              \
  do {                                                             \
    ::sp::count_launch();                                          \
    ::sp::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, \
                     __LINE__);                                    \
  } while (0)

namespace sp {
// Programmatic dependent launch (sm_90+): a kernel launched this way may be
// scheduled while its stream predecessor's last blocks still run; it must
// call pdl_wait() before touching anything the predecessor writes (a no-op
// when launched normally). cfg3 D=1 iteration 3.817 -> 3.803 ms with the
// sort's P2-P4 and the SGD carry pass launched this way.
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...), "pdl launch",
             __FILE__, __LINE__);
  count_launch();
}
}  // namespace sp
