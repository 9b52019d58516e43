// Per-CTA timeline stamps for latency studies (%globaltimer, ns). Compiled in
// only with -DAVEC_TRACE (a separate, non-product build, tools/trace_op.sh);
// the stamps of the launch that ran with g_trace_on set are read back with
// avec_trace_dump.
#pragma once
#include <cstdint>

#ifdef AVEC_TRACE
#include <cuda_runtime.h>
namespace avec {
namespace {  // one buffer per translation unit (no relocatable device code)
__device__ unsigned long long g_trace[148 * 2 * 16];
__device__ int g_trace_on = 0;
}  // namespace
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// host side (conv_pm.cu, conv_tc.cu): arm the next launches / read the stamps back
void conv_pm_trace(int on, cudaStream_t st);
int conv_pm_trace_dump(unsigned long long* host, int n);
void conv_tc_trace(int on, cudaStream_t st);
int conv_tc_trace_dump(unsigned long long* host, int n);
}  // namespace avec
#define AVEC_STAMP(slot)                                                                  \
  do {                                                                                    \
    if (avec::g_trace_on && blockIdx.x < 296) avec::g_trace[blockIdx.x * 16 + (slot)] = avec::gtimer(); \
  } while (0)
#else
#define AVEC_STAMP(slot) \
  do {                   \
  } while (0)
#endif
