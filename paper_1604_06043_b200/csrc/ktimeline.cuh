// ktimeline.cuh — optional in-kernel timeline probes (developer build: make timeline, which
// defines MSTAB_TIMELINE). Each probe folds %globaltimer (ns) or clock64 into a slot of a
// device buffer bound with mstab_timeline_bind(); the product build compiles them to nothing.
// Used to split a launch into ramp / stream / reduction / dense-step phases.
#pragma once
#include <cuda_runtime.h>

namespace mstab_b200 {
#ifdef MSTAB_TIMELINE
namespace {
__device__ unsigned long long* g_tl = nullptr;
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
}  // namespace
#define TL_MIN(i) \
  do { if (::mstab_b200::g_tl) atomicMin(::mstab_b200::g_tl + (i), ::mstab_b200::tl_now()); } while (0)
#define TL_MAX(i) \
  do { if (::mstab_b200::g_tl) atomicMax(::mstab_b200::g_tl + (i), ::mstab_b200::tl_now()); } while (0)
#define TL_SET(i) \
  do { if (::mstab_b200::g_tl) ::mstab_b200::g_tl[i] = ::mstab_b200::tl_now(); } while (0)
#define TL_CLK(i) \
  do { if (::mstab_b200::g_tl) ::mstab_b200::g_tl[i] = (unsigned long long)clock64(); } while (0)
#define TL_BIND_FN(name) \
  void name(unsigned long long* p) { cudaMemcpyToSymbol(g_tl, &p, sizeof(p)); }
#else
#define TL_MIN(i) do {} while (0)
#define TL_MAX(i) do {} while (0)
#define TL_SET(i) do {} while (0)
#define TL_CLK(i) do {} while (0)
#define TL_BIND_FN(name) \
  void name(unsigned long long*) {}
#endif
}  // namespace mstab_b200
