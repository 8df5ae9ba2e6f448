// Error reporting and version for the libbddc C ABI (include/bddc.h).
#include <string.h>
#include <stdio.h>
#include "common.cuh"

static thread_local char g_msg[512] = "";
static thread_local int g_code = 0;

extern "C" int bddc_set_error(int code, const char* msg) {
  g_code = code;
  snprintf(g_msg, sizeof(g_msg), "%s", msg ? msg : "");
  return code;
}

extern "C" const char* bddc_last_error(void) { return g_msg; }

extern "C" int bddc_version(void) { return 1; }

extern "C" size_t bddc_geom_size(void) { return sizeof(bddc_geom); }

// Number of kernel launches issued through this library (every launch site
// is followed by LAUNCH_OK, which counts it).  Used by bench.py.
static unsigned long long g_launches = 0;
extern "C" void bddc_count_launch(void) { __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED); }
static int g_pdl = 1;
extern "C" int bddc_pdl_enabled(void) { return g_pdl; }
extern "C" void bddc_set_pdl(int on) { g_pdl = on ? 1 : 0; }
static int g_pdl_pcg = 31;   // bit mask: 1 phi, 2 gemv, 4 projection+dot, 8 CG update, 16 p update
extern "C" int bddc_pdl_pcg_enabled(void) { return g_pdl_pcg; }
extern "C" void bddc_set_pdl_pcg(int mask) { g_pdl_pcg = mask; }
extern "C" unsigned long long bddc_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

// Page-lock / release a caller-owned host array (the per-solve source upload
// becomes one async DMA).  A failed registration (already registered by another
// owner, unaligned or unsupported memory) is cleared from this runtime's sticky
// error state here, so it can never surface at an unrelated later launch.
extern "C" int bddc_host_register(void* p, size_t bytes) {
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return bddc_set_error(BDDC_ERR_CUDA, cudaGetErrorString(e));
  }
  return 0;
}

extern "C" int bddc_host_unregister(void* p) {
  cudaError_t e = cudaHostUnregister(p);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return bddc_set_error(BDDC_ERR_CUDA, cudaGetErrorString(e));
  }
  return 0;
}
