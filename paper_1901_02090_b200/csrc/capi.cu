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
