// api.cu -- the non-kernel parts of the C ABI (include/fiber.h): errors, device check,
// segment storage views, normal decoding.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "fiber.h"
#include "fiber_internal.h"

static thread_local char g_msg[512] = "no error";

int set_error(int code, const char* msg) {
  snprintf(g_msg, sizeof(g_msg), "%s", msg);
  return code;
}

int check_device() {
  // the compute capability of each device, queried once (immutable)
  static int major_of[64];
  int dev = 0, major = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess && dev >= 0 && dev < 64 && __atomic_load_n(&major_of[dev], __ATOMIC_ACQUIRE))
    major = major_of[dev];
  else if (e == cudaSuccess) {
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e == cudaSuccess && dev >= 0 && dev < 64)
      __atomic_store_n(&major_of[dev], major, __ATOMIC_RELEASE);
  }
  if (e != cudaSuccess) {
    char buf[400];
    snprintf(buf, sizeof(buf), "CUDA: %s", cudaGetErrorString(e));
    return set_error(FIBER_ECUDA, buf);
  }
  if (major != 10) {
    char buf[200];
    snprintf(buf, sizeof(buf), "device %d is sm_%d*, this library is built for sm_100a", dev, major);
    return set_error(FIBER_EDEVICE, buf);
  }
  return FIBER_OK;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[400];
    snprintf(buf, sizeof(buf), "%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
    return set_error(FIBER_ECUDA, buf);
  }
  return FIBER_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t fiber_segments_bytes(int64_t n) {
  if (n < 0) return 0;
  return 4 * align256((size_t)n * 16) + align256((size_t)n * 4);
}

extern "C" int fiber_segments_view(void* storage, int64_t n, fiber_segments* out) {
  if (!out || n < 0 || n >= ((int64_t)1 << 32) || (n > 0 && !storage) ||
      ((uintptr_t)storage & 255u) != 0)
    return set_error(FIBER_EINVAL, "fiber_segments_view: bad arguments");
  char* b = (char*)storage;
  size_t plane = align256((size_t)n * 16);
  out->p0 = b;
  out->p1 = b + plane;
  out->p2 = b + 2 * plane;
  out->p3 = b + 3 * plane;
  out->flags = (uint32_t*)(b + 4 * plane);
  out->n = n;
  return FIBER_OK;
}

extern "C" const char* fiber_error_string(int code) {
  switch (code) {
    case FIBER_OK: return "ok";
    case FIBER_EINVAL:
    case FIBER_ECUDA:
    case FIBER_EDEVICE: return g_msg;
    default: return "unknown fiber_status";
  }
}

extern "C" void fiber_decode_normal(uint32_t n_oct, float out[3]) {
  float x = (float)(int16_t)(n_oct & 0xffffu) / 32767.0f;
  float y = (float)(int16_t)(n_oct >> 16) / 32767.0f;
  float z = 1.0f - fabsf(x) - fabsf(y);
  if (z < 0.0f) {
    float ox = (1.0f - fabsf(y)) * copysignf(1.0f, x);
    float oy = (1.0f - fabsf(x)) * copysignf(1.0f, y);
    x = ox;
    y = oy;
  }
  float l = sqrtf(x * x + y * y + z * z);
  out[0] = x / l;
  out[1] = y / l;
  out[2] = z / l;
}

extern "C" int fiber_abi_version(void) { return 101; }
