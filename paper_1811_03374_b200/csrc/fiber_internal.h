// fiber_internal.h -- host-side helpers shared by the C-ABI translation units of libfiber.
#pragma once
#include <cuda_runtime.h>

#include "fiber.h"

// Record `code` with a message in the calling thread's error slot and return it.
int set_error(int code, const char* msg);
// FIBER_OK if the current device is an sm_100 GPU, else FIBER_EDEVICE / FIBER_ECUDA.
int check_device();
// Turn cudaGetLastError() after a launch into FIBER_OK / FIBER_ECUDA.
int check_launch(const char* what);
// K2 + K3 on device pairs with nearest keys only (intersect.cu): mode bit 0 = the running
// t_max bound of fiber_intersect_closest, bit 1 = keys carry the segment index.
int launch_intersect_mode(const fiber_ray* rays, int64_t n_rays, const fiber_segments* segs,
                          const fiber_pair* pairs, int64_t n_pairs, int max_depth,
                          uint64_t* nearest, void* stream, int mode);
// The library's private stream-ordered scratch pool of device `dev` (intersect.cu): keeps its
// memory between calls, so per-call scratch needs no system calls after warm-up.
cudaMemPool_t scratch_pool(int dev);
