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
