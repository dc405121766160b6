// Internal declarations shared by the libgjinv translation units (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gjinv.h"

namespace gj {

struct BatchedArgs {
  int n;
  int64_t batch;
  const void* A;
  void* Ainv;          // may be null (determinant-only)
  int32_t* ipiv;       // may be null
  double* logabsdet;   // may be null
  int8_t* sign;        // may be null
  void* det;           // may be null
  int32_t* info;       // may be null
  double tol;          // >= 0 (default already resolved)
};

// K1/K2 launchers (gj_batched.cu). Return cudaSuccess or the launch error.
cudaError_t launch_batched(gj_dtype dt, const BatchedArgs& a, cudaStream_t s);

// Number of SMs of the current device (cached per device).
int device_sm_count();

}  // namespace gj
