// Device-resident numeric setup (dsetup.cu).
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "patches.hpp"

namespace rm {

struct NumericError : std::runtime_error {   // non-positive pivot -> RM_ENUMERIC
  using std::runtime_error::runtime_error;
};

// Computes every value block of a family built with SetupInput::defer_numeric on the current
// device: block f (PatchFamily::fclass / foff / fcells) is written as its stream layout to
// vals + fdst[f].  sc_dinv / sc_c / sc_w (device, sized like the host arrays; sc_c for Cartesian,
// sc_w for trilinear families, null otherwise) receive the static-condensation cell data when
// sc_dinv is non-null.  Synchronises st.  Throws NumericError on a failed factorization (after the
// reading-G7 restarts for ICC-SC), std::runtime_error on CUDA errors.  *sigma_max = the largest
// restart shift used (0 if none).
void device_numeric_setup(const PatchFamily& P, const std::vector<long long>& fdst, double* vals, double* sc_dinv,
                          double* sc_c, double* sc_w, cudaStream_t st, double* sigma_max);

}  // namespace rm
