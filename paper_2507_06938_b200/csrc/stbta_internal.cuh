// Internal (C++) interfaces shared by the stbta translation units.
#pragma once

#include <cuda_runtime.h>

#include "gemm.cuh"

namespace stbta {

}  // namespace stbta
