// multi-material (binned / divergent) kernels — see nmq_abi.cu
#include "nmq_internal.h"
