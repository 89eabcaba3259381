// inst_radix_u32.cu -- explicit instantiations of the radix-pipeline (u32 keys, RadixDigitizer) launch templates
// (isort_launch.cuh): one translation unit per key type / digitizer family so the
// kernels compile in parallel.
#define ISORT_LAUNCH_DEFINITIONS
#include "isort_launch.cuh"

namespace isort {
using RDz = RadixDigitizer<uint32_t>;
ISORT_INST_PIPELINE(uint32_t, false, RDz)
ISORT_INST_PIPELINE(uint32_t, true, RDz)
}  // namespace isort
