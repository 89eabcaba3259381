// inst_radix_u64.cu -- explicit instantiations of the radix-pipeline (u64 keys, RadixDigitizer) launch templates
// (isort_launch.cuh): one translation unit per key type / digitizer family so the
// kernels compile in parallel.
#define ISORT_LAUNCH_DEFINITIONS
#include "isort_launch.cuh"

namespace isort {
using RDz = RadixDigitizer<uint64_t>;
ISORT_INST_PIPELINE(uint64_t, false, RDz)
ISORT_INST_PIPELINE(uint64_t, true, RDz)
}  // namespace isort
