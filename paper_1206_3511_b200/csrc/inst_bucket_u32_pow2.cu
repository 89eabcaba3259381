// inst_bucket_u32_pow2.cu -- explicit instantiations of the bucket-sort (u32 keys, kPow2Narrow bucket index) launch templates
// (isort_launch.cuh): one translation unit per key type / digitizer family so the
// kernels compile in parallel.
#define ISORT_LAUNCH_DEFINITIONS
#include "isort_launch.cuh"

namespace isort {
using BDz = BucketDigitizer<uint32_t, kPow2Narrow>;
ISORT_INST_PIPELINE(uint32_t, false, BDz)
ISORT_INST_PIPELINE(uint32_t, true, BDz)
ISORT_INST_SEGMENTS(uint32_t, BDz, false)
ISORT_INST_SEGMENTS(uint32_t, BDz, true)
}  // namespace isort
