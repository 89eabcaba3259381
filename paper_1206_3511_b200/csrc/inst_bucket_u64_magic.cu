// inst_bucket_u64_magic.cu -- explicit instantiations of the bucket-sort (u64 keys, kMagicNarrow bucket index) launch templates
// (isort_launch.cuh): one translation unit per key type / digitizer family so the
// kernels compile in parallel.
#define ISORT_LAUNCH_DEFINITIONS
#include "isort_launch.cuh"

namespace isort {
using BDz = BucketDigitizer<uint64_t, kMagicNarrow>;
ISORT_INST_PIPELINE(uint64_t, false, BDz)
ISORT_INST_PIPELINE(uint64_t, true, BDz)
ISORT_INST_SEGMENTS(uint64_t, BDz, false)
ISORT_INST_SEGMENTS(uint64_t, BDz, true)
}  // namespace isort
