// inst_partition_u32.cu -- explicit instantiations of the key-range partition (u32 keys, DestDigitizer) launch templates
// (isort_launch.cuh): one translation unit per key type / digitizer family so the
// kernels compile in parallel.
#define ISORT_LAUNCH_DEFINITIONS
#include "isort_launch.cuh"

namespace isort {
using DDz = DestDigitizer<uint32_t>;
using C1 = PassCfg<uint32_t, false, 1>;
using C2 = PassCfg<uint32_t, false, ISORT_PASS_CHUNKS>;
using C1V = PassCfg<uint32_t, true, 1>;
using C2V = PassCfg<uint32_t, true, ISORT_PASS_CHUNKS>;
ISORT_INST_PIPELINE(uint32_t, false, DDz)
ISORT_INST_PIPELINE(uint32_t, true, DDz)
ISORT_INST_HISTOGRAM(uint32_t, DDz)
ISORT_INST_PASSES(uint32_t, false, DDz, C1, true)
ISORT_INST_PASSES(uint32_t, false, DDz, C2, true)
ISORT_INST_PASSES(uint32_t, true, DDz, C1V, true)
ISORT_INST_PASSES(uint32_t, true, DDz, C2V, true)
}  // namespace isort
