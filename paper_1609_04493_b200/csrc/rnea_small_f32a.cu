// rnea_small_f32a.cu -- the fp32 register kernels, n = 1..16 (rnea_small.cuh), one TU per range so the build runs them in parallel.
#include "rnea_small.cuh"

namespace rd {
RD_SMALL_INST(float, 1)
RD_SMALL_INST(float, 2)
RD_SMALL_INST(float, 3)
RD_SMALL_INST(float, 4)
RD_SMALL_INST(float, 5)
RD_SMALL_INST(float, 6)
RD_SMALL_INST(float, 7)
RD_SMALL_INST(float, 8)
RD_SMALL_INST(float, 9)
RD_SMALL_INST(float, 10)
RD_SMALL_INST(float, 11)
RD_SMALL_INST(float, 12)
RD_SMALL_INST(float, 13)
RD_SMALL_INST(float, 14)
RD_SMALL_INST(float, 15)
RD_SMALL_INST(float, 16)
}  // namespace rd
