// rnea_small_f32b.cu -- the fp32 register kernels, n = 17..32 (rnea_small.cuh), one TU per range so the build runs them in parallel.
#include "rnea_small.cuh"

namespace rd {
RD_SMALL_INST(float, 17)
RD_SMALL_INST(float, 18)
RD_SMALL_INST(float, 19)
RD_SMALL_INST(float, 20)
RD_SMALL_INST(float, 21)
RD_SMALL_INST(float, 22)
RD_SMALL_INST(float, 23)
RD_SMALL_INST(float, 24)
RD_SMALL_INST(float, 25)
RD_SMALL_INST(float, 26)
RD_SMALL_INST(float, 27)
RD_SMALL_INST(float, 28)
RD_SMALL_INST(float, 29)
RD_SMALL_INST(float, 30)
RD_SMALL_INST(float, 31)
RD_SMALL_INST(float, 32)
}  // namespace rd
