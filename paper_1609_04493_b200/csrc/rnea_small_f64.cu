// rnea_small_f64.cu -- the fp64 register kernels, n = 1..16 (rnea_small.cuh), one TU per range so the build runs them in parallel.
#include "rnea_small.cuh"

namespace rd {
RD_SMALL_INST(double, 1)
RD_SMALL_INST(double, 2)
RD_SMALL_INST(double, 3)
RD_SMALL_INST(double, 4)
RD_SMALL_INST(double, 5)
RD_SMALL_INST(double, 6)
RD_SMALL_INST(double, 7)
RD_SMALL_INST(double, 8)
RD_SMALL_INST(double, 9)
RD_SMALL_INST(double, 10)
RD_SMALL_INST(double, 11)
RD_SMALL_INST(double, 12)
RD_SMALL_INST(double, 13)
RD_SMALL_INST(double, 14)
RD_SMALL_INST(double, 15)
RD_SMALL_INST(double, 16)
}  // namespace rd
