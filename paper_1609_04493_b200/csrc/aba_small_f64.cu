// aba_small_f64.cu -- the fp64 register-resident ABA kernels, n = 1..16 (aba_small.cuh).
#include "aba_small.cuh"

namespace rd {
RD_ABA_SMALL_INST(double, 1)
RD_ABA_SMALL_INST(double, 2)
RD_ABA_SMALL_INST(double, 3)
RD_ABA_SMALL_INST(double, 4)
RD_ABA_SMALL_INST(double, 5)
RD_ABA_SMALL_INST(double, 6)
RD_ABA_SMALL_INST(double, 7)
RD_ABA_SMALL_INST(double, 8)
RD_ABA_SMALL_INST(double, 9)
RD_ABA_SMALL_INST(double, 10)
RD_ABA_SMALL_INST(double, 11)
RD_ABA_SMALL_INST(double, 12)
RD_ABA_SMALL_INST(double, 13)
RD_ABA_SMALL_INST(double, 14)
RD_ABA_SMALL_INST(double, 15)
RD_ABA_SMALL_INST(double, 16)
}  // namespace rd
