// aba_small_f32.cu -- the fp32 register-resident ABA kernels, n = 1..20 (aba_small.cuh).
#include "aba_small.cuh"

namespace rd {
RD_ABA_SMALL_INST(float, 1)
RD_ABA_SMALL_INST(float, 2)
RD_ABA_SMALL_INST(float, 3)
RD_ABA_SMALL_INST(float, 4)
RD_ABA_SMALL_INST(float, 5)
RD_ABA_SMALL_INST(float, 6)
RD_ABA_SMALL_INST(float, 7)
RD_ABA_SMALL_INST(float, 8)
RD_ABA_SMALL_INST(float, 9)
RD_ABA_SMALL_INST(float, 10)
RD_ABA_SMALL_INST(float, 11)
RD_ABA_SMALL_INST(float, 12)
RD_ABA_SMALL_INST(float, 13)
RD_ABA_SMALL_INST(float, 14)
RD_ABA_SMALL_INST(float, 15)
RD_ABA_SMALL_INST(float, 16)
RD_ABA_SMALL_INST(float, 17)
RD_ABA_SMALL_INST(float, 18)
RD_ABA_SMALL_INST(float, 19)
RD_ABA_SMALL_INST(float, 20)
}  // namespace rd
