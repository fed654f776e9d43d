// fp32 step kernels, hidden size 4 (see lstm_f32.cuh).
#include "lstm_f32.cuh"

ACKPT_INSTANTIATE_F32(4)
