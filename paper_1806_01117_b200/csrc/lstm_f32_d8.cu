// fp32 step kernels, hidden size 8 (see lstm_f32.cuh).
#include "lstm_f32.cuh"

ACKPT_INSTANTIATE_F32(8)
