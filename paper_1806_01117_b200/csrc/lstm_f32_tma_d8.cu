// TMA-pipelined fp32 step kernels, hidden size 8 (see lstm_f32_tma.cuh).
#include "lstm_f32_tma.cuh"

ACKPT_INSTANTIATE_TMA(8, ackpt::tma::kFwd, 256, 3)
ACKPT_INSTANTIATE_TMA(8, ackpt::tma::kBwd, 256, 3)
ACKPT_INSTANTIATE_TMA(8, ackpt::tma::kBwd, 256, 2)
ACKPT_INSTANTIATE_TMA(8, ackpt::tma::kFwd, 128, 4)
ACKPT_INSTANTIATE_TMA(8, ackpt::tma::kBwd, 128, 3)
