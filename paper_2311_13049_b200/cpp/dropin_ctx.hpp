// dropin_ctx.hpp — the drop-in's device context, shared by the operator entry points
// (flap_gpu.cpp) and the FFTW3 entry points (fftw_gpu.cpp): one fw_ctx (device FW_DEVICE,
// default 0) created on first use, and the lock that serialises calls on it.
#pragma once

#include <mutex>

#include "fw_capi.h"

namespace fwave {
namespace gpu_dropin {
fw_ctx context();
std::mutex& mutex();
}  // namespace gpu_dropin
}  // namespace fwave
