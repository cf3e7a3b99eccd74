// libvpe runtime bookkeeping: kernel-launch accounting across eager launches and graph replays.
#pragma once
#include <stdint.h>

namespace vpe {
// called by every enqueue path with the number of kernels it enqueued
void count_launches(int64_t n);
}  // namespace vpe
