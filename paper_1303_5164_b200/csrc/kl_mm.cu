// kl_mm.cu -- MM on the 5th-generation tensor cores: placeholder until the tcgen05
// kernel lands (the runtime reports KL_EINVAL for KL_MM submissions meanwhile).
#include <cuda_runtime.h>
#include "kl_internal.h"

int kl_mm_info(KlKindInfo*) { return -2; }
int kl_mm_prepare(const void*, uint32_t, void*, uint32_t) { return -2; }
int kl_mm_launch_persistent(const void*, const KlLaunch&, uint32_t, void*) { return -2; }
int kl_mm_launch_plain(const void*, uint32_t, uint32_t, void*) { return -2; }
