// mu_fused.h -- the 1-pass fused short-wide MU kernel (mu_fused.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ntt {

struct FusedCtx {
  int dummy = 0;
};

bool fused_supported(int64_t m, int64_t n, int r);
int fused_grid(int64_t m, int64_t n, int r, int num_sms);
size_t fused_scratch_bytes(int64_t m, int64_t n, int r, int grid);
void fused_destroy(FusedCtx& c);

}  // namespace ntt
