// hcran_k512.cu -- the 512-thread instantiation of the solve kernel (one instance per CTA).
#include "hcran_kernel.cuh"

namespace hcran {
KernelFn kernel_512_512() { return hcran_solve_kernel<512, 512>; }

void phase_cycles_512(unsigned long long* out32, int reset) {
#if defined(HCRAN_PROFILE)
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out32, g_phase_cycles, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
#else
  for (int i = 0; i < 32; ++i) out32[i] = 0;
  (void)reset;
#endif
}
}  // namespace hcran
