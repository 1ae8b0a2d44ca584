// hcran_k256.cu -- the 256-thread instantiation of the solve kernel (one instance per CTA).
#include "hcran_kernel.cuh"

namespace hcran {
KernelFn kernel_256_256() { return hcran_solve_kernel<256, 256>; }
}  // namespace hcran
