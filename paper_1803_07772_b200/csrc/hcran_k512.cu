// hcran_k512.cu -- the 512-thread instantiation of the solve kernel (one instance per CTA).
#include "hcran_kernel.cuh"

namespace hcran {
KernelFn kernel_512_512() { return hcran_solve_kernel<512, 512>; }
}  // namespace hcran
