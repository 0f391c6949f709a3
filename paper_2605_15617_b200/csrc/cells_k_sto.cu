// cells_k_sto.cu — instantiation unit of the cell kernel (cell_kernel.cuh), variant
// SH=true (sharded), PR=false (per-rank durations), MS=false (multi-stream), tp = 1..8.
#ifndef PRISM_CELL_STATS
#include "cell_kernel.cuh"

namespace prism {

const void *cell_kernel_get_sto(int tp, int ks) {
  if (ks == 8) {  // EP CTAs: eight replica cells of tp-width R per CTA
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, true, false, false, 8>;
      case 4: return (const void *)cell_kernel<4, true, false, false, 8>;
      case 8: return (const void *)cell_kernel<8, true, false, false, 8>;
      default: return nullptr;
    }
  }
  if (ks == 16) {  // EP CTAs of sixteen narrower replica cells
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, true, false, false, 16>;
      case 4: return (const void *)cell_kernel<4, true, false, false, 16>;
      default: return nullptr;
    }
  }
  if (ks != 1) return nullptr;
  switch (tp) {
    case 1: return (const void *)cell_kernel<1, true, false, false>;
    case 2: return (const void *)cell_kernel<2, true, false, false>;
    case 3: return (const void *)cell_kernel<3, true, false, false>;
    case 4: return (const void *)cell_kernel<4, true, false, false>;
    case 5: return (const void *)cell_kernel<5, true, false, false>;
    case 6: return (const void *)cell_kernel<6, true, false, false>;
    case 7: return (const void *)cell_kernel<7, true, false, false>;
    case 8: return (const void *)cell_kernel<8, true, false, false>;
    default: return nullptr;
  }
}

}  // namespace prism
#endif
