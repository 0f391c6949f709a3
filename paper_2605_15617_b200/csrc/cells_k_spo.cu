// cells_k_spo.cu — instantiation unit of the cell kernel (cell_kernel.cuh), variant
// SH=true (sharded), PR=true (per-rank durations), MS=false (multi-stream), tp = 1..8.
#ifndef PRISM_CELL_STATS
#include "cell_kernel.cuh"

namespace prism {

const void *cell_kernel_get_spo(int tp, int ks) {
  if (ks == 8) {  // EP CTAs: eight replica cells of tp-width R per CTA
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, true, true, false, 8>;
      case 4: return (const void *)cell_kernel<4, true, true, false, 8>;
      case 8: return (const void *)cell_kernel<8, true, true, false, 8>;
      default: return nullptr;
    }
  }
  if (ks == 16) {  // EP CTAs of sixteen narrower replica cells
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, true, true, false, 16>;
      case 4: return (const void *)cell_kernel<4, true, true, false, 16>;
      default: return nullptr;
    }
  }
  if (ks != 1) return nullptr;
  switch (tp) {
    case 1: return (const void *)cell_kernel<1, true, true, false>;
    case 2: return (const void *)cell_kernel<2, true, true, false>;
    case 3: return (const void *)cell_kernel<3, true, true, false>;
    case 4: return (const void *)cell_kernel<4, true, true, false>;
    case 5: return (const void *)cell_kernel<5, true, true, false>;
    case 6: return (const void *)cell_kernel<6, true, true, false>;
    case 7: return (const void *)cell_kernel<7, true, true, false>;
    case 8: return (const void *)cell_kernel<8, true, true, false>;
    default: return nullptr;
  }
}

}  // namespace prism
#endif
