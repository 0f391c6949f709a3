// cells_k_upm.cu — instantiation unit of the cell kernel (cell_kernel.cuh), variant
// SH=false (sharded), PR=true (per-rank durations), MS=true (multi-stream), tp = 1..8.
#ifndef PRISM_CELL_STATS
#include "cell_kernel.cuh"

namespace prism {

const void *cell_kernel_get_upm(int tp, int ks) {
  if (ks == 8) {  // EP CTAs: eight replica cells of tp-width R per CTA
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, false, true, true, 8>;
      case 4: return (const void *)cell_kernel<4, false, true, true, 8>;
      case 8: return (const void *)cell_kernel<8, false, true, true, 8>;
      default: return nullptr;
    }
  }
  if (ks == 16) {  // EP CTAs of sixteen narrower replica cells
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, false, true, true, 16>;
      case 4: return (const void *)cell_kernel<4, false, true, true, 16>;
      default: return nullptr;
    }
  }
  if (ks != 1) return nullptr;
  switch (tp) {
    case 1: return (const void *)cell_kernel<1, false, true, true>;
    case 2: return (const void *)cell_kernel<2, false, true, true>;
    case 3: return (const void *)cell_kernel<3, false, true, true>;
    case 4: return (const void *)cell_kernel<4, false, true, true>;
    case 5: return (const void *)cell_kernel<5, false, true, true>;
    case 6: return (const void *)cell_kernel<6, false, true, true>;
    case 7: return (const void *)cell_kernel<7, false, true, true>;
    case 8: return (const void *)cell_kernel<8, false, true, true>;
    default: return nullptr;
  }
}

}  // namespace prism
#endif
