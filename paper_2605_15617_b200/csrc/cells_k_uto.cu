// cells_k_uto.cu — instantiation unit of the cell kernel (cell_kernel.cuh), variant
// SH=false (sharded), PR=false (per-rank durations), MS=false (multi-stream), tp = 1..8.
#ifndef PRISM_CELL_STATS
#include "cell_kernel.cuh"

namespace prism {

const void *cell_kernel_get_uto(int tp, int ks) {
  if (ks == 8) {  // EP CTAs: eight replica cells of tp-width R per CTA
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, false, false, false, 8>;
      case 4: return (const void *)cell_kernel<4, false, false, false, 8>;
      case 8: return (const void *)cell_kernel<8, false, false, false, 8>;
      default: return nullptr;
    }
  }
  if (ks == 16) {  // EP CTAs of sixteen narrower replica cells
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, false, false, false, 16>;
      case 4: return (const void *)cell_kernel<4, false, false, false, 16>;
      default: return nullptr;
    }
  }
  if (ks != 1) return nullptr;
  switch (tp) {
    case 1: return (const void *)cell_kernel<1, false, false, false>;
    case 2: return (const void *)cell_kernel<2, false, false, false>;
    case 3: return (const void *)cell_kernel<3, false, false, false>;
    case 4: return (const void *)cell_kernel<4, false, false, false>;
    case 5: return (const void *)cell_kernel<5, false, false, false>;
    case 6: return (const void *)cell_kernel<6, false, false, false>;
    case 7: return (const void *)cell_kernel<7, false, false, false>;
    case 8: return (const void *)cell_kernel<8, false, false, false>;
    default: return nullptr;
  }
}

const void *cell_kernel_get_sto(int tp, int ks);
const void *cell_kernel_get_upo(int tp, int ks);
const void *cell_kernel_get_spo(int tp, int ks);
const void *cell_kernel_get_utm(int tp, int ks);
const void *cell_kernel_get_stm(int tp, int ks);
const void *cell_kernel_get_upm(int tp, int ks);
const void *cell_kernel_get_spm(int tp, int ks);

const void *cell_kernel_get(int tp, bool sh, bool pr, bool ms, int ks) {
  switch ((sh ? 1 : 0) | (pr ? 2 : 0) | (ms ? 4 : 0)) {
    case 0: return cell_kernel_get_uto(tp, ks);
    case 1: return cell_kernel_get_sto(tp, ks);
    case 2: return cell_kernel_get_upo(tp, ks);
    case 3: return cell_kernel_get_spo(tp, ks);
    case 4: return cell_kernel_get_utm(tp, ks);
    case 5: return cell_kernel_get_stm(tp, ks);
    case 6: return cell_kernel_get_upm(tp, ks);
    case 7: return cell_kernel_get_spm(tp, ks);
    default: return nullptr;
  }
}

}  // namespace prism
#endif
