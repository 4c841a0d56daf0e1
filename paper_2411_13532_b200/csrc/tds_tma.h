// Host-side helpers shared by the TMA-staged kernels (k_tma, k_dd).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "tds_internal.h"

namespace tds {

struct TmaArgs {
    FastArgs f;
    CUtensorMap map;
    int boxr;          // rows per TMA box (divides rows)
    int store_cs;      // streaming stores (A/B knob TDS_STCS)
};

PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
size_t tma_smem(const FastArgs& a);
int box_rows(int rows, int M);
int store_policy();
// 3-D tensor map (lanes, rows, groups) over the field a.u; box 16 x boxr x 1
int encode_field_map(const FastArgs& a, int M, CUtensorMap* map, int* boxr);

}  // namespace tds
