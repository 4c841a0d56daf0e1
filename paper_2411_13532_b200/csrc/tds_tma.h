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
    int tab_smem;      // TAB_GLOBAL: per-row table staged in shared memory
    int band;          // banded reduced map (FastArgs::Hb)
};

// lines per tile (8 or 16; 0 = not TMA-eligible) and tiles per CTA
struct TileCfg {
    int tl;
    int tpc;
};

PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
TileCfg tile_cfg(const FastArgs& a);   // A/B knob TDS_TL=8|16
size_t tma_smem(const FastArgs& a, TileCfg c);
int box_rows(int rows, int M);
int store_policy();
// 3-D tensor map (lanes, rows, groups) over the field a.u; box tl x boxr x 1
int encode_field_map(const FastArgs& a, int M, int tl, CUtensorMap* map, int* boxr);
// cudaFuncAttributeMaxDynamicSharedMemorySize of `fn` raised to >= smem on
// the CURRENT device (the attribute is per device context; cached per
// (function, device), thread-safe)
int ensure_smem(const void* fn, size_t smem, const char* what);
// persistent grid: resident CTAs x SMs of the current device, capped by
// `items` and (if > 0) by max_ctas; 0 if the kernel does not fit an SM
long long persistent_grid(const void* fn, int threads, size_t smem, long long items,
                          int max_ctas);

// 4-D view (lane, x, y-group, z) of an x-layout (nx, ny, nz) block, box tl
// lanes x 1 x 1 x boxr z-rows: the z lines read in place (tds_transport.cu)
int encode_xz_map(const double* u, int nx, int ny, int nz, int sz, int M, int tl,
                  CUtensorMap* map, int* boxr);

// long lines split over a thread-block cluster (tds_cluster.cu)
bool tmc_eligible(int M, bool uniform, const FastArgs& a);
int launch_tmc(int M, bool uniform, const FastArgs& a, cudaStream_t s);

}  // namespace tds
