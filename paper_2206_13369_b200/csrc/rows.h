// Warp-per-row streaming fine kernels (rows.cu).
#pragma once
#include "cpcp.h"
#include "pcp.h"

namespace mlr {
// True when every coarse support fits the two-chunk ring buffer.
bool rows_warp_ok(const ChainDev& ch, bool f32);
// mode: 0 start, 1 update, 2 output (see pcp.cu RowMode)
int pcp_rows(PcpPlan* p, int mode, const void* D, int64_t ldd, const void* Yin, void* Yout, int64_t ldy, void* Lout,
             void* Sout, int64_t ldo, cudaStream_t st);
// mode: 0 init, 1 update, 2 output (see cpcp.cu CpMode)
int cp_rows(CpcpPlan* p, int mode, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S,
            int64_t lds, void* Lout, int64_t ldl, cudaStream_t st);
int cp_dots_rows(CpcpPlan* p, cudaStream_t st);
}  // namespace mlr
