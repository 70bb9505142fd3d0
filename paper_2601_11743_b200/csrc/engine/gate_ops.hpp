// Driver-API stream memory operations used by the launch gate, resolved at
// run time through cudaGetDriverEntryPoint (no link-time libcuda dependency).
#pragma once

#include <cuda.h>

#include <cstdint>

namespace nixie::b200 {
bool gate_mem_ops_available();
CUresult gate_write(CUstream s, CUdeviceptr addr, std::uint64_t v);
CUresult gate_wait_geq(CUstream s, CUdeviceptr addr, std::uint64_t v);
}  // namespace nixie::b200
