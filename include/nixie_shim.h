/* nixie-b200 — the interposer shim (paper_2601_11743_b200/lib/libnixie_shim.so).
 *
 * LD_PRELOAD it into an unmodified CUDA application that links the CUDA
 * runtime dynamically, with NIXIE_SOCKET naming a running nixied's socket
 * (paper_2601_11743_b200/lib/nixied). Without NIXIE_SOCKET it is inert (every
 * call passes straight through).
 *
 * It exports the CUDA runtime/driver entry points below with their own
 * signatures (cuda_runtime_api.h / cuda.h); this header only lists them and
 * the two probes. Reference anchors: the paper's shim; the
 * registry entry points it feeds, MemState::allocate / free_chunk
 * (proj/src/mem_model.cpp:48-116); the grant it enforces,
 * MlfqScheduler::on_grant_start / on_grant_end (proj/src/mlfq.cpp:188-194).
 *
 *   allocation   cudaMalloc, cudaFree, cudaMallocAsync, cudaFreeAsync, cudaMallocPitch, cudaMalloc3D,
 *                cuMemAlloc_v2, cuMemFree_v2, cuMemAllocPitch_v2, cuMemAllocAsync, cuMemFreeAsync
 *   memory info  cudaMemGetInfo (budget as total; managed + passthrough + implicit bytes as used)
 *   implicit     cudaStreamCreate, cudaStreamCreateWithFlags, cudaStreamCreateWithPriority,
 *   allocations  cudaStreamDestroy, cudaGraphInstantiate, cudaGraphInstantiateWithFlags,
 *                cudaGraphExecDestroy, cudaDeviceSetLimit, cuStreamCreate, cuStreamCreateWithPriority,
 *                cuStreamDestroy_v2, cublasCreate_v2, cublasDestroy_v2, cublasLtCreate, cublasLtDestroy,
 *                cudnnCreate, cudnnDestroy (the device memory each call takes is charged to the app:
 *                PAPER.md:137, "APIs that implicitly allocate memory (e.g., cudaStreamCreate)")
 *   launch gate  cudaLaunchKernel, cudaLaunchKernelExC, cudaLaunchCooperativeKernel,
 *                cudaGraphLaunch, cuLaunchKernel, cuLaunchKernelEx, cuLaunchCooperativeKernel,
 *                cuGraphLaunch, cudaMemcpy, cudaMemcpyAsync, cudaMemcpy2D, cudaMemcpy2DAsync,
 *                cudaMemcpy3D, cudaMemcpy3DAsync, cudaMemcpyPeer, cudaMemcpyPeerAsync,
 *                cudaMemcpy3DPeer, cudaMemcpy3DPeerAsync, cudaMemset, cudaMemsetAsync, cudaMemset2D,
 *                cudaMemset2DAsync, cudaMemset3D, cudaMemset3DAsync
 *                (and the _ptds / _ptsz per-thread-stream variants of each runtime call;
 *                the batched-copy entry points are not wrapped: the GPU pool closed
 *                them)
 *                cuMemcpy, cuMemcpyAsync, cuMemcpyHtoD_v2, cuMemcpyDtoH_v2, cuMemcpyDtoD_v2,
 *                cuMemcpyHtoDAsync_v2, cuMemcpyDtoHAsync_v2, cuMemcpyDtoDAsync_v2, cuMemcpy2D_v2,
 *                cuMemcpy2DUnaligned_v2, cuMemcpy2DAsync_v2, cuMemcpy3D_v2, cuMemcpy3DAsync_v2,
 *                cuMemcpyPeer, cuMemcpyPeerAsync, cuMemsetD8_v2, cuMemsetD16_v2, cuMemsetD32_v2,
 *                cuMemsetD8Async, cuMemsetD16Async, cuMemsetD32Async, cuMemsetD2D8_v2,
 *                cuMemsetD2D16_v2, cuMemsetD2D32_v2 (driver entry points; the same set, plus the
 *                2D/3D/peer async copies and 2D memsets, is wrapped in the table
 *                cuGetProcAddress hands to cudart and libraries)
 *                cublasLtMatmul, cublasGemmEx, cublasGemmStridedBatchedEx, cublasSgemm_v2,
 *                cublasSgemmStridedBatched, cudnnBackendExecute (cuBLAS and cuDNN launch
 *                through their static runtimes' private driver tables)
 *   blocking     cudaDeviceSynchronize, cudaStreamSynchronize, cudaEventSynchronize
 *   capture      cudaStreamBeginCapture, cudaStreamEndCapture (launches recorded into a
 *                capture are not gated but count as activity)
 */
#ifndef NIXIE_SHIM_H
#define NIXIE_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

/* 1 when the shim is connected to a daemon (NIXIE_SOCKET set and reachable). */
int nixie_shim_active(void);
/* The daemon's id for this process (its AppId), or 0xFFFFFFFF when inactive. */
unsigned nixie_shim_app(void);

#ifdef __cplusplus
}
#endif

#endif /* NIXIE_SHIM_H */
