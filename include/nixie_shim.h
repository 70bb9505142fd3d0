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
 *   allocation   cudaMalloc, cudaFree, cudaMallocAsync, cudaFreeAsync, cuMemAlloc_v2, cuMemFree_v2
 *   memory info  cudaMemGetInfo
 *   launch gate  cudaLaunchKernel, cudaLaunchKernelExC, cudaLaunchCooperativeKernel,
 *                cudaGraphLaunch, cuLaunchKernel, cudaMemcpy, cudaMemcpyAsync,
 *                cudaMemcpy2D, cudaMemcpy2DAsync, cudaMemset, cudaMemsetAsync
 *                (and the _ptsz per-thread-stream variants of each runtime call)
 *                cublasLtMatmul, cublasGemmEx, cublasGemmStridedBatchedEx, cublasSgemm_v2,
 *                cublasSgemmStridedBatched, cudnnBackendExecute (cuBLAS and cuDNN launch
 *                through their static runtimes' private driver tables)
 *   blocking     cudaDeviceSynchronize, cudaStreamSynchronize, cudaEventSynchronize
 *   capture      cudaStreamBeginCapture, cudaStreamEndCapture
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
