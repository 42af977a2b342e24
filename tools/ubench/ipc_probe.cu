// Probe: two processes on ONE GPU exchange data through CUDA IPC mappings, synchronised only by
// stream memory operations (cuStreamWriteValue32 on the peer's flag, cuStreamWaitValue32 on the
// local flag) -- the transport the peer-memory USP path uses.  Prints errors and the round-trip time.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <sys/wait.h>
#include <unistd.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("rank %d: %s -> %s\n", rank, #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void fill(int* p, int n, int v) { for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v; }
__global__ void check(const int* p, int n, int v, int* err) { for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) if (p[i] != v) atomicAdd(err, 1); }

int main() {
  int p01[2], p10[2];
  if (pipe(p01) || pipe(p10)) return 1;
  int rank = 0;
  pid_t kid = fork();
  if (kid == 0) rank = 1;
  const int wfd = rank == 0 ? p01[1] : p10[1], rfd = rank == 0 ? p10[0] : p01[0];
  CK(cudaSetDevice(0));
  PFN_cuStreamWaitValue32_v11070 waitv; PFN_cuStreamWriteValue32_v11070 writev;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&waitv, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&writev, cudaEnableDefault, &q));
  int attr = -1; cuDeviceGetAttribute(&attr, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, 0);
  printf("rank %d: can_flush_remote_writes=%d\n", rank, attr);
  const int n = 1 << 20;
  int *buf, *flag, *err;
  CK(cudaMalloc(&buf, n * 4)); CK(cudaMalloc(&flag, 256)); CK(cudaMalloc(&err, 4));
  CK(cudaMemset(buf, 0, n * 4)); CK(cudaMemset(flag, 0, 256)); CK(cudaMemset(err, 0, 4));
  CK(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h[2], ph[2];
  CK(cudaIpcGetMemHandle(&h[0], buf)); CK(cudaIpcGetMemHandle(&h[1], flag));
  if (write(wfd, h, sizeof h) != sizeof h) return 2;
  if (read(rfd, ph, sizeof ph) != sizeof ph) return 3;
  int *pbuf, *pflag;
  CK(cudaIpcOpenMemHandle((void**)&pbuf, ph[0], cudaIpcMemLazyEnablePeerAccess));
  CK(cudaIpcOpenMemHandle((void**)&pflag, ph[1], cudaIpcMemLazyEnablePeerAccess));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 200;
  cudaEventRecord(e0, st);
  for (int it = 1; it <= iters; ++it) {
    fill<<<64, 256, 0, st>>>(pbuf, n, it * 2 + rank);  // into the peer's buffer
    if (writev(st, (CUdeviceptr)pflag, it, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) { printf("writev fail\n"); return 4; }
    if (waitv(st, (CUdeviceptr)flag, it, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) { printf("waitv fail\n"); return 5; }
    check<<<64, 256, 0, st>>>(buf, n, it * 2 + (1 - rank), err);
    // the peer may overwrite my buf only after I checked it: second flag (ack)
    if (writev(st, (CUdeviceptr)(pflag + 1), it, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) return 6;
    if (waitv(st, (CUdeviceptr)(flag + 1), it, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) return 7;
  }
  cudaEventRecord(e1, st);
  CK(cudaStreamSynchronize(st));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int herr; cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
  printf("rank %d: %d iterations, %d mismatches, %.3f ms per iteration\n", rank, iters, herr, ms / iters);
  cudaIpcCloseMemHandle(pbuf); cudaIpcCloseMemHandle(pflag);
  if (kid) { int s; waitpid(kid, &s, 0); printf("child exit %d\n", WEXITSTATUS(s)); }
  return herr ? 9 : 0;
}
