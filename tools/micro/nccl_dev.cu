// NCCL 2.28 device API smoke test (the in-graph min-loc exchange's building
// blocks): a communicator, a symmetric window, a device communicator with one
// LSA barrier, and a kernel that stores a record into every peer's window slot,
// syncs the LSA barrier and reads all slots back -- captured in a CUDA graph.
// Runs with 1 rank (one GPU) or under torchrun-style env (RANK/WORLD_SIZE and
// a shared id file) with one process per GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I$NCCL/include nccl_dev.cu -L$NCCL/lib -l:libnccl.so.2 -o nccl_dev
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
#define NK(x) do { ncclResult_t e = (x); if (e != ncclSuccess) { std::printf("%s: %s\n", #x, ncclGetErrorString(e)); return 1; } } while (0)

__global__ void exch(ncclDevComm dc, ncclWindow_t win, int rounds, double* out) {
  const int rank = dc.rank, world = dc.nRanks;
  for (int it = 0; it < rounds; ++it) {
    const size_t slot = size_t((it & 1) * world + rank) * sizeof(double);
    if (threadIdx.x < world) {
      double* p = static_cast<double*>(ncclGetLsaPointer(win, slot, threadIdx.x));
      *p = 100.0 * it + rank;
    }
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamLsa(dc), dc.lsaBarrier, 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    if (threadIdx.x == 0) {
      double s = 0;
      for (int q = 0; q < world; ++q)
        s += *static_cast<double*>(ncclGetLocalPointer(win, size_t((it & 1) * world + q) * sizeof(double)));
      out[it] = s;
    }
    __syncthreads();
  }
}

int main() {
  const int rank = std::getenv("RANK") ? std::atoi(std::getenv("RANK")) : 0;
  const int world = std::getenv("WORLD_SIZE") ? std::atoi(std::getenv("WORLD_SIZE")) : 1;
  CK(cudaSetDevice(rank));
  ncclUniqueId id;
  if (world == 1) {
    NK(ncclGetUniqueId(&id));
  } else {  // rank 0 writes the id to a file the others read
    const char* f = std::getenv("NCCL_ID_FILE");
    if (rank == 0) {
      NK(ncclGetUniqueId(&id));
      FILE* fp = std::fopen(f, "wb");
      std::fwrite(&id, sizeof id, 1, fp);
      std::fclose(fp);
    } else {
      FILE* fp = nullptr;
      while (!(fp = std::fopen(f, "rb"))) {}
      while (std::fread(&id, sizeof id, 1, fp) != 1) std::rewind(fp);
      std::fclose(fp);
    }
  }
  ncclComm_t comm;
  NK(ncclCommInitRank(&comm, world, id, rank));
  void* buf = nullptr;
  const size_t bytes = 4096;
  NK(ncclMemAlloc(&buf, bytes));
  ncclWindow_t win;
  NK(ncclCommWindowRegister(comm, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC));
  ncclDevCommRequirements req{};  // zero: no resources, teams or GIN
  req.lsaBarrierCount = 1;
  ncclDevComm dc;
  NK(ncclDevCommCreate(comm, &req, &dc));
  double* out;
  CK(cudaMalloc(&out, 64 * sizeof(double)));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  // plain launch, then the same kernel captured in a graph
  exch<<<1, 128, 0, st>>>(dc, win, 8, out);
  CK(cudaStreamSynchronize(st));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  exch<<<1, 128, 0, st>>>(dc, win, 8, out);
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  double h[8];
  CK(cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int it = 0; it < 8; ++it) {
    double want = 0;
    for (int q = 0; q < world; ++q) want += 100.0 * it + q;
    bad += h[it] != want;
  }
  std::printf("rank %d/%d: device-API exchange %s (round 7 sum %.0f)\n", rank, world, bad ? "FAILED" : "ok", h[7]);
  NK(ncclDevCommDestroy(comm, &dc));
  NK(ncclCommWindowDeregister(comm, win));
  NK(ncclMemFree(buf));
  NK(ncclCommDestroy(comm));
  return bad ? 1 : 0;
}
