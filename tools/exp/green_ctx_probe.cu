// Experiment: can runtime-API launches target a green-context stream (SM
// partition) while the primary context stays current, with cudaMalloc memory?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

__global__ void smid_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
  long long t0 = clock64();
  while (clock64() - t0 < 200000) {}
}

template <typename F>
F get(const char* n) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(n, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    printf("no entry %s\n", n);
    return nullptr;
  }
  return reinterpret_cast<F>(p);
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  auto getRes = get<PFN_cuDeviceGetDevResource_v12040>("cuDeviceGetDevResource");
  auto split = get<PFN_cuDevSmResourceSplitByCount_v12040>("cuDevSmResourceSplitByCount");
  auto gen = get<PFN_cuDevResourceGenerateDesc_v12040>("cuDevResourceGenerateDesc");
  auto gcreate = get<PFN_cuGreenCtxCreate_v12040>("cuGreenCtxCreate");
  auto gstream = get<PFN_cuGreenCtxStreamCreate_v12050>("cuGreenCtxStreamCreate");
  CUdevResource all{}, part[1]{}, rest{};
  printf("getres %d\n", getRes(0, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("all sms %u\n", all.sm.smCount);
  unsigned n = 1;
  printf("split %d\n", split(part, &n, &all, &rest, 0, 32));
  printf("part %u rest %u groups %u\n", part[0].sm.smCount, rest.sm.smCount, n);
  CUdevResourceDesc d1, d2;
  printf("gen %d %d\n", gen(&d1, part, 1), gen(&d2, &rest, 1));
  CUgreenCtx g1, g2;
  printf("gctx %d %d\n", gcreate(&g1, d1, 0, CU_GREEN_CTX_DEFAULT_STREAM), gcreate(&g2, d2, 0, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s1, s2;
  printf("gstream %d %d\n", gstream(&s1, g1, CU_STREAM_NON_BLOCKING, 0), gstream(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
  int* buf;
  cudaMalloc(&buf, 4096 * sizeof(int));
  smid_kernel<<<512, 32, 0, (cudaStream_t)s1>>>(buf);
  printf("launch1 %s\n", cudaGetErrorString(cudaGetLastError()));
  printf("sync1 %s\n", cudaGetErrorString(cudaStreamSynchronize((cudaStream_t)s1)));
  std::vector<int> h(512);
  cudaMemcpy(h.data(), buf, 512 * sizeof(int), cudaMemcpyDeviceToHost);
  std::set<int> sms(h.begin(), h.end());
  printf("green1 used %zu distinct SMs\n", sms.size());
  smid_kernel<<<512, 32, 0, (cudaStream_t)s2>>>(buf + 1024);
  cudaStreamSynchronize((cudaStream_t)s2);
  cudaMemcpy(h.data(), buf + 1024, 512 * sizeof(int), cudaMemcpyDeviceToHost);
  std::set<int> sms2(h.begin(), h.end());
  int overlap = 0;
  for (int s : sms2) overlap += sms.count(s);
  printf("green2 used %zu distinct SMs, overlap %d\n", sms2.size(), overlap);
  // events across green / primary streams
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  cudaEventRecord(ev, (cudaStream_t)s1);
  cudaStreamWaitEvent(0, ev, 0);
  printf("cross %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  // graph capture on a green stream
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture((cudaStream_t)s1, cudaStreamCaptureModeRelaxed);
  smid_kernel<<<8, 32, 0, (cudaStream_t)s1>>>(buf);
  printf("endcap %s\n", cudaGetErrorString(cudaStreamEndCapture((cudaStream_t)s1, &g)));
  printf("inst %s\n", cudaGetErrorString(cudaGraphInstantiate(&ge, g, 0)));
  printf("glaunch %s\n", cudaGetErrorString(cudaGraphLaunch(ge, (cudaStream_t)s1)));
  printf("gsync %s\n", cudaGetErrorString(cudaStreamSynchronize((cudaStream_t)s1)));
  return 0;
}
