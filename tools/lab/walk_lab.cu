// Experiment harness (not product code): reads the STS walk's per-level timing record.
#include "../../paper_2210_05105_b200/csrc/sts_walk.cu"
extern "C" int lab_walk_prof(void *d_ws, int64_t J, int64_t n, int leaf, int R,
                             unsigned long long *h_out) {
  WalkWs L(J, rcp_sts_depth(n, leaf), R);
  return (int)cudaMemcpy(h_out, (char *)d_ws + L.o_prof, kProfBytes, cudaMemcpyDeviceToHost);
}

// grid barrier cost: `iters` cooperative-groups grid syncs by the walk's launch shape
__global__ void __launch_bounds__(512, 2) gsync_probe_kernel(int iters, int *sink) {
  cg::grid_group grid = cg::this_grid();
  for (int i = 0; i < iters; ++i) grid.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

extern "C" int lab_gsync_probe(int iters, int *d_sink, float *ms_out) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gsync_probe_kernel, 512, 100 * 1024);
  const int grid = 2 * sm_count();
  void *args[] = {(void *)&iters, (void *)&d_sink};
  cudaFuncSetAttribute(gsync_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((const void *)gsync_probe_kernel, dim3(grid), dim3(512), args,
                                100 * 1024, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  *ms_out = best;
  return (int)cudaGetLastError();
}
