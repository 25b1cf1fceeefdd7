// Experiment harness (not product code): reads the STS walk's per-level timing record.
#include "../../paper_2210_05105_b200/csrc/sts_walk.cu"
extern "C" int lab_walk_prof(void *d_ws, int64_t J, int64_t n, int leaf, int R,
                             unsigned long long *h_out) {
  WalkWs L(J, rcp_sts_depth(n, leaf), R);
  return (int)cudaMemcpy(h_out, (char *)d_ws + L.o_prof, kProfBytes, cudaMemcpyDeviceToHost);
}
