// Diagnostics: pure HBM streaming with the same mechanism the decode GEMM
// uses (one producer thread per CTA, cp.async.bulk of `chunk` bytes into an
// S-stage shared-memory ring, mbarrier completion), without the MMA.  Used to
// separate the memory pipeline's ceiling from the GEMM's own overheads.
#include "common.cuh"

namespace exg {
namespace {
__global__ void stream_probe_kernel(const uint8_t* __restrict__ src, int64_t bytes_per_cta, int chunk, int stages,
                                    int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16];
  const uint8_t* base = src + (int64_t)blockIdx.x * bytes_per_cta;
  const int n = (int)(bytes_per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n && i < stages; ++i) {
      mbar_arrive_expect_tx(&full[i], chunk);
      bulk_load(sm + i * chunk, base + (int64_t)i * chunk, chunk, &full[i]);
    }
    int acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += sm[s * chunk + (i & 63)];
      if (i + stages < n) {
        mbar_arrive_expect_tx(&full[s], chunk);
        bulk_load(sm + s * chunk, base + (int64_t)(i + stages) * chunk, chunk, &full[s]);
      }
    }
    if (acc == 0x7fffffff) *sink = acc;
  }
}
}  // namespace

void stream_probe(const void* src, int64_t bytes_per_cta, int ctas, int chunk, int stages, int* sink,
                  cudaStream_t st) {
  const int smem = chunk * stages;
  EXG_CUDA(cudaFuncSetAttribute(stream_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  stream_probe_kernel<<<ctas, 32, smem, st>>>((const uint8_t*)src, bytes_per_cta, chunk, stages, sink);
  EXG_CHECK_LAUNCH();
}

}  // namespace exg

extern "C" int exg_diag_stream_probe(const void* src, int64_t bytes_per_cta, int ctas, int chunk, int stages,
                                     int* sink, void* stream) {
  try {
    exg::stream_probe(src, bytes_per_cta, ctas, chunk, stages, sink, (cudaStream_t)stream);
    return 0;
  } catch (...) {
    return 3;
  }
}
