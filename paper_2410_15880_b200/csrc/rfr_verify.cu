// rfr_verify.cu -- batched candidate verification on sm_100a, one warp per
// candidate.  Replaces the reference's per-candidate Python loop
// build_candidate -> trace_test -> round_and_divide (pkg/src/polyfactor/
// verify.py:60-155, driven at :267-286):
//   1. pick the smaller-degree side of {pattern, complement} (both are
//      factors or neither is);
//   2. multiply out its linear (x - u) and quadratic (x^2 - t x + m) pieces in
//      double-double (~106 bits), lane-parallel over the coefficients;
//   3. bound every coefficient's error from the roots' error bound and the
//      arithmetic (a magnitude polynomial evaluated with perturbed roots), and
//      reject any coefficient farther from an integer than its bound (the
//      reference's eps test, verify.py:145-148, with a derived tolerance);
//   4. trial-divide the input p by the rounded monic q modulo three primes
//      2^61 - 1, 2^62 - 57, 2^63 - 25 (two-fold reduction, no division) (the reference's divide_exact, polynomial.py:155-183, as a
//      filter; the host confirms survivors exactly with the certificate).
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rfr.h"
#include "rfr_common.cuh"
#include "rfr_internal.h"
#include "rfr_verify.cuh"

namespace rfr {

__global__ void __launch_bounds__(kVerifyWarps * 32) verify_kernel(VerifyArgs A) {
  __shared__ WarpBuf bufs[kVerifyWarps];
  __shared__ ProfSmem PS;
  pdl_wait();  // programmatic launch: the previous kernel is complete
  pdl_trigger();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long mm = A.m;
  if (A.m_dev) mm = min(mm, (long long)*A.m_dev);
  const long long k0 = A.m_begin_dev ? min((long long)*A.m_begin_dev, mm) : 0ll;
  // grid sized by a row bound, count on the device: idle CTAs leave before
  // staging the profile (uniform per CTA, ahead of the barrier)
  if (k0 + (long long)blockIdx.x * kVerifyWarps >= mm) return;
  stage_profile_smem(PS, A, threadIdx.x, blockDim.x);
  __syncthreads();
  WarpBuf& B = bufs[w];
  // grid-stride over the candidates (one warp each): the fused search+verify
  // sizes the grid by SMs, the count being known on the device only
  for (long long k = k0 + (long long)blockIdx.x * kVerifyWarps + w; k < mm;
       k += (long long)gridDim.x * kVerifyWarps) {
    __syncwarp();  // the warp's buffer is reused candidate after candidate
    verify_one(A, PS, B, k, lane);
    __syncwarp();
  }
}

cudaError_t launch_verify(const VerifyArgs& A, cudaStream_t s) {
  if (A.m <= 0) return cudaSuccess;
  long long blocks = (A.m + kVerifyWarps - 1) / kVerifyWarps;
  if (A.m_dev) {  // count on the device: enough warps to cover a typical set, grid-stride beyond
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (blocks > 8LL * nsm) blocks = 8LL * nsm;
  }
  const cudaError_t e = launch_pdl(verify_kernel, dim3((unsigned)blocks), dim3(kVerifyWarps * 32), 0, s, A);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace rfr
