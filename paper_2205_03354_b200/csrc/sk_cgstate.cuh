// Device-resident CG scalars (sk_cg.cu), shared with the fused matrix-free
// CG apply of the 2D stencil kernel (sk_stencil_kernels.cuh, Mode::CgApply).
#pragma once

#include <cstdint>

namespace sk {

enum : int { kCgRunning = 0, kCgCheck = 1, kCgNotPD = 2, kCgMaxIter = 3 };

struct CgState {
  double rho, pq, alpha, beta, target;
  double scalar_out;  // result slot of auxiliary reductions
  int64_t it, max_iter;
  int status;
  int pad;
  unsigned counter[4];
};

// Last CTA of the q = A p pass: pq = p.q, "not positive definite"
// (linalg.cpp:50-51) or alpha = rho / pq (:52).
__device__ __forceinline__ void cg_publish_pq(CgState* st, double pq) {
  st->pq = pq;
  if (pq <= 0) st->status = kCgNotPD;
  else st->alpha = st->rho / pq;
}

}  // namespace sk
