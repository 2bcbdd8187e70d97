// srtt_fast.cu -- blocked fast path for srdct/srft (see srtt_sketch.cu).
#include "nsk_internal.hpp"

namespace nsk {

int srtt_direct_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                      int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);

int srtt_fast_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                    int64_t lda, double* SA, int64_t ldsa, cudaStream_t st) {
  return srtt_direct_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
}

}  // namespace nsk
