// quant.cu -- INT8 QAT path (placeholder translation unit; see sparse_i8 in a later revision).
#include "kernels.h"
namespace sla2dev {
cudaError_t launch_quant_prep(const QuantLaunch&, cudaStream_t, int*) { return cudaErrorNotSupported; }
cudaError_t launch_sparse_i8(const SparseI8Launch&, cudaStream_t, int*) { return cudaErrorNotSupported; }
}  // namespace sla2dev
