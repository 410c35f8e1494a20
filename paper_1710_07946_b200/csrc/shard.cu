// shard.cu — helpers of the row-sharded path (§8(e)): each rank writes the
// entries of a C-A block that it owns into a zeroed global-size buffer; an NCCL sum then
// assembles the block exactly on every rank (x + 0 + ... + 0 = x), so the replicated maxvol
// sees the same bits for any number of ranks and its pivots are identical for G = 1..8.
#include "kernels.cuh"

namespace lra {

// dst (m_global x q col-major) rows [row0, row0 + m_local) <- src (m_local x q col-major, ld)
__global__ void k_scatter_rows(const double *src, int64_t ld, int64_t m_local, int q, int64_t row0,
                               int64_t m_global, double *dst) {
  const int64_t tot = m_local * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m_local, j = e / m_local;
    dst[j * m_global + row0 + i] = src[j * ld + i];
  }
}

// vertical block C = W[:, J] (m_global x q col-major): local rows from the local operand
__global__ void k_scatter_wcols(OpView op, const int64_t *J, int q, int64_t row0, int64_t m_global, double *dst) {
  const int64_t tot = op.m * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % op.m, j = e / op.m;
    dst[j * m_global + row0 + i] = op.at(i, J[j]);
  }
}

// horizontal block R^T = W[I, :]^T (n x q col-major): slots whose row this rank owns
__global__ void k_scatter_wrows(OpView op, const int64_t *I, int q, int64_t row0, double *dst) {
  const int s = blockIdx.y;
  const int64_t gi = I[s] - row0;
  if (gi < 0 || gi >= op.m) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += (int64_t)gridDim.x * blockDim.x)
    dst[(int64_t)s * op.n + j] = op.at(gi, j);
}

// generator G = W[I, J] (k x l col-major): owned rows
__global__ void k_scatter_g(OpView op, const int64_t *I, const int64_t *J, int k, int l, int64_t row0, double *dst) {
  for (int e = threadIdx.x; e < k * l; e += blockDim.x) {
    const int s = e % k, j = e / k;
    const int64_t gi = I[s] - row0;
    if (gi >= 0 && gi < op.m) dst[e] = op.at(gi, J[j]);
  }
}

cudaError_t launch_scatter_rows(const double *src, int64_t ld, int64_t m_local, int q, int64_t row0,
                                int64_t m_global, double *dst, cudaStream_t st) {
  k_scatter_rows<<<592, 256, 0, st>>>(src, ld, m_local, q, row0, m_global, dst);
  return cudaGetLastError();
}
cudaError_t launch_scatter_wcols(const OpView &op, const int64_t *J, int q, int64_t row0, int64_t m_global,
                                 double *dst, cudaStream_t st) {
  k_scatter_wcols<<<592, 256, 0, st>>>(op, J, q, row0, m_global, dst);
  return cudaGetLastError();
}
cudaError_t launch_scatter_wrows(const OpView &op, const int64_t *I, int q, int64_t row0, double *dst,
                                 cudaStream_t st) {
  k_scatter_wrows<<<dim3(32, (unsigned)q), 256, 0, st>>>(op, I, q, row0, dst);
  return cudaGetLastError();
}
cudaError_t launch_scatter_g(const OpView &op, const int64_t *I, const int64_t *J, int k, int l, int64_t row0,
                             double *dst, cudaStream_t st) {
  k_scatter_g<<<1, 256, 0, st>>>(op, I, J, k, l, row0, dst);
  return cudaGetLastError();
}

}  // namespace lra
