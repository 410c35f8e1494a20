// shard.cu — helpers of the row-sharded path (§8(e)).  The blocks whose rows are
// the sharded rows of W (the sketch Y, W[:,J]) are assembled by an NCCL allgather of equal
// chunks (each rank's rows packed, zero-padded to cm = ceil(m / G) rows) and an unpack into the
// m x q column-major block; the blocks with data-dependent ownership (W[I,:]^T, W[I,J]: row
// I[s] lives on one rank) by owner scatter into a zeroed buffer and an NCCL sum (exact:
// x + 0 + ... + 0 = x).  Either way every rank holds the same bits, the replicated maxvol picks
// the same pivots for G = 1..8, and the chain is driven by device-side control flags (no host
// synchronization): k_ctl_step after every maxvol, k_ctl_combine at the end.
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

// chunk (cm x q col-major) <- local rows of src (m_local x q, ld), zero rows beyond m_local
__global__ void k_pack_rows(const double *src, int64_t ld, int64_t m_local, int q, int64_t cm, double *chunk) {
  const int64_t tot = cm * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % cm, j = e / cm;
    chunk[e] = i < m_local ? src[j * ld + i] : 0.0;
  }
}
// chunk (cm x q col-major) <- local rows of W[:, J]
__global__ void k_pack_wcols(OpView op, const int64_t *J, int q, int64_t cm, double *chunk) {
  const int64_t tot = cm * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % cm, j = e / cm;
    chunk[e] = i < op.m ? op.at(i, J[j]) : 0.0;
  }
}
// dst (m_global x q col-major) <- the gathered chunks (rank g's rows g cm ..)
__global__ void k_unpack_chunks(const double *gathered, int64_t cm, int q, int nranks, int64_t m_global, double *dst) {
  const int64_t tot = m_global * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m_global, j = e / m_global;
    const int64_t g = i / cm, il = i % cm;
    dst[e] = gathered[(g * q + j) * cm + il];
  }
}

// After the maxvol number idx of the chain (kind 0 = sketch, 1 = horizontal, 2 = vertical, loop):
// ctl[0] = first failure status, ctl[1] = converged (a loop after the first swapped nothing,
// reading C13), ctl[3] = number of maxvol calls that ran.  A maxvol launched after either flag
// was set did nothing (CAArgs::skip), and its step leaves ctl unchanged.
__global__ void k_ctl_step(const lra_ca_stats *sts, int idx, int kind, int loop, int32_t *ctl) {
  if (ctl[0] != 0 || ctl[1] != 0) return;
  ctl[3] = idx + 1;
  if (sts[idx].status != LRA_OK) {
    ctl[0] = sts[idx].status;
    return;
  }
  if (kind == 2 && loop > 0 && sts[idx].swaps == 0 && sts[idx - 1].swaps == 0) ctl[1] = 1;
}

// The per-call statistics of the calls that ran, combined as the fused kernel reports them.
__global__ void k_ctl_combine(const lra_ca_stats *sts, const int32_t *ctl, int has_y, lra_ca_stats *out) {
  lra_ca_stats o{};
  o.status = LRA_OK;
  o.logvol_final = __longlong_as_double(0x7ff8000000000000LL);       // filled by the nucleus
  o.min_pivot_margin = __longlong_as_double(0x7ff8000000000000LL);   // not measured here
  for (int i = 0; i < ctl[3]; ++i) {
    const lra_ca_stats &x = sts[i];
    if (x.status != LRA_OK) o.status = x.status;
    o.lu_steps += x.lu_steps;
    o.swaps += x.swaps;
    o.cap_hits += x.cap_hits;
    if (has_y && i == 0) {
      o.sketch_swaps = x.swaps;
    } else if (((has_y ? i - 1 : i) % 2) == 0) {
      o.cert_cols = x.cert_rows;
    } else {
      o.cert_rows = x.cert_rows;
      o.loops_done += 1;
    }
  }
  *out = o;
}

cudaError_t launch_pack_rows(const double *src, int64_t ld, int64_t m_local, int q, int64_t cm, double *chunk,
                             cudaStream_t st) {
  k_pack_rows<<<592, 256, 0, st>>>(src, ld, m_local, q, cm, chunk);
  return cudaGetLastError();
}
cudaError_t launch_pack_wcols(const OpView &op, const int64_t *J, int q, int64_t cm, double *chunk, cudaStream_t st) {
  k_pack_wcols<<<592, 256, 0, st>>>(op, J, q, cm, chunk);
  return cudaGetLastError();
}
cudaError_t launch_unpack_chunks(const double *gathered, int64_t cm, int q, int nranks, int64_t m_global, double *dst,
                                 cudaStream_t st) {
  k_unpack_chunks<<<592, 256, 0, st>>>(gathered, cm, q, nranks, m_global, dst);
  return cudaGetLastError();
}
cudaError_t launch_ctl_step(const lra_ca_stats *sts, int idx, int kind, int loop, int32_t *ctl, cudaStream_t st) {
  k_ctl_step<<<1, 1, 0, st>>>(sts, idx, kind, loop, ctl);
  return cudaGetLastError();
}
cudaError_t launch_ctl_combine(const lra_ca_stats *sts, const int32_t *ctl, int has_y, lra_ca_stats *out,
                               cudaStream_t st) {
  k_ctl_combine<<<1, 1, 0, st>>>(sts, ctl, has_y, out);
  return cudaGetLastError();
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
