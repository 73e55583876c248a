// Tensor-product Q_p mesh generation on the GPU.
//
// Same numbering as the host tf_mesh_tensor (symbolic.cpp) and the reference's
// 1D Mesh (fem.py:59-80): elements in Morton order, every grid point owned by
// element min(i / p, n - 1) per axis, a DOF's global index = its owner's first
// index (exclusive scan of owned-point counts in Morton order) + its
// lexicographic offset inside the owner (x fastest), 1-based.
//   1. Morton key of every element (bit b of axis a at position dim*b + a);
//   2. radix sort of (key, element) -> Morton order, and its inverse (rank);
//   3. owned-point counts in Morton order, exclusive scan -> first indices;
//   4. one thread per (element, local point): owner, offset, global index.
// Element values of graded / weighted meshes: scale(e) * reference matrix,
// scale = product of the element's widths times its density.
#include <cub/cub.cuh>

#include "common.cuh"

namespace tfb {

struct MeshDims {
  int dim, p;
  long long n[3];
};

__device__ __forceinline__ void mesh_coords(const MeshDims& M, long long e, long long c[3]) {
  c[0] = e % M.n[0];
  c[1] = (e / M.n[0]) % M.n[1];
  c[2] = e / (M.n[0] * M.n[1]);
}

__global__ void mesh_keys_kernel(MeshDims M, long long n_elem, unsigned long long* keys,
                                 long long* idx) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n_elem;
       e += (long long)gridDim.x * blockDim.x) {
    long long c[3];
    mesh_coords(M, e, c);
    unsigned long long key = 0;
    for (int b = 0; b < 21; b++)
      for (int a = 0; a < M.dim; a++) key |= (unsigned long long)((c[a] >> b) & 1) << (M.dim * b + a);
    keys[e] = key;
    idx[e] = e;
  }
}

__global__ void mesh_rank_kernel(MeshDims M, long long n_elem, const long long* order,
                                 long long* rank, long long* owned) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n_elem;
       j += (long long)gridDim.x * blockDim.x) {
    const long long e = order[j];
    rank[e] = j;
    long long c[3];
    mesh_coords(M, e, c);
    long long o = 1;
    for (int a = 0; a < M.dim; a++) o *= M.p + (c[a] == M.n[a] - 1 ? 1 : 0);
    owned[j] = o;
  }
}

__global__ void mesh_dofs_kernel(MeshDims M, long long n_elem, int nloc, const long long* order,
                                 const long long* rank, const long long* first,
                                 int32_t* __restrict__ out) {
  const long long total = n_elem * nloc;
  const long long np1 = M.p + 1;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / nloc, loc = t - j * nloc;
    long long c[3];
    mesh_coords(M, order[j], c);
    const long long al[3] = {loc % np1, (loc / np1) % np1, loc / (np1 * np1)};
    long long owner[3] = {0, 0, 0}, off[3] = {0, 0, 0}, w[3] = {1, 1, 1};
    for (int a = 0; a < M.dim; a++) {
      const long long i = c[a] * M.p + al[a];
      owner[a] = min(i / M.p, M.n[a] - 1);
      off[a] = i - owner[a] * M.p;
      w[a] = M.p + (owner[a] == M.n[a] - 1 ? 1 : 0);
    }
    const long long oe = owner[0] + M.n[0] * (owner[1] + M.n[1] * owner[2]);
    const long long lr = off[0] + w[0] * (off[1] + w[1] * off[2]);
    out[t] = (int32_t)(first[rank[oe]] + lr + 1);
  }
}

__global__ void mesh_values_kernel(MeshDims M, long long n_elem, int nloc2, const long long* order,
                                   const double* nodes, const double* density,
                                   const double* ref, double* __restrict__ vals) {
  const long long total = n_elem * nloc2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / nloc2;
    const int q = (int)(t - j * nloc2);
    double s = 1.0;  // same multiplication order as TensorMesh.element_values
    long long c[3];
    mesh_coords(M, order[j], c);
    long long base = 0;
    for (int a = 0; a < M.dim; a++) {
      s *= nodes ? nodes[base + c[a] + 1] - nodes[base + c[a]] : 1.0 / (double)M.n[a];
      base += M.n[a] + 1;
    }
    if (density) s *= density[j];
    vals[t] = s * ref[q];
  }
}

static bool mesh_dims(int32_t dim, const int64_t* ns, int32_t p, MeshDims& M, long long& n_elem,
                      long long& n_dof) {
  if (dim < 1 || dim > 3 || p < 1 || !ns) return false;
  M.dim = dim;
  M.p = p;
  M.n[0] = M.n[1] = M.n[2] = 1;
  n_elem = 1;
  n_dof = 1;
  for (int a = 0; a < dim; a++) {
    if (ns[a] < 1 || ns[a] > (1 << 21)) return false;
    M.n[a] = ns[a];
    n_elem *= ns[a];
    n_dof *= ns[a] * p + 1;
  }
  return n_dof < (long long)INT32_MAX;
}

static int key_bits(const MeshDims& M) {
  long long mx = std::max(M.n[0], std::max(M.n[1], M.n[2]));
  int b = 1;
  while ((1LL << b) < mx) b++;
  return M.dim * b;
}

// workspace: keys[2n] (u64), idx[2n], rank[n], owned[n], first[n] (i64), cub temp
static size_t cub_temp_bytes(long long n, int bits) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (long long*)nullptr,
                                  (long long*)nullptr, (int)n, 0, bits);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (long long*)nullptr, (long long*)nullptr, (int)n);
  return std::max(a, b);
}

}  // namespace tfb

using namespace tfb;

extern "C" int64_t tf_mesh_tensor_device_workspace(int32_t dim, const int64_t* ns, int32_t p) {
  MeshDims M;
  long long n_elem, n_dof;
  if (!mesh_dims(dim, ns, p, M, n_elem, n_dof) || n_elem >= INT32_MAX) return -1;
  return (int64_t)(7 * 8 * n_elem + cub_temp_bytes(n_elem, key_bits(M)) + 256);
}

extern "C" int tf_mesh_tensor_device(int32_t dim, const int64_t* ns, int32_t p,
                                     int32_t* elem_dofs, int64_t* order_out, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  MeshDims M;
  long long n_elem, n_dof;
  if (!mesh_dims(dim, ns, p, M, n_elem, n_dof) || !elem_dofs || !workspace) return TF_ERR_INVALID;
  if (workspace_bytes < tf_mesh_tensor_device_workspace(dim, ns, p)) return TF_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  auto* keys = (unsigned long long*)w;
  auto* keys2 = keys + n_elem;
  auto* idx = (long long*)(keys2 + n_elem);
  auto* order = idx + n_elem;
  auto* rank = order + n_elem;
  auto* owned = rank + n_elem;
  auto* first = owned + n_elem;
  void* temp = (void*)(((uintptr_t)(first + n_elem) + 255) & ~(uintptr_t)255);
  size_t temp_bytes = cub_temp_bytes(n_elem, key_bits(M));
  const unsigned g = (unsigned)std::min<long long>((n_elem + 255) / 256, 148 * 16);
  mesh_keys_kernel<<<g, 256, 0, st>>>(M, n_elem, keys, idx);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys2, idx, order,
                                                  (int)n_elem, 0, key_bits(M), st);
  if (e != cudaSuccess) return TF_ERR_CUDA;
  mesh_rank_kernel<<<g, 256, 0, st>>>(M, n_elem, order, rank, owned);
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, owned, first, (int)n_elem, st);
  if (e != cudaSuccess) return TF_ERR_CUDA;
  int nloc = 1;
  for (int a = 0; a < dim; a++) nloc *= p + 1;
  const unsigned g2 = (unsigned)std::min<long long>((n_elem * nloc + 255) / 256, 148 * 32);
  mesh_dofs_kernel<<<g2, 256, 0, st>>>(M, n_elem, nloc, order, rank, first, elem_dofs);
  if (order_out)
    cudaMemcpyAsync(order_out, order, sizeof(long long) * n_elem, cudaMemcpyDeviceToDevice, st);
  return cudaGetLastError() == cudaSuccess ? TF_OK : TF_ERR_CUDA;
}

extern "C" int tf_mesh_element_values_device(int32_t dim, const int64_t* ns, int32_t p,
                                             const int64_t* order, const double* nodes,
                                             const double* density, const double* ref,
                                             double* values, void* stream) {
  MeshDims M;
  long long n_elem, n_dof;
  if (!mesh_dims(dim, ns, p, M, n_elem, n_dof) || !order || !ref || !values)
    return TF_ERR_INVALID;
  int nloc = 1;
  for (int a = 0; a < dim; a++) nloc *= p + 1;
  const unsigned g = (unsigned)std::min<long long>((n_elem * nloc * nloc + 255) / 256, 148 * 32);
  mesh_values_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(
      M, n_elem, nloc * nloc, reinterpret_cast<const long long*>(order), nodes, density, ref,
      values);
  return cudaGetLastError() == cudaSuccess ? TF_OK : TF_ERR_CUDA;
}
