// mesh.cu -- the evaluation side after training: the grid of query points,
// zero-level-set extraction and the paper's reconstruction metrics (§4: Chamfer
// Distance x10^3, F1 x10^2, Normal Consistency x10^2; the Hausdorff distance of the Fig. 1 error
// maps).  Readings: DESIGN.md §2 items 17-21.
//
//   extraction  marching tetrahedra: each grid cell split into the 6 Kuhn tetrahedra around its
//               main diagonal (shared faces triangulated identically: watertight), a vertex on
//               every sign-changing edge by linear interpolation t = f_a / (f_a - f_b), inside =
//               f < 0, triangles oriented from the inside corners to the outside ones.  Two
//               passes (per-cell triangle counts -> exclusive scan -> emission), so the output
//               order is fixed: cells x-fastest, tetrahedra, triangles -- deterministic.
//   metrics     nsample points area-weighted on the triangles (inverse CDF of the fp64 cumulative
//               areas, counter-based SplitMix64 randoms), brute-force nearest neighbours both ways
//               (shared-memory tiles of the reference set; ties -> the lowest index), and
//               fixed-order fp64 reductions of the distances, threshold counts and |cos| of the
//               matched normals.
#include <cub/cub.cuh>

#include "../../include/fdsdf.h"
#include "common.cuh"
#include "fdepi.cuh"

namespace fdsdf {

// the 6 Kuhn tetrahedra of a cell (corner b = (b & 1, (b >> 1) & 1, (b >> 2) & 1))
__constant__ int kKuhn[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

struct V3 {
  float x, y, z;
};
__device__ __forceinline__ V3 lerp_edge(const V3& a, const V3& b, float fa, float fb) {
  const float t = fa / (fa - fb);
  return V3{fmaf(t, b.x - a.x, a.x), fmaf(t, b.y - a.y, a.y), fmaf(t, b.z - a.z, a.z)};
}

// triangles of one tetrahedron (0, 1 or 2) into tri[..][3]
__device__ __forceinline__ int tet_triangles(const float (&f)[4], const V3 (&p)[4], V3 (&tri)[2][3]) {
  int mask = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) mask |= (f[q] < 0.f) << q;
  if (mask == 0 || mask == 15) return 0;
  int in[4], out[4], ni = 0, no = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if ((mask >> q) & 1)
      in[ni++] = q;
    else
      out[no++] = q;
  }
  int nt;
  if (ni == 1 || ni == 3) {
    const int lone = ni == 1 ? in[0] : out[0];
    int o[3], k = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q != lone) o[k++] = q;
    for (int j = 0; j < 3; ++j) tri[0][j] = lerp_edge(p[lone], p[o[j]], f[lone], f[o[j]]);
    nt = 1;
  } else {
    const int a = in[0], b = in[1], c = out[0], d = out[1];
    const V3 ac = lerp_edge(p[a], p[c], f[a], f[c]), ad = lerp_edge(p[a], p[d], f[a], f[d]);
    const V3 bd = lerp_edge(p[b], p[d], f[b], f[d]), bc = lerp_edge(p[b], p[c], f[b], f[c]);
    tri[0][0] = ac, tri[0][1] = ad, tri[0][2] = bd;
    tri[1][0] = ac, tri[1][1] = bd, tri[1][2] = bc;
    nt = 2;
  }
  // orientation: normal from the inside corners towards the outside ones
  float gx = 0.f, gy = 0.f, gz = 0.f;
  for (int q = 0; q < 4; ++q) {
    const float w = ((mask >> q) & 1) ? -1.f / ni : 1.f / no;
    gx = fmaf(w, p[q].x, gx);
    gy = fmaf(w, p[q].y, gy);
    gz = fmaf(w, p[q].z, gz);
  }
  for (int s = 0; s < nt; ++s) {
    const V3 e1{tri[s][1].x - tri[s][0].x, tri[s][1].y - tri[s][0].y, tri[s][1].z - tri[s][0].z};
    const V3 e2{tri[s][2].x - tri[s][0].x, tri[s][2].y - tri[s][0].y, tri[s][2].z - tri[s][0].z};
    const float nx = e1.y * e2.z - e1.z * e2.y, ny = e1.z * e2.x - e1.x * e2.z, nz = e1.x * e2.y - e1.y * e2.x;
    if (nx * gx + ny * gy + nz * gz < 0.f) {
      const V3 t = tri[s][1];
      tri[s][1] = tri[s][2];
      tri[s][2] = t;
    }
  }
  return nt;
}

struct Grid {
  const float* f;
  int nx, ny, nz;
  float ox, oy, oz, sp;
};

__device__ __forceinline__ void cell_corners(const Grid& g, int64_t cell, float (&cf)[8], V3 (&cp)[8]) {
  const int cx = g.nx - 1, cy = g.ny - 1;
  const int i = (int)(cell % cx), j = (int)((cell / cx) % cy), k = (int)(cell / ((int64_t)cx * cy));
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const int di = b & 1, dj = (b >> 1) & 1, dk = (b >> 2) & 1;
    cf[b] = g.f[(i + di) + (int64_t)g.nx * ((j + dj) + (int64_t)g.ny * (k + dk))];
    cp[b] = V3{g.ox + g.sp * (float)(i + di), g.oy + g.sp * (float)(j + dj), g.oz + g.sp * (float)(k + dk)};
  }
}

__global__ void mt_count_kernel(const Grid g, int64_t ncell, int* counts) {
  for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell < ncell;
       cell += (int64_t)gridDim.x * blockDim.x) {
    float cf[8];
    V3 cp[8];
    cell_corners(g, cell, cf, cp);
    int n = 0;
    for (int t = 0; t < 6; ++t) {
      int mask = 0;
      for (int q = 0; q < 4; ++q) mask |= (cf[kKuhn[t][q]] < 0.f) << q;
      const int ni = __popc(mask);
      n += (ni == 0 || ni == 4) ? 0 : (ni == 2 ? 2 : 1);
    }
    counts[cell] = n;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[ncell] = 0;
}

__global__ void mt_emit_kernel(const Grid g, int64_t ncell, const int64_t* offsets, float* tris) {
  for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell < ncell;
       cell += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offsets[cell];
    if (offsets[cell + 1] == o) continue;
    float cf[8];
    V3 cp[8];
    cell_corners(g, cell, cf, cp);
    for (int t = 0; t < 6; ++t) {
      float f[4];
      V3 p[4];
      for (int q = 0; q < 4; ++q) {
        f[q] = cf[kKuhn[t][q]];
        p[q] = cp[kKuhn[t][q]];
      }
      V3 tri[2][3];
      const int nt = tet_triangles(f, p, tri);
      for (int s = 0; s < nt; ++s, ++o)
        for (int v = 0; v < 3; ++v) {
          tris[o * 9 + v * 3 + 0] = tri[s][v].x;
          tris[o * 9 + v * 3 + 1] = tri[s][v].y;
          tris[o * 9 + v * 3 + 2] = tri[s][v].z;
        }
    }
  }
}

__global__ void grid_points_kernel(int nx, int ny, int nz, float ox, float oy, float oz, float sp, float* x) {
  const int64_t n = (int64_t)nx * ny * nz;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % nx), j = (int)((q / nx) % ny), k = (int)(q / ((int64_t)nx * ny));
    x[q * 3 + 0] = ox + sp * (float)i;
    x[q * 3 + 1] = oy + sp * (float)j;
    x[q * 3 + 2] = oz + sp * (float)k;
  }
}

// ----------------------------------------------------------------------------- metrics

__global__ void tri_area_kernel(const float* tris, int64_t nt, double* area) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    const float* v = tris + t * 9;
    const double e1x = (double)v[3] - v[0], e1y = (double)v[4] - v[1], e1z = (double)v[5] - v[2];
    const double e2x = (double)v[6] - v[0], e2y = (double)v[7] - v[1], e2z = (double)v[8] - v[2];
    const double cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
    area[t] = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
  }
}

__device__ __forceinline__ double counter_u01(uint64_t seed, uint64_t k) {
  return (double)(mix64(seed + (k + 1ull) * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
}

__global__ void sample_kernel(const float* tris, int64_t nt, const double* cum, int64_t ns, uint64_t seed, float* P,
                              float* Pn) {
  const double total = cum[nt - 1];
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < ns; s += (int64_t)gridDim.x * blockDim.x) {
    const double u0 = counter_u01(seed, 3 * s), u1 = counter_u01(seed, 3 * s + 1), u2 = counter_u01(seed, 3 * s + 2);
    const double target = u0 * total;
    int64_t lo = 0, hi = nt;  // first t with cum[t] > target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cum[mid] > target)
        hi = mid;
      else
        lo = mid + 1;
    }
    const int64_t t = lo < nt ? lo : nt - 1;
    const float* v = tris + t * 9;
    const double r1 = sqrt(u1);
    const double w0 = 1.0 - r1, w1 = r1 * (1.0 - u2), w2 = r1 * u2;
    for (int d = 0; d < 3; ++d) P[s * 3 + d] = (float)(w0 * v[d] + w1 * v[3 + d] + w2 * v[6 + d]);
    const double e1x = (double)v[3] - v[0], e1y = (double)v[4] - v[1], e1z = (double)v[5] - v[2];
    const double e2x = (double)v[6] - v[0], e2y = (double)v[7] - v[1], e2z = (double)v[8] - v[2];
    double cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
    const double inv = 1.0 / sqrt(cx * cx + cy * cy + cz * cz);
    Pn[s * 3 + 0] = (float)(cx * inv);
    Pn[s * 3 + 1] = (float)(cy * inv);
    Pn[s * 3 + 2] = (float)(cz * inv);
  }
}

// brute-force nearest neighbour of every query in the reference set: d = min |q - r|, idx = the
// lowest index attaining it
constexpr int NN_TILE = 2048;
__global__ void __launch_bounds__(256) nn_kernel(const float* Q, int64_t nq, const float* R, int64_t nr, float* dist,
                                                 int* idx) {
  __shared__ float rs[NN_TILE * 3];
  for (int64_t qb = blockIdx.x * (int64_t)blockDim.x; qb < nq; qb += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = qb + threadIdx.x;
    const bool ok = q < nq;
    const float qx = ok ? Q[q * 3] : 0.f, qy = ok ? Q[q * 3 + 1] : 0.f, qz = ok ? Q[q * 3 + 2] : 0.f;
    float best = INFINITY;
    int bi = 0;
    for (int64_t r0 = 0; r0 < nr; r0 += NN_TILE) {
      const int m = (int)(nr - r0 < NN_TILE ? nr - r0 : NN_TILE);
      __syncthreads();
      for (int i = threadIdx.x; i < m * 3; i += blockDim.x) rs[i] = R[r0 * 3 + i];
      __syncthreads();
      for (int i = 0; i < m; ++i) {
        const float dx = qx - rs[i * 3], dy = qy - rs[i * 3 + 1], dz = qz - rs[i * 3 + 2];
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        if (d2 < best) {
          best = d2;
          bi = (int)(r0 + i);
        }
      }
    }
    if (ok) {
      dist[q] = sqrtf(best);
      idx[q] = bi;
    }
  }
}

// fixed-order fp64 partial sums over contiguous ranges: [sum d, count d < tau, sum |n_q . n_r[idx]|, max d]
constexpr int RED_BLOCKS = 256;
__global__ void __launch_bounds__(256) nn_reduce_kernel(const float* dist, const int* idx, const float* Qn,
                                                        const float* Rn, int64_t nq, float tau, double* part) {
  __shared__ double sh[4][256];
  const int64_t per = (nq + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = (b0 + per < nq) ? b0 + per : nq;
  double s = 0.0, c = 0.0, n = 0.0, mx = 0.0;
  for (int64_t q = b0 + threadIdx.x; q < b1; q += blockDim.x) {
    const double d = dist[q];
    s += d;
    c += d < (double)tau ? 1.0 : 0.0;
    const int r = idx[q];
    n += fabs((double)Qn[q * 3] * Rn[r * 3] + (double)Qn[q * 3 + 1] * Rn[r * 3 + 1] + (double)Qn[q * 3 + 2] * Rn[r * 3 + 2]);
    mx = fmax(mx, d);
  }
  sh[0][threadIdx.x] = s;
  sh[1][threadIdx.x] = c;
  sh[2][threadIdx.x] = n;
  sh[3][threadIdx.x] = mx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + w];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + w];
      sh[2][threadIdx.x] += sh[2][threadIdx.x + w];
      sh[3][threadIdx.x] = fmax(sh[3][threadIdx.x], sh[3][threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) part[blockIdx.x * 4 + k] = sh[k][0];
}

__global__ void final_reduce_kernel(const double* part, int nb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0, c = 0.0, n = 0.0, mx = 0.0;
    for (int b = 0; b < nb; ++b) {
      s += part[b * 4];
      c += part[b * 4 + 1];
      n += part[b * 4 + 2];
      mx = fmax(mx, part[b * 4 + 3]);
    }
    out[0] = s;
    out[1] = c;
    out[2] = n;
    out[3] = mx;
  }
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static size_t mt_scan_temp(int64_t ncell) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int*)nullptr, (int64_t*)nullptr, (int)(ncell + 1));
  return t;
}

static size_t cum_scan_temp(int64_t nt) {
  size_t t = 0;
  cub::DeviceScan::InclusiveSum(nullptr, t, (const double*)nullptr, (double*)nullptr, (int)nt);
  return t;
}

static int blocks_for(int64_t n, int per = 256) { return (int)std::max<int64_t>(1, std::min<int64_t>(4096, (n + per - 1) / per)); }

}  // namespace fdsdf

using namespace fdsdf;

extern "C" {

fdsdf_status fdsdf_grid_points(int nx, int ny, int nz, float ox, float oy, float oz, float spacing, float* d_x,
                               void* stream) {
  if (nx < 1 || ny < 1 || nz < 1 || !d_x || !(spacing > 0.f)) return FDSDF_E_INVALID;
  const int64_t n = (int64_t)nx * ny * nz;
  grid_points_kernel<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(nx, ny, nz, ox, oy, oz, spacing, d_x);
  return cudaGetLastError() == cudaSuccess ? FDSDF_OK : FDSDF_E_CUDA;
}

size_t fdsdf_mesh_work_bytes(int nx, int ny, int nz) {
  if (nx < 2 || ny < 2 || nz < 2) return 0;
  const int64_t ncell = (int64_t)(nx - 1) * (ny - 1) * (nz - 1);
  return align256((ncell + 1) * sizeof(int)) + align256((ncell + 1) * sizeof(int64_t)) + align256(mt_scan_temp(ncell));
}

fdsdf_status fdsdf_mesh_extract(const float* d_f, int nx, int ny, int nz, float ox, float oy, float oz,
                                float spacing, float* d_tris, int64_t max_tris, int64_t* h_ntris, void* d_work,
                                size_t work_bytes, void* stream) {
  if (!d_f || !h_ntris || nx < 2 || ny < 2 || nz < 2 || !(spacing > 0.f) || max_tris < 0) return FDSDF_E_INVALID;
  if (!d_work || work_bytes < fdsdf_mesh_work_bytes(nx, ny, nz)) return FDSDF_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ncell = (int64_t)(nx - 1) * (ny - 1) * (nz - 1);
  unsigned char* w = static_cast<unsigned char*>(d_work);
  int* counts = reinterpret_cast<int*>(w);
  int64_t* offsets = reinterpret_cast<int64_t*>(w + align256((ncell + 1) * sizeof(int)));
  void* temp = w + align256((ncell + 1) * sizeof(int)) + align256((ncell + 1) * sizeof(int64_t));
  size_t tb = mt_scan_temp(ncell);
  const Grid g{d_f, nx, ny, nz, ox, oy, oz, spacing};
  mt_count_kernel<<<blocks_for(ncell), 256, 0, st>>>(g, ncell, counts);
  if (cudaGetLastError() != cudaSuccess) return FDSDF_E_CUDA;
  if (cub::DeviceScan::ExclusiveSum(temp, tb, counts, offsets, (int)(ncell + 1), st) != cudaSuccess) return FDSDF_E_CUDA;
  int64_t total = 0;
  if (cudaMemcpyAsync(&total, offsets + ncell, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return FDSDF_E_CUDA;
  *h_ntris = total;
  if (total > max_tris || (total > 0 && !d_tris)) return FDSDF_E_INVALID;  // *h_ntris tells the size needed
  if (total > 0) {
    mt_emit_kernel<<<blocks_for(ncell), 256, 0, st>>>(g, ncell, offsets, d_tris);
    if (cudaGetLastError() != cudaSuccess) return FDSDF_E_CUDA;
  }
  return FDSDF_OK;
}

size_t fdsdf_metrics_work_bytes(int64_t ntris, int64_t nsample, int64_t ngt) {
  if (ntris < 1 || nsample < 1 || ngt < 1) return 0;
  return 2 * align256(ntris * sizeof(double)) + align256(cum_scan_temp(ntris)) + 2 * align256(nsample * 3 * sizeof(float)) +
         align256(nsample * sizeof(float)) + align256(nsample * sizeof(int)) + align256(ngt * sizeof(float)) +
         align256(ngt * sizeof(int)) + align256(2 * RED_BLOCKS * 4 * sizeof(double)) + align256(8 * sizeof(double));
}

fdsdf_status fdsdf_mesh_metrics(const float* d_tris, int64_t ntris, const float* d_gt, const float* d_gt_normals,
                                int64_t ngt, int64_t nsample, uint64_t seed, float tau, double* h_out, void* d_work,
                                size_t work_bytes, void* stream) {
  if (!d_tris || !d_gt || !d_gt_normals || !h_out || ntris < 1 || ngt < 1 || nsample < 1 || !(tau > 0.f))
    return ntris == 0 ? FDSDF_E_EMPTY : FDSDF_E_INVALID;
  if (ntris > INT32_MAX || ngt > INT32_MAX || nsample > INT32_MAX) return FDSDF_E_INVALID;
  if (!d_work || work_bytes < fdsdf_metrics_work_bytes(ntris, nsample, ngt)) return FDSDF_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char* w = static_cast<unsigned char*>(d_work);
  auto take = [&](size_t b) {
    unsigned char* p = w;
    w += align256(b);
    return p;
  };
  double* area = reinterpret_cast<double*>(take(ntris * sizeof(double)));
  double* cum = reinterpret_cast<double*>(take(ntris * sizeof(double)));
  size_t tb = cum_scan_temp(ntris);
  void* temp = take(tb);
  float* P = reinterpret_cast<float*>(take(nsample * 3 * sizeof(float)));
  float* Pn = reinterpret_cast<float*>(take(nsample * 3 * sizeof(float)));
  float* dp = reinterpret_cast<float*>(take(nsample * sizeof(float)));
  int* ip = reinterpret_cast<int*>(take(nsample * sizeof(int)));
  float* dg = reinterpret_cast<float*>(take(ngt * sizeof(float)));
  int* ig = reinterpret_cast<int*>(take(ngt * sizeof(int)));
  double* part = reinterpret_cast<double*>(take(2 * RED_BLOCKS * 4 * sizeof(double)));
  double* res = reinterpret_cast<double*>(take(8 * sizeof(double)));
  tri_area_kernel<<<blocks_for(ntris), 256, 0, st>>>(d_tris, ntris, area);
  if (cub::DeviceScan::InclusiveSum(temp, tb, area, cum, (int)ntris, st) != cudaSuccess) return FDSDF_E_CUDA;
  sample_kernel<<<blocks_for(nsample), 256, 0, st>>>(d_tris, ntris, cum, nsample, seed, P, Pn);
  nn_kernel<<<blocks_for(nsample), 256, 0, st>>>(P, nsample, d_gt, ngt, dp, ip);
  nn_kernel<<<blocks_for(ngt), 256, 0, st>>>(d_gt, ngt, P, nsample, dg, ig);
  nn_reduce_kernel<<<RED_BLOCKS, 256, 0, st>>>(dp, ip, Pn, d_gt_normals, nsample, tau, part);
  nn_reduce_kernel<<<RED_BLOCKS, 256, 0, st>>>(dg, ig, d_gt_normals, Pn, ngt, tau, part + RED_BLOCKS * 4);
  final_reduce_kernel<<<1, 32, 0, st>>>(part, RED_BLOCKS, res);
  final_reduce_kernel<<<1, 32, 0, st>>>(part + RED_BLOCKS * 4, RED_BLOCKS, res + 4);
  if (cudaGetLastError() != cudaSuccess) return FDSDF_E_CUDA;
  double r[8];
  if (cudaMemcpyAsync(r, res, sizeof(r), cudaMemcpyDeviceToHost, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
    return FDSDF_E_CUDA;
  const double prec = r[1] / (double)nsample, rec = r[5] / (double)ngt;
  h_out[0] = 0.5 * (r[0] / (double)nsample + r[4] / (double)ngt);   // CD
  h_out[1] = prec + rec > 0.0 ? 2.0 * prec * rec / (prec + rec) : 0.0;  // F1
  h_out[2] = 0.5 * (r[2] / (double)nsample + r[6] / (double)ngt);   // NC
  h_out[3] = r[3] > r[7] ? r[3] : r[7];                              // Hausdorff
  h_out[4] = prec;
  h_out[5] = rec;
  return FDSDF_OK;
}

}  // extern "C"
