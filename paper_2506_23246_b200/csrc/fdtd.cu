// Yee TEz FDTD reference solver on the periodic unit cell.
//
// Reference: fdtd.py:115-181 (run_reference), :194-211 (energy).  Ez at nodes
// (x_i, y_j), Hx at (x_i, y_j + dy/2), Hy at (x_i + dx/2, y_j), H leapfrogged
// at half steps, a pointwise epsilon in the Ez update, snapshots collocated to
// the Ez nodes by temporal and spatial two-point averages of H.
//
// Every thread owns one cell per step, recomputes the two neighbouring new H
// values its Ez update needs (stencil radius 1) and writes the next (Ez, Hx,
// Hy) into the other buffer set; all steps run in one cooperative launch with
// a grid barrier between steps (per-step launches as the fallback).
// float64 throughout, every operation rounded separately (explicit _rn
// intrinsics, no FMA contraction) and in numpy's order, so the fields equal
// the reference's bit for bit given the same initial state.
#include <cooperative_groups.h>

#include <cmath>

#include "gates.cuh"

namespace qpinn {

struct FdtdDev {
  int nx, ny;
  double dt, dx, dy;
  double cx, cy;  // dt/dx, dt/dy
};

__device__ __forceinline__ double hx_next(const double* __restrict__ ez,
                                          const double* __restrict__ hx, int nx, int ny, int j,
                                          int i, double cy) {
  const int jn = j + 1 == ny ? 0 : j + 1;  // roll(ez, -1, axis=0)
  const double e = ez[j * nx + i];
  return __dsub_rn(hx[j * nx + i], __dmul_rn(cy, __dsub_rn(ez[jn * nx + i], e)));
}
__device__ __forceinline__ double hy_next(const double* __restrict__ ez,
                                          const double* __restrict__ hy, int nx, int j, int i,
                                          double cx) {
  const int in = i + 1 == nx ? 0 : i + 1;  // roll(ez, -1, axis=1)
  const double e = ez[j * nx + i];
  return __dadd_rn(hy[j * nx + i], __dmul_rn(cx, __dsub_rn(ez[j * nx + in], e)));
}

// one cell of one leapfrog step (fdtd.py:160-174), optionally recording the
// collocated snapshot
__device__ __forceinline__ void fdtd_cell(const FdtdDev& p, int c, const double* __restrict__ eps,
                                          const double* __restrict__ ez,
                                          const double* __restrict__ hx,
                                          const double* __restrict__ hy, double* __restrict__ ez_o,
                                          double* __restrict__ hx_o, double* __restrict__ hy_o,
                                          double* __restrict__ rec_ez, double* __restrict__ rec_hx,
                                          double* __restrict__ rec_hy) {
  const int j = c / p.nx, i = c % p.nx;
  const int jm = j == 0 ? p.ny - 1 : j - 1, im = i == 0 ? p.nx - 1 : i - 1;
  const double hxn = hx_next(ez, hx, p.nx, p.ny, j, i, p.cy);
  const double hyn = hy_next(ez, hy, p.nx, j, i, p.cx);
  const double hxn_m = hx_next(ez, hx, p.nx, p.ny, jm, i, p.cy);  // roll(hx_new, 1, axis=0)
  const double hyn_m = hy_next(ez, hy, p.nx, j, im, p.cx);         // roll(hy_new, 1, axis=1)
  if (rec_ez) {
    rec_ez[c] = ez[c];
    const double hxm = __dmul_rn(0.5, __dadd_rn(hx[c], hxn));
    const double hxm_m = __dmul_rn(0.5, __dadd_rn(hx[jm * p.nx + i], hxn_m));
    const double hym = __dmul_rn(0.5, __dadd_rn(hy[c], hyn));
    const double hym_m = __dmul_rn(0.5, __dadd_rn(hy[j * p.nx + im], hyn_m));
    rec_hx[c] = __dmul_rn(0.5, __dadd_rn(hxm, hxm_m));
    rec_hy[c] = __dmul_rn(0.5, __dadd_rn(hym, hym_m));
  }
  const double curl = __dsub_rn(__ddiv_rn(__dsub_rn(hyn, hyn_m), p.dx),
                                __ddiv_rn(__dsub_rn(hxn, hxn_m), p.dy));
  ez_o[c] = __dadd_rn(ez[c], __dmul_rn(__ddiv_rn(p.dt, eps[c]), curl));
  hx_o[c] = hxn;
  hy_o[c] = hyn;
}

__global__ void fdtd_step(FdtdDev p, const double* __restrict__ eps, const double* __restrict__ ez,
                          const double* __restrict__ hx, const double* __restrict__ hy,
                          double* __restrict__ ez_o, double* __restrict__ hx_o,
                          double* __restrict__ hy_o, double* __restrict__ rec_ez,
                          double* __restrict__ rec_hx, double* __restrict__ rec_hy) {
  const int n = p.nx * p.ny;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    fdtd_cell(p, c, eps, ez, hx, hy, ez_o, hx_o, hy_o, rec_ez, rec_hx, rec_hy);
}

// all steps in one cooperative launch: a grid-wide barrier between steps
// replaces a kernel launch per step (the per-step work is L2-resident and
// microseconds long, so launches dominated)
struct FdtdBufs {
  double* f[2][3];
  double* rec[3];
};
__global__ void fdtd_persistent(FdtdDev p, const double* __restrict__ eps, FdtdBufs b,
                                const int32_t* __restrict__ snaps, int n_snaps, int steps) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int n = p.nx * p.ny;
  int k = 0;
  for (int s = 0; s <= steps; ++s) {
    const int cur = s & 1;
    const bool snap = k < n_snaps && snaps[k] == s;
    const size_t ro = (size_t)k * n;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
      fdtd_cell(p, c, eps, b.f[cur][0], b.f[cur][1], b.f[cur][2], b.f[cur ^ 1][0],
                b.f[cur ^ 1][1], b.f[cur ^ 1][2], snap ? b.rec[0] + ro : nullptr,
                snap ? b.rec[1] + ro : nullptr, snap ? b.rec[2] + ro : nullptr);
    if (snap) ++k;
    grid.sync();
  }
}

// initial state (fdtd.py:140-153) and the epsilon map (physics.py:45-49)
__global__ void fdtd_init(FdtdDev p, int ic, double cx0, double cy0, double sx, double sy,
                          int dielectric, double eps_r, double slab_x0, double* __restrict__ eps,
                          double* __restrict__ ez, double* __restrict__ hx,
                          double* __restrict__ hy) {
  const int n = p.nx * p.ny;
  auto xs = [&](int i) { return __dadd_rn(-1.0, __dmul_rn(p.dx, (double)i)); };
  auto ys = [&](int j) { return __dadd_rn(-1.0, __dmul_rn(p.dy, (double)j)); };
  auto pulse = [&](int j, int i) {
    const double ux = __ddiv_rn(__dsub_rn(xs(i), cx0), sx);
    const double uy = __ddiv_rn(__dsub_rn(ys(j), cy0), sy);
    return exp(__dmul_rn(-25.0, __dadd_rn(__dmul_rn(ux, ux), __dmul_rn(uy, uy))));
  };
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int j = c / p.nx, i = c % p.nx;
    const double x = xs(i);
    eps[c] = dielectric && x >= slab_x0 ? eps_r : 1.0;
    if (ic == 1) {  // plane wave Ez = Hy = cos(pi (x + t))
      ez[c] = cos(__dmul_rn(kPi, __dadd_rn(x, 0.0)));
      hx[c] = 0.0;
      hy[c] = cos(__dmul_rn(kPi, __dadd_rn(__dadd_rn(x, __ddiv_rn(p.dx, 2.0)),
                                           -__ddiv_rn(p.dt, 2.0))));
    } else {  // H(-dt/2) = -(dt/2) dH/dt|0 by the discrete curls of Ez(0)
      const double e = pulse(j, i);
      const int jn = j + 1 == p.ny ? 0 : j + 1, in = i + 1 == p.nx ? 0 : i + 1;
      const double h = __ddiv_rn(p.dt, 2.0);
      ez[c] = e;
      hx[c] = __ddiv_rn(__dmul_rn(h, __dsub_rn(pulse(jn, i), e)), p.dy);
      hy[c] = __ddiv_rn(__dmul_rn(-h, __dsub_rn(pulse(j, in), e)), p.dx);
    }
  }
}

// U = 0.5 sum (eps Ez^2 + Hx^2 + Hy^2) dx dy per snapshot (fdtd.py:194-197); one block
// per snapshot, fixed-order tree (deterministic)
__global__ void field_energy(int n, const double* __restrict__ eps, const double* __restrict__ ez,
                             const double* __restrict__ hx, const double* __restrict__ hy,
                             double dxdy, double* __restrict__ u) {
  __shared__ double red[256];
  const size_t off = (size_t)blockIdx.x * n;
  double v = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double e = ez[off + c], a = hx[off + c], b = hy[off + c];
    v += 0.5 * (eps[c] * e * e + a * a + b * b);
  }
  red[threadIdx.x] = v;
  __syncthreads();
  for (int m = blockDim.x / 2; m > 0; m >>= 1) {
    if (threadIdx.x < m) red[threadIdx.x] += red[threadIdx.x + m];
    __syncthreads();
  }
  if (threadIdx.x == 0) u[blockIdx.x] = red[0] * dxdy;
}

}  // namespace qpinn

using namespace qpinn;

extern "C" {

size_t qpinn_fdtd_workspace_bytes(int nx, int ny) {
  // eps + two field sets, plus room for a snapshot schedule of up to 2^16 steps
  return nx < 1 || ny < 1 ? 0 : (size_t)7 * nx * ny * sizeof(double) + 65536 * sizeof(int32_t);
}

int qpinn_fdtd_run(int nx, int ny, int steps, double dt, int ic, const double* pulse,
                   int dielectric, double eps_r, double slab_x0, const int32_t* snap_steps,
                   int n_snaps, double* rec_ez, double* rec_hx, double* rec_hy,
                   double* energy, void* workspace, size_t workspace_bytes, void* stream) {
  if (nx < 2 || ny < 2 || steps < 1 || !(dt > 0.0) || (ic != 0 && ic != 1) || n_snaps < 0)
    return fail(QPINN_ERR_CONFIG, "fdtd: bad configuration");
  if (workspace_bytes < qpinn_fdtd_workspace_bytes(nx, ny))
    return fail(QPINN_ERR_CONFIG, "fdtd: workspace too small");
  for (int k = 0; k < n_snaps; ++k)
    if (snap_steps[k] < 0 || snap_steps[k] > steps || (k && snap_steps[k] <= snap_steps[k - 1]))
      return fail(QPINN_ERR_CONFIG, "fdtd: snapshot steps must be increasing within [0, steps]");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)nx * ny;
  double* eps = (double*)workspace;
  double* buf[2][3] = {{eps + n, eps + 2 * n, eps + 3 * n}, {eps + 4 * n, eps + 5 * n, eps + 6 * n}};
  FdtdDev p{nx, ny, dt, 2.0 / nx, 2.0 / ny, 0.0, 0.0};
  p.cx = dt / p.dx;
  p.cy = dt / p.dy;
  const double pc[4] = {pulse ? pulse[0] : 0.0, pulse ? pulse[1] : 0.0, pulse ? pulse[2] : 1.0,
                        pulse ? pulse[3] : 1.0};
  const int threads = 256;
  const int blocks = (int)((n + threads - 1) / threads < 4096 ? (n + threads - 1) / threads : 4096);
  fdtd_init<<<blocks, threads, 0, st>>>(p, ic, pc[0], pc[1], pc[2], pc[3], dielectric, eps_r,
                                        slab_x0, eps, buf[0][0], buf[0][1], buf[0][2]);
  QPINN_CUDA_CHECK(cudaGetLastError());
  int coop = 0, dev = 0, per_sm = 0;
  QPINN_CUDA_CHECK(cudaGetDevice(&dev));
  QPINN_CUDA_CHECK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  QPINN_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fdtd_persistent,
                                                                 threads, 0));
  if (coop && per_sm > 0 && n_snaps <= 65536) {
    int32_t* snaps = (int32_t*)(eps + 7 * n);
    if (n_snaps)
      QPINN_CUDA_CHECK(cudaMemcpyAsync(snaps, snap_steps, n_snaps * sizeof(int32_t),
                                       cudaMemcpyHostToDevice, st));
    FdtdBufs b{{{buf[0][0], buf[0][1], buf[0][2]}, {buf[1][0], buf[1][1], buf[1][2]}},
               {rec_ez, rec_hx, rec_hy}};
    int grid = per_sm * num_sms();
    const int need = (int)((n + threads - 1) / threads);
    if (grid > need) grid = need;
    int ns = n_snaps;
    int nsteps = steps;
    void* args[] = {(void*)&p, (void*)&eps, (void*)&b, (void*)&snaps, (void*)&ns,
                    (void*)&nsteps};
    QPINN_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)fdtd_persistent, grid, threads,
                                                 args, 0, st));
  } else {
    int k = 0;
    for (int s = 0; s <= steps; ++s) {
      const int cur = s & 1;
      const bool snap = k < n_snaps && snap_steps[k] == s;
      fdtd_step<<<blocks, threads, 0, st>>>(
          p, eps, buf[cur][0], buf[cur][1], buf[cur][2], buf[cur ^ 1][0], buf[cur ^ 1][1],
          buf[cur ^ 1][2], snap ? rec_ez + k * n : nullptr, snap ? rec_hx + k * n : nullptr,
          snap ? rec_hy + k * n : nullptr);
      if (snap) ++k;
    }
  }
  QPINN_CUDA_CHECK(cudaGetLastError());
  if (energy && n_snaps > 0) {
    field_energy<<<n_snaps, 256, 0, st>>>((int)n, eps, rec_ez, rec_hx, rec_hy, p.dx * p.dy,
                                          energy);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return QPINN_OK;
}

}  // extern "C"
