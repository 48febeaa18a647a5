// sqv_ray.cu — ray_iou over label grids: one thread per
// (frame, ray) walks pred and gt by a 3D DDA to the first occupied voxel,
// then the per-threshold TP/FP/FN tallies are reduced per block and added to
// int64 counts (exact, order-independent).  FP64 with explicit _rn
// intrinsics (no FMA contraction): the same expressions, in the same order,
// as the CPU checker used by the tests, so hit distances are bit-identical.
#include "sqv_kernels.cuh"

namespace sqv {

namespace {

constexpr int kRayThreads = 128;

struct RayGrid {
  const uint8_t* lab;
  int dims[3];
  double org[3];
  double res;
  int C;
};

__device__ __forceinline__ double bound_t(const RayGrid& g, int a, int cell, double O, double D) {
  // (org + cell * res - O) / D, rounded step by step
  return __ddiv_rn(__dsub_rn(__dadd_rn(g.org[a], __dmul_rn((double)cell, g.res)), O), D);
}

__device__ int first_hit(const RayGrid& g, const double O[3], const double D[3], double* d_out,
                         int* c_out) {
  double t0 = 0.0, t1 = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double lo = g.org[a], hi = __dadd_rn(g.org[a], __dmul_rn((double)g.dims[a], g.res));
    if (D[a] == 0.0) {
      if (!(O[a] >= lo && O[a] < hi)) return 0;
    } else {
      double ta = __ddiv_rn(__dsub_rn(lo, O[a]), D[a]), tb = __ddiv_rn(__dsub_rn(hi, O[a]), D[a]);
      if (ta > tb) {
        const double s = ta;
        ta = tb;
        tb = s;
      }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
    }
  }
  if (!(t0 < t1)) return 0;
  int i[3], step[3];
  double tmax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double p = __dadd_rn(O[a], __dmul_rn(t0, D[a]));
    double f = floor(__ddiv_rn(__dsub_rn(p, g.org[a]), g.res));
    if (f < 0.0) f = 0.0;
    if (f > (double)(g.dims[a] - 1)) f = (double)(g.dims[a] - 1);
    i[a] = (int)f;
    step[a] = D[a] > 0.0 ? 1 : (D[a] < 0.0 ? -1 : 0);
    tmax[a] = step[a] == 0 ? INFINITY : bound_t(g, a, i[a] + (step[a] > 0), O[a], D[a]);
  }
  double t = t0;
  for (;;) {
    const uint8_t l =
        __ldg(g.lab + i[0] + (int64_t)g.dims[0] * (i[1] + (int64_t)g.dims[1] * i[2]));
    if (l < g.C) {
      *d_out = t;
      *c_out = l;
      return 1;
    }
    int a = 0;
    if (tmax[1] < tmax[a]) a = 1;
    if (tmax[2] < tmax[a]) a = 2;
    if (!(tmax[a] < t1)) return 0;
    t = tmax[a];
    i[a] += step[a];
    if (i[a] < 0 || i[a] >= g.dims[a]) return 0;
    tmax[a] = bound_t(g, a, i[a] + (step[a] > 0), O[a], D[a]);
  }
}

__global__ void __launch_bounds__(kRayThreads) ray_iou_kernel(RayArgs A) {
  __shared__ unsigned long long s_cnt[kMaxRayThr * 3];
  for (int k = threadIdx.x; k < A.n_thr * 3; k += blockDim.x) s_cnt[k] = 0ull;
  __syncthreads();
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)A.n_frames * A.n_rays;
  if (gid < total) {
    const int64_t f = gid / A.n_rays, r = gid - f * A.n_rays;
    const int64_t V = (int64_t)A.dims[0] * A.dims[1] * A.dims[2];
    RayGrid g;
    g.dims[0] = A.dims[0];
    g.dims[1] = A.dims[1];
    g.dims[2] = A.dims[2];
    g.org[0] = A.org[0];
    g.org[1] = A.org[1];
    g.org[2] = A.org[2];
    g.res = A.res;
    g.C = A.n_classes;
    const double O[3] = {A.origins[3 * r], A.origins[3 * r + 1], A.origins[3 * r + 2]};
    const double D[3] = {A.dirs[3 * r], A.dirs[3 * r + 1], A.dirs[3 * r + 2]};
    double dp = 0.0, dg = 0.0;
    int cp = -1, cg = -1;
    g.lab = A.pred + f * V;
    const int hp = first_hit(g, O, D, &dp, &cp);
    g.lab = A.gt + f * V;
    const int hg = first_hit(g, O, D, &dg, &cg);
    if (A.d_pred) {
      A.d_pred[gid] = hp ? dp : -1.0;
      A.c_pred[gid] = hp ? cp : -1;
      A.d_gt[gid] = hg ? dg : -1.0;
      A.c_gt[gid] = hg ? cg : -1;
    }
    for (int j = 0; j < A.n_thr; ++j) {
      if (hp && hg) {
        if (cp == cg && fabs(__dsub_rn(dp, dg)) <= A.thr[j]) {
          atomicAdd(&s_cnt[3 * j], 1ull);
        } else {
          atomicAdd(&s_cnt[3 * j + 1], 1ull);
          atomicAdd(&s_cnt[3 * j + 2], 1ull);
        }
      } else if (hp) {
        atomicAdd(&s_cnt[3 * j + 1], 1ull);
      } else if (hg) {
        atomicAdd(&s_cnt[3 * j + 2], 1ull);
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < A.n_thr * 3; k += blockDim.x)
    if (s_cnt[k]) atomicAdd(A.counts + k, s_cnt[k]);
}

}  // namespace

int ray_iou_launch(const RayArgs& A, cudaStream_t s) {
  const int64_t total = (int64_t)A.n_frames * A.n_rays;
  if (total <= 0) return SQV_OK;
  ray_iou_kernel<<<(unsigned)((total + kRayThreads - 1) / kRayThreads), kRayThreads, 0, s>>>(A);
  count_launch();
  return check_launch("ray_iou_kernel");
}

}  // namespace sqv
