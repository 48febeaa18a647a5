/*
 * sqv_oracle.c — CPU FP64 restatement of the SuperQuadricOcc voxelization path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for the B200 library.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the product
 * path (paper_2511_17361_b200) never does.
 *
 * What it follows (all paths under /root/reference):
 *   - SuperQuadric validation + eps clamp ........ pkg/src/sqocc/core.py:143-173
 *   - quat_normalize ............................. pkg/src/sqocc/core.py:30-35
 *   - quat_to_matrix / world_to_local_matrix ..... pkg/src/sqocc/core.py:55-65,183-185
 *   - to_local ................................... pkg/src/sqocc/core.py:237-244
 *   - inside_outside (abs, exponents, F_CAP) ..... pkg/src/sqocc/core.py:254-273
 *   - density = exp(-F) .......................... pkg/src/sqocc/core.py:276-282
 *   - voxelize window + scatter .................. SPEC.md:345-353, ledger SPEC.md:382-385
 *   - voxelize_bruteforce (whole-grid window) .... SPEC.md:355-363
 *   - finalize (tau, argmax lowest index) ........ SPEC.md:365-373
 *   - bins (tile -> ascending primitive ids) ..... SPEC.md:385 (tile shape pinned in include/sqv.h)
 *   - confusion counts for IoU / mIoU ............ SPEC.md:494-512,532
 *   - ray_iou: DDA first hits, TP/FP/FN per threshold
 *
 * Parity pin: tests/golden/make_golden.py evaluates the reference's own
 * sqocc.core functions (imported from /root/reference) on seeded inputs and
 * commits the results under tests/golden/; tests/test_oracle_golden.py checks
 * this file against them (1e-12 relative, windows/bins/labels exact).
 *
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).  FP contraction
 * is off so every expression rounds like NumPy's float64 ufuncs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TX 8  /* SQV_TILE_X */
#define TY 8  /* SQV_TILE_Y */
#define TZ 16 /* SQV_TILE_Z */

static const double EPS_MIN = 0.2; /* core.py:18 */
static const double EPS_MAX = 2.0; /* core.py:19 */
static const double F_CAP = 1e30;  /* core.py:23 */

typedef struct {
  double origin[3];
  int32_t dims[3];
  double res;
} ogrid;

typedef struct {
  double tau;
  int32_t radius;
  int32_t truncate;
  int32_t prob_sum;
  int32_t free_label;
  double extent;
} ocfg;

/* Prepared primitive: what SuperQuadric holds after __post_init__ plus the
 * world->local matrix and the voxel window. */
typedef struct {
  double mu[3], scale[3];
  double Rwl[9]; /* world_to_local_matrix(), row-major */
  double a, b, c; /* 2/eps2, eps2/eps1, 2/eps1 (core.py:267-269) */
  double sigma;
  int32_t lo[3], hi[3]; /* clipped window, empty if lo > hi */
  int32_t live;         /* window non-empty and sigma > 0 */
} oprim;

int sqvo_abi(void) { return 1; }

int sqvo_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void sqvo_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* quat_to_matrix (core.py:55-65): local-to-world rotation of unit q=(w,x,y,z). */
static void quat_to_matrix(const double q[4], double R[9]) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double xx = x * x, yy = y * y, zz = z * z;
  double wx = w * x, wy = w * y, wz = w * z;
  double xy = x * y, xz = x * z, yz = y * z;
  R[0] = 1.0 - 2.0 * (yy + zz); R[1] = 2.0 * (xy - wz);       R[2] = 2.0 * (xz + wy);
  R[3] = 2.0 * (xy + wz);       R[4] = 1.0 - 2.0 * (xx + zz); R[5] = 2.0 * (yz - wx);
  R[6] = 2.0 * (xz - wy);       R[7] = 2.0 * (yz + wx);       R[8] = 1.0 - 2.0 * (xx + yy);
}

/* Validation + normalisation + clamp of one primitive, in the order of
 * SuperQuadric.__post_init__ (core.py:143-173).  Returns failure bits (the
 * same bits as include/sqv.h SQV_BAD_*). */
static int prep_one(const double* mu, const double* scale, const double* rot, double opacity,
                    const double* eps, const double* logits, int C, oprim* P) {
  int bad = 0;
  for (int k = 0; k < 3; ++k)
    if (!isfinite(mu[k]) || !isfinite(scale[k])) bad |= 1;
  if (!bad)
    for (int k = 0; k < 3; ++k)
      if (!(scale[k] > 0.0)) bad |= 2;
  for (int k = 0; k < C; ++k)
    if (!isfinite(logits[k])) bad |= 4;
  if (!(opacity >= 0.0 && opacity <= 1.0)) bad |= 8;
  /* quat_normalize (core.py:30-35) */
  double n = sqrt(rot[0] * rot[0] + rot[1] * rot[1] + rot[2] * rot[2] + rot[3] * rot[3]);
  if (!(n >= 1e-12)) bad |= 16;
  if (!isfinite(eps[0]) || !isfinite(eps[1])) bad |= 32;
  if (bad) return bad;
  double q[4] = {rot[0] / n, rot[1] / n, rot[2] / n, rot[3] / n};
  double R[9];
  quat_to_matrix(q, R);
  /* world_to_local_matrix = quat_to_matrix(rot).T (core.py:183-185) */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) P->Rwl[3 * i + j] = R[3 * j + i];
  /* eps clamp (core.py:160-165) */
  double e1 = fmin(fmax(eps[0], EPS_MIN), EPS_MAX);
  double e2 = fmin(fmax(eps[1], EPS_MIN), EPS_MAX);
  P->a = 2.0 / e2;
  P->b = e2 / e1;
  P->c = 2.0 / e1;
  for (int k = 0; k < 3; ++k) {
    P->mu[k] = mu[k];
    P->scale[k] = scale[k];
  }
  P->sigma = opacity;
  return 0;
}

/* Voxel window of SPEC.md:348 with the ledger expansion of SPEC.md:382:
 * centre voxel c = floor((mu - origin)/res), radius r = N + ceil(max(s)*K/res),
 * window [c-r, c+r] per axis (Chebyshev) clipped to the grid.  The device
 * prep kernel evaluates the same IEEE expressions in the same order. */
static void window_of(oprim* P, const ogrid* g, const ocfg* cfg) {
  if (!cfg->truncate) {
    for (int k = 0; k < 3; ++k) {
      P->lo[k] = 0;
      P->hi[k] = g->dims[k] - 1;
    }
    return;
  }
  double smax = fmax(fmax(P->scale[0], P->scale[1]), P->scale[2]);
  double r = (double)cfg->radius + ceil(smax * cfg->extent / g->res);
  for (int k = 0; k < 3; ++k) {
    double c = floor((P->mu[k] - g->origin[k]) / g->res);
    double lo = fmax(c - r, 0.0);
    double hi = fmin(c + r, (double)(g->dims[k] - 1));
    if (lo > hi) {
      P->lo[k] = 1;
      P->hi[k] = 0;
    } else {
      P->lo[k] = (int32_t)lo;
      P->hi[k] = (int32_t)hi;
    }
  }
}

static int is_live(const oprim* P) {
  return P->sigma > 0.0 && P->lo[0] <= P->hi[0] && P->lo[1] <= P->hi[1] && P->lo[2] <= P->hi[2];
}

/* to_local (core.py:237-244) + inside_outside (core.py:254-273). */
static double field_F(const oprim* P, double px, double py, double pz) {
  double d0 = px - P->mu[0], d1 = py - P->mu[1], d2 = pz - P->mu[2];
  double l0 = d0 * P->Rwl[0] + d1 * P->Rwl[1] + d2 * P->Rwl[2];
  double l1 = d0 * P->Rwl[3] + d1 * P->Rwl[4] + d2 * P->Rwl[5];
  double l2 = d0 * P->Rwl[6] + d1 * P->Rwl[7] + d2 * P->Rwl[8];
  double ax = fabs(l0) / P->scale[0];
  double ay = fabs(l1) / P->scale[1];
  double az = fabs(l2) / P->scale[2];
  double f = pow(pow(ax, P->a) + pow(ay, P->a), P->b) + pow(az, P->c);
  return fmin(f, F_CAP);
}

/* ---- per-primitive preparation for a batch --------------------------- */

static int prep_batch(int F, int N, int C, const double* mu, const double* scale, const double* rot,
                      const double* opacity, const double* eps, const double* logits,
                      const int32_t* n_valid, const ogrid* g, const ocfg* cfg, oprim* P,
                      int64_t* bad_prim, int32_t* bad_bits) {
  int64_t first_bad = -1;
  int32_t first_bits = 0;
  for (int f = 0; f < F; ++f) {
    int nv = n_valid ? n_valid[f] : N;
    for (int i = 0; i < N; ++i) {
      int64_t gi = (int64_t)f * N + i;
      oprim* p = &P[gi];
      memset(p, 0, sizeof(*p));
      p->lo[0] = 1; p->hi[0] = 0;
      if (i >= nv) continue;
      int bad = prep_one(mu + 3 * gi, scale + 3 * gi, rot + 4 * gi, opacity[gi], eps + 2 * gi,
                         logits + (int64_t)C * gi, C, p);
      if (bad) {
        if (first_bad < 0) {
          first_bad = gi;
          first_bits = bad;
        }
        p->sigma = 0.0;
        continue;
      }
      window_of(p, g, cfg);
      p->live = is_live(p);
    }
  }
  if (bad_prim) *bad_prim = first_bad;
  if (bad_bits) *bad_bits = first_bits;
  return first_bad < 0 ? 0 : -4;
}

/* Per-primitive class weights: raw logits (logit-sum) or softmax (prob-sum,
 * SPEC.md:339,383). */
static void class_weights(const double* logits, int C, int prob_sum, double* out) {
  if (!prob_sum) {
    for (int k = 0; k < C; ++k) out[k] = logits[k];
    return;
  }
  double m = logits[0];
  for (int k = 1; k < C; ++k) m = fmax(m, logits[k]);
  double s = 0.0;
  for (int k = 0; k < C; ++k) {
    out[k] = exp(logits[k] - m);
    s += out[k];
  }
  for (int k = 0; k < C; ++k) out[k] /= s;
}

/* ---- exported entry points ------------------------------------------- */

/* Windows [F][N][6] and validation, no voxel work. */
int sqvo_prep(int F, int N, int C, const double* mu, const double* scale, const double* rot,
              const double* opacity, const double* eps, const double* logits,
              const int32_t* n_valid, const double* origin, const int32_t* dims, double res,
              double tau, int32_t radius, int32_t truncate, int32_t prob_sum, int32_t free_label,
              double extent, int32_t* windows, int64_t* bad_prim, int32_t* bad_bits) {
  ogrid g = {{origin[0], origin[1], origin[2]}, {dims[0], dims[1], dims[2]}, res};
  ocfg cfg = {tau, radius, truncate, prob_sum, free_label, extent};
  oprim* P = (oprim*)malloc(sizeof(oprim) * (size_t)F * (size_t)(N > 0 ? N : 1));
  int rc = prep_batch(F, N, C, mu, scale, rot, opacity, eps, logits, n_valid, &g, &cfg, P,
                      bad_prim, bad_bits);
  for (int64_t gi = 0; gi < (int64_t)F * N; ++gi) {
    const oprim* p = &P[gi];
    int32_t* w = windows + 6 * gi;
    if (p->live) {
      for (int k = 0; k < 3; ++k) {
        w[k] = p->lo[k];
        w[3 + k] = p->hi[k];
      }
    } else {
      w[0] = w[1] = w[2] = 1;
      w[3] = w[4] = w[5] = 0;
    }
  }
  free(P);
  return rc;
}

/* Bins: for every (frame, tile) the ascending list of frame-local ids of
 * live primitives whose window overlaps the tile.  tile_off has F*T+1
 * entries; prim_ids needs capacity >= entries (returns -6 otherwise and
 * still fills tile_off). */
int sqvo_bins(int F, int N, const int32_t* windows, const int32_t* dims, int32_t* tile_off,
              int32_t* prim_ids, int64_t capacity, int64_t* n_entries) {
  int ntx = (dims[0] + TX - 1) / TX, nty = (dims[1] + TY - 1) / TY, ntz = (dims[2] + TZ - 1) / TZ;
  int64_t T = (int64_t)ntx * nty * ntz;
  int64_t* cnt = (int64_t*)calloc((size_t)(F * T + 1), sizeof(int64_t));
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < N; ++i) {
      const int32_t* w = windows + 6 * ((int64_t)f * N + i);
      if (w[0] > w[3] || w[1] > w[4] || w[2] > w[5]) continue;
      for (int tz = w[2] / TZ; tz <= w[5] / TZ; ++tz)
        for (int ty = w[1] / TY; ty <= w[4] / TY; ++ty)
          for (int tx = w[0] / TX; tx <= w[3] / TX; ++tx)
            cnt[f * T + tx + (int64_t)ntx * (ty + (int64_t)nty * tz)]++;
    }
  int64_t run = 0;
  for (int64_t t = 0; t < F * T; ++t) {
    int64_t c = cnt[t];
    tile_off[t] = (int32_t)run;
    cnt[t] = run;
    run += c;
  }
  tile_off[F * T] = (int32_t)run;
  *n_entries = run;
  if (run > capacity) {
    free(cnt);
    return -6;
  }
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < N; ++i) {
      const int32_t* w = windows + 6 * ((int64_t)f * N + i);
      if (w[0] > w[3] || w[1] > w[4] || w[2] > w[5]) continue;
      for (int tz = w[2] / TZ; tz <= w[5] / TZ; ++tz)
        for (int ty = w[1] / TY; ty <= w[4] / TY; ++ty)
          for (int tx = w[0] / TX; tx <= w[3] / TX; ++tx)
            prim_ids[cnt[f * T + tx + (int64_t)ntx * (ty + (int64_t)nty * tz)]++] = i;
    }
  free(cnt);
  return 0;
}

/*
 * voxelize in FP64: for each primitive in ascending order
 * (sigma > 0, non-empty window), for each voxel centre p = origin +
 * (idx + 0.5)*res in the window: w = exp(-F(to_local(p))),
 * v_o += sigma*w, v_c += w*c.  Parallel over (frame, z-layer) slabs
 * (SPEC.md:385,389): every voxel accumulates in primitive order, so the
 * result is independent of the thread count.  Then finalize.
 * v_o [F][V], v_c [F][V][C] (nullable), labels [F][V] (u8, nullable).
 * Returns -4 on invalid primitive (outputs untouched), else 0.
 */
int sqvo_voxelize(int F, int N, int C, const double* mu, const double* scale, const double* rot,
                  const double* opacity, const double* eps, const double* logits,
                  const int32_t* n_valid, const double* origin, const int32_t* dims, double res,
                  double tau, int32_t radius, int32_t truncate, int32_t prob_sum,
                  int32_t free_label, double extent, double* v_o, double* v_c, uint8_t* labels,
                  int64_t* n_pairs, int64_t* bad_prim, int32_t* bad_bits) {
  ogrid g = {{origin[0], origin[1], origin[2]}, {dims[0], dims[1], dims[2]}, res};
  ocfg cfg = {tau, radius, truncate, prob_sum, free_label, extent};
  int64_t FN = (int64_t)F * N;
  oprim* P = (oprim*)malloc(sizeof(oprim) * (size_t)(FN > 0 ? FN : 1));
  int rc = prep_batch(F, N, C, mu, scale, rot, opacity, eps, logits, n_valid, &g, &cfg, P,
                      bad_prim, bad_bits);
  if (rc) {
    free(P);
    return rc;
  }
  double* cw = (double*)malloc(sizeof(double) * (size_t)(FN > 0 ? FN : 1) * (size_t)C);
  for (int64_t gi = 0; gi < FN; ++gi) class_weights(logits + C * gi, C, prob_sum, cw + C * gi);
  const int64_t nx = dims[0], ny = dims[1], nz = dims[2];
  const int64_t V = nx * ny * nz;
  int64_t pairs = 0;
  double* vo_buf = v_o;
  double* vo_own = NULL;
  if (!vo_buf) vo_buf = vo_own = (double*)malloc(sizeof(double) * (size_t)(F * V));
  double* vc_buf = v_c;
  double* vc_own = NULL;
  if (!vc_buf && labels) vc_buf = vc_own = (double*)malloc(sizeof(double) * (size_t)(F * V * C));
  memset(vo_buf, 0, sizeof(double) * (size_t)(F * V));
  if (vc_buf) memset(vc_buf, 0, sizeof(double) * (size_t)(F * V * C));

#pragma omp parallel for collapse(2) schedule(dynamic, 1) reduction(+ : pairs)
  for (int f = 0; f < F; ++f)
    for (int z = 0; z < (int)nz; ++z) {
      double* vo = vo_buf + f * V;
      double* vc = vc_buf ? vc_buf + f * V * C : NULL;
      for (int i = 0; i < N; ++i) {
        const oprim* p = &P[(int64_t)f * N + i];
        if (!p->live) continue;
        if (z < p->lo[2] || z > p->hi[2]) continue;
        const double* c = cw + C * ((int64_t)f * N + i);
        double pz = g.origin[2] + ((double)z + 0.5) * g.res;
        for (int y = p->lo[1]; y <= p->hi[1]; ++y) {
          double py = g.origin[1] + ((double)y + 0.5) * g.res;
          for (int x = p->lo[0]; x <= p->hi[0]; ++x) {
            double px = g.origin[0] + ((double)x + 0.5) * g.res;
            double w = exp(-field_F(p, px, py, pz));
            int64_t v = x + nx * (y + ny * (int64_t)z);
            vo[v] += p->sigma * w;
            if (vc) {
              double* o = vc + v * C;
              for (int k = 0; k < C; ++k) o[k] += w * c[k];
            }
            pairs++;
          }
        }
      }
    }
  if (n_pairs) *n_pairs = pairs;
  if (labels) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < F * V; ++v) {
      /* finalize: free if v_o < tau, else first argmax */
      if (vo_buf[v] < tau) {
        labels[v] = (uint8_t)free_label;
      } else {
        const double* o = vc_buf + v * C;
        int best = 0;
        for (int k = 1; k < C; ++k)
          if (o[k] > o[best]) best = k;
        labels[v] = (uint8_t)best;
      }
    }
  }
  free(vo_own);
  free(vc_own);
  free(cw);
  free(P);
  return 0;
}

/* finalize on FP64 dense grids. */
void sqvo_finalize(const double* v_o, const double* v_c, int64_t n, int C, double tau,
                   int32_t free_label, uint8_t* labels) {
  for (int64_t v = 0; v < n; ++v) {
    if (v_o[v] < tau) {
      labels[v] = (uint8_t)free_label;
    } else {
      int best = 0;
      for (int k = 1; k < C; ++k)
        if (v_c[v * C + k] > v_c[v * C + best]) best = k;
      labels[v] = (uint8_t)best;
    }
  }
}

/* Confusion counts ("confusion-matrix oracle"): row = gt,
 * column = pred, index C = free (any label >= C).  Accumulates. */
void sqvo_confusion(const uint8_t* pred, const uint8_t* gt, int64_t n, int C, int64_t* cm) {
  for (int64_t v = 0; v < n; ++v) {
    int p = pred[v] < C ? pred[v] : C;
    int t = gt[v] < C ? gt[v] : C;
    cm[t * (C + 1) + p]++;
  }
}

/* Point-wise F and density for primitive `prim` of a 1-frame batch
 * (core.py:254-282).  Returns validation bits of that primitive. */
int sqvo_density(int N, int C, const double* mu, const double* scale, const double* rot,
                 const double* opacity, const double* eps, const double* logits,
                 const double* points, const int32_t* pair_prim, int64_t n_points, double* F,
                 double* density) {
  oprim* P = (oprim*)malloc(sizeof(oprim) * (size_t)(N > 0 ? N : 1));
  int any_bad = 0;
  for (int i = 0; i < N; ++i) {
    memset(&P[i], 0, sizeof(oprim));
    any_bad |= prep_one(mu + 3 * i, scale + 3 * i, rot + 4 * i, opacity[i], eps + 2 * i,
                        logits + (int64_t)C * i, C, &P[i]);
  }
  if (!any_bad)
    for (int64_t k = 0; k < n_points; ++k) {
      const oprim* p = &P[pair_prim[k]];
      double f = field_F(p, points[3 * k], points[3 * k + 1], points[3 * k + 2]);
      F[k] = f;
      density[k] = exp(-f);
    }
  free(P);
  return any_bad;
}

/* ---- ray_iou ----------------------------------------
 * First occupied voxel (label < C) of a label grid [nz][ny][nx] (x-fastest,
 * SPEC.md:392) along O + t*D, t >= 0, by a 3D DDA (Amanatides-Woo): slab
 * entry into the grid box, start voxel by floor, then step the axis whose
 * next boundary is nearest (ties: lowest axis).  Boundary times are
 * recomputed from the lattice each step (no accumulated increments).  The
 * hit distance is the t at which the ray enters the voxel (0 when the origin
 * lies inside it).  FP64, no contraction: the device kernel evaluates the
 * same expressions in the same order. */
static int ray_first_hit(const uint8_t* lab, const int32_t* dims, const double* org, double res,
                         int C, const double* O, const double* D, double* d_out, int* c_out) {
  double t0 = 0.0, t1 = INFINITY;
  for (int a = 0; a < 3; ++a) {
    const double lo = org[a], hi = org[a] + (double)dims[a] * res;
    if (D[a] == 0.0) {
      if (!(O[a] >= lo && O[a] < hi)) return 0;
    } else {
      double ta = (lo - O[a]) / D[a], tb = (hi - O[a]) / D[a];
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
  for (int a = 0; a < 3; ++a) {
    const double p = O[a] + t0 * D[a];
    double f = floor((p - org[a]) / res);
    if (f < 0.0) f = 0.0;
    if (f > (double)(dims[a] - 1)) f = (double)(dims[a] - 1);
    i[a] = (int)f;
    step[a] = D[a] > 0.0 ? 1 : (D[a] < 0.0 ? -1 : 0);
    tmax[a] = step[a] == 0 ? INFINITY
                           : (org[a] + (double)(i[a] + (step[a] > 0)) * res - O[a]) / D[a];
  }
  double t = t0;
  for (;;) {
    const uint8_t l = lab[i[0] + (int64_t)dims[0] * (i[1] + (int64_t)dims[1] * i[2])];
    if (l < C) {
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
    if (i[a] < 0 || i[a] >= dims[a]) return 0;
    tmax[a] = (org[a] + (double)(i[a] + (step[a] > 0)) * res - O[a]) / D[a];
  }
}

/* Per-ray hits of pred and gt for F frames x R rays (frame-major outputs,
 * class -1 = no hit) and the matching counts of SPEC.md:519-521 per
 * threshold: counts[k][0..2] += TP, FP, FN.  A ray with both hits that fail
 * to match (class or |d_pred - d_gt| > thr) is one FP and one FN. */
void sqvo_ray_iou(int F, const uint8_t* pred, const uint8_t* gt, const int32_t* dims,
                  const double* org, double res, int C, int64_t R, const double* origins,
                  const double* dirs, int n_thr, const double* thr, int64_t* counts,
                  double* d_pred, int32_t* c_pred, double* d_gt, int32_t* c_gt) {
  const int64_t V = (int64_t)dims[0] * dims[1] * dims[2];
  for (int f = 0; f < F; ++f)
    for (int64_t r = 0; r < R; ++r) {
      double dp = 0.0, dg = 0.0;
      int cp = -1, cg = -1;
      const int hp = ray_first_hit(pred + f * V, dims, org, res, C, origins + 3 * r, dirs + 3 * r,
                                   &dp, &cp);
      const int hg = ray_first_hit(gt + f * V, dims, org, res, C, origins + 3 * r, dirs + 3 * r,
                                   &dg, &cg);
      const int64_t k = (int64_t)f * R + r;
      if (d_pred) {
        d_pred[k] = hp ? dp : -1.0;
        c_pred[k] = hp ? cp : -1;
        d_gt[k] = hg ? dg : -1.0;
        c_gt[k] = hg ? cg : -1;
      }
      for (int j = 0; j < n_thr; ++j) {
        int64_t* c = counts + 3 * j;
        if (hp && hg) {
          if (cp == cg && fabs(dp - dg) <= thr[j])
            c[0]++;
          else {
            c[1]++;
            c[2]++;
          }
        } else if (hp) {
          c[1]++;
        } else if (hg) {
          c[2]++;
        }
      }
    }
}
