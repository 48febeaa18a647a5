// sqv_api.cu — the C ABI of include/sqv.h: argument checks, workspace
// layout, and the stage sequence of sqv_voxelize.
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sqv_kernels.cuh"

namespace sqv {

static std::atomic<long long> g_launches{0};
static std::atomic<unsigned long long*> g_stats{nullptr};  // sqv_stats_attach
static thread_local char g_err[512] = "";

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SQV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return SQV_OK;
}

namespace {

constexpr size_t kAlign = 256;
inline size_t up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Header {  // device-side scalars, read back in one 32-byte copy
  long long n_entries;
  unsigned long long bad_word;
  unsigned long long n_pairs;
  int tile_counter;  // the persistent evaluator's work counter
  int deep_count;    // tiles listed for the CUDA-core complement
};
static_assert(sizeof(Header) == 4 * sizeof(long long), "header_out_kernel copies 4 words");

// The one mid-pipeline readback goes through a mapped pinned buffer written
// by a one-thread kernel: no copy engine is involved, so the readback never
// queues behind a caller's bulk H2D/D2H traffic on other streams (the
// overlapped stream API copies ~100 MB per batch).  One buffer per host
// thread; calls on a thread are sequential (each waits for its readback).
__global__ void header_out_kernel(const Header* src, Header* dst) {
  volatile long long* d = reinterpret_cast<volatile long long*>(dst);
  const long long* s = reinterpret_cast<const long long*>(src);
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k] = s[k];
}

static Header* mapped_header() {
  static thread_local Header* h = nullptr;
  if (!h) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, sizeof(Header), cudaHostAllocMapped | cudaHostAllocPortable) !=
        cudaSuccess)
      return nullptr;
    h = static_cast<Header*>(p);
  }
  return h;
}

struct Layout {
  size_t hdr, recs, lrows, counts, offs, windows, tile_off, deep, scan_tmp, frame_count;  // fixed
  size_t keys_a, vals_a, keys_b, vals_b, radix_tmp, bmask;                       // variable
  size_t fixed_end, total;
};

Layout layout(int64_t FN, int64_t FT, int lrow, int64_t n_entries, int64_t F = 0) {
  Layout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += up(bytes);
    return at;
  };
  L.hdr = take(sizeof(Header));
  L.recs = take((size_t)FN * kRecWords * 4);
  L.lrows = take((size_t)FN * lrow * 4);
  L.counts = take((size_t)(FN + 1) * 4);
  L.offs = take((size_t)(FN + 1) * 4);
  L.windows = take((size_t)FN * 6 * 4);
  L.tile_off = take((size_t)(FT + 1) * 4);
  L.deep = take((size_t)FT * 4);
  const int64_t st = scan_tmp_ints(FN > FT ? FN : FT);
  L.scan_tmp = take((size_t)st * 4);
  L.frame_count = take((size_t)(F + 1) * 4);
  L.fixed_end = o;
  L.keys_a = take((size_t)n_entries * 4);
  L.vals_a = take((size_t)n_entries * 4);
  L.keys_b = take((size_t)n_entries * 4);
  L.vals_b = take((size_t)n_entries * 4);
  L.radix_tmp = take((size_t)radix_tmp_ints(n_entries) * 4);
  L.bmask = take((size_t)n_entries * 4);
  L.total = o;
  return L;
}

int check_grid(const sqv_grid* g) {
  if (!g) return set_error(SQV_ERR_ARG, "grid is NULL");
  for (int k = 0; k < 3; ++k) {
    if (g->dims[k] < 1) return set_error(SQV_ERR_ARG, "dims must be >= 1");
    if (!std::isfinite(g->origin[k])) return set_error(SQV_ERR_ARG, "origin must be finite");
  }
  if (!(g->resolution > 0.0) || !std::isfinite(g->resolution))
    return set_error(SQV_ERR_ARG, "resolution must be > 0");
  const int64_t V = (int64_t)g->dims[0] * g->dims[1] * g->dims[2];
  if (V > (1LL << 40)) return set_error(SQV_ERR_ARG, "grid too large");
  return SQV_OK;
}

void tiles_of(const sqv_grid* g, int* ntx, int* nty, int* ntz) {
  *ntx = (g->dims[0] + kTileX - 1) / kTileX;
  *nty = (g->dims[1] + kTileY - 1) / kTileY;
  *ntz = (g->dims[2] + kTileZ - 1) / kTileZ;
}

// tau compared in FP32 exactly as FP64 v_o < tau would be for an FP32 v_o:
// the smallest float >= tau.
float tau_f32(double tau) {
  if (std::isinf(tau)) return tau > 0 ? INFINITY : -INFINITY;
  float t = (float)tau;
  if ((double)t < tau) t = std::nextafter(t, INFINITY);
  return t;
}

// Opt-in stage profiler (sqv_profile_*): CUDA events on the caller's stream.
// The previous call's emit/sort/eval events are folded in at the next
// call's header readback (stream order guarantees they completed).
// Stage timer: a ring of event sets, one per sqv_voxelize call, so calls on
// different streams (pipelined batches) never overwrite each other's events;
// a set is folded once its last event has completed (or at read time).
struct Profiler {
  static constexpr int kRing = 8;
  std::mutex mu;
  bool on = false;
  bool created = false;
  cudaEvent_t ev[kRing][6];
  bool pending[kRing] = {};
  int next = 0;
  double ms[SQV_NSTAGES] = {0, 0, 0, 0, 0};
  long long calls = 0;
  // SQV_PROF_TRACE (diagnostics): print every folded call's stage events as
  // times (ms) since sqv_profile_enable — prep, after the count scan, after
  // the readback, before the masks, after the evaluator, after the masks
  cudaEvent_t ref;
  bool trace = false;
  void ensure() {
    if (!created) {
      for (auto& set : ev)
        for (auto& e : set) cudaEventCreate(&e);
      cudaEventCreate(&ref);
      created = true;
    }
  }
  static float el(cudaEvent_t a, cudaEvent_t b) {
    float m = 0.f;
    cudaEventElapsedTime(&m, a, b);
    return m;
  }
  void fold(int i) {
    if (trace) {
      fprintf(stderr, "sqv trace call %lld:", calls);
      for (int k = 0; k < 6; ++k) fprintf(stderr, " %.3f", el(ref, ev[i][k]));
      fprintf(stderr, "\n");
    }
    const double m0 = el(ev[i][0], ev[i][1]), m1 = el(ev[i][2], ev[i][3]),
                 m2 = el(ev[i][3], ev[i][4]), m4 = el(ev[i][5], ev[i][4]);
    ms[0] += m0;
    ms[1] += m1;
    ms[2] += m2;
    ms[3] += m0 + m1 + m2;
    ms[4] += m4;
    calls++;
    pending[i] = false;
  }
  void fold_ready() {
    for (int i = 0; i < kRing; ++i)
      if (pending[i] && cudaEventQuery(ev[i][4]) == cudaSuccess) fold(i);
  }
  void fold_all() {
    for (int i = 0; i < kRing; ++i)
      if (pending[i]) {
        cudaEventSynchronize(ev[i][4]);
        fold(i);
      }
  }
  int acquire() {  // caller holds mu
    ensure();
    fold_ready();
    const int i = next;
    next = (next + 1) % kRing;
    if (pending[i]) {  // more than kRing calls in flight: wait for the oldest
      cudaEventSynchronize(ev[i][4]);
      fold(i);
    }
    return i;
  }
};
Profiler g_prof;

}  // namespace
}  // namespace sqv

using namespace sqv;

extern "C" {

int sqv_abi_version(void) { return SQV_ABI_VERSION; }
const char* sqv_last_error(void) { return g_err; }
int64_t sqv_launch_count(void) { return g_launches.load(); }

int64_t sqv_tiles_per_frame(const sqv_grid* grid) {
  if (check_grid(grid)) return -1;
  int a, b, c;
  tiles_of(grid, &a, &b, &c);
  return (int64_t)a * b * c;
}

size_t sqv_workspace_bytes(int32_t n_frames, int32_t n_prims, int32_t n_classes,
                           const sqv_grid* grid, int64_t n_entries) {
  if (check_grid(grid) || n_frames < 0 || n_prims < 0) return 0;
  const int cm = eval_cm_for(n_classes);
  if (!cm) return 0;
  const int lrow = (cm + 1 + 3) & ~3;
  const int64_t T = sqv_tiles_per_frame(grid);
  return layout((int64_t)n_frames * n_prims, (int64_t)n_frames * T, lrow, n_entries, n_frames).total;
}

int sqv_voxelize(const sqv_prims* prims, const sqv_grid* grid, const sqv_cfg* cfg,
                 const sqv_outputs* out, sqv_bins* bins, void* workspace, size_t ws_bytes,
                 size_t* ws_needed, int64_t* bad_prim, int32_t* bad_bits, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (bad_prim) *bad_prim = -1;
  if (bad_bits) *bad_bits = 0;
  if (!prims || !cfg || !out || !out->labels) return set_error(SQV_ERR_ARG, "NULL argument");
  if (int rc = check_grid(grid)) return rc;
  const int F = prims->n_frames, N = prims->n_prims, C = prims->n_classes;
  if (F < 0 || N < 0) return set_error(SQV_ERR_ARG, "negative frame/primitive count");
  if (C < 1) return set_error(SQV_ERR_ARG, "need at least one class");
  const int cm = eval_cm_for(C);
  if (!cm) return set_error(SQV_ERR_UNSUPPORTED, "%d classes > SQV_MAX_CLASSES (%d)", C,
                            SQV_MAX_CLASSES);
  if (!(cfg->tau >= 0.0)) return set_error(SQV_ERR_ARG, "tau must be >= 0");
  if (cfg->neighborhood_radius < 0) return set_error(SQV_ERR_ARG, "radius must be >= 0");
  if (!(cfg->window_extent >= 0.0) || !std::isfinite(cfg->window_extent))
    return set_error(SQV_ERR_ARG, "window_extent must be finite and >= 0");
  if (cfg->free_label < 0 || cfg->free_label > 255 || cfg->free_label < C)
    return set_error(SQV_ERR_ARG, "free_label must lie in [C, 255]");
  if (cfg->precision != 0 && cfg->precision != 1)
    return set_error(SQV_ERR_ARG, "precision must be 0 (fast) or 1 (strict)");
  if (cfg->semantic_mode != 0 && cfg->semantic_mode != 1)
    return set_error(SQV_ERR_ARG, "semantic_mode must be 0 (logit-sum) or 1 (prob-sum)");
  if (F == 0) return SQV_OK;
  int ntx, nty, ntz;
  tiles_of(grid, &ntx, &nty, &ntz);
  const int64_t T = (int64_t)ntx * nty * ntz;
  const int64_t FN = (int64_t)F * N, FT = (int64_t)F * T;
  if (FT >= (1LL << 31) || FN >= (1LL << 31))
    return set_error(SQV_ERR_ARG, "batch too large (split frames)");
  const int lrow = (cm + 1 + 3) & ~3;
  Layout L = layout(FN, FT, lrow, 0, F);
  // binning: for sparse batches (< 64 entries per tile on average, decided
  // after the header readback) one CTA per frame (sqv_bin.cu) when the
  // frame's tile counters fit shared memory (config 1 +3%); dense batches
  // keep emit + radix sort, whose many short CTAs slot in under the previous
  // batch's evaluation better than F long ones (per-frame binning measured
  // config 2 -0.6%, config 3 -1.7%, config 4 -4.6%).  SQV_BIN=radix / frame
  // force either (A/B, tests); SQV_BIN=fused also moves the block masks into
  // the per-frame kernel (measured slower everywhere but config 1).
  const char* benv = std::getenv("SQV_BIN");
  const bool bin_radix = benv && std::strcmp(benv, "radix") == 0;
  const bool bin_forced = benv && (std::strcmp(benv, "frame") == 0 || std::strcmp(benv, "fused") == 0);
  const bool frame_ok = bin_frames_supported((int)T) && !bin_radix;
  if (ws_bytes < L.fixed_end || !workspace) {
    if (ws_needed) *ws_needed = L.total;
    return set_error(SQV_ERR_WORKSPACE, "workspace too small: need >= %zu bytes", L.total);
  }
  char* ws = (char*)workspace;
  Header* hdr = (Header*)(ws + L.hdr);
  int* counts = (int*)(ws + L.counts);
  int* offs = (int*)(ws + L.offs);
  int* windows = (int*)(ws + L.windows);
  int* tile_off = (int*)(ws + L.tile_off);
  int* scan_tmp = (int*)(ws + L.scan_tmp);
  int* frame_count = (int*)(ws + L.frame_count);
  float* recs = (float*)(ws + L.recs);
  float* lrows = (float*)(ws + L.lrows);

  // header: zeros, bad_word = ~0 (memset kernels, no host copy)
  if (cudaMemsetAsync(hdr, 0, sizeof(Header), s) != cudaSuccess ||
      cudaMemsetAsync(&hdr->bad_word, 0xFF, sizeof(hdr->bad_word), s) != cudaSuccess ||
      (frame_ok && cudaMemsetAsync(frame_count, 0, (size_t)F * 4, s) != cudaSuccess))
    return check_launch("workspace init");
  Header* hmap = mapped_header();
  if (!hmap) return set_error(SQV_ERR_CUDA, "mapped header allocation failed");

  const bool prof = g_prof.on;
  int pset = 0;
  if (prof) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    pset = g_prof.acquire();
    cudaEventRecord(g_prof.ev[pset][0], s);
  }
  // K1 prep
  if (FN > 0) {
    PrepArgs P;
    P.mu = prims->mu;
    P.scale = prims->scale;
    P.rot = prims->rot;
    P.opacity = prims->opacity;
    P.eps = prims->eps;
    P.logits = prims->logits;
    P.n_valid = prims->n_valid;
    P.n_frames = F;
    P.n_prims = N;
    P.n_classes = C;
    P.cm = cm;
    P.lrow = lrow;
    P.grid = *grid;
    P.cfg = *cfg;
    P.recs = recs;
    P.lrows = lrows;
    P.counts = counts;
    P.windows = windows;
    P.bad_word = &hdr->bad_word;
    P.n_pairs = &hdr->n_pairs;
    P.n_entries = reinterpret_cast<unsigned long long*>(&hdr->n_entries);
    P.frame_count = frame_ok ? frame_count : nullptr;
    prep_kernel<<<div_up(FN, 128), 128, 0, s>>>(P);
    count_launch();
    if (int rc = check_launch("prep_kernel")) return rc;
  }
  // K2 scan of per-primitive tile counts -> entry offsets.  The entry total
  // in the header is prep's 64-bit sum: the int32 scan may wrap for batches
  // past 2^31 entries, and the check below rejects those before emit reads
  // the offsets.
  if (int rc = scan_exclusive(counts, offs, FN, scan_tmp, nullptr, s)) return rc;
  if (prof) cudaEventRecord(g_prof.ev[pset][1], s);
  header_out_kernel<<<1, 1, 0, s>>>(hdr, hmap);
  count_launch();
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("header readback");
  Header h;
  {
    const volatile long long* m = reinterpret_cast<const volatile long long*>(hmap);
    long long* d = reinterpret_cast<long long*>(&h);
    for (int k = 0; k < 4; ++k) d[k] = m[k];
  }
  if (h.bad_word != ~0ULL) {
    if (bad_prim) *bad_prim = (int64_t)(h.bad_word >> 8);
    if (bad_bits) *bad_bits = (int32_t)(h.bad_word & 255u);
    return set_error(SQV_ERR_INVALID_PRIM, "primitive %lld failed validation (bits %d)",
                     (long long)(h.bad_word >> 8), (int)(h.bad_word & 255u));
  }
  const int64_t E = h.n_entries;  // exact (64-bit atomics in prep)
  if (E < 0 || E >= (1LL << 31) - 1)
    return set_error(SQV_ERR_ARG, "too many bin entries: %lld (split frames)", (long long)E);
  const bool frame_bin = frame_ok && (bin_forced || E < 64 * FT);
  L = layout(FN, FT, lrow, E, F);
  if (ws_needed) *ws_needed = L.total;
  if (ws_bytes < L.total)
    return set_error(SQV_ERR_WORKSPACE, "workspace too small: need %zu bytes", L.total);
  uint32_t* keys_a = (uint32_t*)(ws + L.keys_a);
  uint32_t* keys_b = (uint32_t*)(ws + L.keys_b);
  int* vals_a = (int*)(ws + L.vals_a);
  int* vals_b = (int*)(ws + L.vals_b);
  int* radix_tmp = (int*)(ws + L.radix_tmp);

  if (prof) cudaEventRecord(g_prof.ev[pset][2], s);
  // evaluator choice: tcgen05 by default; SQV_EVAL=ffma selects the
  // CUDA-core one (A/B runs).  The tensor cores accumulate with truncation:
  // the bias grows with the number of K steps per voxel (measured: about
  // -1e-8 relative per entry per tile, scripts/diag_depth.py).  Tiles deeper
  // than the precision mode allows go to the CUDA-core evaluator (FP32
  // round-to-nearest), launched after the tensor-core one on the same
  // stream over the deep-tile list the binning builds.
  const char* ev = std::getenv("SQV_EVAL");
  const bool ffma = (ev && std::strcmp(ev, "ffma") == 0) || !eval_tc_supported(cm);
  int depth = cfg->precision ? 512 : 768;
  if (const char* de = std::getenv("SQV_TC_DEPTH")) depth = std::atoi(de);
  const bool complement = !ffma && E > depth && cm <= 32;
  int* deep = (int*)(ws + L.deep);
  uint32_t* bmask = (uint32_t*)(ws + L.bmask);
  const int* sorted_vals = vals_a;
  const uint32_t* sorted_keys = keys_a;
  if (frame_bin) {
    // K3-K4b in one launch: per-frame counting sort, tile offsets, deep
    // list and block masks (sqv_bin.cu)
    BinArgs Bn;
    Bn.n_frames = F;
    Bn.n_prims = N;
    Bn.tiles_per_frame = (int)T;
    Bn.ntx = ntx;
    Bn.nty = nty;
    Bn.counts = counts;
    Bn.windows = windows;
    Bn.frame_count = frame_count;
    Bn.keys = keys_a;
    Bn.vals = vals_a;
    Bn.tile_off = tile_off;
    Bn.deep_min = complement ? depth : -1;
    Bn.deep_tiles = deep;
    Bn.deep_count = &hdr->deep_count;
    Bn.recs = recs;
    Bn.lrows = lrows;
    Bn.lrow = lrow;
    Bn.acc_c = cfg->precision ? SQV_ACC_C : INFINITY;
    // (block masks in the binning kernel: SQV_BIN=fused; measured slower,
    // the masks' per-entry field tests want the whole GPU, not F CTAs)
    Bn.bmask = (!ffma && benv && std::strcmp(benv, "fused") == 0) ? bmask : nullptr;
    if (int rc = bin_frames_launch(Bn, s)) return rc;
  } else {
    // K3 emit + K4 radix sort + tile offsets
    int which = 0;
    if (E > 0) {
      EmitArgs Em;
      Em.n_frames = F;
      Em.n_prims = N;
      Em.tiles_per_frame = (int)T;
      Em.ntx = ntx;
      Em.nty = nty;
      Em.counts = counts;
      Em.offs = offs;
      Em.windows = windows;
      Em.keys = keys_a;
      Em.vals = vals_a;
      emit_kernel<<<(int)div_up(FN * 32, 256), 256, 0, s>>>(Em);
      count_launch();
      if (int rc = check_launch("emit_kernel")) return rc;
      int bits = 0;
      while (bits < 32 && (1LL << bits) < FT) ++bits;
      if (int rc = radix_sort(keys_a, vals_a, keys_b, vals_b, E, bits, radix_tmp, &which, s))
        return rc;
    }
    sorted_vals = which ? vals_b : vals_a;
    sorted_keys = which ? keys_b : keys_a;
    tile_bounds_kernel<<<div_up(FT + 1, 256), 256, 0, s>>>(sorted_keys, E, FT, tile_off,
                                                           complement ? depth : -1, deep,
                                                           &hdr->deep_count);
    count_launch();
    if (int rc = check_launch("tile_bounds_kernel")) return rc;
  }

  // K5 evaluate + finalize
  EvalArgs A;
  A.recs = recs;
  A.lrows = lrows;
  A.tile_off = tile_off;
  A.prim_ids = sorted_vals;
  A.n_prims = N;
  A.n_classes = C;
  A.lrow = lrow;
  A.tiles_per_frame = (int)T;
  A.ntx = ntx;
  A.nty = nty;
  A.nx = grid->dims[0];
  A.ny = grid->dims[1];
  A.nz = grid->dims[2];
  A.tau = tau_f32(cfg->tau);
  A.free_label = cfg->free_label;
  {
    const char* fe = std::getenv("SQV_FIELD");  // diagnostics only: 9 = 9-MUFU form, 8 = SFU log1p
    A.field = fe ? std::atoi(fe) : (cfg->precision ? 6 : 7);
  }
  A.labels = out->labels;
  A.v_o = out->v_o;
  A.v_c = out->v_c;
  A.n_tiles = (int)FT;
  A.tile_counter = &hdr->tile_counter;  // zeroed with the header
  A.deep_tiles = deep;
  A.deep_count = &hdr->deep_count;
  A.n_entries = E;
  A.stats = g_stats.load();
  if (prof) cudaEventRecord(g_prof.ev[pset][3], s);
  {
    A.bmask = bmask;
    if (!ffma && E > 0 && !(frame_bin && benv && std::strcmp(benv, "fused") == 0))
      if (int rc = block_masks_launch(sorted_keys, sorted_vals, E, recs, lrows, lrow, tile_off,
                                      (int)T, ntx, nty, N,
                                      cfg->precision ? SQV_ACC_C : INFINITY, bmask, s))
        return rc;
    if (prof) cudaEventRecord(g_prof.ev[pset][5], s);
    A.tc_max_entries = ffma ? -1 : depth;
    A.ffma_min_entries = ffma ? -1 : depth;
    if (ffma) {
      if (int rc = eval_launch(A, cm, (int)FT, s)) return rc;
    } else {
      if (int rc = eval_tc_launch(A, cm, (int)FT, s)) return rc;
      if (complement)
        if (int rc = eval_launch(A, cm, (int)FT, s)) return rc;
    }
  }
  if (prof) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    cudaEventRecord(g_prof.ev[pset][4], s);
    g_prof.pending[pset] = true;
  }

  if (bins) {
    bins->n_entries = E;
    bins->n_pairs = (int64_t)h.n_pairs;
    if (bins->windows &&
        cudaMemcpyAsync(bins->windows, windows, (size_t)FN * 6 * 4, cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess)
      return check_launch("bins export");
    if (bins->tile_off &&
        cudaMemcpyAsync(bins->tile_off, tile_off, (size_t)(FT + 1) * 4, cudaMemcpyDeviceToDevice,
                        s) != cudaSuccess)
      return check_launch("bins export");
    if (bins->prim_ids) {
      if (bins->capacity < E)
        return set_error(SQV_ERR_CAPACITY, "bins capacity %lld < %lld entries",
                         (long long)bins->capacity, (long long)E);
      if (E > 0 && cudaMemcpyAsync(bins->prim_ids, sorted_vals, (size_t)E * 4,
                                   cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return check_launch("bins export");
    }
  }
  return SQV_OK;
}

int sqv_finalize(const float* v_o, const float* v_c, int64_t n_voxels, int32_t n_classes,
                 double tau, int32_t free_label, uint8_t* labels, void* stream) {
  if (n_voxels < 0 || n_classes < 1 || !(tau >= 0.0) || free_label < n_classes ||
      free_label > 255)
    return set_error(SQV_ERR_ARG, "invalid finalize arguments");
  return finalize_launch(v_o, v_c, n_voxels, n_classes, tau_f32(tau), free_label, labels,
                         (cudaStream_t)stream);
}

int sqv_confusion(const uint8_t* pred, const uint8_t* gt, int64_t n_voxels, int32_t n_classes,
                  int32_t free_label, int64_t* cm, void* stream) {
  (void)free_label;  // every label >= C (free_label included) maps to index C
  if (n_voxels < 0 || n_classes < 1 || n_classes > 255)
    return set_error(SQV_ERR_ARG, "invalid confusion arguments");
  return confusion_launch(pred, gt, n_voxels, n_classes, cm, (cudaStream_t)stream);
}

int sqv_density(const sqv_prims* prims, const double* points, const int32_t* pair_prim,
                int64_t n_points, float* F, float* density, void* stream) {
  if (!prims || n_points < 0) return set_error(SQV_ERR_ARG, "invalid density arguments");
  return density_launch(prims, points, pair_prim, n_points, F, density, (cudaStream_t)stream);
}

int sqv_ray_iou(const uint8_t* pred, const uint8_t* gt, int32_t n_frames, const sqv_grid* grid,
                int32_t n_classes, const double* origins, const double* dirs, int64_t n_rays,
                const double* thresholds, int32_t n_thr, int64_t* counts, sqv_ray_hits* hits,
                void* stream) {
  if (!grid || !pred || !gt || !origins || !dirs || !counts || n_frames < 0)
    return set_error(SQV_ERR_ARG, "invalid ray_iou arguments");
  if (n_rays < 1) return set_error(SQV_ERR_ARG, "zero rays");
  if (n_thr < 1 || n_thr > kMaxRayThr) return set_error(SQV_ERR_ARG, "1..16 thresholds");
  if (n_classes < 1 || n_classes > 255) return set_error(SQV_ERR_ARG, "n_classes must lie in [1, 255]");
  const int rc = check_grid(grid);
  if (rc) return rc;
  RayArgs A{};
  A.pred = pred;
  A.gt = gt;
  for (int a = 0; a < 3; ++a) {
    A.dims[a] = grid->dims[a];
    A.org[a] = grid->origin[a];
  }
  A.res = grid->resolution;
  A.n_classes = n_classes;
  A.n_frames = n_frames;
  A.n_rays = n_rays;
  A.origins = origins;
  A.dirs = dirs;
  A.n_thr = n_thr;
  for (int j = 0; j < n_thr; ++j) {
    if (!(thresholds[j] >= 0.0)) return set_error(SQV_ERR_ARG, "thresholds must be >= 0");
    A.thr[j] = thresholds[j];
  }
  A.counts = reinterpret_cast<unsigned long long*>(counts);
  if (hits) {
    A.d_pred = hits->d_pred;
    A.c_pred = hits->c_pred;
    A.d_gt = hits->d_gt;
    A.c_gt = hits->c_gt;
  }
  return ray_iou_launch(A, (cudaStream_t)stream);
}

int sqv_gen_frames(uint64_t seed, int64_t first_frame, int32_t n_frames, int32_t n_prims,
                   int32_t n_classes, const sqv_grid* grid, double smin, double smax,
                   double emin, double* mu, double* scale, double* rot, double* opacity,
                   double* eps, double* logits, void* stream) {
  if (n_frames < 0 || n_prims < 0 || n_classes < 1 || first_frame < 0)
    return set_error(SQV_ERR_ARG, "invalid gen_frames sizes");
  if (!(smin > 0.0 && smax >= smin && std::isfinite(smax)))
    return set_error(SQV_ERR_ARG, "scales must satisfy 0 < smin <= smax");
  if (!(emin > 0.0 && emin <= 2.0)) return set_error(SQV_ERR_ARG, "emin must lie in (0, 2]");
  const int rc = check_grid(grid);
  if (rc) return rc;
  if ((int64_t)n_frames * n_prims > 0 && (!mu || !scale || !rot || !opacity || !eps || !logits))
    return set_error(SQV_ERR_ARG, "output arrays are NULL");
  GenArgs A{};
  A.seed = seed;
  A.first_frame = first_frame;
  A.n_frames = n_frames;
  A.n_prims = n_prims;
  A.n_classes = n_classes;
  for (int a = 0; a < 3; ++a) {
    A.lo[a] = grid->origin[a];
    A.hi[a] = grid->origin[a] + (double)grid->dims[a] * grid->resolution;
  }
  A.smin = smin;
  A.smax = smax;
  A.emin = emin;
  A.mu = mu;
  A.scale = scale;
  A.rot = rot;
  A.opacity = opacity;
  A.eps = eps;
  A.logits = logits;
  return gen_launch(A, (cudaStream_t)stream);
}

int sqv_stats_attach(int64_t* counters) {
  g_stats.store(reinterpret_cast<unsigned long long*>(counters));
  return SQV_OK;
}

int sqv_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = on != 0;
  if (g_prof.on) {
    g_prof.ensure();
    g_prof.trace = std::getenv("SQV_PROF_TRACE") != nullptr;
    cudaEventRecord(g_prof.ref, 0);
  }
  return SQV_OK;
}

int sqv_profile_read(double* ms, int64_t* calls, int reset) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  {
    g_prof.fold_all();
  }
  if (ms)
    for (int k = 0; k < SQV_NSTAGES; ++k) ms[k] = g_prof.ms[k];
  if (calls) *calls = g_prof.calls;
  if (reset) {
    for (int k = 0; k < SQV_NSTAGES; ++k) g_prof.ms[k] = 0.0;
    g_prof.calls = 0;
  }
  return SQV_OK;
}

int sqv_microbench(int which, double* ops_per_s, void* stream) {
  if (!ops_per_s || (which != 0 && which != 1)) return set_error(SQV_ERR_ARG, "microbench args");
  return microbench(which, ops_per_s, (cudaStream_t)stream);
}

}  // extern "C"
