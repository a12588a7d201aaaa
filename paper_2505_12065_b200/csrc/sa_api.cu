// sa_api.cu -- the C ABI (include/sa.h): validation, index object, search planner,
// NCCL plumbing and kernel accounting.  Every step of the path runs in this
// library's kernels; there is no host or library fallback.
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels/flat_scan.cuh"
#include "kernels/merge.cuh"
#include "kernels/score_gemm.cuh"

// ====================================================================== errors
static thread_local std::string g_last_error;

namespace sa {

sa_status set_error(sa_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

sa_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SA_OK;
  if (e == cudaErrorMemoryAllocation)
    return set_error(SA_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  return set_error(SA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ====================================================================== TMA
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

sa_status make_tmap_bf16(CUtensorMap* m, const void* base, int64_t rows, int32_t cols,
                         int32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return set_error(SA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(SA_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return SA_OK;
}

// ====================================================================== profiler
// Kernel accounting: every launch site calls note_launch() (kernels/launch.cuh); the launch is
// counted under the kind of the calling thread's OUTERMOST open ProfRegion (OTHER outside any
// region), and each outermost region is timed with a pair of CUDA events on its stream.  So a
// kind's launches and its time always cover the same kernels (inner regions are absorbed).
namespace {
struct Prof {
  std::mutex mu;
  bool on = false;
  int64_t launches[SA_KERNEL_KINDS] = {};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[SA_KERNEL_KINDS];
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
Prof g_prof;
thread_local int t_depth = 0;            // open regions on this thread
thread_local int t_kind = SA_KERNEL_OTHER;   // kind of the outermost one
thread_local bool t_capturing = false;   // inside a graph capture: no events; tally launches
thread_local int64_t t_tally[SA_KERNEL_KINDS];
}  // namespace

void set_capturing(bool on) {
  t_capturing = on;
  if (on)
    for (int i = 0; i < SA_KERNEL_KINDS; ++i) t_tally[i] = 0;
}
void capture_tally(int64_t out[SA_KERNEL_KINDS]) {
  for (int i = 0; i < SA_KERNEL_KINDS; ++i) out[i] = t_tally[i];
}
void prof_add_launches(const int64_t counts[SA_KERNEL_KINDS]) {
  std::lock_guard<std::mutex> l(g_prof.mu);
  for (int i = 0; i < SA_KERNEL_KINDS; ++i) g_prof.launches[i] += counts[i];
}

void note_launch() {
  const int kind = t_depth > 0 ? t_kind : SA_KERNEL_OTHER;
  if (t_capturing) {
    ++t_tally[kind];
    return;
  }
  std::lock_guard<std::mutex> l(g_prof.mu);
  g_prof.launches[kind]++;
}

ProfRegion::ProfRegion(int kind, cudaStream_t s) : owner_(t_depth++ == 0), s_(s) {
  if (!owner_) return;
  t_kind = kind;
  if (t_capturing) return;
  std::lock_guard<std::mutex> l(g_prof.mu);
  if (!g_prof.on) return;
  begin_ = g_prof.get();
  cudaEventRecord(begin_, s);
}

ProfRegion::~ProfRegion() {
  --t_depth;
  if (!owner_ || !begin_) return;
  std::lock_guard<std::mutex> l(g_prof.mu);
  cudaEvent_t e = g_prof.get();
  cudaEventRecord(e, s_);
  g_prof.ev[t_kind].push_back({begin_, e});
}

// Raise a kernel's dynamic shared-memory limit once per (device, kernel); thread-safe.
cudaError_t ensure_max_smem(const void* func, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, size_t>> done;
  std::lock_guard<std::mutex> l(mu);
  for (auto& d : done)
    if (d.first.first == dev && d.first.second == func) {
      if (d.second >= bytes) return cudaSuccess;
      e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e == cudaSuccess) d.second = bytes;
      return e;
    }
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.push_back({{dev, func}, bytes});
  return e;
}

// ====================================================================== tuning switches
// Timing experiments (SA_EXPERIMENT skips score processing -- invalid results; SA_NO_SEED,
// SA_SEED_ROWS, SA_SEED_RECURSE, SA_LOCKSTEP_LAG change the schedule) are read only by a
// library built with -DSA_TUNING_BUILD (build.py --tuning, written to libsa_tuning.so); the
// product library ignores them, so no environment can change what it computes.
const char* tuning_env(const char* name) {
#ifdef SA_TUNING_BUILD
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// ====================================================================== helpers
static sa_status check_device(int* dev_out, int* sms_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  int major = 0, minor = 0, sms = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (major != 10 || minor != 0)
    return set_error(SA_ERR_UNSUPPORTED, "libsa is built for sm_100a (B200); device is sm_" +
                                             std::to_string(major) + std::to_string(minor));
  if (dev_out) *dev_out = dev;
  if (sms_out) *sms_out = sms;
  return SA_OK;
}

// ====================================================================== flat search
// Plan of one flat scan: units (CTAs or CTA pairs), corpus slices and grid.
struct FlatPlan {
  int cg, QP, S, grid;
};
static FlatPlan plan_flat(int64_t n_rows, int num_sms, int64_t nq_pad) {
  FlatPlan p;
  p.cg = nq_pad > 128 ? 2 : 1;
  const int64_t T = (n_rows + FS_BN - 1) / FS_BN;
  p.QP = (int)(nq_pad / (FS_BM * p.cg));
  const int units = num_sms / p.cg;
  int64_t S = std::max<int64_t>(1, units / p.QP);
  S = std::min<int64_t>(S, T);
  p.S = (int)S;
  p.grid = (int)std::min<int64_t>(units, (int64_t)p.QP * S) * p.cg;
  return p;
}

namespace {
// hint[q] = ordered score of the k-th key of query q's sorted list (0 when fewer than k)
__global__ void hint_from_keys_kernel(const uint64_t* __restrict__ keys, int64_t nq, int k,
                                      uint32_t* __restrict__ hint) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x)
    hint[q] = (uint32_t)(keys[q * k + k - 1] >> 32);
}
}  // namespace

sa_status flat_search_view(const CorpusView& cv, int num_sms, const __nv_bfloat16* Qs, int64_t nq,
                           int32_t k, const SearchOut& out, cudaStream_t s, bool prepass) {
  const int64_t nq_pad = padded_nq(nq);
  const FlatPlan p = plan_flat(cv.n_rows, num_sms, nq_pad);
  StreamFreer f{s};
  uint64_t *part, *heap = nullptr;
  SA_TRY(f.alloc(&part, (size_t)nq_pad * p.S * FS_LISTS_PER_ITEM * k, "alloc partials"));
  if (k > fs_heap_smem_cap(cv.d_pad))
    SA_TRY(f.alloc(&heap, (size_t)p.grid * k * FS_EPI_THREADS, "alloc heaps"));
  // Shared per-query pruning bounds, useful when a query's rows are split over slices:
  // q_hint (max of the heap roots) and q_max (each heap's best score; the kernel's bound warp
  // takes the k-th largest of them).
  const int H = (p.S * FS_LISTS_PER_ITEM + 3) / 4 * 4;   // q_max row stride (16-byte rows)
  uint32_t *hint = nullptr, *qmax = nullptr;
  if (p.S > 1) {
    SA_TRY(f.alloc(&hint, (size_t)nq, "alloc hints"));
    SA_CUDA(cudaMemsetAsync(hint, 0, nq * sizeof(uint32_t), s), "memset");
    static const bool no_bound = [] {   // SA_NO_BOUND=1: tuning experiments only
      const char* e = tuning_env("SA_NO_BOUND");
      return e && e[0] == '1';
    }();
    if (k <= 16 && p.S * FS_LISTS_PER_ITEM >= k && !no_bound) {
      SA_TRY(f.alloc(&qmax, (size_t)nq * H, "alloc heap maxima"));
      SA_CUDA(cudaMemsetAsync(qmax, 0, (size_t)nq * H * sizeof(uint32_t), s), "memset");
    }
    // Seed the bound before the scan: the k-th best score over the first m rows (a
    // sub-scan, ~1/32 of the corpus up to 2^18 rows) is a lower bound of the final k-th
    // score, so the running heaps start pruning at once instead of each filling its own k
    // entries first (that warm-up dominated the insert work: ~40% of the e4m3 scan).
    // 2^18 rows (bf16) / 2^19 (e4m3, whose scan is cheaper): measured best of 2^16..2^20
    static const int64_t seed_env = [] {   // SA_SEED_ROWS: tuning experiments only
      const char* e = tuning_env("SA_SEED_ROWS");
      return e ? atoll(e) : (int64_t)0;
    }();
    const int64_t seed_rows = seed_env > 0 ? seed_env : (int64_t)(cv.fp8 ? 1 << 19 : 1 << 18);
    static const bool seed_recurse = [] {
      const char* e = tuning_env("SA_SEED_RECURSE");
      return !(e && e[0] == '0');
    }();
    const int64_t m = std::min<int64_t>(cv.n_rows / 32, seed_rows) / FS_BN * FS_BN;
    static const bool no_seed = [] {   // SA_NO_SEED=1: timing experiments only
      const char* e = tuning_env("SA_NO_SEED");
      return e && e[0] == '1';
    }();
    // worth it only for long scans: the sub-scans cost ~0.3-0.5 ms whatever the corpus and
    // save ~7% (bf16) / ~11% (e4m3) of the scan (C3 one-GPU emulations of 2-8 shards)
    const int64_t min_rows = cv.fp8 ? (4ll << 20) : (8ll << 20);
    if (prepass && !no_seed && m >= 8 * FS_BN && (cv.n_rows >= min_rows || seed_env > 0)) {
      CorpusView pv = cv;
      pv.n_rows = m;
      uint64_t* pk;
      SA_TRY(f.alloc(&pk, (size_t)nq * k, "alloc hint keys"));
      ProfRegion region(SA_KERNEL_OTHER, s);   // the seed sub-scans count as OTHER
      SearchOut po;
      po.keys = pk;
      // the sub-scan seeds its own bound the same way (m / 32 rows, ...): without it its
      // heaps would pay the whole warm-up themselves
      SA_TRY(flat_search_view(pv, num_sms, Qs, nq, k, po, s, seed_recurse));
      hint_from_keys_kernel<<<(unsigned)std::min<int64_t>((nq + 255) / 256, 1024), 256, 0, s>>>(
          pk, nq, k, hint);
      note_launch();
      SA_CUDA(cudaGetLastError(), "hint seed");
    }
  }
  // soft lockstep of units sharing a corpus slice (see flat_scan.cu)
  int32_t* progress = nullptr;
  const int units = p.grid / p.cg;
  if (p.QP > 1 && p.S > 1 && (int64_t)p.QP * p.S <= units) {
    SA_TRY(f.alloc(&progress, (size_t)units, "alloc progress"));
    SA_CUDA(cudaMemsetAsync(progress, 0, units * sizeof(int32_t), s), "memset");
  }
  FlatScanArgs a{};
  if (const char* e = tuning_env("SA_FS_COUNT"))   // device pointer, [4] u64 (tuning only)
    a.counters = reinterpret_cast<unsigned long long*>(strtoull(e, nullptr, 0));
  a.progress = progress;
  a.q_hint = hint;
  a.q_max = qmax;
  a.q_max_stride = H;
  a.Q = Qs;
  a.nq = nq;
  a.nq_pad = nq_pad;
  a.d_pad = cv.d_pad;
  a.n_rows = cv.n_rows;
  a.QP = p.QP;
  a.S = p.S;
  a.k = k;
  a.row_ids = cv.row_ids;
  a.id_base = cv.id_base;
  a.part = part;
  a.heap_g = heap;
  a.mode = FS_MODE_TOPK;
  a.fp8 = cv.fp8 ? 1 : 0;
  {
    static const int experiment = [] {
      const char* e = tuning_env("SA_EXPERIMENT");   // results invalid: timing only
      return e ? atoi(e) : 0;
    }();
    a.experiment = experiment;
    static const int lag = [] {   // SA_LOCKSTEP_LAG: tuning experiments only
      const char* e = tuning_env("SA_LOCKSTEP_LAG");
      return e ? atoi(e) : 0;
    }();
    a.lockstep_lag = lag;
  }
  CUtensorMap tmap_q;
  SA_TRY(make_tmap_bf16(&tmap_q, Qs, nq, cv.d_pad, FS_BM));
  const CUtensorMap& tm = p.cg == 2 ? *cv.tmap2 : *cv.tmap1;
  {
    ProfRegion region(SA_KERNEL_FLAT_SCAN, s);
    SA_CUDA(launch_flat_scan(tm, tmap_q, a, p.cg, p.grid, s), "flat search launch");
  }
  MergeArgs mg{};
  mg.cand = part;
  mg.groups = p.S * FS_LISTS_PER_ITEM;
  mg.k = k;
  mg.qstride = (int64_t)p.S * FS_LISTS_PER_ITEM * k;
  mg.gstride = k;
  mg.out_keys = out.keys;
  mg.out_ids = out.ids;
  mg.out_scores = out.scores;
  mg.id_offset = 0;
  ProfRegion region(SA_KERNEL_MERGE, s);
  return cuda_status(launch_merge(mg, nq, s), "flat search merge");
}

sa_status flat_scores_view(const CorpusView& cv, int num_sms, const __nv_bfloat16* Qs, int64_t nq,
                           float* out, cudaStream_t s) {
  const int64_t nq_pad = padded_nq(nq);
  const FlatPlan p = plan_flat(cv.n_rows, num_sms, nq_pad);
  FlatScanArgs a{};
  a.Q = Qs;
  a.nq = nq;
  a.nq_pad = nq_pad;
  a.d_pad = cv.d_pad;
  a.n_rows = cv.n_rows;
  a.QP = p.QP;
  a.S = p.S;
  a.k = 1;
  a.dbg = out;
  a.mode = FS_MODE_DEBUG;
  a.fp8 = cv.fp8 ? 1 : 0;
  CUtensorMap tmap_q;
  sa_status st = make_tmap_bf16(&tmap_q, Qs, nq, cv.d_pad, FS_BM);
  if (st != SA_OK) return st;
  if (!cv.fp8 && score_gemm_applies(cv.d_pad)) {
    // a plain streaming GEMM (both operands through one TMA ring): the flat scan's per-unit
    // query staging does not pay off over the few tiles a probe gives each unit
    ScoreGemmArgs g{};
    g.nq = nq;
    g.n_rows = cv.n_rows;
    g.d_pad = cv.d_pad;
    g.out = out;
    g.ldo = cv.n_rows;
    return cuda_status(launch_score_gemm(tmap_q, *cv.tmap1, g, num_sms, s), "score gemm");
  }
  const CUtensorMap& tm = p.cg == 2 ? *cv.tmap2 : *cv.tmap1;
  cudaError_t e = launch_flat_scan(tm, tmap_q, a, p.cg, p.grid, s);
  return cuda_status(e, "score scan");
}

sa_status flat_search(const sa_index* idx, const __nv_bfloat16* Qs, int64_t nq, int64_t nq_pad,
                      int32_t k, const SearchOut& out, cudaStream_t s) {
  (void)nq_pad;
  CorpusView cv{&idx->tmap_x, &idx->tmap_x2, idx->n_local, idx->d_pad, idx->row_ids,
                idx->row_ids ? 0u : (uint32_t)idx->row_offset};
  return flat_search_view(cv, idx->num_sms, Qs, nq, k, out, s);
}

}  // namespace sa

using namespace sa;

extern "C" {

const char* sa_status_string(sa_status s) {
  switch (s) {
    case SA_OK: return "SA_OK";
    case SA_ERR_INVALID_ARG: return "SA_ERR_INVALID_ARG";
    case SA_ERR_STATE: return "SA_ERR_STATE";
    case SA_ERR_OOM: return "SA_ERR_OOM";
    case SA_ERR_CUDA: return "SA_ERR_CUDA";
    case SA_ERR_NCCL: return "SA_ERR_NCCL";
    case SA_ERR_UNSUPPORTED: return "SA_ERR_UNSUPPORTED";
  }
  return "SA_ERR_UNKNOWN";
}

const char* sa_last_error(void) { return g_last_error.c_str(); }

void sa_build_opts_default(sa_build_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->dtype = SA_BF16;
  o->kmeans_iters = 20;
  o->train_per_list = 256;
  o->seed = 0x5A2505ull;
  o->row_offset = 0;
  o->n_total = 0;
  o->comm = nullptr;
  o->stream = nullptr;
  o->centroids = nullptr;
}

sa_status sa_index_build(const void* corpus, int64_t n, int32_t d, int32_t nlist, sa_index** out) {
  sa_build_opts o;
  sa_build_opts_default(&o);
  return sa_index_build_ex(corpus, n, d, nlist, &o, out);
}

static void free_graph_entry(sa_graph_entry& g);

sa_status sa_index_free(sa_index* idx) {
  if (!idx) return SA_OK;
  cudaDeviceSynchronize();
  for (auto& g : idx->graphs) free_graph_entry(g);
  idx->graphs.clear();
  cudaFree(idx->X);
  cudaFree(idx->row_ids);
  cudaFree(idx->centroids);
  cudaFree(idx->centroids_bf16);
  cudaFree(idx->list_off);
  cudaFree(idx->graph);
  cudaFree(idx->graph_knn);
  cudaFree(idx->X8);
  delete idx;
  return SA_OK;
}

sa_status sa_index_build_ex(const void* corpus, int64_t n, int32_t d, int32_t nlist,
                            const sa_build_opts* opts, sa_index** out) {
  if (!corpus || !out || !opts) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (n < 1) return set_error(SA_ERR_INVALID_ARG, "n must be >= 1");
  if (d < 1) return set_error(SA_ERR_INVALID_ARG, "d must be >= 1");
  if (nlist < 0) return set_error(SA_ERR_INVALID_ARG, "nlist must be >= 0");
  if (opts->dtype != SA_BF16 && opts->dtype != SA_F32)
    return set_error(SA_ERR_INVALID_ARG, "bad dtype");
  const int64_t n_total = opts->n_total > 0 ? opts->n_total : n;
  if (opts->row_offset < 0 || opts->row_offset + n > n_total)
    return set_error(SA_ERR_INVALID_ARG, "row_offset + n exceeds n_total");
  if (nlist > n_total) return set_error(SA_ERR_INVALID_ARG, "nlist exceeds n_total");
  if (nlist > 32768) return set_error(SA_ERR_UNSUPPORTED, "nlist > 32768 not supported");
  if (nlist > 0 && (opts->kmeans_iters < 0 || opts->train_per_list < 1))
    return set_error(SA_ERR_INVALID_ARG, "bad k-means options");
  const int32_t d_pad = (d + 63) / 64 * 64;
  if (d_pad > FS_MAX_DPAD) return set_error(SA_ERR_UNSUPPORTED, "d > 768 not supported");
  if (n >= (1ll << 31)) return set_error(SA_ERR_UNSUPPORTED, "n_local >= 2^31");
  if (n_total >= (1ll << 32) - 1) return set_error(SA_ERR_UNSUPPORTED, "n_total >= 2^32");
  const bool list_sharded = opts->list_shard_world > 0;
  if (list_sharded) {
    if (nlist < 1) return set_error(SA_ERR_INVALID_ARG, "list sharding needs nlist >= 1");
    if (opts->list_shard_rank < 0 || opts->list_shard_rank >= opts->list_shard_world)
      return set_error(SA_ERR_INVALID_ARG, "list_shard_rank must be in [0, list_shard_world)");
    if (opts->row_offset != 0 || n_total != n)
      return set_error(SA_ERR_INVALID_ARG, "list sharding takes the full corpus (row_offset 0)");
    if (opts->comm && (opts->comm->world != opts->list_shard_world ||
                       opts->comm->rank != opts->list_shard_rank))
      return set_error(SA_ERR_INVALID_ARG, "list shard (rank, world) differs from the comm's");
  } else if (comm_sharded(opts->comm) && nlist > 0 && opts->n_total <= 0) {
    return set_error(SA_ERR_INVALID_ARG, "sharded IVF build needs n_total");
  }
  int dev = 0, sms = 0;
  sa_status st = check_device(&dev, &sms);
  if (st != SA_OK) return st;

  cudaStream_t s = (cudaStream_t)opts->stream;
  {
    // Search scratch comes from the stream-ordered pool; keep freed blocks cached instead
    // of returning them to the driver at every synchronisation (which would make the next
    // cudaMallocAsync map fresh pages inside the timed search path).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  sa_index* idx = new sa_index;
  idx->device = dev;
  idx->num_sms = sms;
  idx->n_local = n;
  idx->d = d;
  idx->d_pad = d_pad;
  idx->nlist = nlist;
  idx->row_offset = opts->row_offset;
  idx->n_total = n_total;
  idx->comm = opts->comm;
  idx->list_world = opts->list_shard_world;
  idx->list_rank = opts->list_shard_rank;
  st = cuda_status(cudaMalloc(&idx->X, (size_t)n * d_pad * sizeof(__nv_bfloat16)), "alloc corpus");
  if (st == SA_OK) {
    ProfRegion region(SA_KERNEL_STAGE, s);
    st = cuda_status(launch_cast_pad(corpus, opts->dtype == SA_F32, n, d, idx->X, n, d_pad, sms, s),
                     "cast/pad corpus");
  }
  if (st == SA_OK) st = make_tmap_bf16(&idx->tmap_x, idx->X, n, d_pad, FS_BN);
  if (st == SA_OK) st = make_tmap_bf16(&idx->tmap_x2, idx->X, n, d_pad, FS_BN / 2);
  if (st == SA_OK) st = make_tmap_bf16(&idx->tmap_xt, idx->X, n, d_pad, FS_TAIL_ROWS);
  // ivf_build permutes X list-major and re-encodes the tensor maps
  if (st == SA_OK && nlist > 0) st = ivf_build(idx, *opts, s);
  if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "build sync");
  if (st != SA_OK) {
    sa_index_free(idx);
    return st;
  }
  *out = idx;
  return SA_OK;
}

static sa_status validate_search(const sa_index* idx, const void* q, int64_t nq, int32_t k,
                                 int32_t nprobe, const void* ids, const void* scores) {
  if (!idx || !q || !ids || !scores) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (nq < 1) return set_error(SA_ERR_INVALID_ARG, "nq must be >= 1");
  if (k < 1 || k > 256) return set_error(SA_ERR_INVALID_ARG, "k must be in [1, 256]");
  if (nprobe < 0) return set_error(SA_ERR_INVALID_ARG, "nprobe must be >= 0");
  if (nprobe > 0 && idx->nlist == 0)
    return set_error(SA_ERR_STATE, "nprobe > 0 on a flat-only index (nlist = 0)");
  if (nprobe > idx->nlist) return set_error(SA_ERR_INVALID_ARG, "nprobe > nlist");
  if (nq > (1ll << 31) / 2) return set_error(SA_ERR_UNSUPPORTED, "nq too large");
  return SA_OK;
}

// a4 staging + the rank-local search (flat or IVF) into `out`.
static sa_status search_local(const sa_index* idx, const void* queries, sa_dtype qdtype,
                              int64_t nq, int32_t k, int32_t nprobe, const SearchOut& out,
                              cudaStream_t s) {
  if (nprobe > 0 && ivf_small_applies(idx, nq, k, nprobe))
    return ivf_small_search(idx, queries, qdtype == SA_F32, nq, k, nprobe, out, s);
  const int64_t nq_pad = padded_nq(nq);
  __nv_bfloat16* Qs = nullptr;
  sa_status st = dalloc(&Qs, (size_t)nq_pad * idx->d_pad, s, "alloc staged queries");
  if (st != SA_OK) return st;
  cudaError_t e;
  {
    ProfRegion region(SA_KERNEL_STAGE, s);
    e = launch_cast_pad(queries, qdtype == SA_F32, nq, idx->d, Qs, nq_pad, idx->d_pad,
                        idx->num_sms, s);
  }
  if (e != cudaSuccess) {
    cudaFreeAsync(Qs, s);
    return cuda_status(e, "stage queries");
  }
  st = nprobe == 0 ? flat_search(idx, Qs, nq, nq_pad, k, out, s)
                   : ivf_search(idx, Qs, nq, nq_pad, k, nprobe, out, s);
  cudaFreeAsync(Qs, s);
  return st;
}

static sa_status merge_keys(const uint64_t* keys, int32_t w, int64_t nq, int32_t k,
                            int64_t* out_ids, float* out_scores, cudaStream_t s) {
  MergeArgs m{};
  m.cand = keys;
  m.groups = w;
  m.k = k;
  m.qstride = k;
  m.gstride = nq * k;
  m.out_ids = out_ids;
  m.out_scores = out_scores;
  ProfRegion region(SA_KERNEL_MERGE, s);
  return cuda_status(launch_merge(m, nq, s), "final merge");
}

sa_status sa_search_ex(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                       int32_t k, int32_t nprobe, int64_t* out_ids, float* out_scores,
                       void* stream) {
  sa_status st = validate_search(idx, queries, nq, k, nprobe, out_ids, out_scores);
  if (st == SA_OK && qdtype != SA_BF16 && qdtype != SA_F32)
    st = set_error(SA_ERR_INVALID_ARG, "bad qdtype");
  cudaStream_t s = (cudaStream_t)stream;
  const bool sharded = idx && comm_sharded(idx->comm);
  if (sharded) {
    const int64_t args[kCommArgs] = {0x5a5e, nq, k, nprobe, (int64_t)qdtype, 0};
    st = comm_check_args(idx->comm, args, st, s);
  }
  if (st != SA_OK) return st;
  if (!sharded) {
    SearchOut out;
    out.ids = out_ids;
    out.scores = out_scores;
    return search_local(idx, queries, qdtype, nq, k, nprobe, out, s);
  }
  // a9: rank-local sorted [nq, k] keys (global ids) -> ncclAllGather -> k-way merge.
  uint64_t* keys_local = nullptr;
  st = dalloc(&keys_local, (size_t)nq * k, s, "alloc local keys");
  if (st == SA_OK) {
    SearchOut out;
    out.keys = keys_local;
    st = search_local(idx, queries, qdtype, nq, k, nprobe, out, s);
  }
  if (st == SA_OK) st = gather_merge_keys(idx, keys_local, nq, k, out_ids, out_scores, s);
  if (keys_local) cudaFreeAsync(keys_local, s);
  return st;
}

}  // extern "C"

namespace sa {
sa_status gather_merge_keys(const sa_index* idx, const uint64_t* keys_local, int64_t nq, int32_t k,
                            int64_t* out_ids, float* out_scores, cudaStream_t s) {
  const int w = idx->comm->world;
  uint64_t* keys_all = nullptr;
  sa_status st = dalloc(&keys_all, (size_t)nq * k * w, s, "alloc gathered keys");
  if (st == SA_OK)
    st = comm_allgather_bytes(idx->comm, keys_local, keys_all, (size_t)nq * k * sizeof(uint64_t), s);
  if (st == SA_OK) st = merge_keys(keys_all, w, nq, k, out_ids, out_scores, s);
  if (keys_all) cudaFreeAsync(keys_all, s);
  return st;
}
}  // namespace sa

extern "C" {

sa_status sa_search_keys(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                         int32_t k, int32_t nprobe, uint64_t* out_keys, void* stream) {
  sa_status st = validate_search(idx, queries, nq, k, nprobe, out_keys, out_keys);
  if (st != SA_OK) return st;
  if (qdtype != SA_BF16 && qdtype != SA_F32) return set_error(SA_ERR_INVALID_ARG, "bad qdtype");
  SearchOut out;
  out.keys = out_keys;
  return search_local(idx, queries, qdtype, nq, k, nprobe, out, (cudaStream_t)stream);
}

sa_status sa_merge_keys(const uint64_t* keys, int32_t w, int64_t nq, int32_t k, int64_t* out_ids,
                        float* out_scores, void* stream) {
  if (!keys || !out_ids || !out_scores) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (w < 1 || nq < 1) return set_error(SA_ERR_INVALID_ARG, "w and nq must be >= 1");
  if (k < 1 || k > 256) return set_error(SA_ERR_INVALID_ARG, "k must be in [1, 256]");
  return merge_keys(keys, w, nq, k, out_ids, out_scores, (cudaStream_t)stream);
}

sa_status sa_search(const sa_index* idx, const void* queries, int64_t nq, int32_t k, int32_t nprobe,
                    int64_t* out_ids, float* out_scores, void* stream) {
  return sa_search_ex(idx, queries, SA_BF16, nq, k, nprobe, out_ids, out_scores, stream);
}

static void free_graph_entry(sa_graph_entry& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  cudaFreeHost(g.h_q);
  cudaFreeHost(g.h_ids);
  cudaFreeHost(g.h_sc);
  cudaFree(g.d_q);
  cudaFree(g.d_ids);
  cudaFree(g.d_sc);
  cudaFree(g.small_scratch);
  cudaFreeHost(g.h_done);
  g = sa_graph_entry{};
}

// Capture H2D + search + D2H for one (nq, k, nprobe, qdtype) into a graph.
static sa_status capture_search(const sa_index* idx, sa_graph_entry& g) {
  const size_t qbytes = (size_t)g.nq * idx->d * (g.qdtype == SA_F32 ? 4 : 2);
  const size_t nk = (size_t)g.nq * g.k;
  sa_status st = cuda_status(cudaMallocHost(&g.h_q, qbytes), "pinned staging");
  if (st == SA_OK) st = cuda_status(cudaMallocHost(&g.h_ids, nk * 8), "pinned staging");
  if (st == SA_OK) st = cuda_status(cudaMallocHost(&g.h_sc, nk * 4), "pinned staging");
  if (st == SA_OK) st = cuda_status(cudaMalloc(&g.d_q, qbytes), "graph buffers");
  if (st == SA_OK) st = cuda_status(cudaMalloc(&g.d_ids, nk * 8), "graph buffers");
  if (st == SA_OK) st = cuda_status(cudaMalloc(&g.d_sc, nk * 4), "graph buffers");
  if (st == SA_OK && g.nprobe > 0 && ivf_small_applies(idx, g.nq, g.k, g.nprobe)) {
    st = ivf_small_scratch_alloc(idx, g.nq, g.k, g.nprobe, &g.small_scratch);
    if (st == SA_OK) st = cuda_status(cudaMallocHost(&g.h_done, sizeof(int32_t)), "pinned flag");
    if (st == SA_OK) *g.h_done = 0;
  }
  if (st != SA_OK) return st;
  cudaStream_t cs;
  st = cuda_status(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "capture stream");
  if (st != SA_OK) return st;
  cudaGraph_t graph = nullptr;
  st = cuda_status(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
  if (st == SA_OK) {
    set_capturing(true);
    const bool small = g.nprobe > 0 && ivf_small_applies(idx, g.nq, g.k, g.nprobe);
    // agent-step batch: no copy node -- one CTA of the kernel reads the pinned queries over
    // the host link and hands them to the others through device memory
    sa_status s1 = small ? SA_OK
                         : cuda_status(cudaMemcpyAsync(g.d_q, g.h_q, qbytes,
                                                       cudaMemcpyHostToDevice, cs), "H2D");
    SearchOut out;
    out.ids = g.d_ids;
    out.scores = g.d_sc;
    if (small) {
      // agent-step batch: one kernel on persistent scratch whose final merge writes the
      // results straight into the pinned host buffers (zero-copy: the D2H transfer of
      // nq * k * 12 bytes is the kernel's own stores over the host link)
      out.ids = g.h_ids;
      out.scores = g.h_sc;
      if (s1 == SA_OK)
        s1 = ivf_small_search(idx, g.d_q, g.qdtype == SA_F32, g.nq, g.k, g.nprobe, out, cs,
                              nullptr, g.small_scratch, g.h_done, g.h_q);
    } else {
      if (s1 == SA_OK)
        s1 = search_local(idx, g.d_q, (sa_dtype)g.qdtype, g.nq, g.k, g.nprobe, out, cs);
      if (s1 == SA_OK)
        s1 = cuda_status(cudaMemcpyAsync(g.h_ids, g.d_ids, nk * 8, cudaMemcpyDeviceToHost, cs),
                         "D2H");
      if (s1 == SA_OK)
        s1 = cuda_status(cudaMemcpyAsync(g.h_sc, g.d_sc, nk * 4, cudaMemcpyDeviceToHost, cs),
                         "D2H");
    }
    capture_tally(g.launches);
    set_capturing(false);
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    st = s1 != SA_OK ? s1 : cuda_status(e, "end capture");
  }
  if (st == SA_OK) st = cuda_status(cudaGraphInstantiate(&g.exec, graph, 0), "instantiate");
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  return st;
}

static bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("SA_NO_GRAPH");
    return !(e && atoi(e) != 0);
  }();
  return on;
}

sa_status sa_search_host(const sa_index* idx, const void* queries_host, sa_dtype qdtype,
                         int64_t nq, int32_t k, int32_t nprobe, int64_t* out_ids_host,
                         float* out_scores_host, void* stream) {
  sa_status st = validate_search(idx, queries_host, nq, k, nprobe, out_ids_host, out_scores_host);
  if (st != SA_OK) return st;
  if (qdtype != SA_BF16 && qdtype != SA_F32) return set_error(SA_ERR_INVALID_ARG, "bad qdtype");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t qbytes = (size_t)nq * idx->d * (qdtype == SA_F32 ? 4 : 2);
  const bool sharded = comm_sharded(idx->comm);
  if (!sharded && nq <= 1024 && graphs_enabled()) {
    // Small batches (agent-step retrieval) are launch-bound: replay a captured graph.
    sa_index* mi = const_cast<sa_index*>(idx);
    std::lock_guard<std::mutex> lock(mi->graph_mu);
    sa_graph_entry* g = nullptr;
    for (auto& e : mi->graphs)
      if (e.nq == nq && e.k == k && e.nprobe == nprobe && e.qdtype == (int32_t)qdtype) g = &e;
    if (!g) {
      // bounded cache: evict the least recently used shape (no graph of this index is in
      // flight -- every replay below completes under graph_mu)
      if (mi->graphs.size() >= kMaxCapturedSearches) {
        auto lru = std::min_element(mi->graphs.begin(), mi->graphs.end(),
                                    [](const sa_graph_entry& a, const sa_graph_entry& b) {
                                      return a.last_use < b.last_use;
                                    });
        free_graph_entry(*lru);
        mi->graphs.erase(lru);
      }
      sa_graph_entry e;
      e.nq = nq;
      e.k = k;
      e.nprobe = nprobe;
      e.qdtype = (int32_t)qdtype;
      st = capture_search(idx, e);
      if (st != SA_OK) {
        free_graph_entry(e);
        return st;
      }
      mi->graphs.push_back(e);
      g = &mi->graphs.back();
    }
    g->last_use = ++mi->use_clock;
    std::memcpy(g->h_q, queries_host, qbytes);
    st = cuda_status(cudaGraphLaunch(g->exec, s), "graph launch");
    if (st == SA_OK && g->h_done) {
      // the agent-step kernel signals completion through pinned memory after writing the
      // results there: spin on the flag (no stream-synchronisation wake-up on the critical
      // path); a stream error or a completed stream without the flag is reported
      const int32_t want = ++g->seq;
      for (uint64_t it = 1;; ++it) {
        if (*reinterpret_cast<volatile int32_t*>(g->h_done) == want) break;
        if ((it & 255) == 0) {
          const cudaError_t e = cudaStreamQuery(s);
          if (e == cudaErrorNotReady) continue;
          if (e != cudaSuccess) return cuda_status(e, "search");
          if (*reinterpret_cast<volatile int32_t*>(g->h_done) != want)
            return set_error(SA_ERR_CUDA, "agent-step search finished without its signal");
          break;
        }
      }
    } else if (st == SA_OK) {
      st = cuda_status(cudaStreamSynchronize(s), "search sync");
    }
    if (st != SA_OK) return st;
    std::memcpy(out_ids_host, g->h_ids, (size_t)nq * k * 8);
    std::memcpy(out_scores_host, g->h_sc, (size_t)nq * k * 4);
    prof_add_launches(g->launches);
    return SA_OK;
  }
  void* dq = nullptr;
  int64_t* dids = nullptr;
  float* dsc = nullptr;
  st = cuda_status(cudaMallocAsync(&dq, qbytes, s), "alloc queries");
  if (st == SA_OK) st = dalloc(&dids, (size_t)nq * k, s, "alloc ids");
  if (st == SA_OK) st = dalloc(&dsc, (size_t)nq * k, s, "alloc scores");
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(dq, queries_host, qbytes, cudaMemcpyHostToDevice, s), "H2D");
  if (st == SA_OK) st = sa_search_ex(idx, dq, qdtype, nq, k, nprobe, dids, dsc, stream);
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(out_ids_host, dids, (size_t)nq * k * 8,
                                     cudaMemcpyDeviceToHost, s), "D2H ids");
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(out_scores_host, dsc, (size_t)nq * k * 4,
                                     cudaMemcpyDeviceToHost, s), "D2H scores");
  if (dq) cudaFreeAsync(dq, s);
  if (dids) cudaFreeAsync(dids, s);
  if (dsc) cudaFreeAsync(dsc, s);
  sa_status st2 = cuda_status(cudaStreamSynchronize(s), "search sync");
  return st != SA_OK ? st : st2;
}

sa_status sa_index_info(const sa_index* idx, int64_t* n_local, int32_t* d, int32_t* nlist,
                        int64_t* row_offset) {
  if (!idx) return set_error(SA_ERR_INVALID_ARG, "null index");
  if (n_local) *n_local = idx->n_local;
  if (d) *d = idx->d;
  if (nlist) *nlist = idx->nlist;
  if (row_offset) *row_offset = idx->row_offset;
  return SA_OK;
}

sa_status sa_index_export_centroids(const sa_index* idx, float* host_out) {
  if (!idx || !host_out) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (idx->nlist == 0) return set_error(SA_ERR_STATE, "flat-only index has no centroids");
  cudaError_t e = cudaMemcpy2D(host_out, (size_t)idx->d * 4, idx->centroids, (size_t)idx->d_pad * 4,
                               (size_t)idx->d * 4, idx->nlist, cudaMemcpyDeviceToHost);
  return cuda_status(e, "export centroids");
}

sa_status sa_index_export_lists(const sa_index* idx, int64_t* host_offsets, int64_t* host_ids) {
  if (!idx || !host_offsets || !host_ids) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (idx->nlist == 0) return set_error(SA_ERR_STATE, "flat-only index has no lists");
  std::memcpy(host_offsets, idx->h_list_off.data(), (idx->nlist + 1) * sizeof(int64_t));
  std::vector<int32_t> tmp(idx->n_local);
  cudaError_t e = cudaMemcpy(tmp.data(), idx->row_ids, idx->n_local * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "export lists");
  for (int64_t i = 0; i < idx->n_local; ++i) host_ids[i] = (int64_t)(uint32_t)tmp[i];
  return SA_OK;
}

sa_status sa_search_probes(const sa_index* idx, const void* queries, int64_t nq, int32_t nprobe,
                           int32_t* out_lists, void* stream) {
  if (!idx || !queries || !out_lists) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (nq < 1) return set_error(SA_ERR_INVALID_ARG, "nq must be >= 1");
  if (idx->nlist == 0) return set_error(SA_ERR_STATE, "flat-only index");
  if (nprobe < 1 || nprobe > idx->nlist) return set_error(SA_ERR_INVALID_ARG, "bad nprobe");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nq_pad = padded_nq(nq);
  __nv_bfloat16* Qs = nullptr;
  sa_status st = dalloc(&Qs, (size_t)nq_pad * idx->d_pad, s, "alloc staged queries");
  if (st != SA_OK) return st;
  st = cuda_status(launch_cast_pad(queries, false, nq, idx->d, Qs, nq_pad, idx->d_pad,
                                   idx->num_sms, s), "stage queries");
  if (st == SA_OK) st = ivf_probe(idx, Qs, nq, nq_pad, nprobe, out_lists, s);
  cudaFreeAsync(Qs, s);
  return st;
}

sa_status sa_debug_scores(const sa_index* idx, const void* queries, int64_t nq, float* out_scores,
                          void* stream) {
  if (!idx || !queries || !out_scores) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (nq < 1) return set_error(SA_ERR_INVALID_ARG, "nq must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nq_pad = padded_nq(nq);
  __nv_bfloat16* Qs = nullptr;
  float* dbg = nullptr;
  sa_status st = dalloc(&Qs, (size_t)nq_pad * idx->d_pad, s, "alloc staged queries");
  if (st == SA_OK) st = dalloc(&dbg, (size_t)nq_pad * idx->n_local, s, "alloc debug scores");
  if (st == SA_OK)
    st = cuda_status(launch_cast_pad(queries, false, nq, idx->d, Qs, nq_pad, idx->d_pad,
                                     idx->num_sms, s), "stage queries");
  if (st == SA_OK) {
    CorpusView cv{&idx->tmap_x, &idx->tmap_x2, idx->n_local, idx->d_pad, nullptr, 0u};
    st = flat_scores_view(cv, idx->num_sms, Qs, nq, dbg, s);
  }
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(out_scores, dbg, (size_t)nq * idx->n_local * 4,
                                     cudaMemcpyDeviceToDevice, s), "copy scores");
  if (Qs) cudaFreeAsync(Qs, s);
  if (dbg) cudaFreeAsync(dbg, s);
  return st;
}

sa_status sa_debug_small_phases(const sa_index* idx, const void* queries, int64_t nq, int32_t k,
                                int32_t nprobe, int64_t* out_ids, float* out_scores,
                                int64_t* host_ns, int32_t* host_grid, void* stream) {
  if (!idx || !queries || !out_ids || !out_scores || !host_ns || !host_grid)
    return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (!ivf_small_applies(idx, nq, k, nprobe) || idx->num_sms > 1024)
    return set_error(SA_ERR_UNSUPPORTED, "the one-launch path does not apply");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = idx->num_sms;
  int64_t* dns = nullptr;
  sa_status st = dalloc(&dns, (size_t)grid * 8, s, "alloc debug timestamps");
  if (st != SA_OK) return st;
  st = cuda_status(cudaMemsetAsync(dns, 0, (size_t)grid * 8 * sizeof(int64_t), s), "memset");
  SearchOut out{};
  out.ids = out_ids;
  out.scores = out_scores;
  if (st == SA_OK) st = ivf_small_search(idx, queries, false, nq, k, nprobe, out, s, dns);
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(host_ns, dns, (size_t)grid * 8 * sizeof(int64_t),
                                     cudaMemcpyDeviceToHost, s), "copy timestamps");
  if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "sync");
  cudaFreeAsync(dns, s);
  *host_grid = grid;
  return st;
}

sa_status sa_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> l(g_prof.mu);
  for (int k = 0; k < SA_KERNEL_KINDS; ++k) {
    for (auto& p : g_prof.ev[k]) {
      g_prof.pool.push_back(p.first);
      g_prof.pool.push_back(p.second);
    }
    g_prof.ev[k].clear();
    g_prof.launches[k] = 0;
  }
  g_prof.on = on != 0;
  return SA_OK;
}

sa_status sa_profile_read(int32_t kind, double* ms_total, int64_t* launches) {
  if (kind < 0 || kind >= SA_KERNEL_KINDS) return set_error(SA_ERR_INVALID_ARG, "bad kind");
  std::lock_guard<std::mutex> l(g_prof.mu);
  double tot = 0.0;
  for (auto& p : g_prof.ev[kind]) {
    cudaError_t e = cudaEventSynchronize(p.second);
    if (e != cudaSuccess) return cuda_status(e, "profile sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.first, p.second);
    tot += ms;
  }
  if (ms_total) *ms_total = tot;
  if (launches) *launches = g_prof.launches[kind];
  return SA_OK;
}

}  // extern "C"
