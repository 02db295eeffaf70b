// extern "C" boundary of libtwfa (include/twfa.h). Exceptions stop here and
// become the 0/1/2/3 return codes of the reference's CLI (cli.cpp:462-471).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/twfa.h"
#include "fa_bwd.h"
#include "fa_fwd.h"
#include "lowering.h"

struct twfa_plan {
  twfa::LoweredSchedule sched;
  std::string description;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const twfa::UsageError& e) {
    return fail(TWFA_EUSAGE, e.what());
  } catch (const twfa::DomainError& e) {
    return fail(TWFA_EDOMAIN, e.what());
  } catch (const CudaError& e) {
    return fail(TWFA_ECUDA, e.what());
  } catch (const std::exception& e) {
    return fail(TWFA_EDOMAIN, e.what());
  } catch (...) {
    return fail(TWFA_EDOMAIN, "unknown error");
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library does not link libcuda directly.
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled is unavailable");
  return fn;
}

// bf16 (or fp32) tensor of `rank` dims (innermost first), 128-byte swizzled boxes
CUtensorMap make_map(const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                     const cuuint32_t* box, CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                     CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint32_t elem[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, dtype, static_cast<cuuint32_t>(rank),
                           const_cast<void*>(base), dims, strides_bytes, box, elem,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

// TWFA_KERNEL=interpreter forces the runtime interpreter even for plans that
// have a build-time specialization (tests compare the two realizations).
bool allow_specialized() {
  const char* e = std::getenv("TWFA_KERNEL");
  return !(e && std::strcmp(e, "interpreter") == 0);
}

int sm_count() {
  int dev = 0, n = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
  return n;
}

void require_aligned(const void* p, const char* what) {
  if (p == nullptr) throw twfa::UsageError(std::string(what) + " is NULL");
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0) throw twfa::UsageError(std::string(what) + " is not 16-byte aligned");
}

// Causal work lists. A causal launch has work tiles of very different
// length (query block qb of a (b, h) needs 2 (qb + 1) K / V iterations).
// Tiles are taken in (b, h) groups small enough that the group's K and V
// stay in L2 (<= 48 MiB), longest first inside a group, and each goes to the
// CTA with the least work so far (LPT): the CTAs move through the groups
// together, so the tiles running at any moment share K / V, and their totals
// stay balanced. The lists depend only on (device, B*H, S, grid, group
// budget); they are built once, uploaded on the launch stream (which is then
// synchronized, so the first launch of a shape reads finished lists and the
// host copy may be released) and kept read-only on the device. The cache
// holds at most kMaxWorkLists shapes; the oldest entry is freed (after a
// device synchronize, since an earlier launch may still read it) when a new
// shape would exceed that.
struct WorkLists {
  int* list = nullptr;
  int* off = nullptr;
};
constexpr size_t kMaxWorkLists = 64;

long long work_list_budget() {
  long long mb = 48;  // TWFA_WL_GROUP_MB overrides (measurements); clamped to >= 1 MiB
  if (const char* e = std::getenv("TWFA_WL_GROUP_MB")) mb = std::max(1LL, std::atoll(e));
  return mb * (1LL << 20);
}

// kind 0: forward (tile = 256 queries; causal work index w = (qbl-1-qb)*bh + b,
// 2 (qb + 1) K/V iterations); kind 2: forward on CTA pairs (tile = 512
// queries, 4 (qb + 1) iterations, one list per pair); kind 1: backward (tile =
// 128 keys; causal work index w = j*bh + b, nq - j Q iterations). The group bound applies to the
// streamed operands of one (b, h): K, V (forward) or Q, dO (backward).
WorkLists causal_work_lists(int kind, int bh, int S, int grid, cudaStream_t stream) {
  using Key = std::tuple<int, int, int, int, int, long long>;
  static std::mutex mu;
  static std::map<Key, WorkLists> cache;
  static std::deque<Key> order_of_use;
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  const long long budget = work_list_budget();
  std::lock_guard<std::mutex> lock(mu);
  const Key key = std::make_tuple(kind, dev, bh, S, grid, budget);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int tile = kind == 0 ? 256 : kind == 2 ? 512 : 128;
  const int nt = (S + tile - 1) / tile;  // tiles per (b, h)
  const int num = bh * nt;
  const long long stream_bytes = 2LL * S * 128 * 2;  // the two streamed operands of one (b, h)
  const int group = static_cast<int>(std::max<long long>(1, budget / stream_bytes));
  // candidate order: (b, h) groups, longest first inside a group
  std::vector<int> order;
  order.reserve(static_cast<size_t>(num));
  for (int g0 = 0; g0 < bh; g0 += group)
    for (int rank = 0; rank < nt; ++rank)  // rank 0 = the longest tile of a (b, h)
      for (int b = g0; b < std::min(bh, g0 + group); ++b) order.push_back(rank * bh + b);
  using Load = std::pair<long long, int>;
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int x = 0; x < grid; ++x) heap.push({0, x});
  std::vector<std::vector<int>> per(static_cast<size_t>(grid));
  for (int w : order) {
    const int rank = w / bh;
    long long iters;
    if (kind != 1) {
      const int qb = nt - 1 - rank;
      iters = (std::min<long long>(S, static_cast<long long>(tile) * (qb + 1)) + 127) / 128;
    } else {
      iters = nt - rank;  // K/V tile j = rank sees Q tiles j .. nt-1
    }
    const long long cost = iters + 2;  // iterations + the tile boundary
    Load l = heap.top();
    heap.pop();
    per[static_cast<size_t>(l.second)].push_back(w);
    heap.push({l.first + cost, l.second});
  }
  std::vector<int> list, off(static_cast<size_t>(grid) + 1, 0);
  for (int x = 0; x < grid; ++x) {
    off[static_cast<size_t>(x)] = static_cast<int>(list.size());
    list.insert(list.end(), per[static_cast<size_t>(x)].begin(), per[static_cast<size_t>(x)].end());
  }
  off[static_cast<size_t>(grid)] = static_cast<int>(list.size());
  if (cache.size() >= kMaxWorkLists) {  // evict the oldest shape
    const Key old = order_of_use.front();
    order_of_use.pop_front();
    const WorkLists w = cache[old];
    int cur = 0;
    check(cudaGetDevice(&cur), "cudaGetDevice");
    check(cudaSetDevice(std::get<1>(old)), "cudaSetDevice");
    check(cudaDeviceSynchronize(), "cudaDeviceSynchronize (work-list eviction)");
    cudaFree(w.list);
    cudaFree(w.off);
    check(cudaSetDevice(cur), "cudaSetDevice");
    cache.erase(old);
  }
  WorkLists wl;
  check(cudaMalloc(&wl.list, std::max<size_t>(1, list.size()) * sizeof(int)), "cudaMalloc work list");
  check(cudaMalloc(&wl.off, off.size() * sizeof(int)), "cudaMalloc work offsets");
  check(cudaMemcpyAsync(wl.list, list.data(), list.size() * sizeof(int), cudaMemcpyHostToDevice, stream),
        "H2D work list");
  check(cudaMemcpyAsync(wl.off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice, stream),
        "H2D work offsets");
  check(cudaStreamSynchronize(stream), "work-list upload");
  cache[key] = wl;
  order_of_use.push_back(key);
  return wl;
}

// The device of a caller's buffer becomes the current device for the call
// (sm count, work-list cache, kernel attributes and the launch all follow
// it), and is restored afterwards. A host pointer is a usage error.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard(const void* p, const char* what) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      throw twfa::UsageError(std::string(what) + " is not a CUDA device pointer");
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
      throw twfa::UsageError(std::string(what) + " is not a CUDA device pointer");
    int cur = 0;
    check(cudaGetDevice(&cur), "cudaGetDevice");
    if (cur != at.device) {
      check(cudaSetDevice(at.device), "cudaSetDevice");
      prev = cur;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// CTA pairs (cta_group::2) for the forward when the plan allows them;
// TWFA_PAIR=0 keeps one CTA per work tile (comparison runs)
bool use_pairs(const TwfaDevicePlan& p) {
  if (!twfa::fa_fwd_pair_capable(p)) return false;
  // rings that only fit in shared memory with half K / V tiles per CTA
  if (twfa::fa_fwd_smem_bytes(p, false) > 216 * 1024 + 1024 + 16384) return true;
  const char* e = std::getenv("TWFA_PAIR");
  return !(e && std::strcmp(e, "0") == 0);
}

// TWFA_WORK_LISTS=0 keeps the arithmetic causal order (comparison runs)
bool use_work_lists() {
  const char* e = std::getenv("TWFA_WORK_LISTS");
  return !(e && std::strcmp(e, "0") == 0);
}

int fa_fwd_impl(const twfa_plan* plan, const void* q, const void* k, const void* v, void* o, float* lse, int B,
                int H, int S, int D, int causal, float scale, uint32_t* trace, uint32_t cap, void* stream) {
  if (!plan) throw twfa::UsageError("plan is NULL");
  const TwfaDevicePlan& p = plan->sched.plan;
  if (p.family != TWFA_FAMILY_FA_FWD) throw twfa::UsageError("plan is not an FA-forward plan");
  if (D != 128) throw twfa::UsageError("head dim must be 128");
  if (B < 1 || H < 1 || S < 1) throw twfa::UsageError("B, H, S must be positive");
  if (!(scale > 0.f) || !std::isfinite(scale)) throw twfa::UsageError("softmax_scale must be positive");
  if (p.num_tiles != 2) throw twfa::UsageError("the kernel runs two 128-row Q sub-tiles per CTA");
  require_aligned(q, "q");
  require_aligned(k, "k");
  require_aligned(v, "v");
  require_aligned(o, "o");
  DeviceGuard guard(q, "q");
  const cuuint64_t bh = static_cast<cuuint64_t>(B) * H;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(S), bh};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(S) * D * 2};
  const cuuint32_t box_q[3] = {64, 128, 1};
  const cuuint32_t box_kv[3] = {64, static_cast<cuuint32_t>(p.kv_tile), 1};
  const CUtensorMap tq = make_map(q, 3, dims, strides, box_q);
  const CUtensorMap tv = make_map(v, 3, dims, strides, box_kv);
  const CUtensorMap to = make_map(o, 3, dims, strides, box_q);
  twfa::FaArgs a{};
  a.tm_o = to;
  a.o = static_cast<__nv_bfloat16*>(o);
  a.lse = lse;
  a.trace = trace;
  a.trace_cap = cap;
  a.B = B;
  a.H = H;
  a.S = S;
  a.causal = causal ? 1 : 0;
  a.scale_log2 = scale * 1.4426950408889634f;
  auto launch_as = [&](bool pair) {
    // a CTA of a pair loads half the keys of a K tile (per head-dim half)
    const cuuint32_t box_k[3] = {64, static_cast<cuuint32_t>(pair ? p.kv_tile / 2 : p.kv_tile), 1};
    const CUtensorMap tk = make_map(k, 3, dims, strides, box_k);
    // persistent: one work unit (CTA, or CTA pair of 512 query rows) per SM (pair)
    const int unit_rows = pair ? 512 : 256, cta_per_unit = pair ? 2 : 1;
    const long long work = static_cast<long long>(bh) * ((S + unit_rows - 1) / unit_rows);
    const int units = static_cast<int>(std::min<long long>(work, std::max(1, sm_count() / cta_per_unit)));
    const int grid = units * cta_per_unit;
    a.work_list = nullptr;
    a.work_off = nullptr;
    if (causal && use_work_lists()) {
      const WorkLists wl =
          causal_work_lists(pair ? 2 : 0, static_cast<int>(bh), S, units, static_cast<cudaStream_t>(stream));
      a.work_list = wl.list;
      a.work_off = wl.off;
    }
    return twfa::fa_fwd_launch(tq, tk, tv, p, a, grid, static_cast<cudaStream_t>(stream), allow_specialized(),
                               pair);
  };
  const bool pair = use_pairs(p);
  cudaError_t e = launch_as(pair);
  if (pair && (e == cudaErrorInvalidClusterSize || e == cudaErrorLaunchOutOfResources) &&
      twfa::fa_fwd_smem_bytes(p, false) <= 227 * 1024) {
    // the device cannot co-schedule the CTA pairs (e.g. a partitioned GPU):
    // the same plan as one CTA per tile (bit-identical outputs)
    cudaGetLastError();
    e = launch_as(false);
  }
  check(e, "fa_fwd launch");
  return TWFA_OK;
}

int fa_bwd_impl(const twfa_plan* plan, const void* q, const void* k, const void* v, const void* o,
                const void* dout, const float* lse, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, int B,
                int H, int S, int D, int causal, float scale, void* stream, uint32_t* trace = nullptr,
                uint32_t cap = 0) {
  if (!plan) throw twfa::UsageError("plan is NULL");
  const TwfaDevicePlan& p = plan->sched.plan;
  if (p.family != TWFA_FAMILY_FA_BWD) throw twfa::UsageError("plan is not an FA-backward plan");
  if (D != 128) throw twfa::UsageError("head dim must be 128");
  if (B < 1 || H < 1 || S < 1) throw twfa::UsageError("B, H, S must be positive");
  if (!(scale > 0.f) || !std::isfinite(scale)) throw twfa::UsageError("softmax_scale must be positive");
  for (auto [ptr, name] : {std::pair<const void*, const char*>{q, "q"}, {k, "k"}, {v, "v"}, {o, "o"},
                           {dout, "dout"}, {lse, "lse"}, {dq, "dq"}, {dk, "dk"}, {dv, "dv"}, {ws, "workspace"}})
    require_aligned(ptr, name);
  if (ws_bytes < twfa::fa_bwd_workspace_bytes(B, H, S)) throw twfa::UsageError("workspace too small");
  DeviceGuard guard(q, "q");
  const cuuint64_t bh = static_cast<cuuint64_t>(B) * H;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(S), bh};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(S) * D * 2};
  const cuuint64_t strides32[2] = {static_cast<cuuint64_t>(D) * 4, static_cast<cuuint64_t>(S) * D * 4};
  const cuuint32_t box[3] = {64, 128, 1};
  const cuuint32_t box32[3] = {32, 128, 1};
  const size_t rows = static_cast<size_t>(bh) * S;
  float* dq_acc = static_cast<float*>(ws);
  float* dvec = dq_acc + rows * 128;
  twfa::FaBwdArgs a{};
  a.tm_q = make_map(q, 3, dims, strides, box);
  a.tm_k = make_map(k, 3, dims, strides, box);
  a.tm_v = make_map(v, 3, dims, strides, box);
  a.tm_do = make_map(dout, 3, dims, strides, box);
  a.tm_dq = make_map(dq_acc, 3, dims, strides32, box32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  const cuuint32_t box64[3] = {64, 64, 1};
  a.tm_dq64 = make_map(dq_acc, 3, dims, strides32, box64, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                       CU_TENSOR_MAP_SWIZZLE_NONE);
  a.lse = lse;
  a.dvec = dvec;
  a.dq_acc = dq_acc;
  a.dk = static_cast<__nv_bfloat16*>(dk);
  a.dv = static_cast<__nv_bfloat16*>(dv);
  a.B = B;
  a.H = H;
  a.S = S;
  a.causal = causal ? 1 : 0;
  a.scale = scale;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.trace = trace;
  a.trace_cap = cap;
  const long long work = static_cast<long long>(bh) * ((S + 127) / 128);
  const int grid = static_cast<int>(std::min<long long>(work, sm_count()));
  a.work_list = nullptr;
  a.work_off = nullptr;
  if (causal && use_work_lists()) {
    const WorkLists wl = causal_work_lists(1, static_cast<int>(bh), S, grid, static_cast<cudaStream_t>(stream));
    a.work_list = wl.list;
    a.work_off = wl.off;
  }
  check(twfa::fa_bwd_launch(p, a, static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout),
                            static_cast<__nv_bfloat16*>(dq), grid, static_cast<cudaStream_t>(stream)),
        "fa_bwd launch");
  return TWFA_OK;
}

// Host-buffer pipeline of twfa_fa_fwd_host. The (b, h) pairs are
// independent, so the call streams them in chunks: the caller's (pageable)
// Q, K, V of chunk i are copied by host threads into a pinned staging slot,
// DMA'd to the device on a copy stream, computed on a compute stream, and O
// returns through a pinned slot on a third stream while chunk i + 1 is being
// staged, so host copies, PCIe transfers in both directions and the kernel
// overlap. Resources (device buffers for the whole problem, kStages pinned
// slots, streams, events) are cached per calling thread and grow on demand.
constexpr int kStages = 3;
constexpr size_t kChunkBytes = 64u << 20;  // per tensor per chunk

// memcpy split over host threads (the pageable <-> pinned copies are the
// host-side bound of the pipeline)
void parallel_copy(void* dst, const void* src, size_t bytes) {
  const size_t kMin = 4u << 20;
  unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  nt = static_cast<unsigned>(std::min<size_t>(nt, std::max<size_t>(1, bytes / kMin)));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> ts;
  const size_t part = (bytes + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const size_t a = t * part, b = std::min(bytes, a + part);
    if (a >= b) break;
    ts.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
  }
  for (auto& t : ts) t.join();
}

struct HostPipeline {
  int dev = -1;
  void* dbuf = nullptr;  // q, k, v, o (+ lse) of the whole problem
  size_t dbytes = 0;
  void* pin[kStages] = {};  // per slot: q, k, v chunk in, o chunk out, lse chunk out
  size_t pin_bytes = 0;
  cudaStream_t s_h2d = nullptr, s_cmp = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[kStages] = {}, ev_done[kStages] = {}, ev_out[kStages] = {};
  ~HostPipeline() { release(); }
  void release() {
    if (dev < 0) return;
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    if (dbuf) cudaFree(dbuf);
    for (int i = 0; i < kStages; ++i) {
      if (pin[i]) cudaFreeHost(pin[i]);
      if (ev_in[i]) cudaEventDestroy(ev_in[i]);
      if (ev_done[i]) cudaEventDestroy(ev_done[i]);
      if (ev_out[i]) cudaEventDestroy(ev_out[i]);
      pin[i] = nullptr;
      ev_in[i] = ev_done[i] = ev_out[i] = nullptr;
    }
    for (cudaStream_t st : {s_h2d, s_cmp, s_d2h})
      if (st) cudaStreamDestroy(st);
    s_h2d = s_cmp = s_d2h = nullptr;
    dbuf = nullptr;
    dbytes = pin_bytes = 0;
    dev = -1;
  }
  void prepare(size_t need_dev, size_t need_pin) {
    int cur = 0;
    check(cudaGetDevice(&cur), "cudaGetDevice");
    if (dev != cur) {
      release();
      dev = cur;
      check(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking), "cudaStreamCreate");
      check(cudaStreamCreateWithFlags(&s_cmp, cudaStreamNonBlocking), "cudaStreamCreate");
      check(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking), "cudaStreamCreate");
      for (int i = 0; i < kStages; ++i) {
        check(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming), "cudaEventCreate");
        check(cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming), "cudaEventCreate");
        check(cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming), "cudaEventCreate");
      }
    }
    if (need_dev > dbytes) {
      if (dbuf) cudaFree(dbuf);
      dbuf = nullptr;
      dbytes = 0;
      check(cudaMalloc(&dbuf, need_dev), "cudaMalloc");
      dbytes = need_dev;
    }
    if (need_pin > pin_bytes) {
      for (int i = 0; i < kStages; ++i) {
        if (pin[i]) cudaFreeHost(pin[i]);
        pin[i] = nullptr;
      }
      pin_bytes = 0;
      for (int i = 0; i < kStages; ++i) check(cudaMallocHost(&pin[i], need_pin), "cudaMallocHost");
      pin_bytes = need_pin;
    }
  }
};

int fa_fwd_host_impl(const twfa_plan* plan, const uint16_t* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                     float* lse, int B, int H, int S, int D, int causal, float scale) {
  if (!q || !k || !v || !o) throw twfa::UsageError("NULL host buffer");
  if (B < 1 || H < 1 || S < 1 || D != 128) throw twfa::UsageError("unsupported shape");
  thread_local HostPipeline hp;
  // page-locked caller buffers (cudaMallocHost / cudaHostRegister, e.g.
  // torch pin_memory) are DMA'd directly; pageable ones go through the
  // pinned staging slots
  auto pinned = [](const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool direct = pinned(q) && pinned(k) && pinned(v) && pinned(o) && (!lse || pinned(lse));
  const size_t pairs = static_cast<size_t>(B) * H;
  const size_t pb = static_cast<size_t>(S) * D * 2;  // bytes of one pair of one tensor
  const size_t lb = static_cast<size_t>(S) * 4;      // lse bytes of one pair
  const size_t chunk = std::max<size_t>(1, std::min(pairs, kChunkBytes / pb));
  const size_t tb = pairs * pb;
  // device layout: q | k | v | o | lse, each 256-byte aligned (TMA needs 16)
  auto up = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  const size_t off_k = up(tb), off_v = off_k + up(tb), off_o = off_v + up(tb), off_l = off_o + up(tb);
  const size_t need_dev = off_l + (lse ? up(pairs * lb) : 0);
  // pinned slot layout: q | k | v | o | lse of one chunk
  const size_t cb = chunk * pb, cl = chunk * lb;
  const size_t need_pin = direct ? 0 : 4 * cb + (lse ? cl : 0);
  hp.prepare(need_dev, need_pin);
  uint8_t* d = static_cast<uint8_t*>(hp.dbuf);
  const size_t nchunks = (pairs + chunk - 1) / chunk;
  const uint8_t* src[3] = {reinterpret_cast<const uint8_t*>(q), reinterpret_cast<const uint8_t*>(k),
                           reinterpret_cast<const uint8_t*>(v)};
  const size_t doff[3] = {0, off_k, off_v};
  auto drain = [&](size_t j) {  // chunk j's O (and lse) from its pinned slot to the caller
    const int sl = static_cast<int>(j % kStages);
    const size_t p0 = j * chunk, np = std::min(chunk, pairs - p0);
    check(cudaEventSynchronize(hp.ev_out[sl]), "D2H o");
    if (direct) return;
    uint8_t* pin = static_cast<uint8_t*>(hp.pin[sl]);
    parallel_copy(reinterpret_cast<uint8_t*>(o) + p0 * pb, pin + 3 * cb, np * pb);
    if (lse) std::memcpy(reinterpret_cast<uint8_t*>(lse) + p0 * lb, pin + 4 * cb, np * lb);
  };
  for (size_t i = 0; i < nchunks; ++i) {
    const int sl = static_cast<int>(i % kStages);
    const size_t p0 = i * chunk, np = std::min(chunk, pairs - p0);
    // the slot's previous chunk (i - kStages) has returned its O and left
    // the slot's inputs (its H2D completed before its kernel ran)
    if (i >= static_cast<size_t>(kStages)) drain(i - kStages);
    uint8_t* pin = static_cast<uint8_t*>(hp.pin[sl]);
    if (!direct)
      for (int t = 0; t < 3; ++t) parallel_copy(pin + t * cb, src[t] + p0 * pb, np * pb);
    for (int t = 0; t < 3; ++t)
      check(cudaMemcpyAsync(d + doff[t] + p0 * pb, direct ? src[t] + p0 * pb : pin + t * cb, np * pb,
                            cudaMemcpyHostToDevice, hp.s_h2d),
            "H2D");
    check(cudaEventRecord(hp.ev_in[sl], hp.s_h2d), "cudaEventRecord");
    check(cudaStreamWaitEvent(hp.s_cmp, hp.ev_in[sl], 0), "cudaStreamWaitEvent");
    // chunk i as a [1, np, S, 128] problem: the pairs are independent
    const int rc = fa_fwd_impl(plan, d + p0 * pb, d + off_k + p0 * pb, d + off_v + p0 * pb, d + off_o + p0 * pb,
                               lse ? reinterpret_cast<float*>(d + off_l + p0 * lb) : nullptr, 1, static_cast<int>(np),
                               S, D, causal, scale, nullptr, 0, hp.s_cmp);
    if (rc != TWFA_OK) return rc;
    check(cudaEventRecord(hp.ev_done[sl], hp.s_cmp), "cudaEventRecord");
    check(cudaStreamWaitEvent(hp.s_d2h, hp.ev_done[sl], 0), "cudaStreamWaitEvent");
    uint8_t* o_dst = direct ? reinterpret_cast<uint8_t*>(o) + p0 * pb : pin + 3 * cb;
    uint8_t* l_dst = direct ? reinterpret_cast<uint8_t*>(lse) + p0 * lb : pin + 4 * cb;
    check(cudaMemcpyAsync(o_dst, d + off_o + p0 * pb, np * pb, cudaMemcpyDeviceToHost, hp.s_d2h), "D2H o");
    if (lse) check(cudaMemcpyAsync(l_dst, d + off_l + p0 * lb, np * lb, cudaMemcpyDeviceToHost, hp.s_d2h), "D2H lse");
    check(cudaEventRecord(hp.ev_out[sl], hp.s_d2h), "cudaEventRecord");
  }
  for (size_t j = nchunks > static_cast<size_t>(kStages) ? nchunks - kStages : 0; j < nchunks; ++j) drain(j);
  return TWFA_OK;
}

}  // namespace

extern "C" {

int twfa_abi_version(void) { return 2; }

const char* twfa_last_error(void) { return g_last_error.c_str(); }

int twfa_plan_create(const char* problem_json, const char* solution_json, twfa_plan** out) {
  return guarded([&] {
    if (!problem_json || !solution_json || !out) throw twfa::UsageError("NULL argument");
    auto* p = new twfa_plan{twfa::lower(problem_json, solution_json), {}};
    p->description = twfa::describe(p->sched);
    if (p->sched.plan.family == TWFA_FAMILY_FA_FWD) {  // which kernel realizes it
      const std::string name = twfa::fa_fwd_kernel_name(p->sched.plan);
      const std::string kernel =
          allow_specialized() && name != "interpreter" ? "specialized:" + name : std::string("interpreter");
      p->description.insert(p->description.size() - 1, ",\"kernel\":\"" + kernel + "\",\"cta_pair\":" +
                                                        (use_pairs(p->sched.plan) ? "true" : "false"));
    }
    *out = p;
    return TWFA_OK;
  });
}

void twfa_plan_destroy(twfa_plan* plan) { delete plan; }

int twfa_schedule_validate(const char* problem_json, const char* solution_json, char* buf, size_t cap,
                           size_t* needed) {
  return guarded([&] {
    if (!problem_json || !solution_json) throw twfa::UsageError("NULL argument");
    const twfa::LoweredSchedule s = twfa::parse(problem_json, solution_json);
    const std::string d = twfa::violations_json(twfa::validate_schedule(s));
    if (needed) *needed = d.size() + 1;
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, d.size());
      std::memcpy(buf, d.data(), n);
      buf[n] = '\0';
    }
    return TWFA_OK;
  });
}

int twfa_plan_describe(const twfa_plan* plan, char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    if (!plan) throw twfa::UsageError("plan is NULL");
    const std::string& d = plan->description;
    if (needed) *needed = d.size() + 1;
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, d.size());
      std::memcpy(buf, d.data(), n);
      buf[n] = '\0';
    }
    return TWFA_OK;
  });
}

int twfa_plan_raw(const twfa_plan* plan, void* dst, size_t cap, size_t* needed) {
  return guarded([&] {
    if (!plan) throw twfa::UsageError("plan is NULL");
    if (needed) *needed = sizeof(TwfaDevicePlan);
    if (dst) {
      if (cap < sizeof(TwfaDevicePlan)) throw twfa::UsageError("buffer too small");
      std::memcpy(dst, &plan->sched.plan, sizeof(TwfaDevicePlan));
    }
    return TWFA_OK;
  });
}

int twfa_fa_fwd(const twfa_plan* plan, const void* q, const void* k, const void* v, void* o, float* lse, int B,
                int H, int S, int D, int causal, float softmax_scale, void* stream) {
  return guarded(
      [&] { return fa_fwd_impl(plan, q, k, v, o, lse, B, H, S, D, causal, softmax_scale, nullptr, 0, stream); });
}

int twfa_fa_fwd_traced(const twfa_plan* plan, const void* q, const void* k, const void* v, void* o, float* lse,
                       int B, int H, int S, int D, int causal, float softmax_scale, uint32_t* trace, uint32_t cap,
                       void* stream) {
  return guarded([&] {
    if (!trace || cap < 2) throw twfa::UsageError("trace buffer missing");
    return fa_fwd_impl(plan, q, k, v, o, lse, B, H, S, D, causal, softmax_scale, trace, cap, stream);
  });
}

int twfa_fa_fwd_host(const twfa_plan* plan, const uint16_t* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                     float* lse, int B, int H, int S, int D, int causal, float softmax_scale) {
  return guarded([&] { return fa_fwd_host_impl(plan, q, k, v, o, lse, B, H, S, D, causal, softmax_scale); });
}

int twfa_fa_bwd_workspace_size(int B, int H, int S, int D, size_t* bytes) {
  return guarded([&] {
    if (!bytes) throw twfa::UsageError("NULL argument");
    if (B < 1 || H < 1 || S < 1 || D != 128) throw twfa::UsageError("unsupported shape");
    *bytes = twfa::fa_bwd_workspace_bytes(B, H, S);
    return TWFA_OK;
  });
}

int twfa_fa_bwd(const twfa_plan* plan, const void* q, const void* k, const void* v, const void* o, const void* dout,
                const float* lse, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, int B, int H,
                int S, int D, int causal, float softmax_scale, void* stream) {
  return guarded([&] {
    return fa_bwd_impl(plan, q, k, v, o, dout, lse, dq, dk, dv, workspace, workspace_bytes, B, H, S, D, causal,
                       softmax_scale, stream);
  });
}

int twfa_fa_bwd_traced(const twfa_plan* plan, const void* q, const void* k, const void* v, const void* o,
                       const void* dout, const float* lse, void* dq, void* dk, void* dv, void* workspace,
                       size_t workspace_bytes, int B, int H, int S, int D, int causal, float softmax_scale,
                       uint32_t* trace, uint32_t cap, void* stream) {
  return guarded([&] {
    if (!trace || cap < 2) throw twfa::UsageError("trace buffer missing");
    return fa_bwd_impl(plan, q, k, v, o, dout, lse, dq, dk, dv, workspace, workspace_bytes, B, H, S, D, causal,
                       softmax_scale, stream, trace, cap);
  });
}

int twfa_gemm(const twfa_plan* plan, const void* a, const void* b, void* c, int M, int N, int K, void* stream) {
  return guarded([&] {
    if (!plan) throw twfa::UsageError("plan is NULL");
    const TwfaDevicePlan& p = plan->sched.plan;
    if (p.family != TWFA_FAMILY_GEMM) throw twfa::UsageError("plan is not a GEMM plan");
    if (M <= 0 || N <= 0 || K <= 0 || M % 256 || N % 256 || K % 64)
      throw twfa::UsageError("GEMM needs M % 256 == 0, N % 256 == 0, K % 64 == 0");
    if (p.k_depth < 1 || p.k_depth > 6) throw twfa::UsageError("GEMM ring depth must be 1..6");
    require_aligned(a, "a");
    require_aligned(b, "b");
    require_aligned(c, "c");
    DeviceGuard guard(a, "a");
    const cuuint64_t da[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
    const cuuint64_t db[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N)};
    const cuuint64_t dc[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
    const cuuint64_t st[1] = {static_cast<cuuint64_t>(K) * 2};
    const cuuint64_t stc[1] = {static_cast<cuuint64_t>(N) * 2};
    const cuuint32_t box[2] = {64, 128};  // A, B: 128 rows x 64 k per CTA; C: 128 rows x 64 columns per store
    const CUtensorMap ta = make_map(a, 2, da, st, box);
    const CUtensorMap tb = make_map(b, 2, db, st, box);
    const CUtensorMap tc = make_map(c, 2, dc, stc, box);
    // raster group (pair-tile rows whose A panel stays in L2); TWFA_GEMM_GROUP overrides
    int group_m = 8;
    if (const char* e = std::getenv("TWFA_GEMM_GROUP")) group_m = std::max(1, std::atoi(e));
    int pol_mode = 2;  // A and B evict_last (gemm_sm100.cu)
    if (const char* e = std::getenv("TWFA_GEMM_POL")) pol_mode = std::atoi(e);
    twfa::GemmArgs ga{static_cast<__nv_bfloat16*>(c), M, N, K, group_m, pol_mode};
    // one CTA pair (cluster of 2) per 256 x 256 output tile, persistent
    const int pair_tiles = (M / 256) * (N / 256);
    const int grid = 2 * std::min(pair_tiles, sm_count() / 2);
    check(twfa::gemm_launch(ta, tb, tc, p, ga, grid, static_cast<cudaStream_t>(stream)), "gemm launch");
    return TWFA_OK;
  });
}

int twfa_grid_size(int* out) {
  return guarded([&] {
    if (!out) throw twfa::UsageError("NULL argument");
    *out = sm_count();
    return TWFA_OK;
  });
}

}  // extern "C"
