// libmpcore C ABI: handle table + entry points (include/mpcore.h).
//
// Mirrors the reference's handle-based surface (ffi.py:1-306, build_lib.py:
// 31-208): sequential never-reused uint64 handles, a locked table, a
// mutation latch per object (status 6 on concurrent mutation), exceptions
// mapped to status codes, text in caller-owned buffers.  Objects hold their
// planes in device memory; all compute runs on the library's CUDA stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/mpcore.h"
#include "bignum.h"
#include "internal.h"
#include "longfloat.cuh"
#include "refine_host.h"
#include "testsys.h"
#include "dist.h"
#include <set>

namespace {

constexpr const char *kVersion = "0.1.0";

enum Kind { K_MATRIX = 1, K_VECTOR = 2, K_PIVOT = 3, K_REPORT = 4 };

struct Object {
  int kind = 0;
  int k = 0, rows = 0, cols = 0;
  double *d = nullptr;          // planar device storage (matrix / vector)
  int32_t *dswaps = nullptr;    // pivot record on device
  int32_t *dperm = nullptr;     // composed permutation (PivotRecord.permutation)
  std::vector<int32_t> swaps;   // pivot record on host
  bool busy = false;            // mutation latch (ffi.py:96-105)
  std::unique_ptr<mpr::Report> report;
  cudaEvent_t upload = nullptr; // last asynchronous copy to / from d
  // an asynchronous copy was recorded in `upload` and the library stream
  // has not yet been made to wait for it; set and cleared only under the
  // device lock
  std::atomic<bool> upload_pending{false};
  // MPCORE_DEBUG_GUARD: planes allocated inside guard zones (raw = base
  // of the allocation, d = raw + guard) filled with GUARD_BYTE; checked by
  // mpcore_debug_check_guards
  char *raw = nullptr;
  size_t guard = 0;
  ~Object() {
    if (upload) {  // an asynchronous upload may still target d
      cudaEventSynchronize(upload);
      cudaEventDestroy(upload);
    }
    if (raw) cudaFree(raw);
    else if (d) cudaFree(d);
    if (dswaps) cudaFree(dswaps);
    if (dperm) cudaFree(dperm);
  }
  int64_t count() const { return (int64_t)k * rows * cols; }
};
using ObjPtr = std::shared_ptr<Object>;

// Every handle lookup notes objects with an outstanding asynchronous copy;
// the next DevLock taken by the same thread (before it queues any work on
// the library stream, and never while another thread captures that stream
// into a graph) makes the library stream wait for those copies.
thread_local std::vector<std::shared_ptr<Object>> g_touched;
void object_ready(const std::shared_ptr<Object> &o) {
  if (o->upload_pending.load()) g_touched.push_back(o);
}

struct Table {
  std::mutex mu;
  uint64_t next = 1;
  std::unordered_map<uint64_t, ObjPtr> map;

  uint64_t put(ObjPtr o) {
    std::lock_guard<std::mutex> g(mu);
    uint64_t h = next++;
    map[h] = std::move(o);
    return h;
  }
  ObjPtr get(uint64_t h, int kind) {
    std::lock_guard<std::mutex> g(mu);
    auto it = map.find(h);
    if (it == map.end() || (kind && it->second->kind != kind)) return nullptr;
    object_ready(it->second);
    return it->second;
  }
  bool drop(uint64_t h) {
    std::lock_guard<std::mutex> g(mu);
    return map.erase(h) > 0;
  }
  // -> status; on success o is the latched object
  int latch(uint64_t h, int kind, ObjPtr &o) {
    std::lock_guard<std::mutex> g(mu);
    auto it = map.find(h);
    if (it == map.end() || it->second->kind != kind) return MPCORE_BAD_HANDLE;
    if (it->second->busy) return MPCORE_INTERNAL;
    it->second->busy = true;
    object_ready(it->second);
    o = it->second;
    return MPCORE_OK;
  }
  void unlatch(const ObjPtr &o) {
    std::lock_guard<std::mutex> g(mu);
    o->busy = false;
  }
};

Table &table() {
  static Table t;
  return t;
}

thread_local std::string g_err;

int fail(int st, const std::string &msg) {
  g_err = msg;
  return st;
}

// ---------------------------------------------------------------- device ----
struct Device {
  std::mutex mu;       // serialises device work
  bool tried = false, ok = false;
  int dev = -1, want = -1, sms = 0;
  std::string why;
  cudaStream_t stream = nullptr;
  mpk::LuWork ws;
  mpk::SolveWork sw;
  double *tmp = nullptr;   // scratch vector (aliased solve)
  size_t tmp_bytes = 0;
  int32_t *dswaps = nullptr;  // LU swap output (stable for graph replay)
  int swaps_cap = 0;
  double *aug = nullptr;      // [A | b] workspace of mpcore_solve_system
  size_t aug_bytes = 0;
  // mpcore_set_planes_async: copies on their own stream
  cudaStream_t copy = nullptr;
};

Device &device() {
  static Device d;
  return d;
}

int cuda_fail(cudaError_t e, const char *where) {
  return fail(MPCORE_INTERNAL,
              std::string(where) + ": " + cudaGetErrorString(e));
}

// -> status; initialises the device context once (lock held by caller)
int ensure_device_locked() {
  Device &D = device();
  if (D.tried) return D.ok ? MPCORE_OK : fail(MPCORE_INTERNAL, D.why);
  D.tried = true;
  int want = D.want;
  if (want < 0) {
    const char *env = std::getenv("MPCORE_DEVICE");
    if (env) want = std::atoi(env);
  }
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    D.why = std::string("no CUDA device: ") +
            (e != cudaSuccess ? cudaGetErrorString(e) : "count == 0");
    return fail(MPCORE_INTERNAL, D.why);
  }
  if (want >= 0) {
    e = cudaSetDevice(want);
  } else {
    e = cudaGetDevice(&want);
  }
  if (e != cudaSuccess) {
    D.why = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return fail(MPCORE_INTERNAL, D.why);
  }
  D.dev = want;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, want);
  if (prop.major < 10) {
    D.why = std::string("device ") + prop.name +
            " is not sm_100 class; libmpcore is built for sm_100a only";
    return fail(MPCORE_INTERNAL, D.why);
  }
  D.sms = prop.multiProcessorCount;
  e = cudaStreamCreateWithFlags(&D.stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    D.why = std::string("stream: ") + cudaGetErrorString(e);
    return fail(MPCORE_INTERNAL, D.why);
  }
  if ((e = D.ws.init(D.sms)) != cudaSuccess) {
    D.why = std::string("workspace: ") + cudaGetErrorString(e);
    return fail(MPCORE_INTERNAL, D.why);
  }
  if (const char *t = std::getenv("MPCORE_TRACE_PANEL")) {
    size_t bytes = (size_t)D.sms * 33 * 8 * sizeof(unsigned long long);
    if (cudaMalloc(&D.ws.trace, bytes) == cudaSuccess) {
      cudaMemset(D.ws.trace, 0, bytes);
      D.ws.trace_J = std::atoi(t);
    }
  }
  D.ok = true;
  return MPCORE_OK;
}

cudaEvent_t *event_slots() {
  static cudaEvent_t slots[8] = {};
  return slots;
}

// Holds the device lock; orders the library stream after the asynchronous
// copies of the objects this thread looked up (g_touched).  A flag is
// cleared only once its stream wait has been queued successfully.
struct DevLock {
  std::unique_lock<std::mutex> lk;
  int st;
  DevLock() : lk(device().mu) {
    st = ensure_device_locked();
    std::vector<std::shared_ptr<Object>> touched;
    touched.swap(g_touched);
    if (st) return;
    for (auto &o : touched) {
      if (!o->upload_pending.load()) continue;
      cudaError_t e = cudaStreamWaitEvent(device().stream, o->upload, 0);
      if (e != cudaSuccess) {
        st = cuda_fail(e, "wait for asynchronous copy");
        return;
      }
      o->upload_pending.store(false);
    }
  }
};

int finish(const char *where) {
  Device &D = device();
  cudaError_t e = cudaStreamSynchronize(D.stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, where);
  return MPCORE_OK;
}

int copy_text(const std::string &text, char *buf, int32_t cap) {
  if (buf == nullptr || cap <= 0) return MPCORE_BAD_DIMENSION;
  size_t n = std::min((size_t)(cap - 1), text.size());
  std::memcpy(buf, text.data(), n);
  buf[n] = '\0';
  return n == text.size() ? MPCORE_OK : MPCORE_BAD_DIMENSION;
}

mpk::MatView view(const ObjPtr &o) {
  mpk::MatView v;
  v.p = o->d;
  v.ld = o->cols;
  v.plane = (int64_t)o->rows * o->cols;
  return v;
}

constexpr int kGuardByte = 0xA5;
size_t debug_guard_bytes() {
  const char *g = std::getenv("MPCORE_DEBUG_GUARD");
  return g && *g && *g != '0' ? (size_t)64 * 1024 : 0;
}

int new_container(int kind, int k, int rows, int cols, uint64_t *out) {
  if (out == nullptr) return MPCORE_BAD_DIMENSION;
  *out = 0;
  if (k < 2 || k > 4 || rows < 1 || cols < 1)
    return fail(MPCORE_BAD_DIMENSION, "bad k or shape");
  DevLock L;
  if (L.st) return L.st;
  auto o = std::make_shared<Object>();
  o->kind = kind;
  o->k = k;
  o->rows = rows;
  o->cols = cols;
  size_t bytes = (size_t)o->count() * sizeof(double);
  cudaError_t e;
  if (const size_t g = debug_guard_bytes()) {
    // debug: guard zones on both sides of the planes (write-overrun check)
    e = cudaMalloc(&o->raw, bytes + 2 * g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    o->guard = g;
    o->d = reinterpret_cast<double *>(o->raw + g);
    cudaMemsetAsync(o->raw, kGuardByte, g, device().stream);
    cudaMemsetAsync(o->raw + g + bytes, kGuardByte, g, device().stream);
  } else {
    e = cudaMalloc(&o->d, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  }
  e = cudaMemsetAsync(o->d, 0, bytes, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemset");
  int st = finish("matrix_new");
  if (st) return st;
  *out = table().put(o);
  return MPCORE_OK;
}

ObjPtr container(uint64_t h) {
  ObjPtr o = table().get(h, K_MATRIX);
  if (!o) o = table().get(h, K_VECTOR);
  return o;
}

bool locate(const ObjPtr &o, int i, int j) {
  if (o->kind == K_MATRIX) return 0 <= i && i < o->rows && 0 <= j && j < o->cols;
  return 0 <= i && i < o->rows * o->cols && j == 0;
}

int64_t elem_index(const ObjPtr &o, int i, int j) {
  return o->kind == K_MATRIX ? (int64_t)i * o->cols + j : (int64_t)i;
}

// (device lock held by the caller)
int make_pivot(const std::vector<int32_t> &swaps, uint64_t *out) {
  auto p = std::make_shared<Object>();
  p->kind = K_PIVOT;
  p->rows = (int)swaps.size();
  p->cols = 1;
  p->swaps = swaps;
  cudaError_t e = cudaMalloc(&p->dswaps, swaps.size() * sizeof(int32_t));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(pivot)");
  // uploads on the library stream (where every solve reads them); the
  // host vectors live until finish() below has seen them land
  e = cudaMemcpyAsync(p->dswaps, swaps.data(), swaps.size() * sizeof(int32_t),
                      cudaMemcpyHostToDevice, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "pivot upload");
  // permutation(): position i holds original row order[i] (linalg.py:361-366)
  std::vector<int32_t> order(swaps.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int32_t)i;
  for (size_t j = 0; j < swaps.size(); ++j)
    if (swaps[j] != (int32_t)j) std::swap(order[j], order[swaps[j]]);
  e = cudaMalloc(&p->dperm, order.size() * sizeof(int32_t));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(perm)");
  e = cudaMemcpyAsync(p->dperm, order.data(), order.size() * sizeof(int32_t),
                      cudaMemcpyHostToDevice, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "perm upload");
  int st = finish("pivot upload");
  if (st) return st;
  *out = table().put(p);
  return MPCORE_OK;
}

int default_nb(int k, int n) {
  (void)k;
  (void)n;
  // (experiments: MPCORE_LU_NB overrides the panel width)
  static const int env = [] {
    const char *e = std::getenv("MPCORE_LU_NB");
    return e ? std::atoi(e) : 0;
  }();
  return env > 0 ? env : 32;
}

// factor obj in place; fills swaps; -> status (3 singular)
int factor_locked(const ObjPtr &o, int nb, std::vector<int32_t> &swaps,
                  int32_t *sing) {
  Device &D = device();
  const int n = o->rows;
  cudaError_t e;
  // persistent swap buffer: a stable pointer lets the captured LU graph
  // replay for every matrix of the same shape and address
  if (D.swaps_cap < n) {
    if (D.dswaps) cudaFree(D.dswaps);
    D.dswaps = nullptr;
    D.swaps_cap = 0;
    if ((e = cudaMalloc(&D.dswaps, (size_t)n * sizeof(int32_t))) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc(swaps)");
    D.swaps_cap = n;
  }
  int32_t step = -1;
  e = mpk::lu_factor(o->k, n, n, view(o), D.dswaps,
                     nb > 0 ? nb : default_nb(o->k, n), D.ws, &step, D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "lu_factor");
  swaps.assign(n, 0);
  e = cudaMemcpyAsync(swaps.data(), D.dswaps, n * sizeof(int32_t),
                      cudaMemcpyDeviceToHost, D.stream);
  int st = finish("lu_factor");
  if (st) return st;
  if (e != cudaSuccess) return cuda_fail(e, "swaps download");
  if (sing) *sing = step;
  if (step >= 0)
    return fail(MPCORE_SINGULAR,
                "no nonzero pivot at elimination step " + std::to_string(step));
  return MPCORE_OK;
}

// ---------------------------------------------------------------- prof ----
struct Prof {
  bool on = false;
  struct Rec { int slot; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<int> open;  // stack of indices into recs per slot
  double ms[mpk::PROF_NSLOTS] = {0};
  int64_t launches[mpk::PROF_NSLOTS] = {0};
  int pending[mpk::PROF_NSLOTS];
  cudaEvent_t base = nullptr;     // timeline origin (set by prof_reset)
  std::vector<double> timeline;   // (slot, start us, end us) per launch
  Prof() { for (int &p : pending) p = -1; }
  void collect() {
    for (auto &r : recs) {
      float t = 0;
      if (cudaEventSynchronize(r.b) == cudaSuccess &&
          cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
        ms[r.slot] += t;
        launches[r.slot] += 1;
        float t0 = 0, t1 = 0;
        if (base && timeline.size() < 3 * 200000 &&
            cudaEventElapsedTime(&t0, base, r.a) == cudaSuccess &&
            cudaEventElapsedTime(&t1, base, r.b) == cudaSuccess) {
          timeline.push_back(r.slot);
          timeline.push_back(1e3 * t0);
          timeline.push_back(1e3 * t1);
        }
      }
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    recs.clear();
  }
};
Prof &prof() {
  static Prof p;
  return p;
}

}  // namespace

namespace mpk {
void prof_begin(int slot, cudaStream_t s) {
  Prof &P = prof();
  if (!P.on) return;
  Prof::Rec r;
  r.slot = slot;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s);
  P.pending[slot] = (int)P.recs.size();
  P.recs.push_back(r);
  if (P.recs.size() > 20000) {
    // bound the number of live events
    cudaEventRecord(r.b, s);
    P.pending[slot] = -1;
    P.collect();
  }
}
void prof_end(int slot, cudaStream_t s) {
  Prof &P = prof();
  if (!P.on || P.pending[slot] < 0) return;
  cudaEventRecord(P.recs[P.pending[slot]].b, s);
  P.pending[slot] = -1;
}
bool prof_enabled() { return prof().on; }
int num_sms() { return device().sms > 0 ? device().sms : 148; }
}  // namespace mpk

// ================================================================= ABI ====
extern "C" {

int32_t mpcore_version(char *out, int32_t cap) {
  return copy_text(kVersion, out, cap);
}

int32_t mpcore_simd_enabled(void) {
  const char *v = std::getenv("MPCORE_SIMD");
  if (!v) return 1;
  std::string s(v);
  size_t b = s.find_first_not_of(" \t\r\n"), e = s.find_last_not_of(" \t\r\n");
  s = b == std::string::npos ? "" : s.substr(b, e - b + 1);
  for (auto &c : s) c = (char)std::tolower((unsigned char)c);
  return (s == "0" || s == "off" || s == "false" || s == "no") ? 0 : 1;
}

int32_t mpcore_matrix_new(int32_t k, int32_t rows, int32_t cols,
                          uint64_t *out) {
  return new_container(K_MATRIX, k, rows, cols, out);
}

int32_t mpcore_vector_new(int32_t k, int32_t n, uint64_t *out) {
  return new_container(K_VECTOR, k, n, 1, out);
}

int32_t mpcore_release(uint64_t h) {
  ObjPtr o = table().get(h, 0);
  if (!o) return MPCORE_BAD_HANDLE;
  {
    // free device memory under the device lock (no kernel may be using it)
    DevLock L;
    table().drop(h);
    o.reset();
  }
  return MPCORE_OK;
}

int32_t mpcore_set_element_from_decimal(uint64_t h, int32_t i, int32_t j,
                                        const char *text) {
  if (text == nullptr) return MPCORE_BAD_PARSE;
  ObjPtr o = container(h);
  if (!o) return MPCORE_BAD_HANDLE;
  if (!locate(o, i, j)) return MPCORE_BAD_DIMENSION;
  std::string s(text);
  size_t b = s.find_first_not_of(" \t\r\n\f\v");
  std::string t = b == std::string::npos ? "" : s.substr(b);
  size_t q = t.find_first_not_of("+-");
  bool hex = q != std::string::npos && q + 1 < t.size() && t[q] == '0' &&
             (t[q + 1] == 'x' || t[q + 1] == 'X');
  bn::BF v;
  int st = hex ? bn::parse_hex(s, v) : bn::parse_decimal(s, 53 * o->k + 64, v);
  if (st) return fail(st, "cannot parse element text");
  double comps[4];
  st = bn::to_multicomp(v, o->k, comps);
  if (st) return fail(st, "element does not fit in binary64");
  DevLock L;
  if (L.st) return L.st;
  int64_t idx = elem_index(o, i, j);
  int64_t plane = (int64_t)o->rows * o->cols;
  for (int c = 0; c < o->k; ++c) {
    cudaError_t e = cudaMemcpyAsync(o->d + c * plane + idx, &comps[c],
                                    sizeof(double), cudaMemcpyHostToDevice,
                                    device().stream);
    if (e != cudaSuccess) return cuda_fail(e, "set_element");
  }
  return finish("set_element");
}

int32_t mpcore_get_element_components(uint64_t h, int32_t i, int32_t j,
                                      double *out, int32_t cap) {
  ObjPtr o = container(h);
  if (!o) return MPCORE_BAD_HANDLE;
  if (!locate(o, i, j)) return MPCORE_BAD_DIMENSION;
  if (out == nullptr || cap < o->k) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  int64_t idx = elem_index(o, i, j);
  int64_t plane = (int64_t)o->rows * o->cols;
  for (int c = 0; c < o->k; ++c) {
    cudaError_t e = cudaMemcpyAsync(&out[c], o->d + c * plane + idx,
                                    sizeof(double), cudaMemcpyDeviceToHost,
                                    device().stream);
    if (e != cudaSuccess) return cuda_fail(e, "get_element");
  }
  return finish("get_element");
}

int32_t mpcore_lu_factor_ex(uint64_t h, int32_t nb, uint64_t *piv_out,
                            int32_t *singular_step) {
  if (piv_out == nullptr) return MPCORE_BAD_DIMENSION;
  *piv_out = 0;
  if (singular_step) *singular_step = -1;
  ObjPtr o;
  int st = table().latch(h, K_MATRIX, o);
  if (st) return st;
  struct Unlatch {
    ObjPtr &o;
    ~Unlatch() { table().unlatch(o); }
  } un{o};
  if (o->rows != o->cols)
    return fail(MPCORE_BAD_DIMENSION, "LU needs a square matrix");
  std::vector<int32_t> swaps;
  {
    DevLock L;
    if (L.st) return L.st;
    st = factor_locked(o, nb, swaps, singular_step);
    if (st) return st;
    return make_pivot(swaps, piv_out);
  }
}

static mpk::MatView mv(uint64_t base, int64_t ld, int64_t plane);

// Factor the augmented n x (n+1) matrix [A | b] at aug in place -- the
// right-hand side follows every exchange and update, which is the forward
// substitution of the reference's lu_solve, element by element in its order
// -- then back-substitute into x (planar k x n).  -> status (3 singular)
int solve_augmented_locked(int k, int n, double *aug, int64_t ld,
                           int64_t plane, double *x, int nb,
                           std::vector<int32_t> &swaps, int32_t *sing) {
  Device &D = device();
  cudaError_t e;
  if (D.swaps_cap < n) {
    if (D.dswaps) cudaFree(D.dswaps);
    D.dswaps = nullptr;
    D.swaps_cap = 0;
    if ((e = cudaMalloc(&D.dswaps, (size_t)n * sizeof(int32_t))) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc(swaps)");
    D.swaps_cap = n;
  }
  int32_t step = -1;
  e = mpk::lu_factor(k, n, n + 1, mv((uint64_t)aug, ld, plane), D.dswaps,
                     nb > 0 ? nb : default_nb(k, n), D.ws, &step, D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "lu_factor");
  if (sing) *sing = step;
  if (step >= 0)
    return fail(MPCORE_SINGULAR,
                "no nonzero pivot at elimination step " + std::to_string(step));
  for (int c = 0; c < k && e == cudaSuccess; ++c)
    e = cudaMemcpy2DAsync(x + (size_t)c * n, sizeof(double),
                          aug + (size_t)c * plane + n, (size_t)ld * 8, 8, n,
                          cudaMemcpyDeviceToDevice, D.stream);
  if (e == cudaSuccess)
    e = mpk::lu_solve_back(k, n, mv((uint64_t)aug, ld, plane), x, D.sw,
                           D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "solve_back");
  swaps.assign(n, 0);
  e = cudaMemcpyAsync(swaps.data(), D.dswaps, n * sizeof(int32_t),
                      cudaMemcpyDeviceToHost, D.stream);
  int st = finish("solve_system");
  if (st) return st;
  if (e != cudaSuccess) return cuda_fail(e, "swaps download");
  return MPCORE_OK;
}

int32_t mpcore_lu_factor(uint64_t h, uint64_t *piv_out) {
  return mpcore_lu_factor_ex(h, 0, piv_out, nullptr);
}

int32_t mpcore_lu_solve(uint64_t lu_h, uint64_t piv_h, uint64_t b_h,
                        uint64_t x_h) {
  ObjPtr lu = table().get(lu_h, K_MATRIX);
  ObjPtr piv = table().get(piv_h, K_PIVOT);
  ObjPtr b = table().get(b_h, K_VECTOR);
  if (!lu || !piv || !b) return MPCORE_BAD_HANDLE;
  ObjPtr x;
  int st = table().latch(x_h, K_VECTOR, x);
  if (st) return st;
  struct Unlatch {
    ObjPtr &o;
    ~Unlatch() { table().unlatch(o); }
  } un{x};
  if (x->k != lu->k || b->k != lu->k) return MPCORE_BAD_DIMENSION;
  if (piv->rows != lu->rows || x->rows != lu->rows) return MPCORE_BAD_DIMENSION;
  if (lu->rows != lu->cols) return MPCORE_BAD_DIMENSION;
  if (b->rows != lu->rows) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  const int n = lu->rows;
  cudaError_t e = cudaSuccess;
  const double *src = b->d;
  if (x->d == b->d) {  // in-place solve: stage b in scratch
    size_t bytes = (size_t)b->count() * sizeof(double);
    if (D.tmp_bytes < bytes) {
      if (D.tmp) cudaFree(D.tmp);
      D.tmp = nullptr;
      D.tmp_bytes = 0;
      if ((e = cudaMalloc(&D.tmp, bytes)) != cudaSuccess)
        return cuda_fail(e, "scratch");
      D.tmp_bytes = bytes;
    }
    e = cudaMemcpyAsync(D.tmp, b->d, bytes, cudaMemcpyDeviceToDevice,
                        D.stream);
    if (e != cudaSuccess) return cuda_fail(e, "solve copy");
    src = D.tmp;
  }
  e = mpk::lu_solve(lu->k, n, view(lu), piv->dperm, src, x->d, D.sw,
                    D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "lu_solve");
  return finish("lu_solve");
}

// ------------------------------------------------------------- refine ----
}  // extern "C"

namespace {
// Device buffers of the IR's short side, kept across refinement calls
// (grow-only): the same addresses every call, so the LU's captured launch
// graph (keyed on the matrix pointer) is replayed instead of re-captured.
// One refinement at a time uses it; a concurrent one allocates its own.
struct IrWorkspace {
  std::atomic<bool> busy{false};
  double *a = nullptr, *b = nullptr, *x = nullptr;
  int32_t *perm = nullptr;
  size_t acap = 0, bcap = 0, xcap = 0, pcap = 0;
  // the long residual (residual.cu): page-locked staging of the
  // fixed-width A, its device copy, vectors, and the upload stream
  void *stage = nullptr, *hx = nullptr, *hres = nullptr, *stage_pl = nullptr;
  size_t stagecap = 0, hcap = 0, stage_plcap = 0;
  void *rA = nullptr, *rb = nullptr, *rx = nullptr, *rres = nullptr;
  size_t rAcap = 0, rbcap = 0, rxcap = 0, rrcap = 0;
  // page-locked results of an asynchronous factor_solve: status, swaps, x
  void *hres_fs = nullptr;
  size_t hres_fscap = 0;
  // the device conversion's scratch: bad flag, max exponent, partial sums
  // (device) and their page-locked copies
  void *dconv = nullptr, *hconv = nullptr;
  size_t dconvcap = 0, hconvcap = 0;
  void *rflat = nullptr;  // compact exact values (device)
  size_t rflatcap = 0;
  cudaStream_t up = nullptr;
  cudaEvent_t up_done = nullptr;
};
// (the host's ff::F, uploaded as is)
static_assert(sizeof(lf::DF) == 96 && offsetof(lf::DF, exp) == 8 &&
                  offsetof(lf::DF, m) == 16,
              "lf::DF layout must match ff::F");
constexpr size_t LF_BYTES = sizeof(lf::DF);
cudaError_t grow_dev(void **p, size_t &cap, size_t need) {
  if (cap >= need) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  cap = 0;
  cudaError_t r = cudaMalloc(p, need);
  if (r == cudaSuccess) cap = need;
  return r;
}
cudaError_t grow_host(void **p, size_t &cap, size_t need) {
  if (cap >= need) return cudaSuccess;
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  cap = 0;
  cudaError_t r = cudaHostAlloc(p, need, cudaHostAllocDefault);
  if (r == cudaSuccess) cap = need;
  return r;
}
IrWorkspace &ir_ws() {
  static IrWorkspace w;
  return w;
}

// production variant of the long residual (residual.cu): 5 = products in
// their own kernel, then the chains (default); 2 = products on producer
// warps beside the chain; 0 = warp per row; MPCORE_RESIDUAL_VARIANT
// overrides
int residual_variant() {
  static const int v = [] {
    const char *e = std::getenv("MPCORE_RESIDUAL_VARIANT");
    return e ? std::atoi(e) : 5;
  }();
  return v;
}

// The IR's short side on the GPU: factors stay resident in HBM.
class GpuShortSolver : public mpr::ShortSolver {
 public:
  ~GpuShortSolver() override {
    if (shared_) {
      ir_ws().busy.store(false);
      return;
    }
    if (a_ || perm_ || b_ || x_) {
      // (owned buffers; the shared ones stay in ir_ws() for the next call)
      DevLock L;
      if (a_) cudaFree(a_);
      if (perm_) cudaFree(perm_);
      if (b_) cudaFree(b_);
      if (x_) cudaFree(x_);
    }
  }
  int factor(int k, int n, const double *a,
             std::string &err) override {
    k_ = k;
    n_ = n;
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    cudaError_t e = cudaSuccess;
    size_t mb = (size_t)k * n * n * sizeof(double), vb = (size_t)k * n * 8;
    if ((e = ensure_buffers(mb, vb, (size_t)n * 4)) != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    if ((e = cudaMemcpyAsync(a_, a, mb, cudaMemcpyHostToDevice, D.stream)) !=
            cudaSuccess ||
        (e = cudaStreamSynchronize(D.stream)) != cudaSuccess ||
        (e = start_upload()) != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    auto o = std::make_shared<Object>();  // borrow the factor path
    o->kind = K_MATRIX;
    o->k = k;
    o->rows = o->cols = n;
    o->d = a_;
    std::vector<int32_t> swaps;
    int32_t step = -1;
    int st = factor_locked(o, 0, swaps, &step);
    o->d = nullptr;  // not owned
    if (st) { err = g_err; return st; }
    std::vector<int32_t> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int j = 0; j < n; ++j)
      if (swaps[j] != j) std::swap(order[j], order[swaps[j]]);
    // ordered on the library stream (the solves read perm_ there); the
    // host vector stays alive until the copy has landed
    if ((e = cudaMemcpyAsync(perm_, order.data(), (size_t)n * 4,
                             cudaMemcpyHostToDevice, D.stream)) != cudaSuccess ||
        (e = cudaStreamSynchronize(D.stream)) != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    ld_ = n;
    return MPCORE_OK;
  }
  // factor + first solve in one call: b rides along the factorisation as
  // column n of [A | b] (its forward substitution), then the back
  // substitution (solve_augmented_locked, bitwise factor + solve); the
  // factors stay in place with row stride n + 1 for the later solves
  int factor_solve(int k, int n, const double *a, const std::vector<double> &b,
                   std::vector<double> &x, std::string &err) override {
    k_ = k;
    n_ = n;
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    cudaError_t e = cudaSuccess;
    const size_t plane = (size_t)n * (n + 1);
    const size_t mb = (size_t)k * plane * sizeof(double), vb = (size_t)k * n * 8;
    e = ensure_buffers(mb, vb, (size_t)n * 4);
    for (int c = 0; c < k && e == cudaSuccess; ++c) {
      e = cudaMemcpy2DAsync(a_ + c * plane, (n + 1) * 8, a + (size_t)c * n * n,
                            (size_t)n * 8, (size_t)n * 8, n,
                            cudaMemcpyHostToDevice, D.stream);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(a_ + c * plane + n, (n + 1) * 8,
                              b.data() + (size_t)c * n, 8, 8, n,
                              cudaMemcpyHostToDevice, D.stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(D.stream);
    if (e == cudaSuccess) e = start_upload();
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    std::vector<int32_t> swaps;
    int32_t step = -1;
    int st = solve_augmented_locked(k, n, a_, n + 1, (int64_t)plane, x_, 0,
                                    swaps, &step);
    if (st) { err = g_err; return st; }
    ld_ = n + 1;
    x.resize((size_t)k * n);
    std::vector<int32_t> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int j = 0; j < n; ++j)
      if (swaps[j] != j) std::swap(order[j], order[swaps[j]]);
    if ((e = cudaMemcpyAsync(x.data(), x_, vb, cudaMemcpyDeviceToHost,
                             D.stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(perm_, order.data(), (size_t)n * 4,
                             cudaMemcpyHostToDevice, D.stream)) != cudaSuccess ||
        (e = cudaStreamSynchronize(D.stream)) != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    return MPCORE_OK;
  }
  // the same, asynchronously: the uploads, the LU of [A | b], the back
  // substitution and the copies of status, swaps and x into page-locked
  // memory are enqueued and begin returns; end waits for them
  int factor_solve_begin(int k, int n, const double *a,
                         const std::vector<double> &b,
                         std::string &err) override {
    if (!claim()) return -1;
    k_ = k;
    n_ = n;
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    IrWorkspace &w = ir_ws();
    cudaError_t e = cudaSuccess;
    const size_t plane = (size_t)n * (n + 1);
    const size_t mb = (size_t)k * plane * sizeof(double), vb = (size_t)k * n * 8;
    const size_t hb = 16 + (size_t)n * 4 + vb;
    if ((e = ensure_buffers(mb, vb, (size_t)n * 4)) == cudaSuccess)
      e = grow_host(&w.hres_fs, w.hres_fscap, hb);
    if (e == cudaSuccess && D.swaps_cap < n) {
      if (D.dswaps) cudaFree(D.dswaps);
      D.dswaps = nullptr;
      D.swaps_cap = 0;
      if ((e = cudaMalloc(&D.dswaps, (size_t)n * sizeof(int32_t))) ==
          cudaSuccess)
        D.swaps_cap = n;
    }
    for (int c = 0; c < k && e == cudaSuccess; ++c) {
      // (A's planes are already in place when the device converted them)
      if (!a_on_device_)
        e = cudaMemcpy2DAsync(a_ + c * plane, (n + 1) * 8,
                              a + (size_t)c * n * n, (size_t)n * 8,
                              (size_t)n * 8, n, cudaMemcpyHostToDevice,
                              D.stream);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(a_ + c * plane + n, (n + 1) * 8,
                              b.data() + (size_t)c * n, 8, 8, n,
                              cudaMemcpyHostToDevice, D.stream);
    }
    char *h = static_cast<char *>(w.hres_fs);
    mpk::MatView v{a_, n + 1, (int64_t)plane};
    if (e == cudaSuccess)
      e = mpk::lu_factor_async(k, n, n + 1, v, D.dswaps, default_nb(k, n),
                               D.ws, D.stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h, D.ws.status, 4, cudaMemcpyDeviceToHost,
                          D.stream);
    for (int c = 0; c < k && e == cudaSuccess; ++c)
      e = cudaMemcpy2DAsync(x_ + (size_t)c * n, sizeof(double),
                            a_ + (size_t)c * plane + n, (size_t)(n + 1) * 8, 8,
                            n, cudaMemcpyDeviceToDevice, D.stream);
    // (the back substitution reads garbage after a singular step; end
    // reports the step and never uses it)
    if (e == cudaSuccess) e = mpk::lu_solve_back(k, n, v, x_, D.sw, D.stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h + 16, D.dswaps, (size_t)n * 4,
                          cudaMemcpyDeviceToHost, D.stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h + 16 + (size_t)n * 4, x_, vb,
                          cudaMemcpyDeviceToHost, D.stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    ld_ = n + 1;
    inflight_ = true;
    return MPCORE_OK;
  }
  int factor_solve_end(std::vector<double> &x, std::string &err) override {
    if (!inflight_) { err = "no factorisation in flight"; return MPCORE_INTERNAL; }
    inflight_ = false;
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    cudaError_t e = cudaStreamSynchronize(D.stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    const int n = n_, k = k_;
    const char *h = static_cast<const char *>(ir_ws().hres_fs);
    int32_t step;
    std::memcpy(&step, h, 4);
    if (step >= 0) {
      err = "no nonzero pivot at elimination step " + std::to_string(step);
      return MPCORE_SINGULAR;
    }
    const int32_t *swaps = reinterpret_cast<const int32_t *>(h + 16);
    std::vector<int32_t> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int j = 0; j < n; ++j)
      if (swaps[j] != j) std::swap(order[j], order[swaps[j]]);
    x.resize((size_t)k * n);
    std::memcpy(x.data(), h + 16 + (size_t)n * 4, x.size() * sizeof(double));
    if ((e = cudaMemcpyAsync(perm_, order.data(), (size_t)n * 4,
                             cudaMemcpyHostToDevice, D.stream)) != cudaSuccess ||
        (e = cudaStreamSynchronize(D.stream)) != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    return MPCORE_OK;
  }
  // ---- the long -> short conversion on the device (convert.cu) ----
  bool device_convert_supported(int p) override {
    return p <= 512 && claim();
  }
  int device_convert_begin(int k, int n, int p, const void *flat,
                           bool compact, std::string &err) override {
    if (!claim()) { err = "no conversion workspace"; return MPCORE_INTERNAL; }
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    IrWorkspace &w = ir_ws();
    if (flat != w.stage) { err = "flat input must be staging slot 0"; return MPCORE_INTERNAL; }
    const size_t nn = (size_t)n * n, plane = (size_t)n * (n + 1);
    const size_t sc = 16 + (size_t)mpk::long_to_short_partials() * sizeof(double);
    cudaError_t e = ensure_buffers((size_t)k * plane * sizeof(double),
                                   (size_t)k * n * 8, (size_t)n * 4);
    if (e == cudaSuccess) e = grow_dev(&w.rA, w.rAcap, nn * LF_BYTES);
    if (e == cudaSuccess && compact)
      e = grow_dev(&w.rflat, w.rflatcap, nn * sizeof(mpk::LongFlat9));
    if (e == cudaSuccess) e = grow_dev(&w.dconv, w.dconvcap, sc);
    if (e == cudaSuccess) e = grow_host(&w.hconv, w.hconvcap, sc);
    char *dc = static_cast<char *>(w.dconv);
    if (e == cudaSuccess)
      e = mpk::long_to_short_init(reinterpret_cast<int *>(dc),
                                  reinterpret_cast<int *>(dc + 4), D.stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    ck_ = k;
    cn_ = n;
    cp_ = p;
    compact_ = compact;
    return MPCORE_OK;
  }
  int device_convert_rows(int r0, int r1, std::string &err) override {
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    IrWorkspace &w = ir_ws();
    const int n = cn_;
    const size_t plane = (size_t)n * (n + 1);
    char *dc = static_cast<char *>(w.dconv);
    const size_t rec = compact_ ? sizeof(mpk::LongFlat9) : LF_BYTES;
    const size_t off = (size_t)r0 * n * rec;
    void *dst = compact_ ? w.rflat : w.rA;
    cudaError_t e = cudaMemcpyAsync(static_cast<char *>(dst) + off,
                                    static_cast<char *>(w.stage) + off,
                                    (size_t)(r1 - r0) * n * rec,
                                    cudaMemcpyHostToDevice, D.stream);
    if (e == cudaSuccess)
      e = mpk::long_to_short_rows(ck_, n, cp_, w.rA,
                                  compact_ ? w.rflat : nullptr, r0, r1, a_,
                                  n + 1, (int64_t)plane,
                                  reinterpret_cast<int *>(dc),
                                  reinterpret_cast<int *>(dc + 4), D.stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    return MPCORE_OK;
  }
  int device_convert_end(int *emax, double *hsum, std::string &err) override {
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    IrWorkspace &w = ir_ws();
    const int np = mpk::long_to_short_partials();
    const size_t sc = 16 + (size_t)np * sizeof(double);
    char *dc = static_cast<char *>(w.dconv), *hc = static_cast<char *>(w.hconv);
    cudaError_t e = mpk::long_to_short_stats(
        cn_, a_, cn_ + 1, reinterpret_cast<const int *>(dc + 4),
        reinterpret_cast<double *>(dc + 16), D.stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hc, dc, sc, cudaMemcpyDeviceToHost, D.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(D.stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    int bad;
    std::memcpy(&bad, hc, 4);
    std::memcpy(emax, hc + 4, 4);
    double s = 0.0;
    for (int i = 0; i < np; ++i) {
      double v;
      std::memcpy(&v, hc + 16 + (size_t)i * sizeof(double), sizeof v);
      s += v;
    }
    *hsum = s;
    if (bad) return MPCORE_OVERFLOW;  // a head outside binary64: host path
    rn_ = cn_;
    a_on_device_ = true;
    af_on_device_ = true;
    return MPCORE_OK;
  }
  int download_long_A(void *dst, std::string &err) override {
    if (!af_on_device_) { err = "no device copy of A"; return MPCORE_INTERNAL; }
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    IrWorkspace &w = ir_ws();
    cudaError_t e = cudaMemcpyAsync(dst, w.rA, (size_t)rn_ * rn_ * LF_BYTES,
                                    cudaMemcpyDeviceToHost, device().stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(device().stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    return MPCORE_OK;
  }
  // ---- the long residual on the device (residual.cu) ----
  bool residual_supported(int p) override { return p <= 512 && claim(); }
  void *staging(int slot, size_t bytes) override {
    if (!claim() || slot < 0 || slot > 1) return nullptr;
    DevLock L;
    if (L.st) return nullptr;
    IrWorkspace &w = ir_ws();
    void **p = slot == 0 ? &w.stage : &w.stage_pl;
    size_t &cap = slot == 0 ? w.stagecap : w.stage_plcap;
    if (grow_host(p, cap, bytes) != cudaSuccess) return nullptr;
    return *p;
  }
  int residual_setup(int n, int p, const void *A, const void *b,
                     std::string &err) override {
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    if (!shared_) { err = "no residual workspace"; return MPCORE_INTERNAL; }
    IrWorkspace &w = ir_ws();
    const size_t mb = (size_t)n * n * LF_BYTES, vb = (size_t)n * LF_BYTES;
    cudaError_t e = cudaSuccess;
    if (!w.up) {
      if ((e = cudaStreamCreateWithFlags(&w.up, cudaStreamNonBlocking)) ==
          cudaSuccess)
        e = cudaEventCreateWithFlags(&w.up_done, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = grow_dev(&w.rA, w.rAcap, mb);
    if (e == cudaSuccess) e = grow_dev(&w.rb, w.rbcap, vb);
    if (e == cudaSuccess) e = grow_dev(&w.rx, w.rxcap, vb);
    if (e == cudaSuccess) e = grow_dev(&w.rres, w.rrcap, vb);
    if (e == cudaSuccess) e = grow_host(&w.hx, w.hcap, 2 * vb);
    if (e == cudaSuccess && A != w.stage) e = cudaErrorInvalidValue;
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    std::memcpy(w.hx, b, vb);
    rn_ = n;
    rp_ = p;
    upload_pending_ = true;  // issued once the short matrix is on the GPU
    if (inflight_) {         // (it already is: the factorisation is running)
      if ((e = start_upload()) != cudaSuccess) {
        err = cudaGetErrorString(e);
        return MPCORE_INTERNAL;
      }
    }
    return MPCORE_OK;
  }
  // the long A (page-locked staging) and b to the device, asynchronously:
  // started by factor() right after its own upload, so the two copies do
  // not share the link and this one overlaps the LU
  cudaError_t start_upload() {
    if (!upload_pending_) return cudaSuccess;
    upload_pending_ = false;
    IrWorkspace &w = ir_ws();
    const size_t mb = (size_t)rn_ * rn_ * LF_BYTES, vb = (size_t)rn_ * LF_BYTES;
    cudaError_t e = cudaSuccess;
    if (!af_on_device_)  // (else the device conversion wrote it)
      e = cudaMemcpyAsync(w.rA, w.stage, mb, cudaMemcpyHostToDevice, w.up);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.rb, w.hx, vb, cudaMemcpyHostToDevice, w.up);
    if (e == cudaSuccess) e = cudaEventRecord(w.up_done, w.up);
    return e;
  }
  int residual(const void *x, void *res, std::string &err) override {
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    IrWorkspace &w = ir_ws();
    Device &D = device();
    const size_t vb = (size_t)rn_ * LF_BYTES;
    cudaError_t e = start_upload();  // (if factor() has not started it)
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    // b's upload reads the same page-locked buffer x goes through: let it
    // finish first (a no-op after the first residual)
    e = cudaStreamSynchronize(w.up);
    char *hx = static_cast<char *>(w.hx), *hres = hx + vb;
    std::memcpy(hx, x, vb);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.rx, hx, vb, cudaMemcpyHostToDevice, D.stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(D.stream, w.up_done, 0);
    if (e == cudaSuccess)
      e = mpk::long_residual(rp_, rn_, w.rA, w.rx, w.rb, w.rres, D.stream,
                             residual_variant());
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hres, w.rres, vb, cudaMemcpyDeviceToHost, D.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(D.stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    std::memcpy(res, hres, vb);
    return MPCORE_OK;
  }

  int solve(const std::vector<double> &b, std::vector<double> &x,
            std::string &err) override {
    DevLock L;
    if (L.st) { err = g_err; return L.st; }
    Device &D = device();
    size_t vb = (size_t)k_ * n_ * 8;
    cudaError_t e = cudaMemcpyAsync(b_, b.data(), vb, cudaMemcpyHostToDevice,
                                    D.stream);
    mpk::MatView v{a_, ld_, (int64_t)n_ * ld_};
    if (e == cudaSuccess)
      e = mpk::lu_solve(k_, n_, v, perm_, b_, x_, D.sw, D.stream);
    x.resize((size_t)k_ * n_);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(x.data(), x_, vb, cudaMemcpyDeviceToHost, D.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(D.stream);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return MPCORE_INTERNAL;
    }
    return MPCORE_OK;
  }

 private:
  // device buffers for a factorisation of mb matrix bytes, vb vector bytes
  // and pb permutation bytes: the shared workspace (grow-only) if this
  // solver holds it, else buffers owned by the solver; both are re-checked
  // on every factor / factor_solve, so a larger n or the n x (n+1) layout
  // after an n x n factor never writes past an allocation
  cudaError_t ensure_buffers(size_t mb, size_t vb, size_t pb) {
    cudaError_t e = cudaSuccess;
    if (claim()) {
      IrWorkspace &w = ir_ws();
      if ((e = grow_dev((void **)&w.a, w.acap, mb)) == cudaSuccess &&
          (e = grow_dev((void **)&w.b, w.bcap, vb)) == cudaSuccess &&
          (e = grow_dev((void **)&w.x, w.xcap, vb)) == cudaSuccess)
        e = grow_dev((void **)&w.perm, w.pcap, pb);
      a_ = w.a;
      b_ = w.b;
      x_ = w.x;
      perm_ = w.perm;
      return e;
    }
    if ((e = grow_dev((void **)&a_, acap_, mb)) == cudaSuccess &&
        (e = grow_dev((void **)&b_, bcap_, vb)) == cudaSuccess &&
        (e = grow_dev((void **)&x_, xcap_, vb)) == cudaSuccess)
      e = grow_dev((void **)&perm_, pcap_, pb);
    return e;
  }
  // the shared workspace, if no other refinement holds it (asked once)
  bool claim() {
    if (!tried_) {
      tried_ = true;
      bool expected = false;
      shared_ = ir_ws().busy.compare_exchange_strong(expected, true);
    }
    return shared_;
  }
  int k_ = 0, n_ = 0, rn_ = 0, rp_ = 0;
  int ld_ = 0;  // row stride of the factors (n, or n + 1 after factor_solve)
  bool upload_pending_ = false;
  bool inflight_ = false;  // factor_solve_begin without its end yet
  int ck_ = 0, cn_ = 0, cp_ = 0;  // the conversion in flight
  bool compact_ = false;
  bool a_on_device_ = false;   // device_convert filled a_'s A planes
  bool af_on_device_ = false;  // ... and the rounded long A (w.rA)
  bool tried_ = false;
  bool shared_ = false;  // buffers borrowed from ir_ws()
  double *a_ = nullptr, *b_ = nullptr, *x_ = nullptr;
  int32_t *perm_ = nullptr;
  size_t acap_ = 0, bcap_ = 0, xcap_ = 0, pcap_ = 0;  // owned buffers only
};
}  // namespace

extern "C" {

int32_t mpcore_solve_system(uint64_t a_h, uint64_t b_h, uint64_t x_h,
                            int32_t nb, uint64_t *piv_out,
                            int32_t *singular_step) {
  if (piv_out == nullptr) return MPCORE_BAD_DIMENSION;
  *piv_out = 0;
  if (singular_step) *singular_step = -1;
  ObjPtr b = table().get(b_h, K_VECTOR);
  if (!b) return MPCORE_BAD_HANDLE;
  ObjPtr a, x;
  int st = table().latch(a_h, K_MATRIX, a);
  if (st) return st;
  struct Unlatch {
    ObjPtr &o;
    ~Unlatch() { if (o) table().unlatch(o); }
  } ua{a};
  st = table().latch(x_h, K_VECTOR, x);
  if (st) return st;
  Unlatch ux{x};
  const int n = a->rows, k = a->k;
  if (a->rows != a->cols || b->rows != n || x->rows != n || b->k != k ||
      x->k != k)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  const int64_t ld = n + 1, plane = (int64_t)n * ld;
  const size_t bytes = (size_t)k * plane * sizeof(double);
  cudaError_t e = cudaSuccess;
  if (D.aug_bytes < bytes) {
    if (D.aug) cudaFree(D.aug);
    D.aug = nullptr;
    D.aug_bytes = 0;
    if ((e = cudaMalloc(&D.aug, bytes)) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc(augmented)");
    D.aug_bytes = bytes;
  }
  for (int c = 0; c < k && e == cudaSuccess; ++c) {
    e = cudaMemcpy2DAsync(D.aug + c * plane, ld * 8, a->d + (size_t)c * n * n,
                          (size_t)n * 8, (size_t)n * 8, n,
                          cudaMemcpyDeviceToDevice, D.stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(D.aug + c * plane + n, ld * 8, b->d + (size_t)c * n,
                            8, 8, n, cudaMemcpyDeviceToDevice, D.stream);
  }
  if (e != cudaSuccess) return cuda_fail(e, "augment");
  std::vector<int32_t> swaps;
  st = solve_augmented_locked(k, n, D.aug, ld, plane, x->d, nb, swaps,
                              singular_step);
  if (st) return st;
  // the factors back into A, as mpcore_lu_factor leaves them
  for (int c = 0; c < k && e == cudaSuccess; ++c)
    e = cudaMemcpy2DAsync(a->d + (size_t)c * n * n, (size_t)n * 8,
                          D.aug + c * plane, ld * 8, (size_t)n * 8, n,
                          cudaMemcpyDeviceToDevice, D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "factors copy");
  st = finish("solve_system");
  if (st) return st;
  return make_pivot(swaps, piv_out);
}

int32_t mpcore_dev_solve_system(int32_t k, int32_t n, uint64_t aug,
                                int64_t ld, int64_t plane, int32_t nb,
                                uint64_t x, int32_t *swaps_out,
                                int32_t *singular_step) {
  if (k < 2 || k > 4 || n < 1 || !aug || !x || ld < n + 1 ||
      plane < (int64_t)n * ld)
    return MPCORE_BAD_DIMENSION;
  if (singular_step) *singular_step = -1;
  DevLock L;
  if (L.st) return L.st;
  std::vector<int32_t> swaps;
  int st = solve_augmented_locked(k, n, reinterpret_cast<double *>(aug), ld,
                                  plane, reinterpret_cast<double *>(x), nb,
                                  swaps, singular_step);
  if (st) return st;
  if (swaps_out) std::copy(swaps.begin(), swaps.end(), swaps_out);
  return MPCORE_OK;
}

int32_t mpcore_refine(const char *a_path, const char *b_path, int32_t short_k,
                      int32_t long_bits, const char *rtol, const char *atol,
                      int32_t max_iter, uint64_t *report_out) {
  if (report_out == nullptr) return MPCORE_BAD_DIMENSION;
  *report_out = 0;
  if (!a_path || !b_path || !rtol || !atol) return MPCORE_BAD_PARSE;
  auto rep = std::make_unique<mpr::Report>();
  std::string err;
  GpuShortSolver gpu;
  int st = mpr::refine_files(a_path, b_path, short_k, long_bits, rtol, atol,
                             max_iter, gpu, *rep, err);
  if (st) return fail(st, err);
  auto o = std::make_shared<Object>();
  o->kind = K_REPORT;
  o->report = std::move(rep);
  *report_out = table().put(o);
  return MPCORE_OK;
}

int32_t mpcore_refine_config3(int32_t n, uint64_t seed, double kappa_exp10,
                              int32_t short_k, int32_t long_bits,
                              const char *rtol, const char *atol,
                              int32_t max_iter, int32_t threads,
                              uint64_t *report_out) {
  if (report_out == nullptr) return MPCORE_BAD_DIMENSION;
  *report_out = 0;
  if (!rtol || !atol) return MPCORE_BAD_PARSE;
  if (n < 1 || n > 65536) return MPCORE_BAD_DIMENSION;
  auto rep = std::make_unique<mpr::Report>();
  std::string err;
  std::vector<bn::BF> A, b;
  const auto t0 = std::chrono::steady_clock::now();
  int st = mpr::config3_system(n, seed, long_bits, kappa_exp10, threads, A, b,
                               err);
  if (st) return fail(st, err);
  const double t_gen = std::chrono::duration<double>(
                           std::chrono::steady_clock::now() - t0)
                           .count();
  GpuShortSolver gpu;
  st = mpr::refine_core(A, b, n, short_k, long_bits, rtol, atol, max_iter,
                        threads, gpu, *rep, err);
  if (st) return fail(st, err);
  rep->timings.insert(rep->timings.begin(), t_gen);
  auto o = std::make_shared<Object>();
  o->kind = K_REPORT;
  o->report = std::move(rep);
  *report_out = table().put(o);
  return MPCORE_OK;
}

int32_t mpcore_write_config3(int32_t n, uint64_t seed, double kappa_exp10,
                             int32_t long_bits, int32_t threads,
                             const char *a_path, const char *b_path) {
  if (!a_path || !b_path) return MPCORE_BAD_PARSE;
  if (n < 1 || n > 65536 || long_bits < 2) return MPCORE_BAD_DIMENSION;
  std::string err;
  std::vector<bn::BF> A, b;
  int st = mpr::config3_system(n, seed, long_bits, kappa_exp10, threads, A, b,
                               err);
  if (!st) st = mpr::write_mpmat(a_path, A, n, n, long_bits, err);
  if (!st) st = mpr::write_mpmat(b_path, b, n, 1, long_bits, err);
  if (st) return fail(st, err);
  return MPCORE_OK;
}

static mpr::Report *report_of(uint64_t h) {
  ObjPtr o = table().get(h, K_REPORT);
  return o ? o->report.get() : nullptr;
}

int32_t mpcore_report_timings(uint64_t h, double *out, int32_t cap,
                              int32_t *count) {
  mpr::Report *r = report_of(h);
  if (!r) return MPCORE_BAD_HANDLE;
  if (count) *count = (int32_t)r->timings.size();
  for (int32_t i = 0; out && i < cap && i < (int32_t)r->timings.size(); ++i)
    out[i] = r->timings[i];
  return MPCORE_OK;
}

int32_t mpcore_report_iterations(uint64_t h, int32_t *out) {
  mpr::Report *r = report_of(h);
  if (!r) return MPCORE_BAD_HANDLE;
  if (!out) return MPCORE_BAD_DIMENSION;
  *out = r->iterations;
  return MPCORE_OK;
}

int32_t mpcore_report_stop_reason(uint64_t h, char *out, int32_t cap) {
  mpr::Report *r = report_of(h);
  if (!r) return MPCORE_BAD_HANDLE;
  return copy_text(r->stop_reason, out, cap);
}

int32_t mpcore_report_residual_count(uint64_t h, int32_t *out) {
  mpr::Report *r = report_of(h);
  if (!r) return MPCORE_BAD_HANDLE;
  if (!out) return MPCORE_BAD_DIMENSION;
  *out = (int32_t)r->residuals.size();
  return MPCORE_OK;
}

int32_t mpcore_report_residual_entry(uint64_t h, int32_t idx, int32_t digits,
                                     char *out, int32_t cap) {
  mpr::Report *r = report_of(h);
  if (!r) return MPCORE_BAD_HANDLE;
  if (idx < 0 || idx >= (int32_t)r->residuals.size())
    return MPCORE_BAD_DIMENSION;
  return copy_text(mpr::format_decimal(r->residuals[idx], digits, r->prec), out,
                   cap);
}

int32_t mpcore_report_solution_count(uint64_t h, int32_t *out) {
  mpr::Report *r = report_of(h);
  if (!r) return MPCORE_BAD_HANDLE;
  if (!out) return MPCORE_BAD_DIMENSION;
  *out = (int32_t)r->solution.size();
  return MPCORE_OK;
}

int32_t mpcore_report_solution_entry(uint64_t h, int32_t idx, int32_t digits,
                                     char *out, int32_t cap) {
  mpr::Report *r = report_of(h);
  if (!r) return MPCORE_BAD_HANDLE;
  if (idx < 0 || idx >= (int32_t)r->solution.size())
    return MPCORE_BAD_DIMENSION;
  return copy_text(mpr::format_decimal(r->solution[idx], digits, r->prec), out,
                   cap);
}

// --------------------------------------------------------- extensions ----
int32_t mpcore_object_info(uint64_t h, int32_t *kind, int32_t *k,
                           int32_t *rows, int32_t *cols) {
  ObjPtr o = table().get(h, 0);
  if (!o) return MPCORE_BAD_HANDLE;
  if (kind) *kind = o->kind;
  if (k) *k = o->k;
  if (rows) *rows = o->rows;
  if (cols) *cols = o->cols;
  return MPCORE_OK;
}

int32_t mpcore_set_planes(uint64_t h, const double *planes, int64_t count) {
  ObjPtr o;
  int st = 0;
  o = table().get(h, 0);
  if (!o || (o->kind != K_MATRIX && o->kind != K_VECTOR))
    return MPCORE_BAD_HANDLE;
  st = table().latch(h, o->kind, o);
  if (st) return st;
  struct Unlatch {
    ObjPtr &o;
    ~Unlatch() { table().unlatch(o); }
  } un{o};
  if (planes == nullptr || count != o->count()) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = cudaMemcpyAsync(o->d, planes, (size_t)count * sizeof(double),
                                  cudaMemcpyHostToDevice, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "set_planes");
  return finish("set_planes");
}

// Asynchronous upload: the copy runs on its own stream, overlapping
// whatever the library stream is computing; the next library call that
// looks the object up orders the library stream after it.  The host buffer (page-locked for a
// truly asynchronous copy) must stay unchanged until such a call returns.
int32_t mpcore_set_planes_async(uint64_t h, const double *planes,
                                int64_t count) {
  ObjPtr o = table().get(h, 0);
  if (!o || (o->kind != K_MATRIX && o->kind != K_VECTOR))
    return MPCORE_BAD_HANDLE;
  if (o->busy) return MPCORE_INTERNAL;  // latched by a running mutator
  if (planes == nullptr || count != o->count()) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  cudaError_t e = cudaSuccess;
  if (!D.copy) e = cudaStreamCreateWithFlags(&D.copy, cudaStreamNonBlocking);
  if (e == cudaSuccess && !o->upload)
    e = cudaEventCreateWithFlags(&o->upload, cudaEventDisableTiming);
  // after the library stream's queued work (which may still read the
  // object), then the copy
  cudaEvent_t after = nullptr;
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&after, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(after, D.stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(D.copy, after, 0);
  if (after) cudaEventDestroy(after);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(o->d, planes, (size_t)count * sizeof(double),
                        cudaMemcpyHostToDevice, D.copy);
  if (e == cudaSuccess) e = cudaEventRecord(o->upload, D.copy);
  if (e != cudaSuccess) return cuda_fail(e, "set_planes_async");
  o->upload_pending.store(true);
  return MPCORE_OK;
}

// Asynchronous download: after the library stream's queued work on the
// object, on the copy stream; `out` is valid after mpcore_sync.  Later
// library work that writes the object waits for the copy.
int32_t mpcore_get_planes_async(uint64_t h, double *out, int64_t cap) {
  ObjPtr o = table().get(h, 0);
  if (!o || (o->kind != K_MATRIX && o->kind != K_VECTOR))
    return MPCORE_BAD_HANDLE;
  if (o->busy) return MPCORE_INTERNAL;
  if (out == nullptr || cap < o->count()) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  cudaError_t e = cudaSuccess;
  if (!D.copy) e = cudaStreamCreateWithFlags(&D.copy, cudaStreamNonBlocking);
  if (e == cudaSuccess && !o->upload)
    e = cudaEventCreateWithFlags(&o->upload, cudaEventDisableTiming);
  cudaEvent_t after = nullptr;
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&after, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(after, D.stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(D.copy, after, 0);
  if (after) cudaEventDestroy(after);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, o->d, (size_t)o->count() * sizeof(double),
                        cudaMemcpyDeviceToHost, D.copy);
  if (e == cudaSuccess) e = cudaEventRecord(o->upload, D.copy);
  if (e != cudaSuccess) return cuda_fail(e, "get_planes_async");
  o->upload_pending.store(true);
  return MPCORE_OK;
}

int32_t mpcore_get_planes(uint64_t h, double *out, int64_t cap) {
  ObjPtr o = container(h);
  if (!o) return MPCORE_BAD_HANDLE;
  if (out == nullptr || cap < o->count()) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = cudaMemcpyAsync(out, o->d, (size_t)o->count() * sizeof(double),
                                  cudaMemcpyDeviceToHost, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "get_planes");
  return finish("get_planes");
}

int32_t mpcore_copy(uint64_t src, uint64_t dst) {
  ObjPtr s = container(src);
  ObjPtr d = container(dst);
  if (!s || !d) return MPCORE_BAD_HANDLE;
  if (s->kind != d->kind || s->k != d->k || s->rows != d->rows ||
      s->cols != d->cols)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  if (s->d == d->d) return MPCORE_OK;
  cudaError_t e = cudaMemcpyAsync(d->d, s->d, (size_t)s->count() * sizeof(double),
                                  cudaMemcpyDeviceToDevice, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "copy");
  return finish("copy");
}

int32_t mpcore_pivot_new(int32_t n, const int32_t *swaps, uint64_t *out) {
  if (out == nullptr) return MPCORE_BAD_DIMENSION;
  *out = 0;
  if (n < 1 || swaps == nullptr) return MPCORE_BAD_DIMENSION;
  for (int j = 0; j < n; ++j)
    if (swaps[j] < j || swaps[j] >= n)
      return fail(MPCORE_BAD_DIMENSION, "invalid swap");
  DevLock L;
  if (L.st) return L.st;
  return make_pivot(std::vector<int32_t>(swaps, swaps + n), out);
}

int32_t mpcore_pivot_get(uint64_t h, int32_t *out, int32_t cap) {
  ObjPtr p = table().get(h, K_PIVOT);
  if (!p) return MPCORE_BAD_HANDLE;
  if (out == nullptr || cap < (int32_t)p->swaps.size())
    return MPCORE_BAD_DIMENSION;
  std::memcpy(out, p->swaps.data(), p->swaps.size() * sizeof(int32_t));
  return MPCORE_OK;
}

int32_t mpcore_host_alloc(int64_t bytes, void **out) {
  if (out == nullptr || bytes <= 0) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = cudaMallocHost(out, (size_t)bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  return MPCORE_OK;
}

int32_t mpcore_host_free(void *p) {
  if (p == nullptr) return MPCORE_OK;
  cudaError_t e = cudaFreeHost(p);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFreeHost");
  return MPCORE_OK;
}

int32_t mpcore_mat_mul(uint64_t a, uint64_t b, uint64_t c) {
  ObjPtr A = table().get(a, K_MATRIX), B = table().get(b, K_MATRIX);
  if (!A || !B) return MPCORE_BAD_HANDLE;
  ObjPtr C;
  int st = table().latch(c, K_MATRIX, C);
  if (st) return st;
  struct Unlatch {
    ObjPtr &o;
    ~Unlatch() { table().unlatch(o); }
  } un{C};
  if (A->k != B->k || C->k != A->k) return MPCORE_BAD_DIMENSION;
  if (A->cols != B->rows || C->rows != A->rows || C->cols != B->cols)
    return MPCORE_BAD_DIMENSION;
  if (C->d == A->d || C->d == B->d)
    return fail(MPCORE_BAD_DIMENSION, "output aliases an input");
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = mpk::gemm(A->k, false, true, A->rows, B->cols, A->cols,
                            view(A), view(B), view(C), device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "mat_mul");
  return finish("mat_mul");
}

int32_t mpcore_mat_vec(uint64_t a, uint64_t x, uint64_t y) {
  ObjPtr A = table().get(a, K_MATRIX), X = table().get(x, K_VECTOR);
  if (!A || !X) return MPCORE_BAD_HANDLE;
  ObjPtr Y;
  int st = table().latch(y, K_VECTOR, Y);
  if (st) return st;
  struct Unlatch {
    ObjPtr &o;
    ~Unlatch() { table().unlatch(o); }
  } un{Y};
  if (A->k != X->k || Y->k != A->k) return MPCORE_BAD_DIMENSION;
  if (A->cols != X->rows || Y->rows != A->rows) return MPCORE_BAD_DIMENSION;
  if (Y->d == X->d) return fail(MPCORE_BAD_DIMENSION, "output aliases input");
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = mpk::matvec(A->k, A->rows, A->cols, view(A), X->d, Y->d,
                              device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "mat_vec");
  return finish("mat_vec");
}

int32_t mpcore_elementwise(int32_t op, uint64_t x, uint64_t y, uint64_t out) {
  ObjPtr X = container(x), Y = container(y), O = container(out);
  if (!X || !Y || !O) return MPCORE_BAD_HANDLE;
  if (op < 0 || op > 3) return MPCORE_BAD_DIMENSION;
  if (X->k != Y->k || O->k != X->k || X->count() != Y->count() ||
      O->count() != X->count())
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  if (op >= 2) {
    // division by an exact zero and the square root of a negative value
    // raise in the reference (mcfloat.py:309-310, 325-326)
    const ObjPtr &chk = op == 2 ? Y : X;
    std::vector<double> heads(chk->count() / chk->k);
    cudaError_t e = cudaMemcpyAsync(heads.data(), chk->d,
                                    heads.size() * sizeof(double),
                                    cudaMemcpyDeviceToHost, device().stream);
    if (e != cudaSuccess) return cuda_fail(e, "operand check");
    int st = finish("operand check");
    if (st) return st;
    for (double v : heads) {
      if (op == 2 && v == 0.0)
        return fail(MPCORE_INTERNAL, "division by zero");
      if (op == 3 && v < 0.0)
        return fail(MPCORE_INTERNAL, "square root of a negative value");
    }
  }
  cudaError_t e = mpk::elementwise(X->k, op, X->count() / X->k, X->d, Y->d,
                                   O->d, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "elementwise");
  return finish("elementwise");
}

int32_t mpcore_axpy(const double *alpha, int32_t k, uint64_t x, uint64_t y) {
  ObjPtr X = container(x);
  if (!X) return MPCORE_BAD_HANDLE;
  ObjPtr Y = container(y);
  if (!Y) return MPCORE_BAD_HANDLE;
  if (alpha == nullptr || k != X->k || Y->k != X->k ||
      Y->count() != X->count())
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = mpk::axpy(X->k, X->count() / X->k, alpha, X->d, Y->d,
                            device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "axpy");
  return finish("axpy");
}

int32_t mpcore_generate(uint64_t h, int32_t slot, int64_t system_n,
                        uint64_t seed) {
  ObjPtr o = container(h);
  if (!o) return MPCORE_BAD_HANDLE;
  if (slot < 0 || slot > 3 || system_n < 1) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  int64_t count = (int64_t)o->rows * o->cols;
  cudaError_t e = mpk::generate(o->k, o->d, count, count, slot, system_n, seed,
                                device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "generate");
  return finish("generate");
}

int32_t mpcore_lu_decomp_pm(int32_t k, int32_t n, double *a_planes,
                            int32_t *swaps, int32_t *singular_step) {
  if (a_planes == nullptr || swaps == nullptr) return MPCORE_BAD_DIMENSION;
  uint64_t h = 0, piv = 0;
  int st = mpcore_matrix_new(k, n, n, &h);
  if (st) return st;
  st = mpcore_set_planes(h, a_planes, (int64_t)k * n * n);
  if (!st) st = mpcore_lu_factor_ex(h, 0, &piv, singular_step);
  if (!st) st = mpcore_get_planes(h, a_planes, (int64_t)k * n * n);
  if (!st) st = mpcore_pivot_get(piv, swaps, n);
  mpcore_release(h);
  if (piv) mpcore_release(piv);
  return st;
}

int32_t mpcore_solve_ls_pm(int32_t k, int32_t n, const double *lu_planes,
                           const int32_t *swaps, const double *b_planes,
                           double *x_planes) {
  if (!lu_planes || !swaps || !b_planes || !x_planes) return MPCORE_BAD_DIMENSION;
  uint64_t h = 0, piv = 0, b = 0, x = 0;
  int st = mpcore_matrix_new(k, n, n, &h);
  if (!st) st = mpcore_set_planes(h, lu_planes, (int64_t)k * n * n);
  if (!st) st = mpcore_pivot_new(n, swaps, &piv);
  if (!st) st = mpcore_vector_new(k, n, &b);
  if (!st) st = mpcore_set_planes(b, b_planes, (int64_t)k * n);
  if (!st) st = mpcore_vector_new(k, n, &x);
  if (!st) st = mpcore_lu_solve(h, piv, b, x);
  if (!st) st = mpcore_get_planes(x, x_planes, (int64_t)k * n);
  for (uint64_t hh : {h, piv, b, x})
    if (hh) mpcore_release(hh);
  return st;
}

int32_t mpcore_set_device(int32_t dev) {
  Device &D = device();
  std::lock_guard<std::mutex> g(D.mu);
  if (D.tried) return D.dev == dev ? MPCORE_OK : fail(MPCORE_INTERNAL,
                                                     "device already initialised");
  D.want = dev;
  return MPCORE_OK;
}

int32_t mpcore_device_name(char *out, int32_t cap) {
  DevLock L;
  if (L.st) return L.st;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device().dev);
  return copy_text(p.name, out, cap);
}

int32_t mpcore_sm_count(int32_t *out) {
  if (!out) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  *out = device().sms;
  return MPCORE_OK;
}

int32_t mpcore_last_error(char *out, int32_t cap) {
  return copy_text(g_err, out, cap);
}

int32_t mpcore_sync(void) {
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  if (D.copy) {  // asynchronous uploads / downloads too
    cudaError_t e = cudaStreamSynchronize(D.copy);
    if (e != cudaSuccess) return cuda_fail(e, "sync (copies)");
  }
  return finish("sync");
}

int32_t mpcore_prof_enable(int32_t on) {
  DevLock L;
  if (L.st) return L.st;
  prof().on = on != 0;
  return MPCORE_OK;
}

int32_t mpcore_prof_reset(void) {
  DevLock L;
  if (L.st) return L.st;
  Prof &P = prof();
  P.collect();
  for (int i = 0; i < mpk::PROF_NSLOTS; ++i) {
    P.ms[i] = 0;
    P.launches[i] = 0;
  }
  P.timeline.clear();
  if (!P.base) cudaEventCreate(&P.base);
  cudaEventRecord(P.base, device().stream);
  return MPCORE_OK;
}

int32_t mpcore_debug_timeline(double *out, int64_t cap, int64_t *count) {
  DevLock L;
  if (L.st) return L.st;
  Prof &P = prof();
  P.collect();
  const int64_t n = (int64_t)P.timeline.size();
  if (count) *count = n / 3;
  if (out) {
    for (int64_t i = 0; i < n && i < cap; ++i) out[i] = P.timeline[i];
  }
  return MPCORE_OK;
}

// Device timing on the library stream: CUDA events in 8 slots.
int32_t mpcore_stream_event_record(int32_t slot) {
  DevLock L;
  if (L.st) return L.st;
  static cudaEvent_t ev[8] = {};
  if (slot < 0 || slot >= 8) return MPCORE_BAD_DIMENSION;
  cudaError_t e = cudaSuccess;
  if (!ev[slot]) e = cudaEventCreate(&ev[slot]);
  if (e == cudaSuccess) e = cudaEventRecord(ev[slot], device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "event record");
  event_slots()[slot] = ev[slot];
  return MPCORE_OK;
}

int32_t mpcore_stream_event_elapsed(int32_t a, int32_t b, double *ms) {
  if (ms == nullptr || a < 0 || a >= 8 || b < 0 || b >= 8)
    return MPCORE_BAD_DIMENSION;
  cudaEvent_t ea = event_slots()[a], eb = event_slots()[b];
  if (!ea || !eb) return MPCORE_BAD_DIMENSION;
  cudaError_t e = cudaEventSynchronize(eb);
  float f = 0.0f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&f, ea, eb);
  if (e != cudaSuccess) return cuda_fail(e, "event elapsed");
  *ms = f;
  return MPCORE_OK;
}

// MPCORE_LU_STAMPS diagnostics: out == NULL (re)arms a buffer of len
// entries (4 per column index: panel entry/exit, exchange+U12 entry/exit,
// globaltimer ns; unset entries ~0 / 0); otherwise copies len entries out.
int32_t mpcore_debug_lu_stamps(int64_t len, uint64_t *out) {
  DevLock L;
  if (L.st) return L.st;
  static unsigned long long *buf = nullptr;
  static int64_t cap = 0;
  if (len <= 0 || len % 4) return MPCORE_BAD_DIMENSION;
  cudaError_t e;
  if (out == nullptr) {
    if (len > cap) {
      if (buf) cudaFree(buf);
      buf = nullptr;
      cap = 0;
      if ((e = cudaMalloc(&buf, len * 8)) != cudaSuccess)
        return cuda_fail(e, "stamps");
      cap = len;
    }
    std::vector<unsigned long long> init((size_t)len);
    for (int64_t i = 0; i < len; ++i) init[i] = (i % 2 == 0) ? ~0ull : 0ull;
    if ((e = cudaMemcpy(buf, init.data(), len * 8, cudaMemcpyHostToDevice)) !=
            cudaSuccess ||
        (e = mpk::lu_stamps_enable(buf)) != cudaSuccess)
      return cuda_fail(e, "stamps");
    return MPCORE_OK;
  }
  if (!buf || len > cap) return MPCORE_BAD_DIMENSION;
  if ((e = cudaMemcpy(out, buf, len * 8, cudaMemcpyDeviceToHost)) !=
      cudaSuccess)
    return cuda_fail(e, "stamps");
  return MPCORE_OK;
}

int32_t mpcore_debug_panel_trace(uint64_t *out_ns, int64_t cap) {
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  int64_t count = (int64_t)D.sms * 33 * 8;
  if (!D.ws.trace) return fail(MPCORE_INTERNAL, "MPCORE_TRACE_PANEL not set");
  if (!out_ns || cap < count) return MPCORE_BAD_DIMENSION;
  cudaError_t e = cudaMemcpy(out_ns, D.ws.trace, count * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "trace");
  return MPCORE_OK;
}

int32_t mpcore_debug_long_residual_selftest(int32_t n, int32_t prec,
                                            uint64_t seed, int32_t variant,
                                            int64_t *mismatches) {
  if (!mismatches || variant < 0 || variant > 5 || variant == 3 || variant == 4)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  *mismatches = mpr::long_residual_selftest(n, prec, seed, device().stream,
                                            variant);
  return *mismatches < 0 ? MPCORE_INTERNAL : MPCORE_OK;
}

int32_t mpcore_debug_longfloat_selftest(int64_t iters, uint64_t seed,
                                        int32_t prec, int64_t *mismatches) {
  if (!mismatches) return MPCORE_BAD_DIMENSION;
  *mismatches = mpr::longfloat_selftest(iters, seed, prec);
  return *mismatches < 0 ? MPCORE_BAD_DIMENSION : MPCORE_OK;
}

int32_t mpcore_debug_solve_trace(uint64_t *out_ns, int64_t cap) {
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  if (!D.sw.trace) return fail(MPCORE_INTERNAL, "MPCORE_TRACE_SOLVE not set");
  if (!out_ns || cap < D.sw.trace_len) return MPCORE_BAD_DIMENSION;
  cudaError_t e = cudaMemcpy(out_ns, D.sw.trace,
                             D.sw.trace_len * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "trace");
  return MPCORE_OK;
}

int32_t mpcore_prof_read(double *ms, int64_t *launches, int32_t cap) {
  if (!ms || !launches || cap < mpk::PROF_NSLOTS) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  Prof &P = prof();
  P.collect();
  for (int i = 0; i < mpk::PROF_NSLOTS; ++i) {
    ms[i] = P.ms[i];
    launches[i] = P.launches[i];
  }
  return MPCORE_OK;
}

// ------------------------------------------ device-pointer (expert) API ----
// Building blocks for callers that lay out and move device memory
// themselves (the distributed LU in dist.py).  Pointers are device
// addresses; views are planar (base, row stride, plane stride).

static mpk::MatView mv(uint64_t base, int64_t ld, int64_t plane) {
  mpk::MatView v;
  v.p = reinterpret_cast<double *>(base);
  v.ld = ld;
  v.plane = plane;
  return v;
}

static const int32_t *never_singular() {
  static int32_t *d = nullptr;
  if (!d) {
    cudaMalloc(&d, sizeof(int32_t));
    cudaMemset(d, 0xFF, sizeof(int32_t));
    cudaDeviceSynchronize();
  }
  return d;
}

int32_t mpcore_object_device_ptr(uint64_t h, uint64_t *ptr) {
  ObjPtr o = container(h);
  if (!o) return MPCORE_BAD_HANDLE;
  if (!ptr) return MPCORE_BAD_DIMENSION;
  *ptr = reinterpret_cast<uint64_t>(o->d);
  return MPCORE_OK;
}

int32_t mpcore_dev_lu_block(int32_t k, int32_t m, int32_t ncols, uint64_t base,
                            int64_t ld, int64_t plane, int32_t nb,
                            int32_t *swaps_out, int32_t *singular_step) {
  if (k < 2 || k > 4 || m < 1 || ncols < 1 || ncols > m || !base ||
      !swaps_out)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  cudaError_t e;
  if (D.swaps_cap < ncols) {
    if (D.dswaps) cudaFree(D.dswaps);
    D.dswaps = nullptr;
    D.swaps_cap = 0;
    if ((e = cudaMalloc(&D.dswaps, (size_t)ncols * sizeof(int32_t))) !=
        cudaSuccess)
      return cuda_fail(e, "cudaMalloc(swaps)");
    D.swaps_cap = ncols;
  }
  int32_t step = -1;
  e = mpk::lu_factor(k, m, ncols, mv(base, ld, plane), D.dswaps,
                     nb > 0 ? nb : 32, D.ws, &step, D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "lu_block");
  e = cudaMemcpyAsync(swaps_out, D.dswaps, (size_t)ncols * sizeof(int32_t),
                      cudaMemcpyDeviceToHost, D.stream);
  int st = finish("lu_block");
  if (st) return st;
  if (e != cudaSuccess) return cuda_fail(e, "swaps download");
  if (singular_step) *singular_step = step;
  if (step >= 0)
    return fail(MPCORE_SINGULAR,
                "no nonzero pivot at elimination step " + std::to_string(step));
  return MPCORE_OK;
}

int32_t mpcore_dev_laswp(int32_t k, uint64_t base, int64_t ld, int64_t plane,
                         int32_t col0, int32_t ncols, int32_t row0,
                         const int32_t *swaps, int32_t nswaps) {
  if (k < 2 || k > 4 || !base || (nswaps > 0 && !swaps) || ncols < 0)
    return MPCORE_BAD_DIMENSION;
  if (nswaps <= 0 || ncols == 0) return MPCORE_OK;
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  const int W = mpk::LU_MAX_W, LIST = 4 * W + 1;
  const int chunks = (nswaps + W - 1) / W;
  std::vector<int32_t> host((size_t)chunks * LIST, 0);
  for (int ch = 0; ch < chunks; ++ch) {
    // compose this chunk's exchanges: row cur[i] receives row src[i]
    int32_t *cur = &host[(size_t)ch * LIST], *src = cur + 2 * W;
    int cnt = 0;
    for (int i = ch * W; i < std::min(nswaps, (ch + 1) * W); ++i) {
      const int a = row0 + i, b = swaps[i];
      if (a == b) continue;
      int ia = -1, ib = -1;
      for (int t = 0; t < cnt; ++t) {
        if (cur[t] == a) ia = t;
        if (cur[t] == b) ib = t;
      }
      if (ia < 0) { cur[cnt] = a; src[cnt] = a; ia = cnt++; }
      if (ib < 0) { cur[cnt] = b; src[cnt] = b; ib = cnt++; }
      std::swap(src[ia], src[ib]);
    }
    cur[4 * W] = cnt;
  }
  int32_t *dlist = nullptr;
  cudaError_t e = cudaMallocAsync(&dlist, host.size() * sizeof(int32_t),
                                  D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "laswp list");
  e = cudaMemcpyAsync(dlist, host.data(), host.size() * sizeof(int32_t),
                      cudaMemcpyHostToDevice, D.stream);
  for (int ch = 0; ch < chunks && e == cudaSuccess; ++ch)
    e = mpk::lu_laswp(k, mv(base, ld, plane), col0, col0 + ncols, 0, 0,
                      dlist + (size_t)ch * LIST, never_singular(), D.stream);
  cudaFreeAsync(dlist, D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "laswp");
  return finish("laswp");
}

int32_t mpcore_dev_trsm(int32_t k, int32_t w, int32_t ncols, uint64_t l11,
                        int64_t ldl, int64_t planel, uint64_t u12, int64_t ldu,
                        int64_t planeu) {
  if (k < 2 || k > 4 || w < 1 || ncols < 0 || !l11 || !u12)
    return MPCORE_BAD_DIMENSION;
  if (ncols == 0) return MPCORE_OK;
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  const int W = mpk::LU_MAX_W;
  cudaError_t e = cudaSuccess;
  // blocked: each diagonal 32-block by the wavefront kernel, then the rows
  // below it in the block get that block's contributions (ascending order)
  for (int sb = 0; sb < w && e == cudaSuccess; sb += W) {
    const int wb = std::min(W, w - sb);
    mpk::MatView Ld = mv(l11 + (uint64_t)((sb * ldl + sb) * 8), ldl, planel);
    mpk::MatView Us = mv(u12 + (uint64_t)(sb * ldu * 8), ldu, planeu);
    e = mpk::lu_trsm(k, Ld, Us, wb, ncols, never_singular(), D.stream);
    if (e == cudaSuccess && sb + wb < w) {
      mpk::MatView L21 = mv(l11 + (uint64_t)(((sb + wb) * ldl + sb) * 8), ldl,
                            planel);
      mpk::MatView Ub = mv(u12 + (uint64_t)((sb + wb) * ldu * 8), ldu, planeu);
      e = mpk::lu_update(k, w - sb - wb, ncols, wb, L21, Us, Ub,
                         never_singular(), D.stream);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "trsm");
  return finish("trsm");
}

int32_t mpcore_dev_gemm(int32_t k, int32_t neg_a, int32_t zero_init, int32_t M,
                        int32_t N, int32_t Kd, uint64_t a, int64_t lda,
                        int64_t pa, uint64_t b, int64_t ldb, int64_t pb,
                        uint64_t c, int64_t ldc, int64_t pc) {
  if (k < 2 || k > 4 || M < 0 || N < 0 || Kd < 0 || !a || !b || !c)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = mpk::gemm(k, neg_a != 0, zero_init != 0, M, N, Kd,
                            mv(a, lda, pa), mv(b, ldb, pb), mv(c, ldc, pc),
                            device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "gemm");
  return finish("gemm");
}

int32_t mpcore_dev_copy2d(int32_t k, int32_t rows, int32_t cols, uint64_t dst,
                          int64_t ldd, int64_t pd, uint64_t src, int64_t lds,
                          int64_t ps) {
  if (k < 1 || rows < 0 || cols < 0 || !dst || !src) return MPCORE_BAD_DIMENSION;
  if (rows == 0 || cols == 0) return MPCORE_OK;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = cudaSuccess;
  for (int c = 0; c < k && e == cudaSuccess; ++c)
    e = cudaMemcpy2DAsync(reinterpret_cast<double *>(dst) + c * pd,
                          (size_t)ldd * 8,
                          reinterpret_cast<const double *>(src) + c * ps,
                          (size_t)lds * 8, (size_t)cols * 8, (size_t)rows,
                          cudaMemcpyDeviceToDevice, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "copy2d");
  return finish("copy2d");
}

int32_t mpcore_dev_lu_solve(int32_t k, int32_t n, uint64_t lu, int64_t ld,
                            int64_t plane, const int32_t *swaps, uint64_t b,
                            uint64_t x) {
  if (k < 2 || k > 4 || n < 1 || !lu || !swaps || !b || !x || b == x)
    return MPCORE_BAD_DIMENSION;
  std::vector<int32_t> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int j = 0; j < n; ++j) {
    if (swaps[j] < j || swaps[j] >= n) return MPCORE_BAD_DIMENSION;
    if (swaps[j] != j) std::swap(order[j], order[swaps[j]]);
  }
  DevLock L;
  if (L.st) return L.st;
  Device &D = device();
  int32_t *dperm = nullptr;
  cudaError_t e = cudaMallocAsync(&dperm, (size_t)n * sizeof(int32_t), D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "perm");
  e = cudaMemcpyAsync(dperm, order.data(), (size_t)n * sizeof(int32_t),
                      cudaMemcpyHostToDevice, D.stream);
  if (e == cudaSuccess)
    e = mpk::lu_solve(k, n, mv(lu, ld, plane), dperm,
                      reinterpret_cast<const double *>(b),
                      reinterpret_cast<double *>(x), D.sw, D.stream);
  cudaFreeAsync(dperm, D.stream);
  if (e != cudaSuccess) return cuda_fail(e, "dev_lu_solve");
  return finish("dev_lu_solve");
}

int32_t mpcore_dev_matvec(int32_t k, int32_t rows, int32_t cols, uint64_t a,
                          int64_t ld, int64_t plane, uint64_t x, uint64_t y) {
  if (k < 2 || k > 4 || rows < 1 || cols < 1 || !a || !x || !y || x == y)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = mpk::matvec(k, rows, cols, mv(a, ld, plane),
                              reinterpret_cast<const double *>(x),
                              reinterpret_cast<double *>(y), device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "dev_matvec");
  return finish("dev_matvec");
}

int32_t mpcore_dev_generate_cyclic(int32_t k, uint64_t base, int64_t ld,
                                   int64_t plane, int32_t rows,
                                   int32_t local_cols, int32_t nb,
                                   int32_t world, int32_t rank, int32_t slot,
                                   int64_t system_n, uint64_t seed) {
  if (k < 2 || k > 4 || !base || rows < 0 || local_cols < 0 || nb < 1 ||
      world < 1 || rank < 0 || rank >= world || system_n < 1)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  cudaError_t e = mpk::generate_cyclic(k, mv(base, ld, plane), rows,
                                       local_cols, nb, world, rank, slot,
                                       system_n, seed, device().stream);
  if (e != cudaSuccess) return cuda_fail(e, "generate_cyclic");
  return finish("generate_cyclic");
}


// ------------------------------------------------ distributed LU ----
// NCCL bootstrap (unique id on one rank, shared by the host's own channel,
// then one communicator per rank) and the native distributed driver
// (dist.cu).  Communicator handles are opaque and checked against the
// live set.
static std::set<uint64_t> &live_comms() {
  static std::set<uint64_t> s;
  return s;
}

int32_t mpcore_dist_unique_id(uint8_t *out, int32_t cap) {
  if (!out || cap < 128) return MPCORE_BAD_DIMENSION;
  std::string err;
  if (mpk::nccl_unique_id(out, err)) return fail(MPCORE_INTERNAL, err);
  return MPCORE_OK;
}

int32_t mpcore_dist_comm_init(int32_t world, int32_t rank, const uint8_t *id,
                              int32_t len, uint64_t *comm_out) {
  if (!comm_out) return MPCORE_BAD_DIMENSION;
  *comm_out = 0;
  if (!id || len != 128 || world < 1 || rank < 0 || rank >= world)
    return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  std::string err;
  void *c = mpk::nccl_comm_init(world, rank, id, err);
  if (!c) return fail(MPCORE_INTERNAL, err);
  *comm_out = reinterpret_cast<uint64_t>(c);
  live_comms().insert(*comm_out);
  return MPCORE_OK;
}

int32_t mpcore_dist_comm_destroy(uint64_t comm) {
  DevLock L;
  if (!live_comms().erase(comm)) return MPCORE_BAD_HANDLE;
  mpk::nccl_comm_destroy(reinterpret_cast<void *>(comm));
  return MPCORE_OK;
}

int32_t mpcore_dist_lu_solve(uint64_t comm, int32_t k, int32_t n, int32_t nb,
                             int32_t world, int32_t nlocal,
                             const int32_t *ranks, const uint64_t *bases,
                             const int64_t *lds, const int64_t *planes,
                             const int32_t *cols, const uint64_t *xs,
                             uint64_t stream, int32_t *swaps_out,
                             int32_t *singular_step, double *phase_ms,
                             int64_t *launches) {
  if (singular_step) *singular_step = -1;
  if (k < 2 || k > 4 || n < 1 || nb < 1 || world < 1 || nlocal < 1 ||
      !ranks || !bases || !lds || !planes || !cols || !xs || !swaps_out)
    return MPCORE_BAD_DIMENSION;
  std::vector<mpk::DistRankView> views(nlocal);
  for (int i = 0; i < nlocal; ++i) {
    if (ranks[i] < 0 || ranks[i] >= world || !bases[i] || !xs[i])
      return MPCORE_BAD_DIMENSION;
    views[i].rank = ranks[i];
    views[i].A = mv(bases[i], lds[i], planes[i]);
    views[i].cols = cols[i];
    views[i].x = reinterpret_cast<double *>(xs[i]);
  }
  DevLock L;
  if (L.st) return L.st;
  if (comm && !live_comms().count(comm)) return MPCORE_BAD_HANDLE;
  Device &D = device();
  cudaStream_t caller =
      stream ? reinterpret_cast<cudaStream_t>(stream) : D.stream;
  std::vector<int32_t> sw;
  std::string err;
  int32_t step = -1;
  int st = mpk::dist_lu_solve(reinterpret_cast<void *>(comm), k, n, nb, world,
                              views, D.ws, D.sw, caller, sw, &step, phase_ms,
                              launches, err);
  if (singular_step) *singular_step = step;
  if (st == 0 || st == MPCORE_SINGULAR)
    std::memcpy(swaps_out, sw.data(), (size_t)n * sizeof(int32_t));
  if (st == 2) return fail(MPCORE_BAD_DIMENSION, err);
  if (st == 3) return fail(MPCORE_SINGULAR, err);
  if (st) return fail(MPCORE_INTERNAL, err);
  return MPCORE_OK;
}


// Debug: verify every guarded object's guard zones (MPCORE_DEBUG_GUARD=1 at
// allocation).  *checked = objects with guards, *bad = objects whose zones
// were written.
int32_t mpcore_debug_check_guards(int64_t *checked, int64_t *bad) {
  if (!checked || !bad) return MPCORE_BAD_DIMENSION;
  *checked = *bad = 0;
  std::vector<ObjPtr> objs;
  {
    Table &T = table();
    std::lock_guard<std::mutex> g(T.mu);
    for (auto &kv : T.map)
      if (kv.second->raw) objs.push_back(kv.second);
  }
  DevLock L;
  if (L.st) return L.st;
  for (auto &o : objs) {
    const size_t g = o->guard, bytes = (size_t)o->count() * sizeof(double);
    std::vector<unsigned char> h(2 * g);
    cudaError_t e = cudaMemcpyAsync(h.data(), o->raw, g,
                                    cudaMemcpyDeviceToHost, device().stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h.data() + g, o->raw + g + bytes, g,
                          cudaMemcpyDeviceToHost, device().stream);
    int st = finish("guards");
    if (st) return st;
    if (e != cudaSuccess) return cuda_fail(e, "guards");
    ++*checked;
    for (unsigned char c : h)
      if (c != kGuardByte) {
        ++*bad;
        break;
      }
  }
  return MPCORE_OK;
}


// the device long -> short conversion (convert.cu) against the host's
// fixed-width from_bf + to_multicomp: mismatching values over iters
int32_t mpcore_debug_convert_selftest(int64_t iters, uint64_t seed,
                                      int32_t prec, int32_t k,
                                      int64_t *mismatches) {
  if (!mismatches) return MPCORE_BAD_DIMENSION;
  DevLock L;
  if (L.st) return L.st;
  *mismatches = mpr::convert_selftest(iters, seed, prec, k, device().stream);
  return *mismatches < 0 ? fail(MPCORE_BAD_DIMENSION, "bad selftest arguments")
                         : MPCORE_OK;
}

}  // extern "C"
