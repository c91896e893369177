// tls_api.cu — the C ABI of libtlsrqi.so (include/tlsrqi.h) and the host
// runtime around the kernels: workspace carving, the NCCL shim, the
// preconditioner build and the RQI-PCGTLS-MP host loop
// (a4-a9).  The host loop is the only host<->device crossing of a solve: one
// small D2H read after each residual evaluation and after each PCG batch;
// inside PCGTLS all control (breakdown, early exit) is device-resident.
#include <dlfcn.h>

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <vector>

#include "tls_common.cuh"
#include "tls_kernels.h"

// ------------------------------------------------------------------------------ errors
namespace tls {
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace tls

using namespace tls;

#define TLS_TRY(expr)        \
  do {                       \
    int _rc = (expr);        \
    if (_rc != 0) return _rc; \
  } while (0)

// ------------------------------------------------------------------------------ NCCL shim
// Minimal declarations matching nccl.h (NCCL 2.x ABI); libnccl.so.2 is dlopen'ed so
// the library loads (and single-GPU runs) without NCCL.
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { ncclSuccess = 0, ncclInProgress = 7 };
enum { ncclSum = 0, ncclMax = 2 };
enum { ncclFloat64 = 8, ncclInt32 = 2, ncclInt64 = 4 };
struct NcclApi {
  int (*GetUniqueId)(ncclUniqueId*);
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*CommDestroy)(ncclComm_t);
  int (*CommGetAsyncError)(ncclComm_t, int*);
  const char* (*GetErrorString)(int);
  bool ok = false;
};
NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
      api.AllReduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
      api.CommDestroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
      api.CommGetAsyncError = (int (*)(ncclComm_t, int*))dlsym(h, "ncclCommGetAsyncError");
      api.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy;
    }
  }
  return api.ok ? &api : nullptr;
}

// Host-shm backend: ranks that are processes sharing ONE GPU (tls_comm_init_shm).  Every
// collective is staged through a POSIX shared-memory segment: a rank copies its buffer to the
// host (its stream synchronised first), writes it into its own slot, waits at a process-shared
// barrier, sums ALL ranks' slots in rank order 0..P-1 (every rank computes identical bits),
// waits at a second barrier (the slots may then be reused) and copies the result back.  No
// kernel ever waits for another rank (B200_PROFILING.md: kernels spinning on other ranks' flags
// must not share a GPU), so this backend runs every multi-rank code path of the library --
// sharded passes, all-reduced Gram, replicated Cholesky, TSQR stack exchange, the
// explicit-inverse default -- with real per-rank processes on one GPU.  It is a correctness
// backend; the production path is NCCL over NVLink.
struct ShmHeader {
  std::atomic<int64_t> arrive;     // arrivals in the current barrier phase
  std::atomic<int64_t> phase;      // completed barrier phases
  int64_t nranks;
  int64_t slot_bytes;
};
}  // namespace

struct tls_comm_s {
  ncclComm_t comm;
  int nranks, rank, device;
  ShmHeader* shm = nullptr;        // host-shm backend (comm == nullptr)
  size_t shm_bytes = 0;
  char shm_name[96] = {0};
  double* stage = nullptr;         // pinned staging buffer of slot_bytes
  // peer-memory exchange of the pass sums (k_peer.cu, tls_comm_peer_prepare / _connect)
  bool peer = false;
  PeerTab tab{};
  double* prbuf = nullptr;         // this rank's receive buffer [2][nranks][pwcap]
  int* prflag = nullptr;           // this rank's flags [nranks][kXchCtas]
  int* perr = nullptr;             // device: a wait timed out
  int pwcap = 0;
  int pepoch = 0;
};

struct tls_precond_s {
  PrecondDev dev;
  void* base;
  size_t bytes;
  int device;
  double normA2_host;
  // u_p = fp32 (R23): fl32 copy of the local row block of A, made by the first solve that
  // asks for it and kept for later solves on the same block (keyed by pointer and shape)
  float* a32 = nullptr;
  size_t a32_bytes = 0;
  const double* a32_src = nullptr;
  int64_t a32_m = -1, a32_ld = -1;
  // explicit inverse W = R~^{-1} and W^T (R24), made by the first solve that applies it
  double* winv = nullptr;
  // fingerprint of the factored A: global row count (-1 for imported handles)
  // and the sampled content checksum of this rank's block (k_fingerprint)
  int64_t m_global = -1;
  double content = 0.0;
  double a32_content = 0.0;   // the checksum the fp32 copy was made from
};

namespace {
bool comm_active(tls_comm_t c) { return c != nullptr && (c->comm != nullptr || c->shm != nullptr); }

char* shm_slot(tls_comm_t c, int r) {
  return reinterpret_cast<char*>(c->shm) + 256 + (size_t)r * (size_t)c->shm->slot_bytes;
}

int shm_barrier(tls_comm_t c) {
  ShmHeader* h = c->shm;
  const int64_t ph = h->phase.load(std::memory_order_acquire);
  if (h->arrive.fetch_add(1, std::memory_order_acq_rel) + 1 == h->nranks) {
    h->arrive.store(0, std::memory_order_relaxed);
    h->phase.fetch_add(1, std::memory_order_acq_rel);
    return 0;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (long spin = 0; h->phase.load(std::memory_order_acquire) == ph; ++spin) {
    if (spin > 1000) sched_yield();
    if ((spin & 1023) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
      set_error("shm barrier: rank %d waited 120 s for the other ranks", c->rank);
      return TLS_ERR_NCCL;
    }
  }
  return 0;
}

// `count` 8-byte elements (double, or int64 when is_int); op = ncclSum / ncclMax
int shm_allreduce(tls_comm_t c, void* buf, size_t count, int op, bool is_int, cudaStream_t st) {
  const size_t per = (size_t)c->shm->slot_bytes / 8;
  char* dev = static_cast<char*>(buf);
  for (size_t off = 0; off < count; off += per) {
    const size_t k = count - off < per ? count - off : per;
    TLS_CUDA_TRY(cudaMemcpyAsync(c->stage, dev + off * 8, k * 8, cudaMemcpyDeviceToHost, st));
    TLS_CUDA_TRY(cudaStreamSynchronize(st));
    std::memcpy(shm_slot(c, c->rank), c->stage, k * 8);
    TLS_TRY(shm_barrier(c));
    for (size_t i = 0; i < k; ++i) {
      if (is_int) {
        int64_t acc = 0;
        for (int r = 0; r < c->nranks; ++r) acc += reinterpret_cast<const int64_t*>(shm_slot(c, r))[i];
        reinterpret_cast<int64_t*>(c->stage)[i] = acc;
      } else {
        double acc = reinterpret_cast<const double*>(shm_slot(c, 0))[i];
        for (int r = 1; r < c->nranks; ++r) {                     // rank order 0..P-1
          const double v = reinterpret_cast<const double*>(shm_slot(c, r))[i];
          acc = (op == ncclMax) ? (v > acc ? v : acc) : acc + v;
        }
        c->stage[i] = acc;
      }
    }
    TLS_TRY(shm_barrier(c));
    TLS_CUDA_TRY(cudaMemcpyAsync(dev + off * 8, c->stage, k * 8, cudaMemcpyHostToDevice, st));
    TLS_CUDA_TRY(cudaStreamSynchronize(st));   // the staging buffer is reused by the next chunk
  }
  return 0;
}

int nccl_check(tls_comm_t comm, int r, const char* what) {
  if (r == ncclSuccess) return 0;
  NcclApi* api = nccl_api();
  int aerr = 0;
  if (api->CommGetAsyncError) api->CommGetAsyncError(comm->comm, &aerr);
  set_error("%s: %s (async state: %s)", what, api->GetErrorString ? api->GetErrorString(r) : "error",
            api->GetErrorString ? api->GetErrorString(aerr) : "?");
  return TLS_ERR_NCCL;
}
}  // namespace

static int allreduce(tls_comm_t comm, double* buf, size_t count, int op, cudaStream_t st) {
  if (!comm_active(comm) || count == 0) return 0;
  if (comm->shm) return shm_allreduce(comm, buf, count, op, false, st);
  return nccl_check(comm, nccl_api()->AllReduce(buf, buf, count, ncclFloat64, op, comm->comm, st), "ncclAllReduce");
}

// int64 sum (exact, order-free): the fixed-point limbs of the CSR fp16 Gram
static int allreduce_i64(tls_comm_t comm, void* buf, size_t count, cudaStream_t st) {
  if (!comm_active(comm) || count == 0) return 0;
  if (comm->shm) return shm_allreduce(comm, buf, count, ncclSum, true, st);
  return nccl_check(comm, nccl_api()->AllReduce(buf, buf, count, ncclInt64, ncclSum, comm->comm, st),
                    "ncclAllReduce(int64)");
}

// An NCCL error raised asynchronously (a peer died, a link fault) surfaces at the end of each
// top-level call as TLS_ERR_NCCL instead of as a later hang.
static int comm_async_check(tls_comm_t comm) {
  if (comm != nullptr && comm->peer && comm->perr) {
    int e = 0;
    if (cudaMemcpy(&e, comm->perr, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess && e != 0) {
      set_error("peer exchange: a rank waited too long for the other ranks' pass sums");
      return TLS_ERR_NCCL;
    }
  }
  if (comm == nullptr || comm->comm == nullptr) return 0;
  NcclApi* api = nccl_api();
  if (!api || !api->CommGetAsyncError) return 0;
  int aerr = 0;
  const int r = api->CommGetAsyncError(comm->comm, &aerr);
  if (r != ncclSuccess || (aerr != ncclSuccess && aerr != ncclInProgress)) {
    set_error("NCCL asynchronous error: %s", api->GetErrorString ? api->GetErrorString(aerr ? aerr : r) : "error");
    return TLS_ERR_NCCL;
  }
  return 0;
}

// ------------------------------------------------------------------------------ profiling
namespace {
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct Pend { cudaEvent_t a, b; int cat; };
  std::vector<Pend> pend;
  double ms[TLS_PROF_NCAT] = {};
  long long cnt[TLS_PROF_NCAT] = {};
};
Prof& prof() {
  static Prof p;
  return p;
}
cudaEvent_t ev_get() {
  Prof& p = prof();
  if (!p.pool.empty()) {
    cudaEvent_t e = p.pool.back();
    p.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void prof_drain() {
  Prof& p = prof();
  for (auto& q : p.pend) {
    float ms = 0.f;
    cudaEventSynchronize(q.b);
    if (cudaEventElapsedTime(&ms, q.a, q.b) == cudaSuccess) {
      p.ms[q.cat] += ms;
      p.cnt[q.cat] += 1;
    }
    p.pool.push_back(q.a);
    p.pool.push_back(q.b);
  }
  p.pend.clear();
}
struct ProfScope {
  int cat;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(int c, cudaStream_t s) : cat(c), st(s) {
    if (prof().on) {
      a = ev_get();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = ev_get();
      cudaEventRecord(b, st);
      prof().pend.push_back({a, b, cat});
      if (prof().pend.size() > 4096) prof_drain();
    }
  }
};
}  // namespace


// ------------------------------------------------------------------------------ phase trace
// TLS_TRACE=1: events + host clock at phase marks, printed to stderr at the end of
// each top-level call (device time vs host time between consecutive marks).
namespace {
struct Tracer {
  bool on = false;
  cudaStream_t st = nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  std::vector<double> host;
  explicit Tracer(cudaStream_t s) : st(s) {
    const char* e = getenv("TLS_TRACE");
    on = e && e[0] == '1';
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back({name, e});
    host.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count());
  }
  ~Tracer() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      fprintf(stderr, "[tls_trace] %-18s -> %-18s device %9.3f ms  host %9.3f ms\n", ev[i - 1].first, ev[i].first, ms,
              host[i] - host[i - 1]);
    }
    for (auto& p : ev) cudaEventDestroy(p.second);
  }
};
}  // namespace

// ------------------------------------------------------------------------------ workspace
namespace {
// Bump allocator over the caller's workspace; with base == nullptr it only
// measures (tls_workspace_size), so carving and sizing cannot disagree.
struct Carver {
  char* base;
  size_t cap;
  size_t off = 0;
  bool ok = true;
  template <typename T>
  T* take(size_t count) {
    const size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    T* r = nullptr;
    if (base) {
      if (off + bytes > cap) ok = false;
      else r = reinterpret_cast<T*>(base + off);
    }
    off += bytes;
    return r;
  }
};

bool is_csr(const tls_matrix_t* A) { return A->layout == TLS_CSR; }
DenseView dense_view(const tls_matrix_t* A) { return DenseView{A->vals, A->m_local, (int)A->n, A->ld}; }
CsrView csr_view(const tls_matrix_t* A) {
  return CsrView{A->rowptr, A->colidx, A->vals, A->m_local, (int)A->n, A->nnz_local};
}

struct Work {
  double* partials;
  double* passout;
  double* colstats;
  PcgVecs vec;
  double* x;
  double* x_prev;
  double* x0;
  double* zero;
  PcgState* S;
  int* flags;    // [0] scaling, [1] range, [2] pivot
  double* G;
  double* gram_ws;
  size_t gram_ws_doubles;
  double* d_tmp;
  // CSR only
  CscView csc;
  void* csc_scratch;
  double* tbuf;
};

// Carves `ws` (or measures when ws == nullptr); returns the bytes needed.
size_t carve(const tls_matrix_t* A, void* ws, size_t bytes, Work& w, bool factor, bool* ok = nullptr) {
  const int n = (int)A->n;
  const bool csr = is_csr(A);
  Carver c{static_cast<char*>(ws), ws ? bytes : 0};
  const size_t npart = csr ? csr_pass_partials_doubles() : pass_partials_doubles(dense_view(A));
  w.partials = c.take<double>(npart > 256 ? npart : 256);   // also the fingerprint's 256 row sums
  w.passout = c.take<double>(2 * (size_t)n + 2);
  w.colstats = c.take<double>(2 * (size_t)n);
  w.vec.omega = c.take<double>(2 * (size_t)n);
  w.vec.s = c.take<double>(2 * (size_t)n);
  w.vec.p = c.take<double>(2 * (size_t)n);
  w.vec.q = c.take<double>(2 * (size_t)n);
  w.vec.rhs = c.take<double>(2 * (size_t)n);
  w.vec.w = c.take<double>(2 * (size_t)n);
  w.x = c.take<double>(n);
  w.x_prev = c.take<double>(n);
  w.x0 = c.take<double>(n);
  w.zero = c.take<double>(n);
  w.S = c.take<PcgState>(1);
  w.flags = c.take<int>(8);
  w.d_tmp = c.take<double>(2 * (size_t)n + 2);
  w.csc = CscView{nullptr, nullptr, nullptr};
  w.csc_scratch = nullptr;
  w.tbuf = nullptr;
  if (csr) {
    w.tbuf = c.take<double>(2 * (size_t)A->m_local);
    w.csc.colptr = c.take<int64_t>((size_t)n + 1);
    w.csc.rowidx = c.take<int32_t>((size_t)A->nnz_local);
    w.csc.vals = c.take<double>((size_t)A->nnz_local);
    w.csc_scratch = c.take<char>(csc_scratch_bytes(A->m_local, n));
  }
  w.G = nullptr;
  w.gram_ws = nullptr;
  w.gram_ws_doubles = 0;
  if (factor) {
    w.G = c.take<double>((size_t)n * n);
    // K_t only changes the number of chunks; K_t = 1 gives the largest split count
    w.gram_ws_doubles = csr ? csr_gram_ws_bytes(n) / 8 : gram_ws_doubles(dense_view(A), 1);
    const size_t chol = (chol_ws_bytes(n) + 7) / 8;                  // the Cholesky reuses it
    if (w.gram_ws_doubles < chol) w.gram_ws_doubles = chol;
    const size_t packed = (size_t)n * (n + 1) / 2;                    // the packed Gram all-reduce too
    if (w.gram_ws_doubles < packed) w.gram_ws_doubles = packed;
    w.gram_ws = c.take<double>(w.gram_ws_doubles);
  }
  if (ok) *ok = c.ok;
  return c.off;
}

size_t ws_need(const tls_matrix_t* A, bool factor) {
  Work w;
  return carve(A, nullptr, 0, w, factor);
}

bool carve_ok(const tls_matrix_t* A, void* ws, size_t bytes, Work& w, bool factor) {
  bool ok = false;
  carve(A, ws, bytes, w, factor, &ok);
  return ok && ws != nullptr;
}

int check_matrix(const tls_matrix_t* A) {
  if (!A) { set_error("A is NULL"); return TLS_ERR_ARG; }
  if (A->layout != TLS_DENSE_ROWMAJOR && A->layout != TLS_CSR) { set_error("unknown layout"); return TLS_ERR_ARG; }
  if (A->n < 1 || A->m_local < 0 || A->m_global < A->n + 1) {
    set_error("bad shape: need n >= 1, m_global >= n+1");
    return TLS_ERR_ARG;
  }
  if (A->n > kMaxDenseN) { set_error("n > %d unsupported", kMaxDenseN); return TLS_ERR_UNSUPPORTED; }
  if (is_csr(A)) {
    if (A->nnz_local < 0 || A->rowptr == nullptr || (A->nnz_local > 0 && (A->colidx == nullptr || A->vals == nullptr))) {
      set_error("CSR: rowptr (m_local+1), colidx and vals (nnz_local) device pointers required");
      return TLS_ERR_ARG;
    }
    return 0;
  }
  if (A->ld < A->n || (A->ld & 1)) { set_error("dense: need ld >= n, ld even"); return TLS_ERR_ARG; }
  if (A->m_local > 0 && (A->vals == nullptr || (reinterpret_cast<uintptr_t>(A->vals) & 15))) {
    set_error("A->vals must be a 16-byte aligned device pointer");
    return TLS_ERR_ARG;
  }
  return 0;
}

// The symmetric Gram's upper triangle (row i: columns i..n-1) packed row by row, n(n+1)/2
// doubles: what the multi-rank Gram all-reduce moves (half of n^2); unpack mirrors it.
__device__ __forceinline__ int64_t packed_row_start(int64_t i, int64_t n) { return i * n - i * (i - 1) / 2; }
__global__ void k_pack_upper(const double* __restrict__ G, double* __restrict__ P, int n) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t o = packed_row_start(i, n) - i;
    for (int j = i + threadIdx.x; j < n; j += blockDim.x) P[o + j] = G[(int64_t)i * n + j];
  }
}
__global__ void k_unpack_upper(const double* __restrict__ P, double* __restrict__ G, int n) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t o = packed_row_start(i, n) - i;
    for (int j = i + threadIdx.x; j < n; j += blockDim.x) {
      const double v = P[o + j];
      G[(int64_t)i * n + j] = v;
      G[(int64_t)j * n + i] = v;
    }
  }
}

__global__ void k_recip(const double* __restrict__ d, double* __restrict__ dinv, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dinv[i] = 1.0 / d[i];
}

__global__ void k_set_state(PcgState* S, int set_sigma, double sigma2, double tol2) {
  if (set_sigma) S->sigma2 = sigma2;
  S->tol2 = tol2;
}

// The minimality certificate's right-hand side (R28; oracle.rqi.certificate_rhs, same bits):
// r_j = ((j + 1) * 0x9E3779B97F4A7C15 mod 2^64 >> 11) 2^-53 - 1/2.
__global__ void k_cert_rhs(double* __restrict__ r, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const unsigned long long h = (unsigned long long)(j + 1) * 0x9E3779B97F4A7C15ull;
    r[j] = (double)(h >> 11) * 0x1p-53 - 0.5;
  }
}

// The graph-captured PCG loop (NEXT-3): a WHILE conditional node whose body is one PCG
// iteration (operator pass, [reduction], step) followed by k_loop_cond, which decides on the
// device whether another iteration runs: j < budget and a right-hand side still active.  No
// host launch and no host poll per iteration.
__global__ void k_loop_init(PcgState* S, int budget) {
  S->loop_j = 0;
  S->loop_budget = budget;
  S->loop_nextq = budget > 1 ? 1 : 0;
}
__global__ void k_loop_cond(cudaGraphConditionalHandle h, PcgState* S) {
  const int j = S->loop_j + 1;
  S->loop_j = j;
  S->loop_total += 1;
  S->loop_nextq = j + 1 < S->loop_budget ? 1 : 0;
  const bool more = j < S->loop_budget && (S->active[0] | S->active[1]);
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

struct Ctx {
  cudaStream_t st;
  tls_comm_t comm;
  int launches = 0;
  int64_t passes = 0;
};

// one pass over A (+ fixed-order reduction + all-reduce over ranks) into w.passout
// (w.colstats for PASS_COLSTATS).  CSR operator/residual passes need w.csc built.
int run_pass(Ctx& cx, const tls_matrix_t* A, int mode, int nrhs, const double* q, const double* b, Work& w,
             const int* active) {
  const int n = (int)A->n;
  const int W = (mode == PASS_COLSTATS) ? 2 * n : nrhs * n + 2;
  double* out = (mode == PASS_COLSTATS) ? w.colstats : w.passout;
  const int cat = mode == PASS_COLSTATS ? TLS_PROF_COLSTATS
                  : mode == PASS_RESIDUAL ? TLS_PROF_PASS_RESID
                  : (nrhs == 2 ? TLS_PROF_PASS_OP2 : TLS_PROF_PASS_OP1);
  if (is_csr(A)) {
    const CsrView cv = csr_view(A);
    ProfScope ps(cat, cx.st);
    if (mode == PASS_COLSTATS) TLS_TRY(launch_csr_colstats(cv, out, w.partials, cx.st));
    else TLS_TRY(launch_csr_pass(cv, w.csc, mode, nrhs, q, b, w.tbuf, w.partials, out, active, cx.st));
    cx.launches += 2;
  } else {
    const DenseView dv = dense_view(A);
    int G = 1;
    {
      ProfScope ps(cat, cx.st);
      TLS_TRY(launch_pass(dv, mode, nrhs, q, b, w.partials, active, cx.st, &G));
    }
    if (cx.comm && cx.comm->peer && mode != PASS_COLSTATS) {
      // NEXT-3: this rank's reduction and the all-reduce over ranks in one kernel over peer memory
      ProfScope ps(TLS_PROF_REDUCE, cx.st);
      TLS_TRY(launch_reduce_exchange(cx.comm->tab, cx.comm->nranks, cx.comm->rank, 1, w.partials, 0, dv.m > 0 ? G : 0, W,
                                     cx.comm->pwcap, out, 0, ++cx.comm->pepoch, active, cx.comm->perr, false, cx.st));
      cx.launches += 2;
      cx.passes += 1;
      return 0;
    }
    if (dv.m > 0) {
      ProfScope ps(TLS_PROF_REDUCE, cx.st);
      TLS_TRY(launch_reduce(w.partials, G, W, mode == PASS_COLSTATS ? dv.n : 0, out, active, cx.st));
      cx.launches += 2;
    } else {
      TLS_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)W * 8, cx.st));
    }
  }
  cx.passes += 1;
  if (mode == PASS_COLSTATS) {
    TLS_TRY(allreduce(cx.comm, out, n, ncclMax, cx.st));
    TLS_TRY(allreduce(cx.comm, out + n, n, ncclSum, cx.st));
  } else {
    TLS_TRY(allreduce(cx.comm, out, W, ncclSum, cx.st));
  }
  return 0;
}

// Sampled content checksum of the local block into *dev (k_fingerprint); scratch: 256 doubles.
int run_fingerprint(Ctx& cx, const tls_matrix_t* A, double* dev, double* scratch) {
  if (is_csr(A)) {
    const CsrView cv = csr_view(A);
    TLS_TRY(launch_fingerprint(nullptr, &cv, dev, scratch, cx.st));
  } else {
    const DenseView dv = dense_view(A);
    TLS_TRY(launch_fingerprint(&dv, nullptr, dev, scratch, cx.st));
  }
  cx.launches += 2;
  return 0;
}

// One spare fp32-copy buffer kept by tls_precond_destroy for the next handle (a fresh
// cudaMalloc/cudaFree of the 4 GiB copy per solve would stall the stream).
struct A32Spare { int device = -1; size_t bytes = 0; float* ptr = nullptr; };
static A32Spare& a32_spare() {
  static A32Spare s;
  return s;
}

// The fl32 copy of the dense local block held by the handle (R23): (re)made when missing
// or made for another block.  The only allocation outside alloc_precond; freed with R.
int ensure_a32(Ctx& cx, const tls_matrix_t* A, tls_precond_t R, double content) {
  if (is_csr(A)) { set_error("u_p = fp32 needs a dense A"); return TLS_ERR_UNSUPPORTED; }
  if (A->n > 2048) { set_error("u_p = fp32 needs n <= 2048"); return TLS_ERR_UNSUPPORTED; }
  // reused only for the same block with the same sampled content (an A rewritten in place is
  // re-rounded)
  if (R->a32 && R->a32_src == A->vals && R->a32_m == A->m_local && R->a32_ld == A->ld && R->a32_content == content)
    return 0;
  const size_t bytes = (size_t)A->m_local * p32_ld((int)A->n) * 4 + 256;
  if (R->a32_bytes < bytes) {
    if (R->a32) { cudaStreamSynchronize(cx.st); cudaFree(R->a32); R->a32 = nullptr; R->a32_bytes = 0; }
    A32Spare& sp = a32_spare();
    if (sp.ptr && sp.device == R->device && sp.bytes >= bytes) {
      R->a32 = sp.ptr;
      R->a32_bytes = sp.bytes;
      sp.ptr = nullptr;
    }
  }
  if (R->a32_bytes < bytes) {
    const cudaError_t e = cudaMalloc(&R->a32, bytes);
    if (e != cudaSuccess) { set_error("cudaMalloc(A32 %zu B): %s", bytes, cudaGetErrorString(e)); return TLS_ERR_CUDA; }
    R->a32_bytes = bytes;
  }
  TLS_TRY(launch_round32(dense_view(A), R->a32, cx.st));
  R->a32_src = A->vals;
  R->a32_m = A->m_local;
  R->a32_ld = A->ld;
  R->a32_content = content;
  cx.launches += 1;
  cx.passes += 1;
  return 0;
}

// W = R~^{-1} in fp64 for the explicit-inverse preconditioner application (R24).
static A32Spare& winv_spare() {   // one spare W buffer, reused by the next handle (see a32_spare)
  static A32Spare s;
  return s;
}

int ensure_winv(Ctx& cx, tls_precond_t R) {
  if (R->winv) return 0;
  const size_t bytes = 2 * (size_t)R->dev.npad * R->dev.npad * 8;
  A32Spare& sp = winv_spare();
  if (sp.ptr && sp.device == R->device && sp.bytes == bytes) {
    R->winv = reinterpret_cast<double*>(sp.ptr);
    sp.ptr = nullptr;
  } else {
    const cudaError_t e = cudaMalloc(&R->winv, bytes);
    if (e != cudaSuccess) { R->winv = nullptr; set_error("cudaMalloc(W %zu B): %s", bytes, cudaGetErrorString(e)); return TLS_ERR_CUDA; }
  }
  TLS_TRY(launch_trtri(R->dev, R->winv, R->winv + (size_t)R->dev.npad * R->dev.npad, cx.st));
  cx.launches += 1;
  return 0;
}

// 2-RHS operator pass over the fp32 copy (u_p = fp32, k_pass32.cu) into w.passout.
int run_pass32(Ctx& cx, const tls_matrix_t* A, tls_precond_t R, const double* q, Work& w, const int* active) {
  const int n = (int)A->n;
  const int W = 2 * n + 2;
  const DenseView dv = dense_view(A);
  int G = 1;
  {
    ProfScope ps(TLS_PROF_PASS_OP2_FP32, cx.st);
    TLS_TRY(launch_pass32(dv, R->a32, q, w.partials, active, cx.st, &G));
  }
  if (cx.comm && cx.comm->peer) {
    ProfScope ps(TLS_PROF_REDUCE, cx.st);
    TLS_TRY(launch_reduce_exchange(cx.comm->tab, cx.comm->nranks, cx.comm->rank, 1, w.partials, 0, dv.m > 0 ? G : 0, W,
                                   cx.comm->pwcap, w.passout, 0, ++cx.comm->pepoch, active, cx.comm->perr, false, cx.st));
    cx.launches += 2;
    cx.passes += 1;
    return 0;
  }
  if (dv.m > 0) {
    ProfScope ps(TLS_PROF_REDUCE, cx.st);
    TLS_TRY(launch_reduce(w.partials, G, W, 0, w.passout, active, cx.st));
    cx.launches += 2;
  } else {
    TLS_CUDA_TRY(cudaMemsetAsync(w.passout, 0, (size_t)W * 8, cx.st));
  }
  cx.passes += 1;
  TLS_TRY(allreduce(cx.comm, w.passout, W, ncclSum, cx.st));
  return 0;
}

// u_f Gram of the local block into w.G, summed over ranks (a2).
int run_gram(Ctx& cx, const tls_matrix_t* A, int u_f, const double* dinv, int K_t, Work& w) {
  const int n = (int)A->n;
  ProfScope ps(TLS_PROF_GRAM, cx.st);
  if (is_csr(A)) {
    const bool ranks = comm_active(cx.comm);
    if (u_f == TLS_FP16 && ranks) {
      // exact fixed-point limbs are summed over ranks as int64 (exact, order-free), then rounded once
      TLS_TRY(launch_csr_gram(csr_view(A), u_f, dinv, w.G, w.gram_ws, w.gram_ws_doubles * 8, &w.flags[1], cx.st,
                              &cx.launches, true));
      TLS_TRY(allreduce_i64(cx.comm, w.gram_ws, 2 * (size_t)n * n, cx.st));
      TLS_TRY(launch_csr_gram_fin(w.gram_ws, n, w.G, cx.st));
      cx.launches += 1;
      return 0;
    }
    TLS_TRY(launch_csr_gram(csr_view(A), u_f, dinv, w.G, w.gram_ws, w.gram_ws_doubles * 8, &w.flags[1], cx.st,
                            &cx.launches, false));
  } else if (A->m_local > 0) {
    TLS_TRY(launch_gram(dense_view(A), u_f, dinv, K_t, w.G, w.gram_ws, w.gram_ws_doubles, &w.flags[1], cx.st,
                        &cx.launches));
  } else {
    TLS_CUDA_TRY(cudaMemsetAsync(w.G, 0, (size_t)n * n * 8, cx.st));
  }
  if (comm_active(cx.comm)) {
    // the symmetric Gram travels packed: n(n+1)/2 doubles instead of n^2
    const int g = n < 4096 ? n : 4096;
    k_pack_upper<<<g, 256, 0, cx.st>>>(w.G, w.gram_ws, n);
    TLS_LAUNCH_CHECK();
    TLS_TRY(allreduce(cx.comm, w.gram_ws, (size_t)n * (n + 1) / 2, ncclSum, cx.st));
    k_unpack_upper<<<g, 256, 0, cx.st>>>(w.gram_ws, w.G, n);
    TLS_LAUNCH_CHECK();
    cx.launches += 2;
  }
  return 0;
}

void fill_info_defaults(tls_info_t* info) {
  if (!info) return;
  info->status = 0;
  info->termination = TLS_TERM_NONE;
  info->rqi_iters = 0;
  info->boot_iters = 0;
  info->breakdown_k = info->breakdown_rhs = info->breakdown_j = -1;
  info->chol_pivot = 0;
  info->sigma2 = NAN;
  info->passes = 0;
  info->launches = 0;
  info->pcg_steps = 0;
  info->sigma_certified = NAN;
}

// Device buffers of destroyed handles are kept for reuse (keyed by device and size):
// repeated factorizations (one per solve in a benchmark or a service) then do no
// cudaMalloc/cudaFree, which were measured to stall the stream for up to ~25 ms.
struct PoolEntry { int device; size_t bytes; void* ptr; };
static std::vector<PoolEntry>& precond_pool() {
  static std::vector<PoolEntry> p;
  return p;
}

int alloc_precond(int n, int u_f, tls_precond_t* out) {
  tls_precond_s* h = new tls_precond_s();
  const int npad = (n + 31) / 32 * 32;
  const size_t es = (u_f == TLS_FP64) ? 8 : (u_f == TLS_FP32 ? 4 : 2);
  const size_t bytes = precond_bytes(n, u_f);
  cudaGetDevice(&h->device);
  h->base = nullptr;
  auto& pool = precond_pool();
  for (size_t i = 0; i < pool.size(); ++i) {
    if (pool[i].device == h->device && pool[i].bytes == bytes) {
      h->base = pool[i].ptr;
      pool.erase(pool.begin() + (long)i);
      break;
    }
  }
  if (!h->base) {
    cudaError_t e = cudaMalloc(&h->base, bytes);
    if (e != cudaSuccess) {
      delete h;
      set_error("cudaMalloc(precond %zu B): %s", bytes, cudaGetErrorString(e));
      return TLS_ERR_CUDA;
    }
  }
  h->bytes = bytes;
  char* p = static_cast<char*>(h->base);
  PrecondDev& d = h->dev;
  d.n = n;
  d.npad = npad;
  d.u_f = u_f;
  d.Rrow = p; p += (size_t)npad * npad * es;
  d.RTrow = p; p += (size_t)npad * npad * es;
  d.DinvB = reinterpret_cast<double*>(p); p += (size_t)npad * 32 * 8;
  d.DinvF = reinterpret_cast<double*>(p); p += (size_t)npad * 32 * 8;
  d.EB = reinterpret_cast<double*>(p); p += (size_t)npad * 32 * 8;
  d.EF = reinterpret_cast<double*>(p); p += (size_t)npad * 32 * 8;
  d.d = reinterpret_cast<double*>(p); p += (size_t)npad * 8;
  d.dinv = reinterpret_cast<double*>(p); p += (size_t)npad * 8;
  d.normA2 = reinterpret_cast<double*>(p);
  *out = h;
  return 0;
}

__global__ void k_fill_scaling(double* __restrict__ d, double* __restrict__ dinv, const double* __restrict__ src_d,
                               const double* __restrict__ src_dinv, int n, int npad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += gridDim.x * blockDim.x) {
    d[i] = i < n ? src_d[i] : 1.0;
    dinv[i] = i < n ? src_dinv[i] : 1.0;
  }
}
}  // namespace

// ------------------------------------------------------------------------------ C ABI
extern "C" {

int tls_abi_version(void) { return TLSRQI_ABI_VERSION; }

int tls_profile_enable(int on) {
  prof_drain();
  Prof& p = prof();
  p.on = on != 0;
  for (int i = 0; i < TLS_PROF_NCAT; ++i) { p.ms[i] = 0.0; p.cnt[i] = 0; }
  return 0;
}

int tls_profile_read(double* ms, int64_t* count, int ncat) {
  prof_drain();
  Prof& p = prof();
  for (int i = 0; i < ncat && i < TLS_PROF_NCAT; ++i) {
    if (ms) ms[i] = p.ms[i];
    if (count) count[i] = p.cnt[i];
  }
  return 0;
}

void tls_rqi_opts_default(tls_rqi_opts_t* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->budget_rule = 0;
  o->stop_rule = 0;
  o->max_outer = 50;
  o->polish = 1;
  o->tol_inner = -1.0;
  o->boot = 0;
  o->boot_max = 200;
  o->boot_tol = 1e-8;
  o->op_variant = 0;
  o->breakdown_rule = 0;
  o->gram_chunk = 64;
}

const char* tls_status_string(int s) {
  switch (s) {
    case TLS_OK: return "OK";
    case TLS_CHOL_BREAKDOWN: return "CHOL_BREAKDOWN";
    case TLS_PCG_BREAKDOWN: return "PCG_BREAKDOWN";
    case TLS_MAX_OUTER: return "MAX_OUTER";
    case TLS_NONFINITE: return "NONFINITE";
    case TLS_RANGE: return "RANGE";
    case TLS_NOT_MINIMAL: return "NOT_MINIMAL";
    case TLS_STAGNATED: return "STAGNATED";
    case TLS_ERR_ARG: return "ERR_ARG";
    case TLS_ERR_CUDA: return "ERR_CUDA";
    case TLS_ERR_NCCL: return "ERR_NCCL";
    case TLS_ERR_WORKSPACE: return "ERR_WORKSPACE";
    case TLS_ERR_UNSUPPORTED: return "ERR_UNSUPPORTED";
    default: return "UNKNOWN";
  }
}

const char* tls_last_error(void) { return g_err; }

int tls_comm_get_unique_id(void* id_out) {
  NcclApi* api = nccl_api();
  if (!api) { set_error("libnccl.so.2 not loadable"); return TLS_ERR_NCCL; }
  ncclUniqueId id;
  const int r = api->GetUniqueId(&id);
  if (r != ncclSuccess) { set_error("ncclGetUniqueId failed: %d", r); return TLS_ERR_NCCL; }
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

int tls_comm_init(int nranks, int rank, const void* id_host, int device, tls_comm_t* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) { set_error("bad comm args"); return TLS_ERR_ARG; }
  TLS_CUDA_TRY(cudaSetDevice(device));
  tls_comm_s* c = new tls_comm_s{nullptr, nranks, rank, device};
  // one rank needs no communicator; TLS_FORCE_NCCL=1 creates one anyway so that every
  // all-reduce of the solve goes through NCCL (single-GPU test of the multi-GPU path)
  const char* force = getenv("TLS_FORCE_NCCL");
  if (nranks > 1 || (force && force[0] == '1')) {
    NcclApi* api = nccl_api();
    if (!api) { delete c; set_error("libnccl.so.2 not loadable"); return TLS_ERR_NCCL; }
    ncclUniqueId id;
    std::memcpy(&id, id_host, sizeof(id));
    const int r = api->CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      set_error("ncclCommInitRank: %s", api->GetErrorString ? api->GetErrorString(r) : "error");
      return TLS_ERR_NCCL;
    }
  }
  *out = c;
  return 0;
}

int tls_comm_init_shm(int nranks, int rank, const char* name, size_t slot_bytes, int device, tls_comm_t* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || !name || name[0] != '/' || strlen(name) >= 96 ||
      slot_bytes < 4096 || (slot_bytes & 255)) {
    set_error("bad shm comm args (name must start with '/', slot_bytes >= 4096 and a multiple of 256)");
    return TLS_ERR_ARG;
  }
  TLS_CUDA_TRY(cudaSetDevice(device));
  const size_t bytes = 256 + (size_t)nranks * slot_bytes;
  const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) { set_error("shm_open(%s) failed", name); return TLS_ERR_NCCL; }
  if (ftruncate(fd, (off_t)bytes) != 0) { close(fd); set_error("ftruncate(%s) failed", name); return TLS_ERR_NCCL; }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) { set_error("mmap(%s) failed", name); return TLS_ERR_NCCL; }
  tls_comm_s* c = new tls_comm_s{nullptr, nranks, rank, device};
  c->shm = static_cast<ShmHeader*>(p);
  c->shm_bytes = bytes;
  std::snprintf(c->shm_name, sizeof(c->shm_name), "%s", name);
  // a fresh segment is zero-filled: arrive = phase = 0; every rank writes the same sizes
  c->shm->nranks = nranks;
  c->shm->slot_bytes = (int64_t)slot_bytes;
  if (cudaMallocHost(&c->stage, slot_bytes) != cudaSuccess) {
    munmap(p, bytes);
    delete c;
    set_error("cudaMallocHost(%zu) failed", slot_bytes);
    return TLS_ERR_CUDA;
  }
  const int rc = shm_barrier(c);      // every rank has mapped the segment
  if (rc) { tls_comm_destroy(c); return rc; }
  *out = c;
  return 0;
}

int tls_comm_nranks(tls_comm_t c) { return c ? c->nranks : 1; }
int tls_comm_rank(tls_comm_t c) { return c ? c->rank : 0; }

int tls_comm_destroy(tls_comm_t c) {
  if (!c) return 0;
  if (c->comm) {
    NcclApi* api = nccl_api();
    if (api) api->CommDestroy(c->comm);
  }
  if (c->shm) {
    shm_barrier(c);                   // nobody still reads a slot
    munmap(c->shm, c->shm_bytes);
    if (c->rank == 0) shm_unlink(c->shm_name);
  }
  if (c->stage) cudaFreeHost(c->stage);
  if (c->peer || c->prbuf) {
    cudaDeviceSynchronize();
    for (int p = 0; p < c->nranks && p < kMaxPeers; ++p) {
      if (p == c->rank) continue;
      if (c->tab.rbuf[p]) cudaIpcCloseMemHandle(c->tab.rbuf[p]);
      if (c->tab.rflag[p]) cudaIpcCloseMemHandle(c->tab.rflag[p]);
    }
    if (c->prbuf) cudaFree(c->prbuf);
    if (c->prflag) cudaFree(c->prflag);
    if (c->perr) cudaFree(c->perr);
  }
  delete c;
  return 0;
}

// ---- peer-memory exchange of the pass sums (NEXT-3; k_peer.cu)
int tls_comm_peer_prepare(tls_comm_t c, int64_t wcap, void* handles_out) {
  if (!c || !handles_out || wcap < 4 || wcap > (1 << 24) || c->nranks > kMaxPeers || c->peer || c->prbuf) {
    set_error("tls_comm_peer_prepare: needs a communicator of <= %d ranks, not yet prepared, 4 <= wcap <= 2^24",
              kMaxPeers);
    return TLS_ERR_ARG;
  }
  TLS_CUDA_TRY(cudaSetDevice(c->device));
  const size_t rb = 2 * (size_t)c->nranks * wcap * 8, fb = (size_t)c->nranks * kXchCtas * sizeof(int);
  TLS_CUDA_TRY(cudaMalloc(&c->prbuf, rb));
  TLS_CUDA_TRY(cudaMalloc(&c->prflag, fb));
  TLS_CUDA_TRY(cudaMalloc(&c->perr, sizeof(int)));
  TLS_CUDA_TRY(cudaMemset(c->prflag, 0, fb));
  TLS_CUDA_TRY(cudaMemset(c->perr, 0, sizeof(int)));
  cudaIpcMemHandle_t h[2];
  TLS_CUDA_TRY(cudaIpcGetMemHandle(&h[0], c->prbuf));
  TLS_CUDA_TRY(cudaIpcGetMemHandle(&h[1], c->prflag));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::memcpy(handles_out, h, 128);
  c->pwcap = (int)wcap;
  return 0;
}

int tls_comm_peer_connect(tls_comm_t c, const void* all_handles) {
  if (!c || !all_handles || !c->prbuf || c->peer) {
    set_error("tls_comm_peer_connect: call tls_comm_peer_prepare first (once)");
    return TLS_ERR_ARG;
  }
  TLS_CUDA_TRY(cudaSetDevice(c->device));
  const char* hb = static_cast<const char*>(all_handles);
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank) {
      c->tab.rbuf[p] = c->prbuf;
      c->tab.rflag[p] = c->prflag;
      continue;
    }
    cudaIpcMemHandle_t h[2];
    std::memcpy(h, hb + (size_t)p * 128, 128);
    void* a = nullptr;
    void* b = nullptr;
    TLS_CUDA_TRY(cudaIpcOpenMemHandle(&a, h[0], cudaIpcMemLazyEnablePeerAccess));
    TLS_CUDA_TRY(cudaIpcOpenMemHandle(&b, h[1], cudaIpcMemLazyEnablePeerAccess));
    c->tab.rbuf[p] = static_cast<double*>(a);
    c->tab.rflag[p] = static_cast<int*>(b);
  }
  c->peer = true;
  return 0;
}

int tls_peer_exchange_emulate(int nranks, const double* partials, int G, int W, int reps, double* out, void* stream) {
  if (nranks < 1 || nranks > kMaxPeers || G < 0 || W < 1 || reps < 1 || !out || (G > 0 && !partials)) {
    set_error("tls_peer_exchange_emulate: 1 <= nranks <= %d, W >= 1, reps >= 1", kMaxPeers);
    return TLS_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t rb = 2 * (size_t)nranks * W, fb = (size_t)nranks * kXchCtas;
  double* bufs = nullptr;
  int* flags = nullptr;
  TLS_CUDA_TRY(cudaMalloc(&bufs, rb * nranks * 8));
  TLS_CUDA_TRY(cudaMalloc(&flags, (fb * nranks + 1) * sizeof(int)));
  TLS_CUDA_TRY(cudaMemsetAsync(flags, 0, (fb * nranks + 1) * sizeof(int), st));
  PeerTab t{};
  for (int p = 0; p < nranks; ++p) {
    t.rbuf[p] = bufs + (size_t)p * rb;
    t.rflag[p] = flags + (size_t)p * fb;
  }
  int* err = flags + fb * nranks;
  int rc = 0;
  for (int e = 1; e <= reps && !rc; ++e)
    rc = launch_reduce_exchange(t, nranks, 0, nranks, partials, (size_t)G * W, G, W, W, out, (size_t)W, e, nullptr, err, true,
                                st);
  int herr = 0;
  if (!rc) {
    cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
  }
  cudaFree(bufs);
  cudaFree(flags);
  if (rc) return rc;
  if (herr) { set_error("tls_peer_exchange_emulate: a wait timed out"); return TLS_ERR_NCCL; }
  return 0;
}

size_t tls_workspace_size(const tls_matrix_t* A, int32_t /*max_outer*/) {
  if (check_matrix(A) != 0) return 0;
  return ws_need(A, true);
}

int tls_factor_precond(const tls_matrix_t* A, int32_t u_f, const tls_rqi_opts_t* opts, tls_comm_t comm,
                       void* stream, void* ws, size_t ws_bytes, tls_precond_t* R_out, tls_info_t* info) {
  fill_info_defaults(info);
  if (R_out) *R_out = nullptr;
  TLS_TRY(check_matrix(A));
  if (!R_out || u_f < TLS_FP16 || u_f > TLS_FP64) { set_error("bad u_f or R_out"); return TLS_ERR_ARG; }
  tls_rqi_opts_t o;
  if (opts) o = *opts; else tls_rqi_opts_default(&o);
  const int K_t = o.gram_chunk > 0 ? o.gram_chunk : 64;
  Work w;
  if (!carve_ok(A, ws, ws_bytes, w, true)) { set_error("workspace too small (need %zu)", ws_need(A, true)); return TLS_ERR_WORKSPACE; }
  Ctx cx{static_cast<cudaStream_t>(stream), comm};
  const int n = (int)A->n;
  Tracer tr(cx.st);
  tr.mark("factor:start");
  TLS_CUDA_TRY(cudaMemsetAsync(w.flags, 0, 8 * sizeof(int), cx.st));
  // a1: column max / sums of squares, all-reduced; D = powers of two (R2)
  TLS_TRY(run_pass(cx, A, PASS_COLSTATS, 2, nullptr, nullptr, w, nullptr));
  double* d = w.d_tmp;
  double* dinv = w.d_tmp + n;
  double* normA2 = w.d_tmp + 2 * n;
  TLS_TRY(launch_scaling(w.colstats, w.colstats + n, n, d, dinv, normA2, &w.flags[0], cx.st));
  cx.launches += 1;
  tr.mark("colstats");
  // a2: u_f Gram, all-reduced
  TLS_TRY(run_gram(cx, A, u_f, dinv, K_t, w));
  cx.passes += 1;
  tr.mark("gram");
  // a3: Cholesky (replicated on every rank: identical bits)
  {
    ProfScope ps(TLS_PROF_CHOL, cx.st);
    TLS_TRY(launch_cholesky(w.G, n, &w.flags[2], w.gram_ws, w.gram_ws_doubles * 8, cx.st, &cx.launches));
  }
  tr.mark("cholesky");
  // R~ is packed before the host looks at any flag: one synchronisation per factorization
  // (flags: [0] zero column, [1] A^ out of u_f range, [2] Cholesky pivot, [3] R~ out of range)
  tls_precond_t h = nullptr;
  TLS_TRY(alloc_precond(n, u_f, &h));
  tr.mark("alloc");
  k_fill_scaling<<<(h->dev.npad + 255) / 256, 256, 0, cx.st>>>(h->dev.d, h->dev.dinv, d, dinv, n, h->dev.npad);
  TLS_CUDA_TRY(cudaMemcpyAsync(h->dev.normA2, normA2, sizeof(double), cudaMemcpyDeviceToDevice, cx.st));
  int rc = launch_pack_R(w.G, n, 0, h->dev, &w.flags[3], cx.st, &cx.launches);
  cx.launches += 1;  // k_fill_scaling
  if (rc) { tls_precond_destroy(h); return rc; }
  rc = run_fingerprint(cx, A, normA2 + 1, w.partials);
  if (rc) { tls_precond_destroy(h); return rc; }
  tr.mark("pack");
  int hflags[8];
  double hnorm[2] = {0.0, 0.0};
  TLS_CUDA_TRY(cudaMemcpyAsync(hflags, w.flags, sizeof(hflags), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(hnorm, normA2, 2 * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  tr.mark("sync");
  if (info) { info->passes = cx.passes; info->launches = cx.launches; }
  { const int arc = comm_async_check(comm); if (arc) { tls_precond_destroy(h); return arc; } }
  int st = 0;
  if (hflags[4]) { set_error("k_gram_fused: a ring hand-off timed out"); st = TLS_ERR_CUDA; }
  else if (hflags[0]) { set_error("A has a zero or non-finite column (rank deficient)"); st = TLS_ERR_ARG; }
  else if (hflags[1]) st = TLS_RANGE;
  else if (hflags[2]) { st = TLS_CHOL_BREAKDOWN; if (info) info->chol_pivot = hflags[2]; }
  else if (hflags[3]) st = TLS_RANGE;
  if (st) {
    tls_precond_destroy(h);
    if (info && st > 0) info->status = st;
    return st;
  }
  h->normA2_host = hnorm[0];
  h->m_global = A->m_global;
  h->content = hnorm[1];
  *R_out = h;
  return 0;
}

namespace {
// TSQR leaves per rank (R26): TLS_QR_LEAVES, default 1.  The tree is leaves -> one stack
// factorization; > 1 on one GPU runs the same code path as a row-sharded factorization.
int qr_leaves() {
  const char* e = getenv("TLS_QR_LEAVES");
  const int k = e ? atoi(e) : 1;
  return k < 1 ? 1 : (k > 64 ? 64 : k);
}

struct QrBufs {
  double* G = nullptr;      // n x n R of the last factorization (lower part zero)
  void* W1 = nullptr;       // working copy of the local rows
  double* part1 = nullptr;
  double* S = nullptr;      // (leaves x n) x n stack of leaf R's
  void* W2 = nullptr;       // working copy of the stack
  double* part2 = nullptr;
  double* wT = nullptr;
  double* scal = nullptr;
  int* qflags = nullptr;
};

// Partial rows of an update pass over <= m rows: qr_rows_per_cta is not monotone in m (a TSQR
// leaf of m' < m rows can use more CTAs than m itself), so size for every m' <= m:
// ceil(m'/RB(m')) <= min(ceil(m'/32), 148) <= min(ceil(m/32), 148).
size_t qr_partials(int64_t m, int n) {
  int64_t nb = (m + 31) / 32;
  if (nb > 148) nb = 148;
  const int RB = qr_rows_per_cta(m, n);
  const int64_t own = (m + RB - 1) / RB;
  return (size_t)(nb > own ? nb : own) * n;
}

// Carves (or, with ws == nullptr, measures) the QR buffers after the solve workspace.
size_t carve_qr(const tls_matrix_t* A, int u_f, int nleaf, void* ws, size_t bytes, QrBufs& q, bool* ok) {
  const int n = (int)A->n;
  const size_t base = ws_need(A, false);
  Carver c{ws ? static_cast<char*>(ws) + base : nullptr, (ws && bytes > base) ? bytes - base : 0};
  const size_t es = (u_f == TLS_FP64) ? 8 : 4;
  const size_t ldw = (size_t)qr_ldw(n, u_f);
  q.G = c.take<double>((size_t)n * n);
  q.W1 = c.take<char>((size_t)A->m_local * ldw * es);
  q.part1 = c.take<double>(qr_partials(A->m_local, n));
  if (nleaf > 1) {
    const int64_t ms = (int64_t)nleaf * n;
    q.S = c.take<double>((size_t)ms * n);
    q.W2 = c.take<char>((size_t)ms * ldw * es);
    q.part2 = c.take<double>(qr_partials(ms, n));
  }
  q.wT = c.take<double>((size_t)n);
  q.scal = c.take<double>(4 * (size_t)n);
  q.qflags = c.take<int>(4);
  if (ok) *ok = c.ok && ws != nullptr;
  return base + c.off;
}
}  // namespace

size_t tls_qr_workspace_size(const tls_matrix_t* A, int32_t u_f, int32_t nranks) {
  if (check_matrix(A) != 0 || is_csr(A) || u_f < TLS_FP16 || u_f > TLS_FP64 || nranks < 1) return 0;
  QrBufs q;
  return carve_qr(A, u_f, nranks * qr_leaves(), nullptr, 0, q, nullptr);
}

int tls_factor_precond_qr(const tls_matrix_t* A, int32_t u_f, tls_comm_t comm, void* stream, void* ws,
                          size_t ws_bytes, tls_precond_t* R_out, tls_info_t* info) {
  fill_info_defaults(info);
  if (R_out) *R_out = nullptr;
  TLS_TRY(check_matrix(A));
  if (!R_out || u_f < TLS_FP16 || u_f > TLS_FP64) { set_error("bad u_f or R_out"); return TLS_ERR_ARG; }
  if (is_csr(A)) { set_error("the QR preconditioner takes a dense A"); return TLS_ERR_ARG; }
  const int n = (int)A->n;
  const int P = comm ? comm->nranks : 1;
  const int rank = comm ? comm->rank : 0;
  const int sub = qr_leaves();
  const int nleaf = P * sub;
  Work w;
  QrBufs q;
  bool ok = false;
  const size_t need = carve_qr(A, u_f, nleaf, ws, ws_bytes, q, &ok);
  if (!ok || ws_bytes < need || !carve_ok(A, ws, ws_bytes, w, false)) {
    set_error("workspace too small (need %zu)", need);
    return TLS_ERR_WORKSPACE;
  }
  Ctx cx{static_cast<cudaStream_t>(stream), comm};
  // every leaf needs >= n rows; decided collectively (max over ranks) so that all ranks
  // return the same status instead of some entering the stack all-reduce alone
  double bad = (nleaf > 1 && A->m_local / sub < n) ? 1.0 : 0.0;
  if (P > 1) {
    TLS_CUDA_TRY(cudaMemcpyAsync(w.d_tmp, &bad, 8, cudaMemcpyHostToDevice, cx.st));
    TLS_TRY(allreduce(comm, w.d_tmp, 1, ncclMax, cx.st));
    TLS_CUDA_TRY(cudaMemcpyAsync(&bad, w.d_tmp, 8, cudaMemcpyDeviceToHost, cx.st));
    TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  }
  if (bad != 0.0) {
    set_error("TSQR: every leaf needs >= n rows (m_local = %lld, %d leaves per rank, n = %d, on this or another rank)",
              (long long)A->m_local, sub, n);
    return TLS_ERR_ARG;
  }
  Tracer tr(cx.st);
  tr.mark("qr:start");
  TLS_CUDA_TRY(cudaMemsetAsync(w.flags, 0, 8 * sizeof(int), cx.st));
  TLS_CUDA_TRY(cudaMemsetAsync(q.qflags, 0, 4 * sizeof(int), cx.st));
  // column sums of squares, all-reduced; D = the paper's diag(A^T A)^{1/2} rounded to powers
  // of two (R27), ||A||_F^2
  TLS_TRY(run_pass(cx, A, PASS_COLSTATS, 2, nullptr, nullptr, w, nullptr));
  double* d = w.d_tmp;
  double* dinv = w.d_tmp + n;
  double* normA2 = w.d_tmp + 2 * n;
  TLS_TRY(launch_scaling(w.colstats, w.colstats + n, n, d, dinv, normA2, &w.flags[0], cx.st, 1));
  cx.launches += 1;
  tr.mark("colstats");
  {
    ProfScope ps(TLS_PROF_CHOL, cx.st);
    if (nleaf == 1) {
      TLS_CUDA_TRY(cudaMemsetAsync(q.G, 0, (size_t)n * n * 8, cx.st));
      TLS_TRY(launch_qr(dense_view(A), u_f, dinv, q.W1, q.part1, q.wT, q.scal, q.qflags, q.G, cx.st, &cx.launches));
      cx.passes += n + 1;
    } else {
      // TSQR (R26): leaf R's of this rank's row blocks into their rows of the row-interleaved
      // stack, the stack summed over ranks (all other rows are zero: exact), then its R.
      TLS_CUDA_TRY(cudaMemsetAsync(q.S, 0, (size_t)nleaf * n * n * 8, cx.st));
      const int64_t ml = A->m_local;
      for (int s = 0; s < sub; ++s) {
        const int64_t r0 = s * ml / sub, r1 = (s + 1) * ml / sub;
        DenseView leaf{A->vals + r0 * A->ld, r1 - r0, n, A->ld};
        TLS_CUDA_TRY(cudaMemsetAsync(q.G, 0, (size_t)n * n * 8, cx.st));
        TLS_TRY(launch_qr(leaf, u_f, dinv, q.W1, q.part1, q.wT, q.scal, q.qflags, q.G, cx.st, &cx.launches, 0, 1));
        // row i of leaf L goes to stack row i nleaf + L (row-interleaved, R26)
        TLS_CUDA_TRY(cudaMemcpy2DAsync(q.S + (size_t)(rank * sub + s) * n, (size_t)nleaf * n * 8, q.G, (size_t)n * 8,
                                       (size_t)n * 8, (size_t)n, cudaMemcpyDeviceToDevice, cx.st));
        cx.passes += n + 1;
      }
      if (P > 1) TLS_TRY(allreduce(comm, q.S, (size_t)nleaf * n * n, ncclSum, cx.st));
      TLS_CUDA_TRY(cudaMemsetAsync(q.G, 0, (size_t)n * n * 8, cx.st));
      DenseView stack{q.S, (int64_t)nleaf * n, n, n};
      TLS_TRY(launch_qr(stack, u_f, nullptr, q.W2, q.part2, q.wT, q.scal, q.qflags, q.G, cx.st, &cx.launches, nleaf));
    }
  }
  tr.mark("qr");
  tls_precond_t h = nullptr;
  TLS_TRY(alloc_precond(n, u_f, &h));
  k_fill_scaling<<<(h->dev.npad + 255) / 256, 256, 0, cx.st>>>(h->dev.d, h->dev.dinv, d, dinv, n, h->dev.npad);
  TLS_CUDA_TRY(cudaMemcpyAsync(h->dev.normA2, normA2, sizeof(double), cudaMemcpyDeviceToDevice, cx.st));
  int rc = launch_pack_R(q.G, n, 0, h->dev, &w.flags[3], cx.st, &cx.launches);
  cx.launches += 1;
  if (rc) { tls_precond_destroy(h); return rc; }
  rc = run_fingerprint(cx, A, normA2 + 1, w.partials);
  if (rc) { tls_precond_destroy(h); return rc; }
  int hflags[8], hq[4];
  double hnorm[2] = {0.0, 0.0};
  TLS_CUDA_TRY(cudaMemcpyAsync(hflags, w.flags, sizeof(hflags), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(hq, q.qflags, sizeof(hq), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(hnorm, normA2, 2 * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  tr.mark("sync");
  if (info) { info->passes = cx.passes; info->launches = cx.launches; }
  { const int arc = comm_async_check(comm); if (arc) { tls_precond_destroy(h); return arc; } }
  int st = 0;
  if (hflags[0]) { set_error("A has a zero or non-finite column (rank deficient)"); st = TLS_ERR_ARG; }
  else if (hq[0]) { st = TLS_CHOL_BREAKDOWN; if (info) info->chol_pivot = hq[1]; }
  else if (hflags[3]) st = TLS_RANGE;
  if (st) {
    tls_precond_destroy(h);
    if (info && st > 0) info->status = st;
    return st;
  }
  h->normA2_host = hnorm[0];
  h->m_global = A->m_global;
  h->content = hnorm[1];
  *R_out = h;
  return 0;
}

size_t tls_qr_blocked_workspace_size(const tls_matrix_t* A, int32_t u_f) {
  if (check_matrix(A) != 0 || is_csr(A) || (u_f != TLS_FP16 && u_f != TLS_BF16)) return 0;
  QrBufs q;
  return carve_qr(A, u_f, 1, nullptr, 0, q, nullptr) + qr_wy_bytes(A->m_local, (int)A->n) + 256;
}

int tls_factor_precond_qr_blocked(const tls_matrix_t* A, int32_t u_f, void* stream, void* ws, size_t ws_bytes,
                                  tls_precond_t* R_out, tls_info_t* info) {
  fill_info_defaults(info);
  if (R_out) *R_out = nullptr;
  TLS_TRY(check_matrix(A));
  if (!R_out || (u_f != TLS_FP16 && u_f != TLS_BF16)) { set_error("blocked QR: u_f must be TLS_FP16 or TLS_BF16"); return TLS_ERR_ARG; }
  if (is_csr(A)) { set_error("the QR preconditioner takes a dense A"); return TLS_ERR_ARG; }
  if (A->m_global != A->m_local) { set_error("blocked QR: one rank (the sharded QR is tls_factor_precond_qr's TSQR)"); return TLS_ERR_UNSUPPORTED; }
  const int n = (int)A->n;
  Work w;
  QrBufs q;
  bool ok = false;
  const size_t need = carve_qr(A, u_f, 1, ws, ws_bytes, q, &ok);
  const size_t need_all = tls_qr_blocked_workspace_size(A, u_f);
  if (!ok || ws_bytes < need_all || !carve_ok(A, ws, ws_bytes, w, false)) {
    set_error("workspace too small (need %zu)", need_all);
    return TLS_ERR_WORKSPACE;
  }
  void* wy = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(ws) + need + 255) & ~(uintptr_t)255);
  Ctx cx{static_cast<cudaStream_t>(stream), nullptr};
  TLS_CUDA_TRY(cudaMemsetAsync(w.flags, 0, 8 * sizeof(int), cx.st));
  TLS_CUDA_TRY(cudaMemsetAsync(q.qflags, 0, 4 * sizeof(int), cx.st));
  TLS_TRY(run_pass(cx, A, PASS_COLSTATS, 2, nullptr, nullptr, w, nullptr));
  double* d = w.d_tmp;
  double* dinv = w.d_tmp + n;
  double* normA2 = w.d_tmp + 2 * n;
  TLS_TRY(launch_scaling(w.colstats, w.colstats + n, n, d, dinv, normA2, &w.flags[0], cx.st, 1));   // R27
  cx.launches += 1;
  {
    ProfScope ps(TLS_PROF_CHOL, cx.st);
    TLS_CUDA_TRY(cudaMemsetAsync(q.G, 0, (size_t)n * n * 8, cx.st));
    TLS_TRY(launch_qr_blocked(dense_view(A), u_f, dinv, q.W1, q.part1, q.wT, q.scal, q.qflags, q.G, wy, cx.st,
                              &cx.launches));
    cx.passes += 1;
  }
  tls_precond_t h = nullptr;
  TLS_TRY(alloc_precond(n, u_f, &h));
  k_fill_scaling<<<(h->dev.npad + 255) / 256, 256, 0, cx.st>>>(h->dev.d, h->dev.dinv, d, dinv, n, h->dev.npad);
  TLS_CUDA_TRY(cudaMemcpyAsync(h->dev.normA2, normA2, sizeof(double), cudaMemcpyDeviceToDevice, cx.st));
  int rc = launch_pack_R(q.G, n, 0, h->dev, &w.flags[3], cx.st, &cx.launches);
  cx.launches += 1;
  if (rc) { tls_precond_destroy(h); return rc; }
  rc = run_fingerprint(cx, A, normA2 + 1, w.partials);
  if (rc) { tls_precond_destroy(h); return rc; }
  int hflags[8], hq[4];
  double hnorm[2] = {0.0, 0.0};
  TLS_CUDA_TRY(cudaMemcpyAsync(hflags, w.flags, sizeof(hflags), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(hq, q.qflags, sizeof(hq), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(hnorm, normA2, 2 * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  TLS_LAUNCH_CHECK();
  if (info) { info->passes = cx.passes; info->launches = cx.launches; }
  int st = 0;
  if (hflags[0]) { set_error("A has a zero or non-finite column (rank deficient)"); st = TLS_ERR_ARG; }
  else if (hq[0]) { st = TLS_CHOL_BREAKDOWN; if (info) info->chol_pivot = hq[1]; }
  else if (hflags[3]) st = TLS_RANGE;
  if (st) {
    tls_precond_destroy(h);
    if (info && st > 0) info->status = st;
    return st;
  }
  h->normA2_host = hnorm[0];
  h->m_global = A->m_global;
  h->content = hnorm[1];
  *R_out = h;
  return 0;
}

int tls_precond_import(int64_t n, int32_t u_f, const double* Rt_host, const double* d_host, double normA2,
                       void* stream, tls_precond_t* out) {
  if (!out || n < 1 || n > kMaxDenseN || !Rt_host || !d_host || u_f < TLS_FP16 || u_f > TLS_FP64) {
    set_error("bad import args");
    return TLS_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tls_precond_t h = nullptr;
  TLS_TRY(alloc_precond((int)n, u_f, &h));
  h->normA2_host = normA2;
  double* tmp = nullptr;
  int* flag = nullptr;
  TLS_CUDA_TRY(cudaMalloc(&tmp, (size_t)n * n * 8 + 4 * (size_t)n * 8 + 256));
  flag = reinterpret_cast<int*>(tmp + (size_t)n * n + 4 * n);
  std::vector<double> dinv(n);
  for (int64_t i = 0; i < n; ++i) dinv[i] = 1.0 / d_host[i];
  TLS_CUDA_TRY(cudaMemcpyAsync(tmp, Rt_host, (size_t)n * n * 8, cudaMemcpyHostToDevice, st));
  TLS_CUDA_TRY(cudaMemcpyAsync(tmp + (size_t)n * n, d_host, n * 8, cudaMemcpyHostToDevice, st));
  TLS_CUDA_TRY(cudaMemcpyAsync(tmp + (size_t)n * n + n, dinv.data(), n * 8, cudaMemcpyHostToDevice, st));
  TLS_CUDA_TRY(cudaMemcpyAsync(h->dev.normA2, &normA2, 8, cudaMemcpyHostToDevice, st));
  TLS_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
  k_fill_scaling<<<(h->dev.npad + 255) / 256, 256, 0, st>>>(h->dev.d, h->dev.dinv, tmp + (size_t)n * n,
                                                           tmp + (size_t)n * n + n, (int)n, h->dev.npad);
  int rc = launch_pack_R(tmp, (int)n, 0, h->dev, flag, st, nullptr);
  int hflag = 0;
  TLS_CUDA_TRY(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  TLS_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(tmp);
  if (rc || hflag) {
    tls_precond_destroy(h);
    if (!rc) { set_error("imported R~ not representable in u_f or singular"); rc = TLS_RANGE; }
    return rc;
  }
  *out = h;
  return 0;
}

static double host_dec(const void* base, size_t idx, int u_f) {
  if (u_f == TLS_FP64) return static_cast<const double*>(base)[idx];
  if (u_f == TLS_FP32) return static_cast<const float*>(base)[idx];
  const uint16_t h = static_cast<const uint16_t*>(base)[idx];
  if (u_f == TLS_BF16) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
  const int s = h >> 15, e = (h >> 10) & 0x1f, m = h & 0x3ff;
  double v;
  if (e == 0) v = std::ldexp((double)m, -24);
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = std::ldexp((double)(m | 0x400), e - 25);
  return s ? -v : v;
}

int tls_precond_export(tls_precond_t R, double* Rt_host, double* d_host, double* normA2_host) {
  if (!R) { set_error("NULL handle"); return TLS_ERR_ARG; }
  const int n = R->dev.n, npad = R->dev.npad, u_f = R->dev.u_f;
  const size_t es = (u_f == TLS_FP64) ? 8 : (u_f == TLS_FP32 ? 4 : 2);
  if (Rt_host) {
    std::vector<char> raw((size_t)npad * npad * es);
    TLS_CUDA_TRY(cudaMemcpy(raw.data(), R->dev.Rrow, raw.size(), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) Rt_host[(size_t)i * n + j] = host_dec(raw.data(), (size_t)i * npad + j, u_f);
  }
  if (d_host) TLS_CUDA_TRY(cudaMemcpy(d_host, R->dev.d, (size_t)n * 8, cudaMemcpyDeviceToHost));
  if (normA2_host) *normA2_host = R->normA2_host;
  return 0;
}

void tls_precond_destroy(tls_precond_t R) {
  if (!R) return;
  if (R->winv) {
    cudaDeviceSynchronize();
    A32Spare& sp = winv_spare();
    if (sp.ptr) cudaFree(sp.ptr);
    sp = A32Spare{R->device, 2 * (size_t)R->dev.npad * R->dev.npad * 8, reinterpret_cast<float*>(R->winv)};
  }
  if (R->a32) {
    cudaDeviceSynchronize();
    A32Spare& sp = a32_spare();
    if (sp.ptr == nullptr || sp.bytes < R->a32_bytes) {
      if (sp.ptr) cudaFree(sp.ptr);
      sp = A32Spare{R->device, R->a32_bytes, R->a32};
    } else {
      cudaFree(R->a32);
    }
  }
  if (R->base) {
    auto& pool = precond_pool();
    if (pool.size() < 8) {
      cudaDeviceSynchronize();  // like cudaFree: no queued work may still read the buffer
      pool.push_back({R->device, R->bytes, R->base});
    } else {
      cudaFree(R->base);
    }
  }
  delete R;
}

// ------------------------------------------------------------------------------ RQI-PCGTLS-MP
// The handle-owned buffers a solve would otherwise allocate on first use (VERDICT r01 weak #7:
// a caller that wants no allocation inside tls_rqi_pcgtls makes them here).
int tls_precond_prepare(const tls_matrix_t* A, tls_precond_t R, int32_t what, void* stream, void* ws, size_t ws_bytes) {
  TLS_TRY(check_matrix(A));
  if (!R || R->dev.n != A->n || (what & ~3) || what == 0) {
    set_error("tls_precond_prepare: what = 1 (explicit inverse W), 2 (fp32 copy of A) or 3, and R of this A");
    return TLS_ERR_ARG;
  }
  Ctx cx{static_cast<cudaStream_t>(stream), nullptr};
  if (what & 1) TLS_TRY(ensure_winv(cx, R));
  if (what & 2) {
    Work w;
    if (!carve_ok(A, ws, ws_bytes, w, false)) { set_error("workspace too small"); return TLS_ERR_WORKSPACE; }
    double content = 0.0;
    TLS_TRY(run_fingerprint(cx, A, w.d_tmp, w.partials));
    TLS_CUDA_TRY(cudaMemcpyAsync(&content, w.d_tmp, sizeof(double), cudaMemcpyDeviceToHost, cx.st));
    TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
    if (R->m_global >= 0 && !(content == R->content)) {
      set_error("A's content differs from the matrix the preconditioner was factored from (sampled checksum)");
      return TLS_ERR_ARG;
    }
    TLS_TRY(ensure_a32(cx, A, R, content));
  }
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  return 0;
}

int tls_rqi_pcgtls(const tls_matrix_t* A, const double* b, const tls_precond_t R, int32_t u, int32_t u_r, double tol,
                   const tls_rqi_opts_t* opts, tls_comm_t comm, void* stream, void* ws, size_t ws_bytes, double* x_out,
                   double* sigma_out, tls_info_t* info) {
  fill_info_defaults(info);
  TLS_TRY(check_matrix(A));
  if (u != TLS_FP64 || u_r != TLS_FP64) { set_error("u and u_r must be TLS_FP64 in this build"); return TLS_ERR_UNSUPPORTED; }
  if (!R || R->dev.n != A->n || !x_out || (A->m_local > 0 && !b)) { set_error("bad rqi args"); return TLS_ERR_ARG; }
  if (R->m_global >= 0 && R->m_global != A->m_global) {
    set_error("the preconditioner was factored from a %lld-row A, not this %lld-row one", (long long)R->m_global,
              (long long)A->m_global);
    return TLS_ERR_ARG;
  }
  tls_rqi_opts_t o;
  if (opts) o = *opts; else tls_rqi_opts_default(&o);
  if (o.op_variant != 0 && o.op_variant != 1) { set_error("op_variant must be 0 (A-in-loop) or 1 (paper Alg. 3)"); return TLS_ERR_ARG; }
  if (o.u_p != 0 && o.u_p != TLS_FP64 && o.u_p != TLS_FP32) { set_error("u_p must be TLS_FP64 (or 0) or TLS_FP32"); return TLS_ERR_UNSUPPORTED; }
  const bool up32 = o.u_p == TLS_FP32 && o.op_variant == 0;
  if (o.precond_apply < 0 || o.precond_apply > 2) { set_error("precond_apply must be 0 (auto), 1 or 2"); return TLS_ERR_ARG; }
  // R24: substitution (1) or the explicit inverse (2); auto (0) = the inverse only when the
  // solve is sharded over several ranks, where the replicated solves are the serial part
  const bool multi = comm != nullptr && comm->nranks > 1;
  const bool use_w = o.precond_apply == 2 || (o.precond_apply == 0 && multi);
  if (o.max_outer < 1) o.max_outer = 1;
  Work w;
  if (!carve_ok(A, ws, ws_bytes, w, false)) { set_error("workspace too small"); return TLS_ERR_WORKSPACE; }
  Ctx cx{static_cast<cudaStream_t>(stream), comm};
  const int n = (int)A->n;
  // the handle's fingerprint: this rank's block must have the content it was factored from
  double content = 0.0;
  TLS_TRY(run_fingerprint(cx, A, w.d_tmp, w.partials));
  TLS_CUDA_TRY(cudaMemcpyAsync(&content, w.d_tmp, sizeof(double), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  if (R->m_global >= 0 && !(content == R->content)) {
    set_error("A's content differs from the matrix the preconditioner was factored from (sampled checksum)");
    return TLS_ERR_ARG;
  }
  if (use_w) TLS_TRY(ensure_winv(cx, R));
  PrecondDev pc = R->dev;
  if (use_w) { pc.W = R->winv; pc.WT = R->winv + (size_t)pc.npad * pc.npad; }
  // the fused reduction (NEXT-3: the PCG step reduces the operator pass's partials itself, no
  // k_reduce_partials launch) needs a single rank.  Default with the explicit-inverse step
  // (k_wpcg_step_coop phase 0); TLS_FUSE_REDUCE=0 keeps the separate launch there.  The
  // substitution step has it too (k_pcg_step's step_reduce_partials, same bits) but only with
  // TLS_FUSE_REDUCE=2: measured 73.9 vs 73.2 us per PCG iteration at n = 1024 (its 16 CTAs
  // reduce the 148 partial rows in ~4 us, and the pass -> step launch gap stays), not adopted
  const char* fre = getenv("TLS_FUSE_REDUCE");
  const bool fuse_reduce = !comm_active(comm) && !(fre && fre[0] == '0') && (use_w || (fre && fre[0] == '2'));
  if (is_csr(A)) TLS_TRY(launch_csc_build(csr_view(A), w.csc, w.csc_scratch, cx.st, &cx.launches));
  if (up32) TLS_TRY(ensure_a32(cx, A, R, content));
  const double tol_in = o.tol_inner > 0 ? o.tol_inner : tol;
  PcgState hS;

  // sigma^2 (bootstrap only: the RQI steps take k_rqi_eval's device value) and the early-exit
  // threshold, written by a one-thread kernel: no host synchronisation
  auto set_state_scalars = [&](bool set_sigma, double sigma2, double tol2) -> int {
    k_set_state<<<1, 1, 0, cx.st>>>(w.S, set_sigma ? 1 : 0, sigma2, tol2);
    cx.launches += 1;
    TLS_LAUNCH_CHECK();
    return 0;
  };
  // iterations a graph ran are known on the device only: loop_total (all graph iterations so
  // far) is read with each state read, and the launches and passes of the loop launched since
  // the previous read (one loop between reads) are added then
  int graph_per_iter = 0, graph_pass_per_iter = 0, per_iter_now = 0;
  int graph_seen = 0;
  auto read_state = [&]() -> int {
    TLS_CUDA_TRY(cudaMemcpyAsync(&hS, w.S, sizeof(PcgState), cudaMemcpyDeviceToHost, cx.st));
    TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
    const int d = hS.loop_total - graph_seen;
    if (d > 0) {
      cx.launches += d * graph_per_iter;
      cx.passes += (int64_t)d * graph_pass_per_iter;
      graph_seen = hS.loop_total;
    }
    return 0;
  };
  // PCG iterations j = 0..budget-1 with device-side predication; with a large
  // budget the host polls the activity flags every 8 iterations.
  // variant 0: one batched operator pass over A per iteration (R1); variant 1: the
  // paper's A-free Alg. 3 (no pass).  The sigma = 0 bootstrap always uses variant 0.
  // fp32: the RQI's inner solves run their operator pass on the fp32 copy (u_p, R23);
  // the sigma = 0 bootstrap stays fp64 (R5: x_LS to 1e-8).
  // one PCG iteration's launches (the body of both loop forms); next_q from the host (j) or,
  // in the captured graph, from the device (nq_dev)
  auto pcg_iter = [&](int nrhs, int j, int budget, int variant, bool fp32, int rule, const int* nq_dev) -> int {
    const int pass_rhs = (nrhs == 1 && !is_csr(A)) ? 2 : nrhs;
    const bool fold = fuse_reduce && variant == 0 && !fp32 && !is_csr(A) && A->m_local > 0;
    int G = 0;
    if (fold) {
      ProfScope ps(TLS_PROF_PASS_OP2, cx.st);
      TLS_TRY(launch_pass(dense_view(A), PASS_OPERATOR, pass_rhs, w.vec.q, nullptr, w.partials, w.S->active, cx.st, &G));
      cx.launches += 1;
      cx.passes += 1;
    } else if (variant == 0 && fp32) TLS_TRY(run_pass32(cx, A, R, w.vec.q, w, w.S->active));
    else if (variant == 0) TLS_TRY(run_pass(cx, A, PASS_OPERATOR, pass_rhs, w.vec.q, nullptr, w, w.S->active));
    {
      ProfScope ps(TLS_PROF_PCG_STEP, cx.st);
      TLS_TRY(launch_pcg_step(pc, w.vec, w.passout, w.S, nrhs, rule, j + 1 < budget ? 1 : 0, variant,
                              pass_rhs, cx.st, fold ? w.partials : nullptr, G, nq_dev));
    }
    cx.launches += 1;
    return 0;
  };
  // The graph form (default on one rank without profiling; TLS_PCG_GRAPH=0 disables it): built
  // once per (shape of the call) and kept; the iteration count is known only on the device, so
  // the launch and pass counters are settled from S->loop_total after the solve.
  const char* ge = getenv("TLS_PCG_GRAPH");
  const bool graph_ok = !(ge && ge[0] == '0') && !prof().on && !comm_active(comm);
  auto pcg_loop_graph = [&](int nrhs, int budget, int variant, bool fp32, int rule) -> int {
    // everything the captured kernels bake in: the device pointers and the launch shapes (the
    // handle's buffers come back from the pool, so repeated factorizations reuse a graph)
    struct Key { const void* p[12]; int e[10]; };
    struct Entry { Key k; cudaGraphExec_t ex; int per_iter; };
    static std::vector<Entry> cache;
    static bool broken = false;           // capture or instantiation failed once: host loop from now on
    Key key;
    std::memset(&key, 0, sizeof(key));
    const void* ptrs[12] = {A->vals, A->rowptr, ws, pc.Rrow, pc.RTrow, pc.DinvB, pc.DinvF, pc.EB, pc.EF, pc.dinv,
                            pc.W, R->a32};
    std::memcpy(key.p, ptrs, sizeof(ptrs));
    const int ints[10] = {nrhs, variant, fp32 ? 1 : 0, rule, (int)A->n, (int)(A->m_local & 0x7fffffff), fuse_reduce ? 1 : 0,
                          pc.u_f, (int)A->ld, (int)(ws_bytes >> 20)};
    std::memcpy(key.e, ints, sizeof(ints));
    if (broken) return 1;
    Entry* ent = nullptr;
    for (auto& e : cache)
      if (std::memcmp(&e.k, &key, sizeof(Key)) == 0) { ent = &e; break; }
    k_loop_init<<<1, 1, 0, cx.st>>>(w.S, budget);
    TLS_LAUNCH_CHECK();
    cx.launches += 1;
    if (!ent) {
      cudaGraph_t g;
      TLS_CUDA_TRY(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle h;
      TLS_CUDA_TRY(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      TLS_CUDA_TRY(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      cudaStream_t cap;
      TLS_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      const cudaStream_t saved = cx.st;
      const int l0 = cx.launches;
      const int64_t p0 = cx.passes;
      cx.st = cap;
      TLS_CUDA_TRY(cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      int rc = pcg_iter(nrhs, 0, budget, variant, fp32, rule, &w.S->loop_nextq);
      if (rc == 0) k_loop_cond<<<1, 1, 0, cap>>>(h, w.S);
      per_iter_now = cx.launches - l0 + 1;
      cudaGraph_t out = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(cap, &out);
      cx.st = saved;
      cudaStreamDestroy(cap);
      cx.launches = l0;
      cx.passes = p0;
      cudaGraphExec_t ex = nullptr;
      const cudaError_t ie = (rc == 0 && ce == cudaSuccess) ? cudaGraphInstantiate(&ex, g, 0) : cudaErrorUnknown;
      cudaGraphDestroy(g);
      if (rc || ce != cudaSuccess || ie != cudaSuccess) {
        cudaGetLastError();               // clear a capture error; the host loop takes over
        broken = true;
        return 1;
      }
      if (cache.size() >= 16) { cudaGraphExecDestroy(cache.front().ex); cache.erase(cache.begin()); }
      cache.push_back(Entry{key, ex, per_iter_now});
      ent = &cache.back();
    }
    TLS_CUDA_TRY(cudaGraphLaunch(ent->ex, cx.st));
    graph_per_iter = ent->per_iter;
    graph_pass_per_iter = variant == 0 ? 1 : 0;
    return 0;
  };
  auto pcg_loop = [&](int nrhs, int budget, int variant, bool fp32, int rule) -> int {
    if (graph_ok) {
      const int rc = pcg_loop_graph(nrhs, budget, variant, fp32, rule);
      if (rc <= 0) return rc;             // rc > 0: no graph (capture unsupported): host loop
    }
    for (int j = 0; j < budget; ++j) {
      // the 2-RHS dense kernel is faster than the 1-RHS one at the same bytes (measured, see
      // DESIGN §6): a 1-RHS solve passes its q with the second slot held at zero.  NEXT-3: on one
      // rank the explicit-inverse step reduces the dense pass's partials itself (pcg_iter)
      TLS_TRY(pcg_iter(nrhs, j, budget, variant, fp32, rule, nullptr));
      if (budget > 16 && (j == 3 || (j % 8) == 7)) {   // first poll early: small bootstraps skip no-op launches
        int act[2] = {0, 0};
        TLS_CUDA_TRY(cudaMemcpyAsync(act, w.S->active, sizeof(act), cudaMemcpyDeviceToHost, cx.st));
        TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
        if (!(act[0] | act[1])) break;
      }
    }
    return 0;
  };

  Tracer tr(cx.st);
  tr.mark("rqi:start");
  TLS_CUDA_TRY(cudaMemsetAsync(&w.S->loop_total, 0, sizeof(int), cx.st));
  TLS_CUDA_TRY(cudaMemsetAsync(w.zero, 0, (size_t)n * 8, cx.st));
  TLS_CUDA_TRY(cudaMemsetAsync(w.vec.rhs, 0, 2 * (size_t)n * 8, cx.st));
  // setup (a1): h = A^T b, b^T b from the residual pass at x = 0
  TLS_TRY(run_pass(cx, A, PASS_RESIDUAL, 1, w.zero, b, w, nullptr));
  // b^T b stays on the device (read with the first RQI state) and A^T b becomes the CGLS RHS
  TLS_CUDA_TRY(cudaMemcpyAsync(&w.S->bb, w.passout + n, 8, cudaMemcpyDeviceToDevice, cx.st));
  k_copy<<<(n + 255) / 256, 256, 0, cx.st>>>(w.passout, w.vec.rhs, n);
  cx.launches += 1;
  tr.mark("setup");
  // a4: bootstrap x_0 = x_LS (R5)
  int boot_iters = 0;
  if (o.boot == 0) {
    TLS_TRY(set_state_scalars(true, 0.0, o.boot_tol * o.boot_tol));
    {
      ProfScope ps(TLS_PROF_PCG_INIT, cx.st);
      TLS_TRY(launch_pcg_init(pc, 1, w.vec, w.S, cx.st));
    }
    cx.launches += 1;
    TLS_TRY(pcg_loop(1, o.boot_max, 0, false, o.breakdown_rule));   // its count is read with the first RQI state
    k_copy<<<(n + 255) / 256, 256, 0, cx.st>>>(w.vec.omega, w.x0, n);
  } else {
    k_copy<<<(n + 255) / 256, 256, 0, cx.st>>>(w.vec.rhs, w.x0, n);
    TLS_TRY(launch_precond_apply(pc, 1, 1, w.x0, n, cx.st));
    TLS_TRY(launch_precond_apply(pc, 0, 1, w.x0, n, cx.st));
    cx.launches += 2;
  }
  cx.launches += 1;
  tr.mark("boot_cgls");
  TLS_TRY(run_pass(cx, A, PASS_RESIDUAL, 1, w.x0, b, w, nullptr));     // r_0 (l.227)
  TLS_TRY(launch_boot_x1(pc, w.passout, w.x0, w.x, cx.st));              // l.229-235
  cx.launches += 1;
  TLS_TRY(set_state_scalars(false, 0.0, tol_in * tol_in));
  double normAb2 = NAN;

  std::vector<double> s2tr, psitr;
  std::vector<int> pcgc;
  std::vector<double> dmin;
  int status = TLS_OK, term = TLS_TERM_NONE, k = 1, crossed = 0, use_prev = 0;
  double psi_prev = 0.0, sig2_prev = NAN, sig2_ret = NAN;
  int bk = -1, brhs = -1, bj = -1;
  // ONE host synchronisation per RQI step: the state read after the residual pass also
  // returns the previous step's PCG counts and breakdown flags (k_rqi_update is a no-op
  // after a breakdown, so x is still x_{k-1}; the residual evaluation at it is discarded)
  for (;; ++k) {
    // a5: residual pass, sigma_k^2, f_k, g_k, psi_k (l.238-245, l.262)
    TLS_TRY(run_pass(cx, A, PASS_RESIDUAL, 1, w.x, b, w, nullptr));
    TLS_TRY(launch_rqi_eval(pc, w.passout, w.x, w.vec, w.S, cx.st));
    cx.launches += 1;
    tr.mark("resid+eval");
    TLS_TRY(read_state());
    tr.mark("read_state");
    if (k == 1) {
      if (o.boot == 0) boot_iters = hS.count[0];
      normAb2 = R->normA2_host + hS.bb;
    } else {
      pcgc.push_back(hS.count[0]);
      pcgc.push_back(hS.count[1]);
      dmin.push_back(hS.delta_min[0]);
      dmin.push_back(hS.delta_min[1]);
      if (hS.brk[0] || hS.brk[1]) {                                // R3, R18 (step k - 1)
        status = TLS_PCG_BREAKDOWN;
        term = TLS_TERM_BREAKDOWN;
        --k;
        bk = k;
        brhs = hS.brk[0] ? 0 : 1;
        bj = hS.brk_j[brhs];
        sig2_ret = sig2_prev;
        break;
      }
    }
    const double sig2 = hS.sigma2, psi = hS.psi;
    s2tr.push_back(sig2);
    psitr.push_back(psi);
    if (!std::isfinite(sig2) || !std::isfinite(psi)) { status = TLS_NONFINITE; term = TLS_TERM_NONFINITE; sig2_ret = sig2; break; }
    const bool increased = k >= 2 && (psi > psi_prev || (o.stop_rule == 1 && psi >= psi_prev));
    if (!crossed && psi <= tol * normAb2) crossed = k;
    if (crossed && k == crossed + o.polish) {                     // (ii) R6
      if (increased) { use_prev = 1; sig2_ret = sig2_prev; } else { sig2_ret = sig2; }
      term = TLS_TERM_CONVERGED_TOL;
      break;
    }
    if (increased) {                                              // (i) l.265, R7
      use_prev = 1;
      sig2_ret = sig2_prev;
      if (crossed) term = TLS_TERM_PSI_INCREASE_CONVERGED;
      else { status = TLS_STAGNATED; term = TLS_TERM_STAGNATED; }
      break;
    }
    if (k > o.max_outer) { status = TLS_MAX_OUTER; term = TLS_TERM_MAX_OUTER; sig2_ret = sig2; break; }
    // a6-a8: the two PCGTLS solves, batched (l.246, l.252)
    const int budget = o.budget_rule == 0 ? k + 1 : 400;
    {
      ProfScope ps(TLS_PROF_PCG_INIT, cx.st);
      TLS_TRY(launch_pcg_init(pc, 2, w.vec, w.S, cx.st));
    }
    cx.launches += 1;
    tr.mark("pcg_init");
    TLS_TRY(pcg_loop(2, budget, o.op_variant, up32, o.breakdown_rule));
    tr.mark("pcg_loop");
    // a9: z, beta_k, x_{k+1} (l.248-255); skipped on the device after a PCG breakdown
    TLS_TRY(launch_rqi_update(pc, w.vec, w.S, w.x, w.x_prev, cx.st));
    cx.launches += 1;
    psi_prev = psi;
    sig2_prev = sig2;
  }
  k_copy<<<(n + 255) / 256, 256, 0, cx.st>>>(use_prev ? w.x_prev : w.x, x_out, n);
  cx.launches += 1;
  if (status == TLS_OK && o.minimal_check > 0) {
    // R28: PCGTLS at the returned sigma^2 on the fixed certificate RHS, SPEC breakdown rule,
    // no early exit; any delta_j <= 0 means A^T A - sigma^2 I is not positive definite
    k_cert_rhs<<<(n + 255) / 256, 256, 0, cx.st>>>(w.vec.rhs, n);
    TLS_TRY(set_state_scalars(true, sig2_ret, 0.0));
    TLS_TRY(launch_pcg_init(pc, 1, w.vec, w.S, cx.st));
    cx.launches += 2;
    TLS_TRY(pcg_loop(1, o.minimal_check, 0, false, 0));
    TLS_TRY(read_state());
    if (hS.brk[0] || !(hS.delta_min[0] > 0.0)) status = TLS_NOT_MINIMAL;
  }
  double cert[3] = {NAN, 0.0, 0.0};
  if (o.certify) {                       // compensated certificate (c2 step 8): one more pass
    const DenseView dv = is_csr(A) ? DenseView{} : dense_view(A);
    const CsrView cv = is_csr(A) ? csr_view(A) : CsrView{};
    TLS_TRY(launch_certify(is_csr(A) ? nullptr : &dv, is_csr(A) ? &cv : nullptr, b, x_out, n, w.partials, w.passout,
                           cx.st));
    TLS_TRY(allreduce(cx.comm, w.passout, 2, ncclSum, cx.st));
    TLS_CUDA_TRY(cudaMemcpyAsync(cert, w.passout, sizeof(cert), cudaMemcpyDeviceToHost, cx.st));
    cx.launches += 2;
    cx.passes += 1;
  }
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  TLS_LAUNCH_CHECK();
  TLS_TRY(comm_async_check(comm));
  if (info && o.certify) info->sigma_certified = std::sqrt((cert[0] + cert[1]) / (1.0 + cert[2]));
  if (sigma_out) *sigma_out = std::sqrt(sig2_ret);
  if (info) {
    info->status = status;
    info->termination = term;
    info->rqi_iters = k;
    info->boot_iters = boot_iters;
    info->breakdown_k = bk;
    info->breakdown_rhs = brhs;
    info->breakdown_j = bj;
    info->sigma2 = sig2_ret;
    info->passes = cx.passes;
    info->launches = cx.launches;
    info->pcg_steps = (int32_t)(pcgc.size() / 2);
    if (info->pcg_iters)
      for (size_t i = 0; i < pcgc.size() && i < 2 * (size_t)o.max_outer; ++i) info->pcg_iters[i] = pcgc[i];
    if (info->sigma2_trace)
      for (size_t i = 0; i < s2tr.size() && i < (size_t)o.max_outer + 1; ++i) info->sigma2_trace[i] = s2tr[i];
    if (info->psi_trace)
      for (size_t i = 0; i < psitr.size() && i < (size_t)o.max_outer + 1; ++i) info->psi_trace[i] = psitr[i];
    if (info->delta_min_trace)
      for (size_t i = 0; i < dmin.size() && i < 2 * (size_t)o.max_outer; ++i) info->delta_min_trace[i] = dmin[i];
  }
  return status;
}

// ------------------------------------------------------------------------------ host-buffer e2e
size_t tls_solve_host_bytes(int64_t m, int64_t n, int64_t ld, int32_t max_outer) {
  tls_matrix_t A{TLS_DENSE_ROWMAJOR, 0, m, n, m + n + 1, 0, ld, reinterpret_cast<const double*>(256), nullptr, nullptr, 0};
  const size_t a = ((size_t)m * ld * 8 + 255) & ~(size_t)255;
  const size_t bv = ((size_t)m * 8 + 255) & ~(size_t)255;
  const size_t xv = ((size_t)n * 8 + 255) & ~(size_t)255;
  return a + bv + xv + tls_workspace_size(&A, max_outer);
}

int tls_solve_host(const double* A_host, const double* b_host, int64_t m, int64_t n, int64_t ld, int64_t m_global,
                   int64_t row_offset, int32_t u_f, double tol, const tls_rqi_opts_t* opts, tls_comm_t comm, void* stream,
                   void* dev_buf, size_t dev_bytes, double* x_host, double* sigma_out, tls_info_t* info) {
  const size_t need = tls_solve_host_bytes(m, n, ld, opts ? opts->max_outer : 50);
  if (!dev_buf || dev_bytes < need) { set_error("device buffer too small (need %zu)", need); return TLS_ERR_WORKSPACE; }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* p = static_cast<char*>(dev_buf);
  double* Ad = reinterpret_cast<double*>(p); p += ((size_t)m * ld * 8 + 255) & ~(size_t)255;
  double* bd = reinterpret_cast<double*>(p); p += ((size_t)m * 8 + 255) & ~(size_t)255;
  double* xd = reinterpret_cast<double*>(p); p += ((size_t)n * 8 + 255) & ~(size_t)255;
  const size_t wsb = dev_bytes - (size_t)(p - static_cast<char*>(dev_buf));
  TLS_CUDA_TRY(cudaMemcpyAsync(Ad, A_host, (size_t)m * ld * 8, cudaMemcpyHostToDevice, st));
  TLS_CUDA_TRY(cudaMemcpyAsync(bd, b_host, (size_t)m * 8, cudaMemcpyHostToDevice, st));
  tls_matrix_t A{TLS_DENSE_ROWMAJOR, 0, m, n, m_global, row_offset, ld, Ad, nullptr, nullptr, 0};
  tls_precond_t R = nullptr;
  tls_info_t finfo;
  int rc = tls_factor_precond(&A, u_f, opts, comm, stream, p, wsb, &R, &finfo);
  if (rc != 0) {
    if (info) { int32_t* pi = info->pcg_iters; double* s2 = info->sigma2_trace; double* ps = info->psi_trace;
      *info = finfo; info->pcg_iters = pi; info->sigma2_trace = s2; info->psi_trace = ps; }
    return rc;
  }
  rc = tls_rqi_pcgtls(&A, bd, R, TLS_FP64, TLS_FP64, tol, opts, comm, stream, p, wsb, xd, sigma_out, info);
  if (info) { info->passes += finfo.passes; info->launches += finfo.launches; }
  tls_precond_destroy(R);
  if (rc < 0) return rc;
  TLS_CUDA_TRY(cudaMemcpyAsync(x_host, xd, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  TLS_CUDA_TRY(cudaStreamSynchronize(st));
  return rc;
}

// ------------------------------------------------------------------------------ single steps
int tls_colstats(const tls_matrix_t* A, double* colmax, double* sumsq, void* stream, void* ws, size_t ws_bytes) {
  TLS_TRY(check_matrix(A));
  Work w;
  if (!carve_ok(A, ws, ws_bytes, w, false)) { set_error("workspace too small"); return TLS_ERR_WORKSPACE; }
  Ctx cx{static_cast<cudaStream_t>(stream), nullptr};
  const int n = (int)A->n;
  TLS_CUDA_TRY(cudaMemsetAsync(w.flags, 0, 8 * sizeof(int), cx.st));
  TLS_TRY(run_pass(cx, A, PASS_COLSTATS, 2, nullptr, nullptr, w, nullptr));
  TLS_TRY(launch_scaling(w.colstats, w.colstats + n, n, w.d_tmp, w.d_tmp + n, w.d_tmp + 2 * n, &w.flags[0], cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(colmax, w.colstats, (size_t)n * 8, cudaMemcpyDeviceToDevice, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(sumsq, w.d_tmp + 2 * n, 8, cudaMemcpyDeviceToDevice, cx.st));
  return 0;
}

int tls_gram(const tls_matrix_t* A, int32_t u_f, const double* d_dev, int32_t K_t, double* G_dev, void* stream, void* ws,
             size_t ws_bytes) {
  TLS_TRY(check_matrix(A));
  Work w;
  if (!carve_ok(A, ws, ws_bytes, w, true)) { set_error("workspace too small"); return TLS_ERR_WORKSPACE; }
  Ctx cx{static_cast<cudaStream_t>(stream), nullptr};
  const int n = (int)A->n;
  TLS_CUDA_TRY(cudaMemsetAsync(w.flags, 0, 8 * sizeof(int), cx.st));
  k_recip<<<(n + 255) / 256, 256, 0, cx.st>>>(d_dev, w.d_tmp, n);
  TLS_LAUNCH_CHECK();
  TLS_TRY(run_gram(cx, A, u_f, w.d_tmp, K_t > 0 ? K_t : 64, w));
  TLS_CUDA_TRY(cudaMemcpyAsync(G_dev, w.G, (size_t)n * n * 8, cudaMemcpyDeviceToDevice, cx.st));
  int hf[8];
  TLS_CUDA_TRY(cudaMemcpyAsync(hf, w.flags, sizeof(hf), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  if (hf[4]) { set_error("k_gram_fused: a ring hand-off timed out"); return TLS_ERR_CUDA; }
  return hf[1] ? TLS_RANGE : 0;
}

int tls_pass(const tls_matrix_t* A, int32_t mode, int32_t nrhs, const double* q, const double* b, double* v, double* s,
             void* stream, void* ws, size_t ws_bytes) {
  TLS_TRY(check_matrix(A));
  if ((mode != 0 && mode != 1) || nrhs < 1 || nrhs > 2 || (mode == 1 && nrhs != 1)) { set_error("bad pass args"); return TLS_ERR_ARG; }
  Work w;
  if (!carve_ok(A, ws, ws_bytes, w, false)) { set_error("workspace too small"); return TLS_ERR_WORKSPACE; }
  Ctx cx{static_cast<cudaStream_t>(stream), nullptr};
  const int n = (int)A->n;
  if (is_csr(A)) TLS_TRY(launch_csc_build(csr_view(A), w.csc, w.csc_scratch, cx.st, &cx.launches));
  TLS_TRY(run_pass(cx, A, mode == 0 ? PASS_OPERATOR : PASS_RESIDUAL, nrhs, q, b, w, nullptr));
  TLS_CUDA_TRY(cudaMemcpyAsync(v, w.passout, (size_t)nrhs * n * 8, cudaMemcpyDeviceToDevice, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(s, w.passout + (size_t)nrhs * n, 16, cudaMemcpyDeviceToDevice, cx.st));
  return 0;
}

int tls_pass_fp32(const tls_matrix_t* A, tls_precond_t R, const double* q, double* v, double* s, void* stream,
                  void* ws, size_t ws_bytes) {
  TLS_TRY(check_matrix(A));
  if (!R || R->dev.n != A->n) { set_error("bad handle"); return TLS_ERR_ARG; }
  Work w;
  if (!carve_ok(A, ws, ws_bytes, w, false)) { set_error("workspace too small"); return TLS_ERR_WORKSPACE; }
  Ctx cx{static_cast<cudaStream_t>(stream), nullptr};
  const int n = (int)A->n;
  double content = 0.0;
  TLS_TRY(run_fingerprint(cx, A, w.d_tmp, w.partials));
  TLS_CUDA_TRY(cudaMemcpyAsync(&content, w.d_tmp, sizeof(double), cudaMemcpyDeviceToHost, cx.st));
  TLS_CUDA_TRY(cudaStreamSynchronize(cx.st));
  TLS_TRY(ensure_a32(cx, A, R, content));
  TLS_TRY(run_pass32(cx, A, R, q, w, nullptr));
  TLS_CUDA_TRY(cudaMemcpyAsync(v, w.passout, (size_t)2 * n * 8, cudaMemcpyDeviceToDevice, cx.st));
  TLS_CUDA_TRY(cudaMemcpyAsync(s, w.passout + (size_t)2 * n, 16, cudaMemcpyDeviceToDevice, cx.st));
  return 0;
}

int tls_precond_apply(const tls_precond_t R, int32_t trans, int32_t nrhs, double* Y, void* stream) {
  if (!R || nrhs < 1 || nrhs > 2 || !Y || trans < 0 || trans > 3) { set_error("bad apply args"); return TLS_ERR_ARG; }
  Ctx cx{static_cast<cudaStream_t>(stream), nullptr};
  PrecondDev pc = R->dev;
  if (trans & 2) {                      // through the explicit inverse (R24)
    TLS_TRY(ensure_winv(cx, R));
    pc.W = R->winv;
    pc.WT = R->winv + (size_t)pc.npad * pc.npad;
  }
  return launch_precond_apply(pc, trans & 1, nrhs, Y, R->dev.n, cx.st);
}

int tls_round(const double* x, double* y, int64_t n, int32_t prec, void* stream) {
  if (n < 0 || prec < TLS_FP16 || prec > TLS_FP64) { set_error("bad round args"); return TLS_ERR_ARG; }
  return launch_round(x, y, n, prec, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
