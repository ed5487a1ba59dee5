// bx_core.cu -- context, Algorithm-1 round loop and the C ABI
// (include/boxscreen_b200.h).  Host-side C++; every O(m k) operation is one of
// the kernels of bx_kernels.cuh launched on the context's stream.
//
// Reference mapping (file:line in /root/reference/pkg/src/boxscreen):
//   bx_ctx_create     Problem (model.py:55-87), ScreeningState (screening.py:27-36),
//                     TranslationVector (duality.py:48-59)
//   refresh()         Workspace.refresh (solvers.py:54-65)
//   primal_passes()   pg_step (solvers.py:101-116), cd_sweep (solvers.py:119-137),
//                     FISTA extension
//   dual_screen()     driver.py:183-201 (dual point, reduced dual, clamp_gap) and
//                     driver.py:213-221 (radius, slack, safe_screen_test)
//   compact()         apply_screening (screening.py:72-94) + refresh + step
//                     re-estimate (driver.py:222-235)
//   certified()       _certified_gap (driver.py:112-117)
//   as_step()         active_set_step (solvers.py:151-204), bx_active.cuh
//   bx_solve          solve (driver.py:131-256)
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/boxscreen_b200.h"
#include "bx_kernels.cuh"
#include "bx_cd.cuh"
#include "bx_batched.cuh"
#include "bx_batched2.cuh"
#include "bx_small.cuh"
#include "bx_active.cuh"
#include "bx_exchange.cuh"

using namespace bx;

namespace {

constexpr size_t kAlign = 256;
constexpr int kMaxRanks = 256;
constexpr int kSmallRounds = 1024;  // rounds per device-resident small-round launch
constexpr int kF32CertEvery = 50;   // fp32 storage: rounds between fp64 certificate attempts
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (torch's bundled libnccl.so.2) so the library has
// no link-time dependency; only the symbols the column-sharded path uses.
// ---------------------------------------------------------------------------
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int (*nccl_get_id_fn)(ncclUniqueId*);
typedef int (*nccl_init_rank_fn)(ncclComm_t*, int, ncclUniqueId, int);
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*nccl_destroy_fn)(ncclComm_t);
typedef const char* (*nccl_errstr_fn)(int);
enum { ncclInt32 = 2, ncclFloat32 = 7, ncclFloat64 = 8, ncclInt64 = 4, ncclSum = 0, ncclMax = 2 };

struct Nccl {
  void* h = nullptr;
  nccl_get_id_fn get_id = nullptr;
  nccl_init_rank_fn init_rank = nullptr;
  nccl_allreduce_fn allreduce = nullptr;
  nccl_destroy_fn destroy = nullptr;
  nccl_errstr_fn errstr = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    get_id = (nccl_get_id_fn)dlsym(h, "ncclGetUniqueId");
    init_rank = (nccl_init_rank_fn)dlsym(h, "ncclCommInitRank");
    allreduce = (nccl_allreduce_fn)dlsym(h, "ncclAllReduce");
    destroy = (nccl_destroy_fn)dlsym(h, "ncclCommDestroy");
    errstr = (nccl_errstr_fn)dlsym(h, "ncclGetErrorString");
    return get_id && init_rank && allreduce && destroy;
  }
};
Nccl g_nccl;

}  // namespace

// ---------------------------------------------------------------------------
// collectives of the column-sharded path.  dtype/op use the
// NCCL enums; the in-process group is the test transport on one GPU: ranks
// are threads of one process, each with its own stream, and synchronise only
// through host barriers (no kernel ever waits on another).
// ---------------------------------------------------------------------------
struct bx_group {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<const void*> ptrs;
  // fused reduce + exchange emulated over all ranks in one cooperative launch
  std::vector<void*> xbufs;    // each rank's exchange buffer (registered by bx_peer_open)
  std::vector<XArgs> xargs;    // each rank's arguments of the current call
  XArgs* xargs_dev = nullptr;  // device copy (rank 0 launches)
  // BX_GROUP_XREDUCE=rank: every rank thread launches the PRODUCTION kernel
  // (k_xreduce, the one the NCCL build runs per GPU) on its own stream, the
  // ranks' grids co-resident on this GPU and exchanging through the flags;
  // default: all ranks in one cooperative launch (k_xreduce_group)
  bool per_rank = false;
  ~bx_group() {
    if (xargs_dev) cudaFree(xargs_dev);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long my = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my; });
    }
  }
};

struct Comm {
  virtual ~Comm() {}
  // in-place allreduce of count elements on `stream`; returns 0 on success
  virtual int allreduce(void* buf, size_t count, int dtype, int op, cudaStream_t stream, std::string& err) = 0;
};

// receive buffer of the fused exchange: [2 parities][kXPeers][mp + kXExtra]
// fp64, then the flags [kXPeers][nb_max] u32
inline size_t xrecv_doubles(int64_t mp) { return (size_t)2 * kXPeers * (mp + kXExtra); }
inline size_t xbuf_bytes(int64_t mp, int nb_max) {
  return xrecv_doubles(mp) * 8 + (size_t)kXPeers * nb_max * 4;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm && g_nccl.destroy) g_nccl.destroy(comm);
  }
  int allreduce(void* buf, size_t count, int dtype, int op, cudaStream_t stream, std::string& err) override {
    const int r = g_nccl.allreduce(buf, buf, count, dtype, op, comm, stream);
    if (r != 0) err = std::string("ncclAllReduce: ") + (g_nccl.errstr ? g_nccl.errstr(r) : "error");
    return r;
  }
};

struct LocalComm : Comm {
  bx_group* g = nullptr;
  int rank = 0;
  void* tmp = nullptr;          // device scratch, >= count * 8 bytes
  const void** dptrs = nullptr; // device array of n pointers
  std::vector<const void*> snap;
  int allreduce(void* buf, size_t count, int dtype, int op, cudaStream_t stream, std::string& err) override {
    const int dt = dtype == ncclFloat64 ? 0 : dtype == ncclFloat32 ? 1 : dtype == ncclInt64 ? 2 : 3;
    const int o = op == ncclMax ? 1 : 0;
    const size_t es = (dt == 1 || dt == 3) ? 4 : 8;
    if (cudaStreamSynchronize(stream) != cudaSuccess) {
      err = "LocalComm: stream sync";
      return 1;
    }
    g->ptrs[rank] = buf;
    g->barrier();
    snap = g->ptrs;
    cudaMemcpyAsync(dptrs, snap.data(), g->n * sizeof(void*), cudaMemcpyHostToDevice, stream);
    int nb = (int)((count + 255) / 256);
    if (nb > 1024) nb = 1024;
    if (nb < 1) nb = 1;
    bx::k_group_reduce<<<nb, 256, 0, stream>>>(tmp, dptrs, g->n, (int64_t)count, dt, o);
    if (cudaStreamSynchronize(stream) != cudaSuccess) {
      err = "LocalComm: reduce";
      return 1;
    }
    g->barrier();  // every rank has read every buffer
    cudaMemcpyAsync(buf, tmp, count * es, cudaMemcpyDeviceToDevice, stream);
    return 0;
  }
  // fused reduce + exchange of every rank in ONE cooperative launch over all
  // ranks' buffers (ranks are threads on one GPU; no kernel waits on another)
  int xreduce(XArgs mine, int nb_max, bool f32, cudaStream_t stream, std::string& err) {
    if (cudaStreamSynchronize(stream) != cudaSuccess) {
      err = "LocalComm: stream sync";
      return 1;
    }
    g->xargs[rank] = mine;
    g->barrier();
    int rc = 0;
    if (g->per_rank) {
      // Every rank's pass has completed (stream syncs + barrier above), so the
      // SMs are free and the n grids of nb small CTAs are co-resident: no
      // rank's flag wait can depend on an unscheduled CTA, and the bounded
      // waits turn any surprise into DE_PEER_TIMEOUT instead of a hang.
      XArgs a = mine;
      for (int p = 0; p < g->n; ++p) {
        char* base = static_cast<char*>(g->xbufs[p]);
        a.recv[p] = reinterpret_cast<double*>(base);
        a.flag[p] = reinterpret_cast<unsigned*>(base + xrecv_doubles(a.mp) * 8);
      }
      a.my_recv = a.recv[rank];
      a.my_flag = a.flag[rank];
      void* kargs[] = {(void*)&a};
      const void* fn = f32 ? (const void*)k_xreduce<float> : (const void*)k_xreduce<double>;
      if (cudaLaunchCooperativeKernel(fn, dim3(a.nb), dim3(XT), kargs, 0, stream) != cudaSuccess) rc = 1;
      if (!rc && cudaStreamSynchronize(stream) != cudaSuccess) rc = 1;
      if (rc) err = "LocalComm: per-rank exchange launch";
      g->barrier();
      return rc;
    }
    if (rank == 0) {
      const int n = g->n;
      for (int q = 0; q < n; ++q) {
        XArgs& a = g->xargs[q];
        for (int p = 0; p < n; ++p) {
          char* base = static_cast<char*>(g->xbufs[p]);
          a.recv[p] = reinterpret_cast<double*>(base);
          a.flag[p] = reinterpret_cast<unsigned*>(base + xrecv_doubles(a.mp) * 8);
        }
        a.my_recv = a.recv[q];
        a.my_flag = a.flag[q];
      }
      if (!g->xargs_dev && cudaMalloc(&g->xargs_dev, kXPeers * sizeof(XArgs)) != cudaSuccess) rc = 1;
      if (!rc) cudaMemcpyAsync(g->xargs_dev, g->xargs.data(), n * sizeof(XArgs), cudaMemcpyHostToDevice, stream);
      const XArgs* dev = g->xargs_dev;
      int nb = mine.nb;
      void* kargs[] = {(void*)&dev, (void*)&nb};
      const void* fn = f32 ? (const void*)k_xreduce_group<float> : (const void*)k_xreduce_group<double>;
      if (!rc && cudaLaunchCooperativeKernel(fn, dim3(n * nb), dim3(XT), kargs, 0, stream) != cudaSuccess) rc = 1;
      if (!rc && cudaStreamSynchronize(stream) != cudaSuccess) rc = 1;
      if (rc) err = "LocalComm: fused exchange launch";
      (void)nb_max;
    }
    g->barrier();  // the results are in every rank's buffers
    return rc;
  }
};

// ---------------------------------------------------------------------------
// the context
// ---------------------------------------------------------------------------
// Small pinned host blocks (the per-round scalar mirrors) come from a
// process-wide free list: cudaMallocHost / cudaFreeHost per solve are
// heavyweight driver calls that serialise with anything else holding the
// driver (e.g. an nvidia-smi query) and showed up as 2x outliers in short
// timed solves.
constexpr size_t kPinBlock = 4096;
static std::mutex g_pin_mu;
static std::vector<void*> g_pin_free;
static void* pin_acquire(size_t bytes) {
  if (bytes > kPinBlock) return nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_free.empty()) {
      void* p = g_pin_free.back();
      g_pin_free.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  return cudaMallocHost(&p, kPinBlock) == cudaSuccess ? p : nullptr;
}
static void pin_release(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}

// A communicator that outlives contexts (bx_comm_create): the NCCL
// communicator plus the fused exchange's IPC-mapped receive buffers and
// their epoch counter, set up once per process group and borrowed by every
// sharded solve (a new ncclCommInitRank and IPC mapping per solve costs more
// than a config-4 solve step).
struct bx_comm {
  NcclComm* nc = nullptr;
  int rank = 0, nranks = 1;
  int xmode = 0;                  // 1 once every peer is mapped
  void* xbuf = nullptr;
  int64_t xmp = 0;                // rows the buffer was sized for
  int xnsm = 0;
  double* xpeer_recv[kXPeers] = {};
  unsigned* xpeer_flag[kXPeers] = {};
  std::vector<void*> xopened;
  unsigned xepoch = 0;            // shared by every context: flags only grow
  ~bx_comm() {
    for (void* p : xopened) cudaIpcCloseMemHandle(p);
    if (xbuf) cudaFree(xbuf);
    delete nc;
  }
};

struct bx_ctx {
  int64_t m = 0, n = 0, mp = 0;  // rows, columns, padded rows
  int dtype = BX_F64;
  size_t esz = 8;
  cudaStream_t stream = nullptr;
  int nsm = 148;
  int Gmax = 148;
  size_t smem_cap = 0;

  const void* A = nullptr;  // original matrix (never written)
  int64_t lda = 0;
  void* Aact = nullptr;  // compacted preserved columns
  int64_t ldact = 0;
  bool act_is_orig = true;  // the preserved columns are read from A itself (through idx when not dense)
  bool dense = true;        // preserved columns are contiguous in their buffer (no column map)
  int64_t kphys = 0;        // columns in the physical buffer the act view reads
  int32_t* pos[2] = {nullptr, nullptr};  // physical column of each preserved position (A_act)
  void *scr_dx = nullptr, *scr_dxp = nullptr;  // b - x, b - x_prev of newly screened columns

  // per-row vectors (mp elements)
  void *y = nullptr, *t = nullptr, *negy = nullptr, *z = nullptr, *z2 = nullptr, *off = nullptr, *tgt = nullptr;
  void *r = nullptr, *rprev = nullptr, *rc = nullptr, *theta = nullptr, *thetac = nullptr, *u = nullptr;
  // per-column state (ping-pong for compaction)
  int cur = 0;
  int32_t* idx[2] = {nullptr, nullptr};
  void *x[2] = {}, *xprev[2] = {}, *lo[2] = {}, *hi[2] = {}, *nrm[2] = {}, *att[2] = {};
  void* gprev[2] = {};  // FISTA: gradient at x_prev (g_{k-1}), carried through compaction
  void *g = nullptr, *v = nullptr, *coef = nullptr;
  // speculative round boundary: the round's screening gradient
  // comes from the next round's first step, which keeps what an undo needs
  // (x_{k-1}, g_{k-1} ping-pong with compaction: a step that stands through a
  // screening event can still be dropped at the end of the solve)
  void *xbak[2] = {}, *gbak[2] = {}, *rbak = nullptr;
  double* epart = nullptr;   // epsilon partials of the speculative step
  bool spec_on = true;       // env BX_SPEC=0 disables (a separate dot pass per round)
  bool zskip_on = true;      // env BX_NO_ZSKIP: the axpy of zero coefficients is computed (exactness test)
  bool fuse_on = true;       // env BX_FUSE=0: PG / FISTA passes leave the reduce to k_reduce
  bool spec_pending = false; // the current x has taken the next round's first step
  bool dot_spec = false;     // dot_done's g / epsilon partials came from a speculative step
  int last_kind = BX_APG;    // kind of the last primal passes (fine-grained C ABI)
  void* gram = nullptr;  // CD Gram blocks [ceil(n/32)][32][32]
  bool gram_dirty = true;
  // full-problem vectors
  void *xfull = nullptr, *lofull = nullptr, *hifull = nullptr, *nrmfull = nullptr, *attfull = nullptr;
  void *gfull = nullptr, *vfull = nullptr;
  // screening scratch
  uint8_t* flags = nullptr;
  int32_t* bcnt = nullptr;
  int32_t* scr_idx = nullptr;
  void* scr_val = nullptr;
  int64_t* sat_lo = nullptr;
  int64_t* sat_up = nullptr;
  int* probe = nullptr;
  // partials
  void* part = nullptr;
  int64_t ldp = 0;
  double* bpart = nullptr;   // pass block scalars
  double* bpart2 = nullptr;  // reduce block scalars
  double* bpart3 = nullptr;  // dual block scalars (4 per block)
  DevScalars* sc = nullptr;
  DevScalars* hsc = nullptr;  // pinned mirror

  int64_t k = 0;  // preserved count
  int64_t n_sat_lo = 0, n_sat_up = 0;
  int has_inf = 0;
  int bound_bits = 0;
  bool g_valid = false;
  bool theta_is_cert = false;
  bool have_apg_state = false;
  unsigned* bar = nullptr;  // grid barrier of the cooperative small-round kernel
  int* done = nullptr;      // small-round kernel: completed rounds, event flag, residual parity
  double* dtrace = nullptr; // small-round kernel / graph rounds: per-round records [kSmallRounds][TRACE_W]
  unsigned long long* stamps = nullptr;  // [0] batch start, [1..2] dual point begin / end, [3] excluded ns
  bool dual_stamps = false;  // (graph capture, screening off) stamp the dual point with k_stamp
  std::chrono::steady_clock::time_point batch_t;  // host clock when a device-resident batch was launched
  cudaEvent_t* dual_ev = nullptr;  // (host loop, screening off) events around the dual point
  bool dot_done = false;    // the round kernel already produced g and the eps partials
  int dot_G = 0;
  int64_t graph_body_kernels = 0;  // nodes of the captured round (launch accounting)
  bool small_ok = true;     // cooperative small-round path allowed (env BX_NO_SMALL disables)
  unsigned bar_epoch = 0;   // grid-barrier epochs issued so far
  int64_t launches = 0;
  int last_Gw = 0;  // block count of the last pass's scalar partials (bpart)
  int last_Ge = 0;  // block count of the last speculative step's epsilon partials (epart)
  std::string err;

  // live per-kernel timing (CUDA events on the context stream)
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  struct Pending {
    int slot;
    int e0;
    double bytes;
  };
  std::vector<Pending> pending;
  bx_prof_entry pstat[BX_PROF_SLOTS];

  // active-set solver: caller scratch (bx_ctx_set_active_set_workspace); the
  // passive mask rides in xprev[] (unused by this kind) through compaction
  int pcap = 0;                 // factor capacity min(m, n)
  double* asR = nullptr;        // [pcap][pcap] Cholesky factor, logical column j in slot as_cslot[j]
  int32_t *as_cslot = nullptr, *as_plist = nullptr, *as_hitf = nullptr;
  double *as_avec = nullptr, *as_rhs = nullptr, *as_c = nullptr, *as_b = nullptr, *as_s = nullptr,
         *as_frac = nullptr;
  AsState* as = nullptr;
  AsState* has = nullptr;       // pinned mirror
  bool as_dirty = true;         // the factor no longer matches the passive mask (compaction)
  int as_p = 0;                 // host copy of the factor size

  // fused reduce + peer exchange (bx_peer_alloc / bx_peer_open)
  int xmode = 0;                  // 0: collectives only, 1: IPC peers (GPUs), 2: in-process group
  void* xbuf = nullptr;           // this rank's receive buffer + flags (cudaMalloc: IPC-exportable)
  double* xpeer_recv[kXPeers] = {};
  unsigned* xpeer_flag[kXPeers] = {};
  std::vector<void*> xopened;     // IPC mappings to close
  unsigned xepoch = 0;
  unsigned* xepoch_p = nullptr;   // the epoch counter in use (own, or the borrowed bx_comm's)
  int xnb = 1;
  uint64_t xtimeout_ns = 30ull * 1000000000ull;  // bound of a peer wait (env BX_PEER_TIMEOUT_S)
  bool comm_owned = true;         // false: `comm` belongs to a bx_comm

  // multi-GPU column sharding
  Comm* comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t col_offset = 0, n_global = 0;
  void* rloc = nullptr;    // this rank's A x partial rows (mp elements)
  double* scal = nullptr;  // small cross-rank scalar buffers [16]
  double* dsum = nullptr;  // dual sums [8]
  int64_t* kvec = nullptr; // per-rank preserved counts [kMaxRanks]
  void* grp_tmp = nullptr;
  const void** grp_ptrs = nullptr;
  int val_bits = 0, col_bits = 0;  // validation flags recorded at create
  // an attached communicator always takes the collective code path (even
  // with one rank, which is how the NCCL plumbing is exercised on one GPU)
  bool sharded() const { return comm != nullptr; }
};

namespace {

int fail(bx_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return fail(c, BX_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

// context-free variant (communicator calls): status only
#define CUR(call)                          \
  do {                                     \
    if ((call) != cudaSuccess) return BX_ERR_CUDA; \
  } while (0)

#define LAUNCHED()                                                                                   \
  do {                                                                                               \
    ++c->launches;                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                             \
    if (e_ != cudaSuccess) return fail(c, BX_ERR_CUDA, "launch (%s:%d): %s", __FILE__, __LINE__, \
                                       cudaGetErrorString(e_));                                      \
  } while (0)

#define TRY(expr)            \
  do {                       \
    int s_ = (expr);         \
    if (s_ != BX_OK) return s_; \
  } while (0)

// ---- collectives ---------------------------------------------------------
int allreduce(bx_ctx* c, void* buf, size_t count, int dtype, int op) {
  if (!c->sharded()) return BX_OK;
  std::string e;
  if (c->comm->allreduce(buf, count, dtype, op, c->stream, e) != 0) return fail(c, BX_ERR_CUDA, "%s", e.c_str());
  ++c->launches;
  return BX_OK;
}
template <typename T>
constexpr int nccl_type() {
  return sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
}

// ---- live timing ---------------------------------------------------------
int prof_drain(bx_ctx* c) {
  if (c->pending.empty()) return BX_OK;
  CU(cudaEventSynchronize(c->ev[c->pending.back().e0 + 1]));
  for (const auto& p : c->pending) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, c->ev[p.e0], c->ev[p.e0 + 1]));
    c->pstat[p.slot].launches += 1;
    c->pstat[p.slot].ms += ms;
    c->pstat[p.slot].bytes += p.bytes;
  }
  c->pending.clear();
  return BX_OK;
}

// returns the event index pair to close with prof_end (or -1)
int prof_begin(bx_ctx* c) {
  if (!c->prof) return -1;
  if (c->ev.empty()) {
    c->ev.resize(2 * 2048);
    for (auto& e : c->ev)
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
  }
  if ((int)c->pending.size() * 2 + 2 > (int)c->ev.size()) {
    if (prof_drain(c) != BX_OK) return -1;
  }
  const int e0 = (int)c->pending.size() * 2;
  cudaEventRecord(c->ev[e0], c->stream);
  c->pending.push_back({-1, e0, 0.0});
  return e0;
}

void prof_end(bx_ctx* c, int e0, int slot, double bytes) {
  if (e0 < 0) return;
  cudaEventRecord(c->ev[e0 + 1], c->stream);
  c->pending.back().slot = slot;
  c->pending.back().bytes = bytes;
}

// Workspace carving
struct Carver {
  char* base;
  size_t off = 0;
  size_t cap;
  bool dry;
  void* take(size_t bytes) {
    off = align_up(off, kAlign);
    void* p = dry ? nullptr : base + off;
    off += align_up(bytes, kAlign);
    return p;
  }
};


void carve(bx_ctx* c, Carver& w) {
  const int64_t m = c->m, n = c->n, mp = c->mp;
  const size_t e = 8;       // every vector is fp64
  const size_t ea = c->esz; // storage type of A
  c->Aact = w.take((size_t)c->ldact * n * ea);
  void** rows[] = {&c->y, &c->t, &c->negy, &c->z, &c->z2, &c->off, &c->tgt,
                   &c->r, &c->rprev, &c->rc, &c->theta, &c->thetac, &c->u};
  for (void** p : rows) *p = w.take(mp * e);
  c->scr_dx = w.take(n * 8);
  c->scr_dxp = w.take(n * 8);
  for (int s = 0; s < 2; ++s) {
    c->pos[s] = (int32_t*)w.take(n * 4);
    c->idx[s] = (int32_t*)w.take(n * 4);
    c->x[s] = w.take(n * e);
    c->xprev[s] = w.take(n * e);
    c->lo[s] = w.take(n * e);
    c->hi[s] = w.take(n * e);
    c->nrm[s] = w.take(n * e);
    c->att[s] = w.take(n * e);
    c->gprev[s] = w.take(n * e);
  }
  for (int s = 0; s < 2; ++s) {
    c->xbak[s] = w.take(n * e);
    c->gbak[s] = w.take(n * e);
  }
  c->rbak = w.take(mp * e);
  c->epart = (double*)w.take(4 * c->Gmax * 8);
  c->g = w.take(n * e);
  c->v = w.take(n * e);
  c->coef = w.take(n * e);
  c->gram = w.take((size_t)((n + CD_B - 1) / CD_B) * 2 * CD_B * CD_B * 8);  // G_JJ and the cross block X_J
  c->xfull = w.take(n * e);
  c->lofull = w.take(n * e);
  c->hifull = w.take(n * e);
  c->nrmfull = w.take(n * e);
  c->attfull = w.take(n * e);
  c->gfull = w.take(n * e);
  c->vfull = w.take(n * e);
  c->flags = (uint8_t*)w.take(n);
  c->bcnt = (int32_t*)w.take((n / RT + 2) * 4 * 4);
  c->scr_idx = (int32_t*)w.take(n * 4);
  c->scr_val = w.take(n * e);
  c->sat_lo = (int64_t*)w.take(n * 8);
  c->sat_up = (int64_t*)w.take(n * 8);
  c->probe = (int*)w.take(64);
  c->ldp = mp;
  c->part = w.take((size_t)c->Gmax * c->ldp * 8);  // fp64 sized: also the small-round path's partial rows
  c->bar = (unsigned*)w.take(4 * kMaxRanks * 4);
  c->done = (int*)w.take(64);
  c->dtrace = (double*)w.take(kSmallRounds * TRACE_W * 8);
  c->stamps = (unsigned long long*)w.take(8 * 8);
  c->bpart = (double*)w.take(c->Gmax * 8 * 4);
  c->bpart2 = (double*)w.take(4096 * 8);
  c->bpart3 = (double*)w.take(4096 * 4 * 8);
  c->sc = (DevScalars*)w.take(sizeof(DevScalars));
  c->rloc = w.take(mp * e);
  c->scal = (double*)w.take(16 * 8);
  c->dsum = (double*)w.take(8 * 8);
  c->kvec = (int64_t*)w.take(kMaxRanks * 8);
  c->grp_tmp = w.take(mp * 8 + 4096);
  c->grp_ptrs = (const void**)w.take(kMaxRanks * 8);
  (void)m;
}

void shape_params(bx_ctx* c) {
  c->mp = round_up(c->m, 32);
  c->ldact = c->mp;
  c->Gmax = 2 * c->nsm;
}

// ---------------------------------------------------------------------------
// pass launcher
// ---------------------------------------------------------------------------
int pick_R(int64_t m, size_t esz) {
  const int V = (int)(16 / esz);
  const int64_t per = (int64_t)NT * V;
  // the smallest R with R * NT * V >= m: then every row-vector of the first
  // R - 1 chunks is full (k_pass drops their row guards)
  for (int R = 1; R <= RMAX; ++R)
    if ((int64_t)R * per >= m) return R;
  return -1;
}

template <typename T, int R, bool D, bool X, typename AT = T>
int launch_pass_RDX(bx_ctx* c, const PassArgs<T>& a, int G, size_t smem) {
  static bool attr_set = false;
  auto kern = k_pass<T, R, D, X, AT>;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_cap);
    if (e != cudaSuccess) return fail(c, BX_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  if (a.fuse) {
    // the fused reduce syncs the grid: every CTA must be resident (G <= #SMs,
    // one CTA per SM), which a cooperative launch guarantees
    void* args[] = {(void*)&a};
    CU(cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(NT), args, smem, c->stream));
  } else {
    kern<<<G, NT, smem, c->stream>>>(a);
  }
  LAUNCHED();
  return BX_OK;
}

template <typename T, int R>
int launch_pass_R(bx_ctx* c, const PassArgs<T>& a, bool dot, bool axpy, int G, size_t smem, bool acc64) {
  if constexpr (sizeof(T) == 4) {
    // certificate passes over fp32 storage: fp64 accumulation
    if (acc64 && dot && !axpy) return launch_pass_RDX<T, R, true, false, double>(c, a, G, smem);
    if (acc64 && !dot && axpy) return launch_pass_RDX<T, R, false, true, double>(c, a, G, smem);
  }
  if (dot && axpy) return launch_pass_RDX<T, R, true, true>(c, a, G, smem);
  if (dot) return launch_pass_RDX<T, R, true, false>(c, a, G, smem);
  return launch_pass_RDX<T, R, false, true>(c, a, G, smem);
}

int grid1d(bx_ctx* c, int64_t n) {
  int64_t b = (n + RT - 1) / RT;
  if (b > 4 * c->nsm) b = 4 * c->nsm;
  if (b < 1) b = 1;
  return (int)b;
}

// A "view" of columns the pass streams
template <typename T>
struct View {
  const T* A;
  int64_t ld;
  const int32_t* colmap;
  int64_t k;
};

template <typename T>
View<T> act_view(bx_ctx* c) {
  // lazy compaction: between physical rewrites the preserved columns are read
  // through a column map (each column is one contiguous bulk copy either way)
  if (c->act_is_orig) return View<T>{(const T*)c->A, c->lda, c->dense ? nullptr : c->idx[c->cur], c->k};
  if (!c->dense) return View<T>{(const T*)c->Aact, c->ldact, c->pos[c->cur], c->k};
  return View<T>{(const T*)c->Aact, c->ldact, nullptr, c->k};
}
template <typename T>
View<T> full_view(bx_ctx* c) {
  return View<T>{(const T*)c->A, c->lda, nullptr, c->n};
}

int pass_grid(bx_ctx* c, int64_t k) {
  int64_t G = (k + 7) / 8;
  if (G > c->nsm) G = c->nsm;
  if (G < 1) G = 1;
  return (int)G;
}

// FISTA's per-column gradient state and the speculative round-boundary step
// for a PG / FISTA pass
struct StepExtra {
  double* gprev = nullptr;  // g_{k-1} in, g_k out (U_APG)
  int spec = 0;             // speculative step: keep x_{k-1}/g_{k-1}, emit g_k + epsilon partials
  double* xbak = nullptr;
  double* gbak = nullptr;
  double* epart = nullptr;
  // fused reduce (k_pass reduces its own partial rows; cooperative launch)
  int fuse = 0;
  const double* roff = nullptr;
  double* rout = nullptr;
  double* rsave = nullptr;
  int rmode = 0;
  int rcounter = 0;
};

// Launch one streamed pass.  Returns the grid used through *G_out.
template <typename T>
int run_pass_blocked(bx_ctx* c, const View<T>& vw, int upd, const double* vin, const double* vin_prev, double* x,
                     double* xprev, const double* lo, const double* hi, double* g, const double* att,
                     const double* coef, double* bpart, int has_inf, int* G_out, const double* nrm,
                     const StepExtra& ex);

// One streamed pass over the columns of `vw`, rows [row0, row0 + mrows) (the
// whole column by default).  accumulate >= 0 turns a U_DOT pass into a
// row-block partial dot (0: first block, 1: add).
template <typename T>
int run_pass(bx_ctx* c, const View<T>& vw, int upd, const double* vin, const double* vin_prev, double* x,
             double* xprev, const double* lo, const double* hi, double* g, const double* att, const double* coef,
             double* bpart, int has_inf, int* G_out, const double* nrm = nullptr, int64_t row0 = 0,
             int64_t mrows = -1, int accumulate = -1, bool acc64 = false, const StepExtra& ex = StepExtra()) {
  const int64_t mm = mrows < 0 ? c->m : mrows;
  const int R = pick_R(mm, sizeof(T));
  if (R < 0 && mrows < 0)
    return run_pass_blocked<T>(c, vw, upd, vin, vin_prev, x, xprev, lo, hi, g, att, coef, bpart, has_inf, G_out,
                               nrm, ex);
  if (R < 0) return fail(c, BX_ERR_UNSUPPORTED, "row block of %lld rows", (long long)mm);
  const bool dot = (upd == U_DOT || upd == U_PG || upd == U_APG || upd == U_POWER);
  const bool axpy = (upd != U_DOT);
  const int C = cols_per_slot(R);
  const uint32_t colbytes = (uint32_t)align_up((size_t)mm * sizeof(T), 16);
  const uint32_t colstride = (uint32_t)align_up(colbytes, 128);
  const size_t scratch = SMAX * 8 + (NWARPS * CMAX + 4 * CMAX + 2) * 8 + 64;
  const size_t slot = (size_t)C * colstride;
  const int G = pass_grid(c, vw.k);
  int S = (int)((c->smem_cap - scratch) / slot);
  if (S > SMAX) S = SMAX;
  if (S < 1) return fail(c, BX_ERR_UNSUPPORTED, "column of %u bytes does not fit shared memory", colbytes);
  // stage the per-column state of each CTA when that costs no ring slot below 2
  const int64_t per_cta = (vw.k + G - 1) / G;
  const size_t stage = align_up((size_t)per_cta * PASS_STAGED * 8, 128);
  int pre = 0;
  {
    int S2 = (int)((c->smem_cap - scratch - stage) / slot);
    if (S2 > SMAX) S2 = SMAX;
    if (S2 >= (S < 2 ? S : 2) && S2 >= 1) {
      S = S2;
      pre = (int)per_cta;
    }
  }
  const size_t smem = S * slot + scratch + (pre ? stage : 0);
  PassArgs<T> a;
  a.A = vw.A + row0;
  a.ld = vw.ld;
  a.colmap = vw.colmap;
  a.k = vw.k;
  a.m = mm;
  a.vin = vin ? vin + row0 : nullptr;
  a.vin_prev = vin_prev ? vin_prev + row0 : nullptr;
  a.accumulate = accumulate;
  a.extrap = (upd == U_DOT && accumulate >= 0 && vin_prev != nullptr) ? 1 : 0;
  a.x = x;
  a.xprev = xprev;
  a.lo = lo;
  a.hi = hi;
  a.g = g;
  a.att = att;
  a.nrm = nrm;
  a.coef = coef;
  a.part = (T*)c->part + row0;
  a.ldp = c->ldp;
  a.bpart = bpart;
  a.sc = c->sc;
  a.upd = upd;
  a.has_inf = has_inf;
  a.C = C;
  a.S = S;
  a.colbytes = colbytes;
  a.colstride = colstride;
  a.pre = pre;
  a.gprev = ex.gprev;
  a.spec = ex.spec;
  a.zskip = c->zskip_on ? 1 : 0;
  a.xbak = ex.xbak;
  a.gbak = ex.gbak;
  a.epart = ex.spec ? ex.epart : nullptr;
  a.fuse = ex.fuse;
  a.roff = ex.roff;
  a.rout = ex.rout;
  a.rsave = ex.rsave;
  a.rpart = c->bpart2;
  a.rmode = ex.rmode;
  a.rcounter = ex.rcounter;
  if (G_out) *G_out = G;
  c->last_Gw = G;
  if (ex.spec) c->last_Ge = G;
  const int e0 = prof_begin(c);
  int st = BX_OK;
  switch (R) {
    case 1: st = launch_pass_R<T, 1>(c, a, dot, axpy, G, smem, acc64); break;
    case 2: st = launch_pass_R<T, 2>(c, a, dot, axpy, G, smem, acc64); break;
    case 4: st = launch_pass_R<T, 4>(c, a, dot, axpy, G, smem, acc64); break;
    case 6: st = launch_pass_R<T, 6>(c, a, dot, axpy, G, smem, acc64); break;
    case 8: st = launch_pass_R<T, 8>(c, a, dot, axpy, G, smem, acc64); break;
    case 10: st = launch_pass_R<T, 10>(c, a, dot, axpy, G, smem, acc64); break;
    case 12: st = launch_pass_R<T, 12>(c, a, dot, axpy, G, smem, acc64); break;
#if BX_NT < 512
    case 13: st = launch_pass_R<T, 13>(c, a, dot, axpy, G, smem, acc64); break;
    case 14: st = launch_pass_R<T, 14>(c, a, dot, axpy, G, smem, acc64); break;
    case 15: st = launch_pass_R<T, 15>(c, a, dot, axpy, G, smem, acc64); break;
    case 16: st = launch_pass_R<T, 16>(c, a, dot, axpy, G, smem, acc64); break;
#endif
    case 3: st = launch_pass_R<T, 3>(c, a, dot, axpy, G, smem, acc64); break;
    case 5: st = launch_pass_R<T, 5>(c, a, dot, axpy, G, smem, acc64); break;
    case 7: st = launch_pass_R<T, 7>(c, a, dot, axpy, G, smem, acc64); break;
    case 9: st = launch_pass_R<T, 9>(c, a, dot, axpy, G, smem, acc64); break;
    case 11: st = launch_pass_R<T, 11>(c, a, dot, axpy, G, smem, acc64); break;
    default: st = fail(c, BX_ERR_UNSUPPORTED, "R=%d", R);
  }
  if (e0 >= 0) {
    // algorithmic bytes: every streamed column once, the per-column state the
    // mode touches, the input row vector(s) and the output row vector once
    static const int col_vec[] = {3, 5, 5, 8, 0, 1};  // U_DOT..U_AX, elements per column
    const double es = (double)sizeof(T);  // storage of A; every vector is fp64
    double bytes = (double)vw.k * (double)c->m * es + (double)vw.k * col_vec[upd] * 8.0;
    if (dot) bytes += (double)c->m * 8.0;
    if (axpy) bytes += (double)c->m * 8.0;
    prof_end(c, e0, BX_PROF_PASS_DOT + upd, bytes);
  }
  return st;
}

// Row-blocked step for m beyond the register-resident envelope: the dot is
// accumulated over row blocks, the per-column update runs once the full dot is
// known (k_colupdate), then A x' is formed block by block into the same
// partial-row buffer.  Two reads of A per step instead of one.
template <typename T>
int run_pass_blocked(bx_ctx* c, const View<T>& vw, int upd, const double* vin, const double* vin_prev, double* x,
                     double* xprev, const double* lo, const double* hi, double* g, const double* att,
                     const double* coef, double* bpart, int has_inf, int* G_out, const double* nrm,
                     const StepExtra& ex) {
  constexpr int64_t BR = (int64_t)NT * (16 / sizeof(T)) * 8;  // rows per block (R = 8)
  const bool dot = (upd == U_DOT || upd == U_PG || upd == U_APG || upd == U_POWER);
  const bool axpy = (upd != U_DOT);
  double* gg = g ? g : (double*)c->g;
  int G = 1;
  if (dot) {
    for (int64_t r0 = 0, q = 0; r0 < c->m; r0 += BR, ++q) {
      const int64_t mr = std::min(BR, c->m - r0);
      // FISTA dots the plain residual too (gradient linearity, k_colupdate)
      TRY(run_pass<T>(c, vw, U_DOT, vin, nullptr, nullptr, nullptr, nullptr, hi, gg, att, nullptr, nullptr, 0, &G,
                      nullptr, r0, mr, q ? 1 : 0));
    }
  }
  const double* cf = coef ? coef : x;  // U_AX without coefficients multiplies by x
  int gw = G;
  if (upd != U_AX) {
    const int nb = grid1d(c, vw.k);
    k_colupdate<<<nb, RT, 0, c->stream>>>(upd, vw.k, x, xprev, lo, hi, gg, att, nrm, (double*)c->coef, bpart,
                                          has_inf, c->sc, ex.gprev, ex.spec, ex.xbak, ex.gbak, ex.epart);
    LAUNCHED();
    if (ex.spec) c->last_Ge = nb;
    if (upd == U_DOT) {
      if (G_out) *G_out = nb;
      return BX_OK;
    }
    cf = (const double*)c->coef;
    gw = nb;
  }
  if (axpy) {
    for (int64_t r0 = 0; r0 < c->m; r0 += BR) {
      const int64_t mr = std::min(BR, c->m - r0);
      TRY(run_pass<T>(c, vw, U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, cf,
                      nullptr, 0, &G, nullptr, r0, mr, -1));
    }
  }
  if (G_out) *G_out = G;
  c->last_Gw = gw;  // the reduce reads the k_colupdate block partials
  return BX_OK;
}

template <typename T>
int run_xreduce(bx_ctx* c, int G, const double* off, double* out, int mode, const double* wpart, int Gw,
                int counter, double* save) {
  XArgs a;
  memset(&a, 0, sizeof(a));
  a.save = save;
  a.timeout_ns = c->xtimeout_ns;
  a.part = c->part;
  a.ldp = c->ldp;
  a.G = G;
  a.m = c->m;
  a.mp = c->mp;
  a.off = off;
  a.out = out;
  a.sc = c->sc;
  a.bpart = c->bpart2;
  a.wpart = (wpart && Gw > 0) ? wpart : nullptr;
  a.Gw = Gw;
  a.stride = a.wpart ? ((mode & ~R_SPEC) == R_APG ? 2 : 1) : 0;
  a.mode = mode;
  a.counter = counter;
  a.rank = c->rank;
  a.nranks = c->nranks;
  a.nb = c->xnb;
  a.epoch = ++*(c->xepoch_p ? c->xepoch_p : &c->xepoch);
  const int e0 = prof_begin(c);
  if (c->xmode == 2) {
    std::string e;
    if (static_cast<LocalComm*>(c->comm)->xreduce(a, c->nsm, sizeof(T) == 4, c->stream, e) != 0)
      return fail(c, BX_ERR_CUDA, "%s", e.c_str());
    ++c->launches;
  } else {
    for (int q = 0; q < c->nranks; ++q) {
      a.recv[q] = c->xpeer_recv[q];
      a.flag[q] = c->xpeer_flag[q];
    }
    a.my_recv = c->xpeer_recv[c->rank];
    a.my_flag = c->xpeer_flag[c->rank];
    void* kargs[] = {(void*)&a};
    CU(cudaLaunchCooperativeKernel((const void*)k_xreduce<T>, dim3(c->xnb), dim3(XT), kargs, 0, c->stream));
    LAUNCHED();
  }
  prof_end(c, e0, BX_PROF_REDUCE, (double)c->m * sizeof(T) * G + 8.0 * c->m * (2.0 * c->nranks + 1));
  return BX_OK;
}

template <typename T>
int run_reduce(bx_ctx* c, int G, const double* off, double* out, int mode, const double* wpart, int Gw, int counter,
               double* save = nullptr) {
  // column-sharded with the peer exchange attached: one fused kernel
  if (c->sharded() && c->xmode) return run_xreduce<T>(c, G, off, out, mode, wpart, Gw, counter, save);
  const int64_t rb = 32 * (16 / (int64_t)sizeof(T));
  int nb = (int)((c->m + rb - 1) / rb);
  if (nb > 4 * c->nsm) nb = 4 * c->nsm;
  if (nb < 1) nb = 1;
  if (c->sharded()) {
    // phase A: this rank's partial rows; block scalars folded; both summed
    // over ranks (NCCL allreduce); phase B: offset, objective, mode logic
    k_reduce<T><<<nb, RT, 0, c->stream>>>((const T*)c->part, c->ldp, G, c->m, nullptr, (double*)c->rloc, c->sc,
                                           c->bpart2, nullptr, 0, R_PLAIN, counter, nullptr);
    LAUNCHED();
    const int stride = ((mode & ~R_SPEC) == R_APG) ? 2 : 1;
    if (wpart && Gw > 0) {
      k_fold<<<1, 32, 0, c->stream>>>(wpart, Gw, stride, 0, c->scal);
      LAUNCHED();
    }
    TRY(allreduce(c, c->rloc, (size_t)c->m, ncclFloat64, ncclSum));
    const int nb2 = (int)(((c->m + 63) / 64) < 4 * c->nsm ? (c->m + 63) / 64 : 4 * c->nsm);
    if (wpart && Gw > 0) TRY(allreduce(c, c->scal, (size_t)stride, ncclFloat64, ncclSum));
    k_reduce<double><<<nb2, RT, 0, c->stream>>>((const double*)c->rloc, c->ldp, 1, c->m, off, out, c->sc, c->bpart2,
                                           (wpart && Gw > 0) ? c->scal : nullptr, (wpart && Gw > 0) ? 1 : 0, mode,
                                           counter, save);
    LAUNCHED();
    return BX_OK;
  }
  const int e0 = prof_begin(c);
  k_reduce<T><<<nb, RT, 0, c->stream>>>((const T*)c->part, c->ldp, G, c->m, off, out, c->sc, c->bpart2, wpart, Gw,
                                         mode, counter, save);
  LAUNCHED();
  prof_end(c, e0, BX_PROF_REDUCE, (double)c->m * sizeof(T) * (G + 2 + (off ? 1 : 0)));
  return BX_OK;
}


// ---------------------------------------------------------------------------
// building blocks of a round
// ---------------------------------------------------------------------------
template <typename T>
int sync_scalars(bx_ctx* c) {
  CU(cudaMemcpyAsync(c->hsc, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return prof_drain(c);
}

int check_dev_err(bx_ctx* c) {
  const int e = c->hsc->err;
  if (e == 0) return BX_OK;
  if (e == DE_STEP_TOO_LARGE)
    return fail(c, BX_ERR_STEP_TOO_LARGE, "objective rose from %.6e to %.6e", c->hsc->err_v1, c->hsc->err_v2);
  if (e == DE_INTERNAL_CONSISTENCY) {
    const DualOut& d = c->hsc->act.gap_raw < -1e-9 ? c->hsc->act : c->hsc->cert;
    return fail(c, BX_ERR_INTERNAL_CONSISTENCY, "duality gap %.3e below round-off slack", d.gap_raw);
  }
  if (e == DE_PEER_TIMEOUT)
    return fail(c, BX_ERR_PEER_TIMEOUT, "fused peer exchange: a peer rank did not publish within %.1f s",
                1e-9 * (double)c->xtimeout_ns);
  return fail(c, BX_ERR_CUDA, "device error code %d", e);
}

// residual r = A_act x + (z - y) and its objective (solvers.py:64)
template <typename T>
int refresh_resid(bx_ctx* c) {
  const int s = c->cur;
  int G = 1;
  TRY(run_pass<T>(c, act_view<T>(c), U_AX, nullptr, nullptr, (double*)c->x[s], nullptr, nullptr, nullptr, nullptr,
                  nullptr, nullptr, nullptr, 0, &G));
  TRY(run_reduce<T>(c, G, (const double*)c->off, (double*)c->r, R_SET, nullptr, 0, 0));
  return BX_OK;
}

// FISTA: r_prev = A_act x_prev + (z - y)
template <typename T>
int refresh_rprev(bx_ctx* c) {
  const int s = c->cur;
  int G = 1;
  TRY(run_pass<T>(c, act_view<T>(c), U_AX, nullptr, nullptr, (double*)c->xprev[s], nullptr, nullptr, nullptr, nullptr,
                  nullptr, nullptr, nullptr, 0, &G));
  TRY(run_reduce<T>(c, G, (const double*)c->off, (double*)c->rprev, R_PLAIN, nullptr, 0, 0));
  return BX_OK;
}

// spectral_norm_estimate on the act view (solvers.py:72-86); one fused pass per
// power iteration: w = A'u, acc = A w, u <- acc / ||w||
template <typename T>
int power_iter(bx_ctx* c, int iters, const double* v0_host, double* sigma, int64_t k_global) {
  const int64_t k = c->k;
  if (k_global == 0) {
    *sigma = 0.0;
    return BX_OK;
  }
  if (k > 0) CU(cudaMemcpyAsync(c->coef, v0_host, k * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int G = 1;
  TRY(run_pass<T>(c, act_view<T>(c), U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                  (const double*)c->coef, nullptr, 0, &G));
  TRY(run_reduce<T>(c, G, nullptr, (double*)c->u, R_PLAIN, nullptr, 0, 0));
  CU(cudaMemsetAsync(&c->sc->err, 0, sizeof(int32_t), c->stream));
  double sig = 0.0;
  // chunks of 10 iterations between host checks of the ||w|| == 0 exit
  for (int it = 0; it < iters; ++it) {
    TRY(run_pass<T>(c, act_view<T>(c), U_POWER, (const double*)c->u, nullptr, nullptr, nullptr, nullptr, nullptr,
                    (double*)c->g, nullptr, nullptr, c->bpart, 0, &G));
    TRY(run_reduce<T>(c, G, nullptr, (double*)c->u, R_POWER, c->bpart, c->last_Gw, 1));
  }
  TRY(sync_scalars<T>(c));
  if (c->hsc->err == DE_POWER_ZERO) {
    // ||w|| hit zero: the reference returns 0.0 (solvers.py:82-83)
    CU(cudaMemsetAsync(&c->sc->err, 0, sizeof(int32_t), c->stream));
    *sigma = 0.0;
    return BX_OK;
  }
  sig = c->hsc->sigma;
  *sigma = sig;
  return BX_OK;
}

void internal_start_vector(int64_t k, int64_t seed, double* out) {
  std::mt19937_64 gen((uint64_t)seed);
  std::normal_distribution<double> nd(0.0, 1.0);
  double s = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    out[i] = nd(gen);
    s += out[i] * out[i];
  }
  s = std::sqrt(s);
  for (int64_t i = 0; i < k; ++i) out[i] /= s;
}

// preserved counts of all ranks -> (global count, this rank's offset in the
// global preserved order; ranks own contiguous column blocks)
int global_k(bx_ctx* c, int64_t* kg, int64_t* pos) {
  if (!c->sharded()) {
    *kg = c->k;
    *pos = 0;
    return BX_OK;
  }
  std::vector<int64_t> kv(c->nranks, 0);
  kv[c->rank] = c->k;
  CU(cudaMemcpyAsync(c->kvec, kv.data(), c->nranks * 8, cudaMemcpyHostToDevice, c->stream));
  TRY(allreduce(c, c->kvec, (size_t)c->nranks, ncclInt64, ncclSum));
  CU(cudaMemcpyAsync(kv.data(), c->kvec, c->nranks * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  *kg = 0;
  *pos = 0;
  for (int r = 0; r < c->nranks; ++r) {
    if (r < c->rank) *pos += kv[r];
    *kg += kv[r];
  }
  return BX_OK;
}

template <typename T>
int auto_step(bx_ctx* c, int iters, double alpha, bx_start_vector_fn fn, void* user, double* eta, double* sigma_out) {
  int64_t kg = 0, pos = 0;
  TRY(global_k(c, &kg, &pos));
  // the start vector is drawn over the GLOBAL preserved set in original order
  // (solvers.py:75-76) and this rank takes its slice
  std::vector<double> v0(kg > 0 ? kg : 1);
  if (kg > 0) {
    if (fn)
      fn(kg, 0, v0.data(), user);
    else
      internal_start_vector(kg, 0, v0.data());
  }
  double sig = 0.0;
  TRY(power_iter<T>(c, iters, v0.data() + pos, &sig, kg));
  if (sigma_out) *sigma_out = sig;
  const double s = sig / 0.999;  // solvers.py:95
  *eta = (s == 0.0) ? 1.0 : 0.99 * alpha / (s * s);
  CU(cudaMemcpyAsync(&c->sc->eta, eta, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

// cyclic coordinate descent sweeps on one thread-block cluster (bx_cd.cuh)
template <typename T>
int cd_sweeps(bx_ctx* c, int passes) {
  const int s = c->cur;
  if (c->k == 0) return BX_OK;
  if (!c->dense) {
    // CD reads A_act densely (block copies of consecutive columns): rewrite
    // the preserved columns contiguously first (a state loaded through
    // bx_set_state; the solve loop's compaction does it at every event)
    k_gather<T><<<(int)(c->k < 8 * c->nsm ? c->k : 8 * c->nsm), RT, 0, c->stream>>>(
        (const T*)c->A, c->lda, c->idx[s], c->k, c->m, (T*)c->Aact, c->ldact);
    LAUNCHED();
    c->act_is_orig = false;
    c->dense = true;
    c->kphys = c->k;
    c->gram_dirty = true;
  }
  View<T> vw = act_view<T>(c);
  constexpr int V = 16 / sizeof(T);
  int NC = 8;
  int64_t rows = round_up((c->m + NC - 1) / NC, V);
  const size_t fixed = (2 + 2 * CD_B + 2 * 16 * CD_B + 3 * CD_ST * CD_B) * 8 + 256 + 4096;  // + static smem of k_cd
  // three block slots (blocks J, J+1 and J+2 in flight) when they fit,
  // else two (the next block's copy then waits for this block's axpy)
  int slots = 3;
  auto smem_for = [&](int64_t r) {
    return (size_t)slots * (CD_B * (size_t)r * sizeof(T) + 2 * CD_B * CD_B * 8) + fixed;
  };
  auto fits = [&]() { return rows <= CD_RT * CD_RMAX && smem_for(rows) <= c->smem_cap; };
  if (!fits()) {
    NC = 16;
    rows = round_up((c->m + NC - 1) / NC, V);
  }
  if (!fits()) slots = 2;
  if (!fits())
    return fail(c, BX_ERR_UNSUPPORTED, "coordinate descent: m=%lld exceeds the cluster envelope", (long long)c->m);
  if (c->gram_dirty) {
    const int nblk = (int)((c->k + CD_B - 1) / CD_B);
    const int e0 = prof_begin(c);
    k_gram<T><<<nblk, 256, 0, c->stream>>>(vw.A, vw.ld, c->m, c->k, (double*)c->gram);
    LAUNCHED();
    prof_end(c, e0, BX_PROF_CD, (double)c->k * c->m * sizeof(T));
    c->gram_dirty = false;
  }
  CdArgs<T> a;
  a.A = vw.A;
  a.ld = vw.ld;
  a.m = c->m;
  a.k = c->k;
  a.x = (double*)c->x[s];
  a.x2 = (double*)c->coef;
  a.lo = (const double*)c->lo[s];
  a.hi = (const double*)c->hi[s];
  a.nrm = (const double*)c->nrm[s];
  a.gram = (const double*)c->gram;
  a.r = (double*)c->r;
  a.sc = c->sc;
  a.passes = passes;
  a.rows_per_cta = (int)rows;
  a.slots = slots;
  a.dbg = nullptr;
  {
    // BX_CD_DEBUG=1: per-phase clock sums of the sweep's critical path, printed at exit
    static unsigned long long* g_cd_dbg = nullptr;
    static bool g_cd_dbg_on = getenv("BX_CD_DEBUG") != nullptr;
    if (g_cd_dbg_on && !g_cd_dbg) {
      CU(cudaMalloc(&g_cd_dbg, 16 * 8));
      CU(cudaMemset(g_cd_dbg, 0, 16 * 8));

      static unsigned long long* keep = g_cd_dbg;
      atexit([] {
        unsigned long long h[16];
        if (cudaMemcpy(h, keep, 128, cudaMemcpyDeviceToHost) == cudaSuccess && h[6]) {
          fprintf(stderr, "k_cd row warp per block (clk): dots %.0f | butterfly %.0f | named barrier %.0f | combine+push %.0f | arrive.release %.0f\n",
                  (double)h[8] / h[6], (double)h[9] / h[6], (double)h[10] / h[6], (double)h[11] / h[6], (double)h[12] / h[6]);
          fprintf(stderr, "k_cd warp 0 per block (clk): cluster arrive %.0f | state loads %.0f | 32 dependent steps %.0f\n",
                  (double)h[13] / h[6], (double)h[14] / h[6], (double)h[15] / h[6]);
        }
        if (h[6])
          fprintf(stderr,
                  "k_cd per block (clk): load+sync %.0f | update chain %.0f (prefetch issue %.0f) | cluster wait %.0f | combine+corr %.0f | "
                  "sync %.0f | axpy phase %.0f | total %.0f over %llu blocks\n",
                  (double)h[0] / h[6], (double)h[1] / h[6], (double)h[7] / h[6], (double)h[2] / h[6], (double)h[3] / h[6],
                  (double)h[4] / h[6], (double)h[5] / h[6],
                  (double)(h[0] + h[1] + h[2] + h[3] + h[4] + h[5]) / h[6], h[6]);
      });
    }
    a.dbg = g_cd_dbg;
  }
  const size_t smem = smem_for(rows);
  const bool one_slot = rows <= CD_RT;  // one residual row per row thread: the small instantiation
  auto kern = slots == 3 ? (one_slot ? k_cd<T, 3, 1> : k_cd<T, 3, CD_RMAX>)
                         : (one_slot ? k_cd<T, 2, 1> : k_cd<T, 2, CD_RMAX>);
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(NC, 1, 1);
  lc.blockDim = dim3(CD_NT, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = NC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const int e0 = prof_begin(c);
  CU(cudaLaunchKernelEx(&lc, kern, a));
  LAUNCHED();
  prof_end(c, e0, BX_PROF_CD, 2.0 * (double)passes * c->k * c->m * sizeof(T));
  if (passes & 1) CU(cudaMemcpyAsync(c->x[s], c->coef, c->k * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  c->g_valid = false;
  return BX_OK;
}

// ---- cooperative small-round path (bx_small.cuh) ---------------------------
template <typename T, int R>
int launch_small_R(bx_ctx* c, SmallArgs& a, int G, size_t smem) {
  auto kern = k_round_small<T, R>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {(void*)&a};
  CU(cudaMemsetAsync(a.bar, 0, sizeof(unsigned), c->stream));  // the launch's barrier counter
  c->batch_t = std::chrono::steady_clock::now();
  const int e0 = prof_begin(c);
  CU(cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(SM_NT), args, smem, c->stream));
  LAUNCHED();
  prof_end(c, e0, BX_PROF_SMALL, (double)a.passes * (double)a.k * a.m * sizeof(T));
  return BX_OK;
}

struct SmallLoop {
  int max_rounds = 1;
  double tol = 0.0;
  int relative_gap = 0;
  int screening = 0;
  double slack_scale = 1e-12;
  double alpha = 1.0;
};

// Runs up to lp.max_rounds rounds on the small path.  *ran = 0 when the path
// does not apply.  With max_rounds > 1 the kernel stops at the first event
// round; *done = event-free rounds completed (trace records in c->dtrace) and
// *event = 1 when the following round's passes + dot pass also ran and its
// dual / screening step is left to the host.
template <typename T>
int small_rounds(bx_ctx* c, int kind, int passes, const SmallLoop& lp, int* ran, int* done, int* event,
                 bool dry = false) {
  *ran = 0;
  *done = 0;
  *event = 0;
  // (not while a speculative step is pending: the kernel starts a round from x)
  if (!c->small_ok || c->sharded() || (kind != BX_PG && kind != BX_APG) || c->k == 0 || c->spec_pending)
    return BX_OK;
  constexpr int V = 16 / sizeof(T);
  const int R = (int)((c->m + SM_NT * V - 1) / (SM_NT * V));
  if (R > 4) return BX_OK;
  const int G = c->nsm;
  const int ncmax = (int)((c->k + G - 1) / G);
  if (ncmax > SM_CMAX) return BX_OK;
  if (lp.max_rounds > 1 && (c->m + G - 1) / G > SM_NT) return BX_OK;
  const int colstride = (int)round_up(c->m, 2 * V);
  const size_t scratch = (16 * SM_CMAX + 2 * SM_CMAX + 2 * SM_NT + 8 + 8 * SM_CMAX + SM_NT + round_up(c->m, 8)) * 8 + 256;
  const size_t smem = align_up((size_t)ncmax * colstride * sizeof(T), 128) + scratch;
  if (smem > c->smem_cap) return BX_OK;
  if (dry) {  // would run (the caller only asks)
    *ran = 1;
    return BX_OK;
  }
  const int s = c->cur;
  View<T> vw = act_view<T>(c);
  SmallArgs a;
  a.dbg = nullptr;
  a.zskip = c->zskip_on ? 1 : 0;
  {
    // BX_SMALL_DEBUG=1: per-phase clock sums of a resident step (CTA 0), printed at exit
    static unsigned long long* g_sm_dbg = nullptr;
    static bool g_sm_dbg_on = getenv("BX_SMALL_DEBUG") != nullptr;
    if (g_sm_dbg_on && !g_sm_dbg) {
      CU(cudaMalloc(&g_sm_dbg, 16 * 8));
      CU(cudaMemset(g_sm_dbg, 0, 16 * 8));
      static unsigned long long* keep = g_sm_dbg;
      atexit([] {
        unsigned long long h[16];
        if (cudaMemcpy(h, keep, 128, cudaMemcpyDeviceToHost) == cudaSuccess && h[6])
          fprintf(stderr, "k_round_small thread 0 per step (clk): residual to smem + barrier %.0f | column dot %.0f | update %.0f | fold + partial-row loop %.0f\n",
                  (double)h[8] / h[6], (double)h[9] / h[6], (double)h[10] / h[6], (double)h[11] / h[6]);
        if (h[6])
          fprintf(stderr,
                  "k_round_small per step (clk): dots+update %.0f | partial rows %.0f | barrier 1 %.0f | row reduce %.0f | "
                  "barrier 2 %.0f | residual load + fold %.0f | total %.0f over %llu steps\n",
                  (double)h[0] / h[6], (double)h[1] / h[6], (double)h[2] / h[6], (double)h[3] / h[6],
                  (double)h[4] / h[6], (double)h[5] / h[6],
                  (double)(h[0] + h[1] + h[2] + h[3] + h[4] + h[5]) / h[6], h[6]);
      });
    }
    a.dbg = g_sm_dbg;
  }
  a.A = vw.A;
  a.ld = vw.ld;
  a.colmap = vw.colmap;
  a.k = c->k;
  a.m = (int)c->m;
  a.x = (double*)c->x[s];
  a.xprev = (double*)c->xprev[s];
  a.gprev = (double*)c->gprev[s];
  a.lo = (const double*)c->lo[s];
  a.hi = (const double*)c->hi[s];
  a.nrm = (const double*)c->nrm[s];
  a.att = (const double*)c->att[s];
  a.g = (double*)c->g;
  a.r[0] = (double*)c->r;
  a.r[1] = (double*)c->rprev;
  a.off = (const double*)c->off;
  a.part = (double*)c->part;
  a.ldp = c->ldp;
  a.bpart = c->bpart3;
  a.epart = c->bpart;
  a.sc = c->sc;
  a.bar = c->bar;
  a.passes = passes;
  a.kind = kind;
  a.g_valid = c->g_valid ? 1 : 0;
  a.has_inf = c->has_inf;
  a.do_dot = 1;
  a.rc = 0;
  a.colstride = colstride;
  a.ncmax = ncmax;
  a.max_rounds = lp.max_rounds < kSmallRounds ? lp.max_rounds : kSmallRounds;
  a.t = (const double*)c->t;
  a.tgt = (const double*)c->tgt;
  a.theta = (double*)c->theta;
  a.dpart = c->bpart3 + 8 * c->Gmax;
  a.trace = c->dtrace;
  a.stamp0 = c->stamps;
  a.done = c->done;
  a.tol = lp.tol;
  a.relative_gap = lp.relative_gap;
  a.screening = lp.screening;
  a.slack_scale = lp.slack_scale;
  a.alpha = lp.alpha;
  int st = BX_OK;
  switch (R) {
    case 1: st = launch_small_R<T, 1>(c, a, G, smem); break;
    case 2: st = launch_small_R<T, 2>(c, a, G, smem); break;
    case 3: st = launch_small_R<T, 3>(c, a, G, smem); break;
    default: st = launch_small_R<T, 4>(c, a, G, smem); break;
  }
  if (st != BX_OK) return st;
  int hd[3] = {0, 0, 0};
  CU(cudaMemcpyAsync(hd, c->done, sizeof(hd), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (a.max_rounds <= 1) {
    hd[0] = 0;
    hd[1] = 1;  // the single round's dual / screening step is the host's
    hd[2] = passes & 1;
  }
  if (hd[2] & 1) std::swap(c->r, c->rprev);
  c->dot_done = hd[1] != 0;
  c->dot_spec = false;
  c->dot_G = G;
  c->g_valid = true;
  *ran = 1;
  *done = hd[0];
  *event = hd[1];
  return BX_OK;
}

template <typename T>
int primal_passes(bx_ctx* c, int kind, int passes);
template <typename T>
int dual_screen(bx_ctx* c, int screening, double slack_scale, double alpha);
template <typename T>
int step_pass(bx_ctx* c, int kind, bool spec);
template <typename T>
bool spec_applies(bx_ctx* c, int kind, int passes);

// ---- graph-resident rounds (streamed PG / FISTA and CD) ---------------------
// The round sequence (primal passes, screening dot, dual point, sphere test)
// is captured once into the body of a CUDA-graph WHILE node; a one-thread
// kernel ends each round: it records the trace, and keeps looping while the
// round had no event (nothing screened, gap above tolerance, no error) and
// the round budget lasts.  The host then syncs once per batch instead of
// once per round.  The body must be a steady-state round -- the host state
// the capture leaves behind equals the state it started from (checked).
struct GraphKey {
  int64_t k, kphys;
  const void *r, *rprev, *x, *g;
  int cur, kind, passes, screening, g_valid, dense, act_is_orig, spec_pending;
  bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
static GraphKey graph_key(const bx_ctx* c, int kind, int passes, int screening) {
  GraphKey k;
  memset(&k, 0, sizeof(k));
  k.k = c->k;
  k.kphys = c->kphys;
  k.r = c->r;
  k.rprev = c->rprev;
  k.x = c->x[c->cur];
  k.g = c->g;
  k.cur = c->cur;
  k.kind = kind;
  k.passes = passes;
  k.screening = screening;
  k.g_valid = c->g_valid ? 1 : 0;
  k.dense = c->dense ? 1 : 0;
  k.act_is_orig = c->act_is_orig ? 1 : 0;
  k.spec_pending = c->spec_pending ? 1 : 0;
  return k;
}

struct GraphEndArgs {
  DevScalars* sc;
  double* trace;  // [limit][TRACE_W]
  unsigned long long* stamps;  // [1..2] the round's dual-point stamps, [3] excluded ns so far
  int* done;      // [0] event-free rounds, [1] event flag
  cudaGraphConditionalHandle h;
  const int* limit;  // device: rounds allowed in this launch
  double tol;
  int relative_gap;
  int screening;
  int spec;  // the body ends with a speculative step: the round's momentum is bak_mom_t
};

__global__ void k_graph_round_end(GraphEndArgs a) {
  const int q = a.done[0];
  const DualOut& d = a.sc->act;
  const double tol_r = a.relative_gap ? a.tol * fmax(1.0, fabs(d.primal)) : a.tol;
  const bool ev = a.sc->err != 0 || a.sc->err_spec != 0 || d.gap_raw < -1e-9 || d.gap < tol_r ||
                  (a.screening && (a.sc->g_lo + a.sc->g_up) > 0);
  if (!ev) {
    double* tr = a.trace + TRACE_W * q;
    const unsigned long long now = globaltimer();
    if (!a.screening) a.stamps[3] += a.stamps[2] - a.stamps[1];
    tr[7] = (double)now;
    tr[8] = (double)a.stamps[3];
    tr[0] = d.primal;
    tr[1] = d.dual;
    tr[2] = d.gap;
    tr[3] = d.eps;
    tr[4] = d.radius;
    tr[5] = a.spec ? a.sc->bak_mom_t : a.sc->mom_t;
    tr[6] = (double)(a.spec ? a.sc->bak_restarts : a.sc->restarts);
    a.done[0] = q + 1;
  } else {
    a.done[1] = 1;
  }
  cudaGraphSetConditional(a.h, (!ev && q + 1 < *a.limit) ? 1u : 0u);
}

// private capture / launch streams (+ join events) of the graph path, pooled
// per process like the pinned blocks (no stream / event creation per solve)
struct GraphStream {
  cudaStream_t cs = nullptr;
  cudaEvent_t join[2] = {nullptr, nullptr};
};
static std::mutex g_gs_mu;
static std::vector<GraphStream> g_gs_free;
static bool graph_stream_acquire(GraphStream* out) {
  {
    std::lock_guard<std::mutex> lk(g_gs_mu);
    if (!g_gs_free.empty()) {
      *out = g_gs_free.back();
      g_gs_free.pop_back();
      return true;
    }
  }
  GraphStream g;
  if (cudaStreamCreateWithFlags(&g.cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&g.join[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&g.join[1], cudaEventDisableTiming) != cudaSuccess)
    return false;
  *out = g;
  return true;
}
static void graph_stream_release(const GraphStream& g) {
  if (!g.cs) return;
  std::lock_guard<std::mutex> lk(g_gs_mu);
  g_gs_free.push_back(g);
}

struct GraphState {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  GraphStream gst;            // private capture / launch stream (the caller's may be the legacy default stream)
  cudaStream_t& cs = gst.cs;
  cudaEvent_t* join = gst.join;
  GraphKey key{};
  bool broken = false;  // capture not steady / unsupported: stop trying this solve
  ~GraphState() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    graph_stream_release(gst);
  }
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
  }
};

// Up to `limit` rounds on the graph.  *ran = 0 when the path does not apply;
// otherwise *done event-free rounds (trace in c->dtrace) and *event = 1 when
// the round after them ran and had an event (its dual / screening results are
// in the device scalars; g is valid, dot_done set).
template <typename T>
int graph_rounds(bx_ctx* c, GraphState& gs, int kind, int passes, int limit, double tol, int relative_gap,
                 int screening, double slack_scale, double alpha, int* ran, int* done, int* event) {
  *ran = 0;
  *done = 0;
  *event = 0;
  if (gs.broken || c->prof || c->sharded() || limit < 2 || c->k == 0) return BX_OK;
  if (kind != BX_PG && kind != BX_APG && kind != BX_CD) return BX_OK;
  {
    int r0 = 0, d0 = 0, e0 = 0;
    SmallLoop probe;
    TRY(small_rounds<T>(c, kind, passes, probe, &r0, &d0, &e0, true));
    if (r0) return BX_OK;  // the small-problem kernel owns these rounds
  }
  if (limit > kSmallRounds) limit = kSmallRounds;
  // with the speculative round boundary the body is: the round's remaining
  // steps, the next round's first step (speculative), the dual point of the
  // round -- steady only when the round's first step is already done
  const bool spec = spec_applies<T>(c, kind, passes);
  if (spec && !c->spec_pending) return BX_OK;
  const GraphKey key = graph_key(c, kind, passes, screening);
  if (!gs.cs && !graph_stream_acquire(&gs.gst)) {
    cudaGetLastError();
    gs.broken = true;
    return BX_OK;
  }
  if (!gs.exec || !(gs.key == key)) {
    gs.reset();
    // any failure while building (e.g. a driver without conditional nodes)
    // leaves the host loop in charge
    auto give_up = [&]() {
      cudaGetLastError();
      gs.reset();
      gs.broken = true;
      return BX_OK;
    };
    cudaGraphConditionalHandle h;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphCreate(&gs.graph, 0) != cudaSuccess ||
        cudaGraphConditionalHandleCreate(&h, gs.graph, 1, cudaGraphCondAssignDefault) != cudaSuccess)
      return give_up();
    p.conditional.handle = h;
    if (cudaGraphAddNode(&node, gs.graph, nullptr, 0, &p) != cudaSuccess) return give_up();
    cudaGraph_t body = p.conditional.phGraph_out[0];
    // capture on the private stream (the round functions launch on c->stream)
    cudaStream_t user_stream = c->stream;
    c->stream = gs.cs;
    if (cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) !=
        cudaSuccess) {
      cudaGetLastError();
      c->stream = user_stream;
      gs.reset();
      gs.broken = true;
      return BX_OK;
    }
    const int64_t launches0 = c->launches;
    // host-side state the captured calls advance (restored if the capture is
    // abandoned: nothing captured has run)
    struct {
      void *r, *rprev;
      bool spec_pending, dot_done, dot_spec, g_valid;
      int dot_G, last_Gw, last_Ge, last_kind;
    } saved{c->r, c->rprev, c->spec_pending, c->dot_done, c->dot_spec, c->g_valid, c->dot_G, c->last_Gw,
            c->last_Ge, c->last_kind};
    int st = primal_passes<T>(c, kind, passes);
    if (st == BX_OK && spec) st = step_pass<T>(c, kind, true);
    c->dual_stamps = !screening;
    if (st == BX_OK) st = dual_screen<T>(c, screening, slack_scale, alpha);
    c->dual_stamps = false;
    GraphEndArgs ga;
    ga.sc = c->sc;
    ga.trace = c->dtrace;
    ga.stamps = c->stamps;
    ga.done = c->done;
    ga.h = h;
    ga.limit = c->done + 2;
    ga.tol = tol;
    ga.relative_gap = relative_gap;
    ga.screening = screening;
    ga.spec = spec ? 1 : 0;
    if (st == BX_OK) k_graph_round_end<<<1, 1, 0, c->stream>>>(ga);
    cudaGraph_t cap = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &cap);
    c->stream = user_stream;
    c->launches = launches0;  // captured, not launched
    if (st != BX_OK || ce != cudaSuccess || !(graph_key(c, kind, passes, screening) == key)) {
      // not a steady-state round (or capture failed): stay on the host loop
      cudaGetLastError();
      gs.reset();
      gs.broken = true;
      c->err.clear();
      c->r = saved.r;
      c->rprev = saved.rprev;
      c->spec_pending = saved.spec_pending;
      c->dot_done = saved.dot_done;
      c->dot_spec = saved.dot_spec;
      c->g_valid = saved.g_valid;
      c->dot_G = saved.dot_G;
      c->last_Gw = saved.last_Gw;
      c->last_Ge = saved.last_Ge;
      c->last_kind = saved.last_kind;
      return BX_OK;
    }
    size_t nn = 0;
    if (cudaGraphGetNodes(body, nullptr, &nn) != cudaSuccess ||
        cudaGraphInstantiate(&gs.exec, gs.graph, 0) != cudaSuccess)
      return give_up();
    c->graph_body_kernels = (int64_t)nn;
    gs.key = key;
  }
  const int hd0[3] = {0, 0, limit};
  CU(cudaMemcpyAsync(c->done, hd0, sizeof(hd0), cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemsetAsync(c->stamps, 0, 8 * sizeof(unsigned long long), c->stream));
  c->batch_t = std::chrono::steady_clock::now();
  k_stamp<<<1, 1, 0, c->stream>>>(c->stamps);  // the batch's start on the device clock
  LAUNCHED();
  // run on the private stream, joined both ways with the caller's stream
  CU(cudaEventRecord(gs.join[0], c->stream));
  CU(cudaStreamWaitEvent(gs.cs, gs.join[0], 0));
  CU(cudaGraphLaunch(gs.exec, gs.cs));
  CU(cudaEventRecord(gs.join[1], gs.cs));
  CU(cudaStreamWaitEvent(c->stream, gs.join[1], 0));
  int hd[2] = {0, 0};
  CU(cudaMemcpyAsync(hd, c->done, sizeof(hd), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  // every executed round launched the body's kernels
  c->launches += (int64_t)(hd[0] + hd[1]) * c->graph_body_kernels;
  *ran = 1;
  *done = hd[0];
  *event = hd[1];
  // the event round's g / eps partials are in place (with spec: the round
  // ended with its speculative step, as the capture left the host state)
  if (hd[1]) {
    c->dot_done = true;
    c->dot_spec = spec;
  }
  return BX_OK;
}

// one PG / FISTA step on the act view: pass + reduce.  spec: the
// speculative round-boundary step -- the pass also emits the
// round's screening gradient g_k and epsilon partials and keeps what an undo
// needs (x_k, and for FISTA x_{k-1} / g_{k-1}; the reduce saves r_k and the
// objective / momentum before the step).
template <typename T>
int step_pass(bx_ctx* c, int kind, bool spec) {
  const int s = c->cur;
  int G = 1;
  StepExtra ex;
  ex.spec = spec ? 1 : 0;
  ex.xbak = (double*)c->xbak[s];
  ex.gbak = (double*)c->gbak[s];
  ex.epart = c->epart;
  const int sm = spec ? R_SPEC : 0;
  double* save = spec ? (double*)c->rbak : nullptr;
  // one GPU and the register-resident pass: the pass reduces its own partial
  // rows (no k_reduce launch); sharded: the cross-rank exchange does it
  const bool fuse = c->fuse_on && !c->sharded() && pick_R(c->m, sizeof(T)) > 0;
  ex.fuse = fuse ? 1 : 0;
  ex.roff = (const double*)c->off;
  ex.rout = (double*)c->r;
  ex.rsave = save;
  ex.rcounter = 2;
  if (kind == BX_PG) {
    ex.rmode = R_PG | sm;
    if (c->g_valid && !spec) {
      TRY(run_pass<T>(c, act_view<T>(c), U_PG_G, nullptr, nullptr, (double*)c->x[s], nullptr, (const double*)c->lo[s],
                      (const double*)c->hi[s], (double*)c->g, nullptr, nullptr, nullptr, 0, &G, nullptr, 0, -1, -1,
                      false, ex));
    } else {
      // spec: x_k goes to xprev (unused by PG) for an undo
      TRY(run_pass<T>(c, act_view<T>(c), U_PG, (const double*)c->r, nullptr, (double*)c->x[s], (double*)c->xprev[s],
                      (const double*)c->lo[s], (const double*)c->hi[s], (double*)c->g, (const double*)c->att[s],
                      nullptr, nullptr, c->has_inf, &G, nullptr, 0, -1, -1, false, ex));
    }
    if (!fuse) TRY(run_reduce<T>(c, G, (const double*)c->off, (double*)c->r, R_PG | sm, nullptr, 0, 2, save));
  } else {
    // FISTA by gradient linearity: the pass dots r_k; the new
    // residual is reduced in place
    ex.rmode = R_APG | sm;
    ex.gprev = (double*)c->gprev[s];
    TRY(run_pass<T>(c, act_view<T>(c), U_APG, (const double*)c->r, nullptr, (double*)c->x[s], (double*)c->xprev[s],
                    (const double*)c->lo[s], (const double*)c->hi[s], (double*)c->g, (const double*)c->att[s],
                    nullptr, c->bpart, c->has_inf, &G, (const double*)c->nrm[s], 0, -1, -1, false, ex));
    if (!fuse)
      TRY(run_reduce<T>(c, G, (const double*)c->off, (double*)c->r, R_APG | sm, c->bpart, c->last_Gw, 2, save));
  }
  c->g_valid = false;
  if (spec) {
    c->spec_pending = true;
    c->dot_done = true;  // g_k and its epsilon partials are the round's screening gradient
    c->dot_spec = true;
    c->dot_G = c->last_Ge;
  }
  return BX_OK;
}

// one round's primal passes.  After an accepted speculative step the round's
// first step has already been taken (at the end of the previous round).
template <typename T>
int primal_passes(bx_ctx* c, int kind, int passes) {
  c->last_kind = kind;
  int p0 = 0;
  if (c->spec_pending) {
    p0 = 1;
    c->spec_pending = false;
  } else {
    int ran = 0, done = 0, ev = 0;
    SmallLoop lp;
    TRY(small_rounds<T>(c, kind, passes, lp, &ran, &done, &ev));
    if (ran) return BX_OK;
  }
  if (kind == BX_CD) return cd_sweeps<T>(c, passes);  // all sweeps in one launch
  for (int p = p0; p < passes; ++p) TRY(step_pass<T>(c, kind, false));
  return BX_OK;
}

// Whether the round about to end should evaluate its screening gradient with
// the next round's first step (speculatively) instead of a dot-only pass:
// PG / FISTA on the streamed path, when the next round runs there too.
template <typename T>
bool spec_applies(bx_ctx* c, int kind, int passes) {
  if (!c->spec_on || (kind != BX_PG && kind != BX_APG) || c->k == 0) return false;
  int ran = 0, done = 0, ev = 0;
  SmallLoop lp;
  lp.max_rounds = 2;
  if (small_rounds<T>(c, kind, passes, lp, &ran, &done, &ev, true) != BX_OK) return false;
  return !ran;  // the cooperative small-round kernel owns the next round
}

// Undo the speculative step (k_spec_undo): the state is again the round's
// final iterate x_k with r_k, g_{k-1} and the scalars before the step.
template <typename T>
int spec_undo(bx_ctx* c, int kind) {
  if (!c->spec_pending) return BX_OK;
  const int s = c->cur;
  const int64_t n = c->k > c->m ? c->k : c->m;
  k_spec_undo<<<grid1d(c, n), RT, 0, c->stream>>>(c->k, kind == BX_APG ? 1 : 0, (double*)c->x[s],
                                                  (double*)c->xprev[s], (const double*)c->xbak[s],
                                                  (double*)c->gprev[s], (const double*)c->gbak[s], c->m,
                                                  (double*)c->r, (const double*)c->rbak, c->sc);
  LAUNCHED();
  c->spec_pending = false;
  c->g_valid = false;
  return BX_OK;
}

// ---------------------------------------------------------------------------
// active set (solvers.py:140-204; kernels in bx_active.cuh)
// ---------------------------------------------------------------------------
int as_sync(bx_ctx* c) {
  CU(cudaMemcpyAsync(c->has, c->as, sizeof(AsState), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  TRY(prof_drain(c));
  c->as_p = c->has->p;
  if (c->has->status == AS_SINGULAR)
    return fail(c, BX_ERR_SINGULAR, "passive-column least-squares system is singular (pivot %.3e, %d columns)",
                c->has->d2, c->has->p);
  return BX_OK;
}

// append preserved column j (j < 0: the one k_as_select chose) to the factor
template <typename T>
int as_append(bx_ctx* c, int32_t j) {
  View<T> vw = act_view<T>(c);
  k_as_colcopy<T><<<grid1d(c, c->m), RT, 0, c->stream>>>(vw.A, vw.ld, vw.colmap, c->m, c->as_avec, c->as_plist, c->as,
                                                          j);
  LAUNCHED();
  const int npl = c->as_p + 1;
  k_as_dots<T><<<(npl + 7) / 8, 256, 0, c->stream>>>(vw.A, vw.ld, vw.colmap, c->as_plist, npl, c->as_avec, c->m,
                                                      c->as_c);
  LAUNCHED();
  k_as_append<<<1, AS_NT, 0, c->stream>>>(c->asR, c->pcap, c->pcap, c->as_cslot, c->as, c->as_c);
  LAUNCHED();
  ++c->as_p;  // provisional; as_sync reads the device count
  return BX_OK;
}

// refactor after a compaction: append the passive columns in preserved order
// (the order the reference's flatnonzero gives its Gram matrix)
template <typename T>
int as_rebuild(bx_ctx* c) {
  const int s = c->cur;
  k_as_reset<<<grid1d(c, c->pcap), RT, 0, c->stream>>>(c->pcap, c->as_cslot, c->as);
  LAUNCHED();
  c->as_p = 0;
  std::vector<double> mask(c->k > 0 ? c->k : 1);
  if (c->k > 0) CU(cudaMemcpyAsync(mask.data(), c->xprev[s], c->k * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (int64_t j = 0; j < c->k; ++j)
    if (mask[j] != 0.0) TRY(as_append<T>(c, (int32_t)j));
  TRY(as_sync(c));
  c->as_dirty = false;
  return BX_OK;
}

// One outer iteration; *optimal = true when no bound coordinate violates the
// optimality conditions (the residual and gradient are then unchanged).
template <typename T>
int as_step(bx_ctx* c, bool* optimal) {
  const int s = c->cur;
  *optimal = false;
  if (c->as_dirty) TRY(as_rebuild<T>(c));
  double* pmask = (double*)c->xprev[s];
  if (!c->g_valid) {
    int G = 1;
    TRY(run_pass<T>(c, act_view<T>(c), U_DOT, (const double*)c->r, nullptr, nullptr, nullptr, nullptr,
                    (const double*)c->hi[s], (double*)c->g, nullptr, nullptr, c->bpart, 0, &G));
  }
  const int e0 = prof_begin(c);
  k_as_select<<<1, AS_NT, 0, c->stream>>>(c->k, c->m, (const double*)c->x[s], (const double*)c->lo[s],
                                          (const double*)c->hi[s], (const double*)c->g, (const double*)c->nrm[s],
                                          pmask, (const double*)c->r, c->as_plist, c->as);
  LAUNCHED();
  prof_end(c, e0, BX_PROF_ACTIVE, 8.0 * (6.0 * c->k + c->m));
  TRY(as_sync(c));
  if (c->has->jstar < 0) {
    *optimal = true;
    return BX_OK;
  }
  TRY(as_append<T>(c, -1));
  const int64_t limit = 2 * c->k + 2;  // solvers.py:180
  const int nbk = grid1d(c, c->k);
  for (int64_t it = 0; it < limit; ++it) {
    // rhs = (y - z) - A_F x_F over the fixed (non-passive) columns
    k_as_coef<<<nbk, RT, 0, c->stream>>>(c->k, (const double*)c->x[s], pmask, (double*)c->coef);
    LAUNCHED();
    int G = 1;
    TRY(run_pass<T>(c, act_view<T>(c), U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                    nullptr, (const double*)c->coef, nullptr, 0, &G));
    TRY(run_reduce<T>(c, G, (const double*)c->tgt, c->as_rhs, R_PLAIN, nullptr, 0, 0));
    View<T> vw = act_view<T>(c);
    const int p = c->as_p;
    if (p > 0) {
      k_as_dots<T><<<(p + 7) / 8, 256, 0, c->stream>>>(vw.A, vw.ld, vw.colmap, c->as_plist, p, c->as_rhs, c->m,
                                                        c->as_b);
      LAUNCHED();
    }
    const int e1 = prof_begin(c);
    k_as_solve<<<1, AS_NT, 0, c->stream>>>(c->asR, c->pcap, c->as_cslot, c->as_plist, c->as, c->as_b, c->as_s,
                                           c->as_frac, c->as_hitf, (double*)c->x[s], (const double*)c->lo[s],
                                           (const double*)c->hi[s], pmask);
    LAUNCHED();
    prof_end(c, e1, BX_PROF_ACTIVE, 8.0 * ((double)p * p + 8.0 * p));
    TRY(as_sync(c));
    if (c->has->status == AS_DONE) {
      TRY(refresh_resid<T>(c));  // solvers.py:202-203 (g by the next dot pass)
      c->g_valid = false;
      return BX_OK;
    }
  }
  return fail(c, BX_ERR_SINGULAR, "active-set inner loop failed to make progress");
}

// epsilon (max over ranks), theta, reduced dual, gap, radius (k_dual [+ fin])
template <typename T>
int dual_point(bx_ctx* c, int which, const double* r, const double* tgt, double* theta, const double* g,
               const double* att, const double* lo, const double* hi, double* v, int64_t k, const double* eps_part,
               int Ge, double slack_scale, double alpha) {
  const double* ep = eps_part;
  int ge = Ge;
  if (c->sharded()) {
    k_fold<<<1, 32, 0, c->stream>>>(eps_part, Ge, 1, 1, c->scal + 8);
    LAUNCHED();
    TRY(allreduce(c, c->scal + 8, 1, ncclFloat64, ncclMax));
    ep = c->scal + 8;
    ge = 1;
  }
  int nb = grid1d(c, c->m > k ? c->m : k);
  const int e0 = prof_begin(c);
  k_dual<double><<<nb, RT, 0, c->stream>>>(r, (const double*)c->t, tgt, theta, c->m, g, att, lo, hi, v, k, ep, ge, c->has_inf,
                                       c->sc, which, c->bpart3, slack_scale, alpha, which == 1 ? 5 : 3,
                                       c->sharded() ? c->dsum : nullptr);
  LAUNCHED();
  prof_end(c, e0, BX_PROF_DUAL, 8.0 * (4.0 * c->m + 6.0 * k));
  if (c->sharded()) {
    TRY(allreduce(c, c->dsum + 2, 2, ncclFloat64, ncclSum));  // bound terms are per-rank
    k_dual_fin<<<1, 32, 0, c->stream>>>(c->dsum, c->sc, which, slack_scale, alpha);
    LAUNCHED();
  }
  return BX_OK;
}

// gradient at the round's final iterate + dual point + gap (+ sphere test).
// The gradient is a dot-only pass, or came with the round kernel / the
// speculative step (dot_done; then with dot_spec the round's final iterate
// is x_prev, its residual r_bak and its objective bak_P, and the sphere test
// also counts the "dirty" screened columns that force an undo).
template <typename T>
int dual_screen(bx_ctx* c, int screening, double slack_scale, double alpha) {
  const int s = c->cur;
  int G = 1;
  const bool spec = c->dot_done && c->dot_spec;
  if (c->dot_done) {
    G = c->dot_G;  // g and the eps partials came with the round kernel / the speculative step
    c->dot_done = false;
  } else {
    TRY(run_pass<T>(c, act_view<T>(c), U_DOT, (const double*)c->r, nullptr, nullptr, nullptr, nullptr,
                    (const double*)c->hi[s], (double*)c->g, (const double*)c->att[s], nullptr, c->bpart, c->has_inf,
                    &G));
    c->dot_G = G;  // a later dual_screen on the same g (dot_done) reuses its eps partials
  }
  c->dot_spec = false;
  if (!spec) c->g_valid = true;  // (after a speculative step g is at x_prev, not x)
  const double* r = spec ? (const double*)c->rbak : (const double*)c->r;
  // the gap evaluation proper -- the gradient above is the step's, as in the
  // reference's pg_step -- is what the offline-gap convention excludes
  if (c->dual_stamps) {
    k_stamp<<<1, 1, 0, c->stream>>>(c->stamps + 1);
    LAUNCHED();
  }
  if (c->dual_ev) CU(cudaEventRecord(c->dual_ev[0], c->stream));
  TRY(dual_point<T>(c, spec ? 2 : 0, r, (const double*)c->tgt, (double*)c->theta, (const double*)c->g,
                    (const double*)c->att[s], (const double*)c->lo[s], (const double*)c->hi[s], (double*)c->v, c->k,
                    spec ? c->epart : c->bpart, G, slack_scale, alpha));
  if (c->dual_ev) CU(cudaEventRecord(c->dual_ev[1], c->stream));
  if (c->dual_stamps) {
    k_stamp<<<1, 1, 0, c->stream>>>(c->stamps + 2);
    LAUNCHED();
  }
  c->theta_is_cert = false;
  if (screening && c->k > 0) {
    const int nbs = (int)((c->k + RT - 1) / RT);
    const int e1 = prof_begin(c);
    const bool apg = c->last_kind == BX_APG;
    k_sphere<double><<<nbs, RT, 0, c->stream>>>((const double*)c->v, (const double*)c->nrm[s], (const double*)c->lo[s],
                                            (const double*)c->hi[s], c->k, c->sc, c->flags, c->bcnt,
                                            spec ? (const double*)c->x[s] : nullptr,
                                            spec ? (const double*)c->xprev[s] : nullptr,
                                            (spec && apg) ? (const double*)c->xbak[s] : nullptr);
    LAUNCHED();
    k_scan<<<1, 1024, 0, c->stream>>>(c->bcnt, nbs, c->sc);
    LAUNCHED();
    prof_end(c, e1, BX_PROF_SPHERE, (double)c->k * 25.0);
  } else {
    CU(cudaMemsetAsync(&c->sc->n_keep, 0, 8 * sizeof(int64_t), c->stream));
  }
  if (screening && c->sharded()) TRY(allreduce(c, &c->sc->g_keep, 4, ncclInt64, ncclSum));
  return BX_OK;
}

// _certified_gap (driver.py:112-117): full-problem A x, A'(y - A x), epsilon
// over all infinite-upper columns, dual objective
// The round's final iterate: x, or x_prev while a speculative step is pending.
const double* round_x(const bx_ctx* c) {
  return (const double*)(c->spec_pending ? c->xprev[c->cur] : c->x[c->cur]);
}

// the full-problem certificate of the iterate in x_full
template <typename T>
int certify_full(bx_ctx* c, double alpha);

template <typename T>
int certified(bx_ctx* c, double alpha) {
  const int s = c->cur;
  k_scatter_x<double><<<grid1d(c, c->k), RT, 0, c->stream>>>(c->k, c->idx[s], round_x(c), (double*)c->xfull);
  LAUNCHED();
  return certify_full<T>(c, alpha);
}

template <typename T>
int certify_full(bx_ctx* c, double alpha) {
  int G = 1;
  // fp32 storage: the certificate's A x and A'r accumulate in fp64 (a fp32
  // sum of A x carries ~1e-7 |Ax| of noise, which puts a floor of ~1e-7
  // |Ax|^2 under the computed gap however optimal x is)
  const bool acc64 = sizeof(T) == 4 && c->m <= (int64_t)NT * 4 * 12;
  TRY(run_pass<T>(c, full_view<T>(c), U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                  (const double*)c->xfull, nullptr, 0, &G, nullptr, 0, -1, -1, acc64));
  if (acc64)
    TRY(run_reduce<double>(c, G, (const double*)c->negy, (double*)c->rc, R_CERT, nullptr, 0, 4));
  else
    TRY(run_reduce<T>(c, G, (const double*)c->negy, (double*)c->rc, R_CERT, nullptr, 0, 4));
  TRY(run_pass<T>(c, full_view<T>(c), U_DOT, (const double*)c->rc, nullptr, nullptr, nullptr, nullptr,
                  (const double*)c->hifull, (double*)c->gfull, (const double*)c->attfull, nullptr, c->bpart + c->Gmax, c->has_inf,
                  &G, nullptr, 0, -1, -1, acc64));
  TRY(dual_point<T>(c, 1, (const double*)c->rc, (const double*)c->y, (double*)c->thetac, (const double*)c->gfull,
                    (const double*)c->attfull, (const double*)c->lofull, (const double*)c->hifull, (double*)c->vfull, c->n,
                    c->bpart + c->Gmax, G, 0.0, alpha));
  return BX_OK;
}

template <typename T>
int dot_accumulate(bx_ctx* c, const double* vin, double* g);

// r += A_S (b_S - x_S) (and r_prev += A_S (b_S - x_prev_S)) over the newly
// screened columns: the residual of the snapped iterate without a pass over the
// preserved set.  The reference recomputes it (solvers.py:64); the next step's
// pass recomputes r = A x + z - y from scratch anyway, so only the one dot of
// that step sees the (rounding-level) difference.  Collective in sharded mode
// (every rank contributes its own screened columns, possibly none).
//
// FISTA also carries g_{k-1} = A'r_{k-1} per preserved column; snapping the
// screened x_{k-1} moves r_{k-1} by d = A_S (b_S - x_prev_S), so g_prev gets
// A_act' d (one dot pass over the preserved set with d as the vector).  The
// oracle recomputes g_prev from the snapped x_prev (same quantity).
template <typename T>
int refresh_incremental(bx_ctx* c, int64_t nscr, int kind) {
  View<T> vw{(const T*)c->A, c->lda, c->scr_idx, nscr};
  int G = 1;
  TRY(run_pass<T>(c, vw, U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                  (const double*)c->scr_dx, nullptr, 0, &G));
  TRY(run_reduce<T>(c, G, (const double*)c->r, (double*)c->r, R_SET, nullptr, 0, 0));
  if (kind == BX_APG && c->k > 0) {
    TRY(run_pass<T>(c, vw, U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                    (const double*)c->scr_dxp, nullptr, 0, &G));
    TRY(run_reduce<T>(c, G, nullptr, (double*)c->u, R_PLAIN, nullptr, 0, 0));
    TRY(dot_accumulate<T>(c, (const double*)c->u, (double*)c->gprev[c->cur]));
  }
  return BX_OK;
}

// g[p] += a_p . vin over the preserved set (whole columns, or row blocks
// beyond the register-resident envelope)
template <typename T>
int dot_accumulate(bx_ctx* c, const double* vin, double* g) {
  if (c->k == 0) return BX_OK;
  int G = 1;
  if (pick_R(c->m, sizeof(T)) > 0)
    return run_pass<T>(c, act_view<T>(c), U_DOT, vin, nullptr, nullptr, nullptr, nullptr, nullptr, g, nullptr,
                       nullptr, nullptr, 0, &G, nullptr, 0, c->m, 1);
  constexpr int64_t BR = (int64_t)NT * (16 / sizeof(T)) * 8;
  for (int64_t r0 = 0; r0 < c->m; r0 += BR)
    TRY(run_pass<T>(c, act_view<T>(c), U_DOT, vin, nullptr, nullptr, nullptr, nullptr, nullptr, g, nullptr, nullptr,
                    nullptr, 0, &G, nullptr, r0, std::min(BR, c->m - r0), 1));
  return BX_OK;
}

// apply_screening + Workspace.refresh (screening.py:72-94, solvers.py:54-65).
// clean: a speculative step stands over a screened set that sat at its bound
// on every iterate the step touched -- the residual, g_prev and the step are
// unchanged by the screening, so there is nothing to refresh.
template <typename T>
int compact(bx_ctx* c, int64_t n_lo, int64_t n_up, int64_t n_keep, int kind, bool z_update, bool clean = false) {
  const int s = c->cur, d = 1 - c->cur;
  const int nbs = (int)((c->k + RT - 1) / RT);
  const int64_t nscr = n_lo + n_up;
  if (nscr > 0) {
    // momentum state / passive mask; a standing speculative step also keeps
    // what dropping it at the end of the solve needs (x_k, x_{k-1}, g_{k-1})
    const bool carry2 = kind == BX_APG || kind == BX_ACTIVE_SET || c->spec_pending;
    const bool bak = c->spec_pending && kind == BX_APG;
    ColState<double> src{c->idx[s], (double*)c->x[s], carry2 ? (double*)c->xprev[s] : nullptr,
                         kind == BX_APG ? (double*)c->gprev[s] : nullptr,
                         bak ? (double*)c->xbak[s] : nullptr, bak ? (double*)c->gbak[s] : nullptr,
                         (double*)c->lo[s], (double*)c->hi[s], (double*)c->nrm[s], (double*)c->att[s],
                         c->dense ? nullptr : c->pos[s]};
    ColState<double> dst{c->idx[d], (double*)c->x[d], (double*)c->xprev[d], (double*)c->gprev[d],
                         (double*)c->xbak[d], (double*)c->gbak[d], (double*)c->lo[d], (double*)c->hi[d],
                         (double*)c->nrm[d], (double*)c->att[d], c->act_is_orig ? nullptr : c->pos[d]};
    k_compact<double><<<nbs, RT, 0, c->stream>>>(c->flags, c->bcnt, c->k, src, dst, (double*)c->xfull, c->scr_idx,
                                                 (double*)c->scr_val, n_lo, c->sat_lo + c->n_sat_lo,
                                                 c->sat_up + c->n_sat_up, c->col_offset, (double*)c->scr_dx,
                                                 (double*)c->scr_dxp);
    LAUNCHED();
    c->cur = d;
    c->k = n_keep;
    c->n_sat_lo += n_lo;
    c->n_sat_up += n_up;
    c->dense = false;
    if (kind == BX_ACTIVE_SET) c->as_dirty = true;  // preserved positions moved
  }
  // z += A_S bound_S  (only when some screened bound is nonzero; collective)
  if (z_update) {
    View<T> vw{(const T*)c->A, c->lda, c->scr_idx, nscr};
    int G = 1;
    TRY(run_pass<T>(c, vw, U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                    (const double*)c->scr_val, nullptr, 0, &G));
    TRY(run_reduce<T>(c, G, (const double*)c->z, (double*)c->z2, R_PLAIN, nullptr, 0, 0));
    std::swap(c->z, c->z2);
    k_offsets<double><<<grid1d(c, c->m), RT, 0, c->stream>>>(c->m, (const double*)c->y, (const double*)c->z,
                                                             (double*)c->off, (double*)c->tgt);
    LAUNCHED();
  }
  if (!clean) TRY(refresh_incremental<T>(c, nscr, kind));
  // physical rewrite of the preserved columns (solvers.py:57) once half the
  // physical buffer is dead -- or always for CD, whose kernels read A_act densely
  if (nscr > 0 && (kind == BX_CD || c->k < c->kphys / 2)) {
    if (c->k > 0) {
      int nb = (int)(c->k < 8 * c->nsm ? c->k : 8 * c->nsm);
      const int e0 = prof_begin(c);
      k_gather<T><<<nb, RT, 0, c->stream>>>((const T*)c->A, c->lda, c->idx[c->cur], c->k, c->m, (T*)c->Aact,
                                             c->ldact);
      LAUNCHED();
      prof_end(c, e0, BX_PROF_GATHER, 2.0 * (double)c->k * c->m * sizeof(T));
    }
    c->act_is_orig = false;
    c->dense = true;
    c->kphys = c->k;
  }
  c->gram_dirty = true;
  c->g_valid = false;
  return BX_OK;
}

template <typename T>
int reset_state(bx_ctx* c, int kind, int restart = 0) {
  const int s = 0;
  c->cur = 0;
  c->k = c->n;
  c->n_sat_lo = c->n_sat_up = 0;
  c->act_is_orig = true;
  c->dense = true;
  c->kphys = c->n;
  c->gram_dirty = true;
  c->g_valid = false;
  c->theta_is_cert = false;
  k_init_cols<double><<<grid1d(c, c->n), RT, 0, c->stream>>>(c->n, (const double*)c->lofull, (const double*)c->hifull,
                                                         (double*)c->xfull, c->idx[s], (double*)c->x[s], (double*)c->lo[s],
                                                         (double*)c->hi[s], (const double*)c->nrmfull, (double*)c->nrm[s],
                                                         (const double*)c->attfull, (double*)c->att[s]);
  LAUNCHED();
  if (kind == BX_ACTIVE_SET) {
    // coordinates start on a bound (driver.py:144-147); empty passive set
    CU(cudaMemcpyAsync(c->x[s], c->lo[s], c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemcpyAsync(c->xfull, c->lo[s], c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemsetAsync(c->xprev[s], 0, c->n * sizeof(double), c->stream));
    k_as_reset<<<grid1d(c, c->pcap), RT, 0, c->stream>>>(c->pcap, c->as_cslot, c->as);
    LAUNCHED();
    c->as_p = 0;
    c->as_dirty = false;
  }
  CU(cudaMemsetAsync(c->z, 0, c->mp * sizeof(double), c->stream));
  k_offsets<double><<<grid1d(c, c->m), RT, 0, c->stream>>>(c->m, (const double*)c->y, (const double*)c->z, (double*)c->off, (double*)c->tgt);
  LAUNCHED();
  DevScalars h;
  memset(&h, 0, sizeof(h));
  h.mom_t = 1.0;
  h.P = INFINITY;
  // round-off-sized tolerances: fp64 = the reference / oracle values
  const bool f32 = sizeof(T) == 4;
  h.rise_rel = f32 ? 1e-5 : 0.0;
  h.rs_f = f32 ? 1e-6 : 1e-12;
  // restart = 1 (objective increase only): the gradient test never fires
  h.rs_g = restart ? INFINITY : (f32 ? 1e-5 : 1e-12);
  CU(cudaMemcpyAsync(c->sc, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  TRY(refresh_resid<T>(c));
  if (kind == BX_APG) {
    // x_prev = x_0; g_prev is unused until a step with momentum (t_0 = 1)
    CU(cudaMemcpyAsync(c->xprev[s], c->x[s], c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemsetAsync(c->gprev[s], 0, c->n * sizeof(double), c->stream));
    c->have_apg_state = true;
  }
  c->spec_pending = false;
  c->dot_done = false;
  c->dot_spec = false;
  return BX_OK;
}

template <typename T>
int create_typed(bx_ctx* c, const void* y, const void* lower, const void* upper, const void* t) {
  const int64_t m = c->m, n = c->n;
  CU(cudaMemsetAsync(c->y, 0, c->mp * sizeof(double), c->stream));
  CU(cudaMemcpyAsync(c->y, y, m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  k_neg<double><<<grid1d(c, m), RT, 0, c->stream>>>(c->mp, (const double*)c->y, (double*)c->negy);
  LAUNCHED();
  CU(cudaMemcpyAsync(c->lofull, lower, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemcpyAsync(c->hifull, upper, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemsetAsync(c->probe, 0, 64, c->stream));
  k_bounds_probe<double><<<grid1d(c, n), RT, 0, c->stream>>>(n, (const double*)c->lofull, (const double*)c->hifull, c->probe);
  LAUNCHED();
  int bits = 0;
  CU(cudaMemcpyAsync(&bits, c->probe, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (bits & 32) return fail(c, BX_ERR_INVALID_ARGUMENT, "NaN entries in bounds");
  if (bits & 8) return fail(c, BX_ERR_INVALID_ARGUMENT, "lower bounds must be finite");
  if (bits & 16) return fail(c, BX_ERR_INVALID_ARGUMENT, "need lower_j < upper_j for every coordinate");
  c->bound_bits = bits;
  c->has_inf = (bits & 4) ? 1 : 0;
  // translation vector: neg-ones unless given (duality.py:74-75)
  CU(cudaMemsetAsync(c->t, 0, c->mp * sizeof(double), c->stream));
  if (t) {
    CU(cudaMemcpyAsync(c->t, t, m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  } else {
    k_fill<double><<<grid1d(c, m), RT, 0, c->stream>>>(m, (double*)c->t, T(-1));
    LAUNCHED();
  }
  CU(cudaMemsetAsync(c->probe, 0, 64, c->stream));
  const int nbw = (int)((n * 32 + RT - 1) / RT < 16 * c->nsm ? (n * 32 + RT - 1) / RT : 16 * c->nsm);
  k_colstats<T><<<nbw, RT, 0, c->stream>>>((const T*)c->A, c->lda, n, m, (const double*)c->t, (double*)c->nrmfull,
                                            (double*)c->attfull, 1, c->probe);
  LAUNCHED();
  int cf = 0;
  CU(cudaMemcpyAsync(&cf, c->probe, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  // reported by bx_solve (after agreeing across ranks): the reference raises
  // these from solve(), driver.py:141-152
  c->col_bits = cf;
  return BX_OK;
}

// data validation agreed over ranks: every rank raises the same error and the
// global bound structure (some u infinite, nonzero bounds) drives every rank
int validate(bx_ctx* c) {
  // {some u infinite, some lower != 0, some finite upper != 0, zero column, t not interior}
  int f[5] = {c->has_inf, c->bound_bits & 1, (c->bound_bits >> 1) & 1, c->col_bits & 1, (c->col_bits >> 1) & 1};
  if (c->sharded()) {
    CU(cudaMemcpyAsync(c->probe, f, sizeof(f), cudaMemcpyHostToDevice, c->stream));
    TRY(allreduce(c, c->probe, 5, ncclInt32, ncclMax));
    CU(cudaMemcpyAsync(f, c->probe, sizeof(f), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  c->has_inf = f[0] ? 1 : 0;
  c->bound_bits = (c->bound_bits & ~3) | (f[1] ? 1 : 0) | (f[2] ? 2 : 0);
  // the translation vector is built before the screening state
  // (driver.py:141-152), so NoInteriorPoint takes precedence over ZeroColumn
  if (c->has_inf && f[4]) return fail(c, BX_ERR_NO_INTERIOR, "strategy did not yield a strictly interior t");
  if (f[3]) return fail(c, BX_ERR_ZERO_COLUMN, "zero column in A");
  return BX_OK;
}

// two CUDA events, destroyed with the scope
struct EventPair {
  cudaEvent_t e[2] = {nullptr, nullptr};
  int create(bx_ctx* c) {
    for (auto& x : e) CU(cudaEventCreate(&x));
    return BX_OK;
  }
  cudaEvent_t operator[](int i) const { return e[i]; }
  ~EventPair() {
    for (auto x : e)
      if (x) cudaEventDestroy(x);
  }
};

template <typename T>
int solve_typed(bx_ctx* c, const bx_solve_cfg* cfg, bx_start_vector_fn fn, void* user, bx_trace_rec* trace,
                int64_t cap, bx_solve_out* out) {
  const auto t0 = std::chrono::steady_clock::now();
  const int kind = cfg->kind;
  const int passes = cfg->inner_passes;
  const int64_t n_all = c->sharded() ? c->n_global : c->n;
  const int64_t max_rounds =
      cfg->max_rounds > 0 ? cfg->max_rounds : (kind == BX_ACTIVE_SET ? 10 * n_all : 1000000);  // driver.py:144-150
  const double tol = cfg->gap_tol;
  const double alpha = cfg->alpha > 0 ? cfg->alpha : 1.0;
  const double slack_scale = cfg->slack_scale >= 0 ? cfg->slack_scale : 1e-12;
  const bool auto_eta = !(cfg->step_size > 0);  // NaN or <= 0
  if (kind == BX_CD && c->sharded())
    return fail(c, BX_ERR_UNSUPPORTED, "coordinate descent is sequential: replicas only, no column sharding");
  if (kind == BX_ACTIVE_SET && c->sharded())
    return fail(c, BX_ERR_UNSUPPORTED, "the active set is sequential: replicas only, no column sharding");
  if (kind == BX_ACTIVE_SET && !c->as)
    return fail(c, BX_ERR_WORKSPACE, "active-set scratch not attached (bx_ctx_set_active_set_workspace)");
  TRY(validate(c));
  TRY(reset_state<T>(c, kind, cfg->restart));
  double eta = cfg->step_size;
  double sigma = 0.0;
  int64_t kg = c->sharded() ? c->n_global : c->n;  // global preserved count
  int64_t basis = kg;
  if ((kind == BX_PG || kind == BX_APG)) {
    if (auto_eta) {
      TRY(auto_step<T>(c, cfg->power_iters, alpha, fn, user, &eta, &sigma));
    } else {
      CU(cudaMemcpyAsync(&c->sc->eta, &eta, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    }
  }
  int64_t rounds = 0, iters = 0;
  bool converged = false;
  int64_t spec_kept = 0, spec_undone = 0, last_restarts = 0;
  const bool spec_force_undo = [] {
    const char* e = getenv("BX_SPEC_FORCE_UNDO");  // test switch: every event takes the undo path
    return e && e[0] == '1';
  }();
  double gap_out = INFINITY;
  int64_t ntrace = 0;
  double excluded = 0.0;  // seconds of gap evaluation left out of the trace (screening off)
  EventPair gap_ev;
  if (!cfg->screening) TRY(gap_ev.create(c));
  static const int f32_every = [] {
    const char* e = getenv("BX_F32_CERT_EVERY");  // 0 disables the periodic certificate
    return e ? atoi(e) : kF32CertEvery;
  }();
  const bool f32cert = c->esz == 4 && kind != BX_ACTIVE_SET && f32_every > 0;
  int64_t last_cert = 0;
  int64_t last_event = 0;  // last round the host handled an event in (graph rounds resume 2 later)
  GraphState gstate;
  static const bool graph_off = getenv("BX_NO_GRAPH") != nullptr;
  SmallLoop lp;
  lp.tol = tol;
  lp.relative_gap = cfg->relative_gap;
  lp.screening = cfg->screening;
  lp.slack_scale = slack_scale;
  lp.alpha = alpha;
  for (int64_t rnd = 1; rnd <= max_rounds; ++rnd) {
    rounds = rnd;
    bool optimal = false;
    if (kind == BX_ACTIVE_SET) {
      TRY(as_step<T>(c, &optimal));
      iters += 1;
    } else if (!c->prof) {
      // small problems: device-resident rounds until the next event
      lp.max_rounds = (int)std::min<int64_t>(max_rounds - rnd + 1, kSmallRounds);
      if (f32cert) lp.max_rounds = (int)std::min<int64_t>(lp.max_rounds, last_cert + f32_every - rnd);
      int ran = 0, done = 0, ev = 0;
      if (lp.max_rounds > 1) TRY(small_rounds<T>(c, kind, passes, lp, &ran, &done, &ev));
      if (!ran && lp.max_rounds > 1 && rnd >= 2 && rnd - last_event >= 2 && !graph_off)
        TRY(graph_rounds<T>(c, gstate, kind, passes, lp.max_rounds, tol, cfg->relative_gap, cfg->screening,
                            slack_scale, alpha, &ran, &done, &ev));
      if (ran) {
        if (done > 0) {
          std::vector<double> tr(TRACE_W * (size_t)done);
          unsigned long long stamp0 = 0;
          CU(cudaMemcpyAsync(tr.data(), c->dtrace, tr.size() * 8, cudaMemcpyDeviceToHost, c->stream));
          CU(cudaMemcpyAsync(&stamp0, c->stamps, sizeof(stamp0), cudaMemcpyDeviceToHost, c->stream));
          CU(cudaStreamSynchronize(c->stream));
          // each round's elapsed from the device clock: the batch's host
          // launch time + the round's end on the device clock, minus the gap
          // evaluations excluded so far (screening off)
          const double tb = std::chrono::duration<double>(c->batch_t - t0).count();
          for (int q = 0; q < done && trace && ntrace < cap; ++q) {
            const double* row = tr.data() + (size_t)TRACE_W * q;
            bx_trace_rec& t = trace[ntrace++];
            t.round = rnd + q;
            t.elapsed = tb + 1e-9 * (row[7] - (double)stamp0) - excluded - 1e-9 * row[8];
            t.primal = row[0];
            t.dual = row[1];
            t.gap = row[2];
            t.preserved_count = kg;
            t.newly_screened_lower = t.newly_screened_upper = 0;
            t.eps = row[3];
            t.radius = row[4];
            t.step = eta;
            t.certified_gap = NAN;
            t.momentum = row[5];
            t.restarts = (int64_t)row[6];
          }
          excluded += 1e-9 * tr[(size_t)TRACE_W * (done - 1) + 8];
          gap_out = tr[(size_t)TRACE_W * (done - 1) + 2];
          last_restarts = (int64_t)tr[(size_t)TRACE_W * (done - 1) + 6];
          iters += (int64_t)done * passes;
          rnd += done;
          rounds = rnd - 1;
        }
        if (!ev) {
          --rnd;  // the for loop's ++rnd resumes at the next undone round
          continue;
        }
        rounds = rnd;
        iters += passes;  // the event round's passes + dot pass ran on the device
      } else {
        TRY(primal_passes<T>(c, kind, passes));
        iters += passes;
        if (spec_applies<T>(c, kind, passes)) TRY(step_pass<T>(c, kind, true));
      }
    } else {
      TRY(primal_passes<T>(c, kind, passes));
      iters += passes;
      if (spec_applies<T>(c, kind, passes)) TRY(step_pass<T>(c, kind, true));
    }
    // offline-gap convention (driver.py:180-181, 237-238): without screening
    // the gap evaluation is excluded from the trace's elapsed time -- here the
    // device time of the dual-point / certificate kernels, bracketed by events
    // (the gradient is the step's own, as in the reference's pg_step)
    c->dual_ev = cfg->screening ? nullptr : gap_ev.e;
    TRY(dual_screen<T>(c, cfg->screening, slack_scale, alpha));
    c->dual_ev = nullptr;
    TRY(sync_scalars<T>(c));
    TRY(check_dev_err(c));
    if (!cfg->screening) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, gap_ev[0], gap_ev[1]));
      excluded += 1e-3 * ms;
    }
    const DualOut act = c->hsc->act;
    gap_out = act.gap;
    double cert_gap = NAN;
    const double tol_r = cfg->relative_gap ? tol * fmax(1.0, fabs(act.primal)) : tol;
    // fp32 storage: the reduced gap of the fp32-accumulated residual has a
    // floor of ~1e-7 |Ax|^2, so the fp64-accumulated certificate is also
    // tried every kF32CertEvery rounds (it alone decides convergence)
    if (act.gap < tol_r || (f32cert && rnd >= last_cert + f32_every)) {
      last_cert = rnd;
      last_event = rnd;
      if (!cfg->screening) CU(cudaEventRecord(gap_ev[0], c->stream));
      TRY(certified<T>(c, alpha));
      if (!cfg->screening) CU(cudaEventRecord(gap_ev[1], c->stream));
      TRY(sync_scalars<T>(c));
      if (!cfg->screening) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, gap_ev[0], gap_ev[1]));
        excluded += 1e-3 * ms;
      }
      TRY(check_dev_err(c));
      cert_gap = c->hsc->cert.gap;
      gap_out = cert_gap;
      c->theta_is_cert = true;
      const double tol_c = cfg->relative_gap ? tol * fmax(1.0, fabs(c->hsc->cert.primal)) : tol;
      if (cert_gap < tol_c) converged = true;
    }
    // the round's momentum / restart count (before a speculative step)
    const double mom_round = c->spec_pending ? c->hsc->bak_mom_t : c->hsc->mom_t;
    const int64_t restarts_round = c->spec_pending ? c->hsc->bak_restarts : c->hsc->restarts;
    last_restarts = restarts_round;
    int64_t n_lo = 0, n_up = 0;
    if (cfg->screening && kg > 0) {
      n_lo = c->hsc->g_lo;
      n_up = c->hsc->g_up;
      if (n_lo || n_up) {
        last_event = rnd;
        const bool z_update = ((c->bound_bits & 1) && n_lo > 0) || ((c->bound_bits & 2) && n_up > 0);
        const int64_t kg_new = c->hsc->g_keep;
        const bool reestimate =
            (kind == BX_PG || kind == BX_APG) && auto_eta && (double)kg_new < 0.5 * (double)basis;
        // the speculative step stands only if screening leaves the problem it
        // was taken on unchanged (no screened coordinate off its bound on any
        // iterate the step touched) and the step size stays
        const bool was_spec = c->spec_pending;
        const bool clean = was_spec && !converged && c->hsc->g_dirty == 0 && !reestimate && !spec_force_undo;
        if (c->spec_pending && !clean) TRY(spec_undo<T>(c, kind));
        TRY(compact<T>(c, c->hsc->n_lo, c->hsc->n_up, c->hsc->n_keep, kind, z_update, clean));
        kg = kg_new;
        if (reestimate) {
          TRY(auto_step<T>(c, cfg->power_iters, alpha, fn, user, &eta, &sigma));
          basis = kg;
        }
        if (clean)
          ++spec_kept;
        else if (was_spec && !converged)
          ++spec_undone;
      }
    }
    if (trace && ntrace < cap) {
      bx_trace_rec& tr = trace[ntrace++];
      tr.round = rnd;
      tr.elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() - excluded;
      tr.primal = act.primal;
      tr.dual = act.dual;
      tr.gap = act.gap;
      tr.preserved_count = kg;
      tr.newly_screened_lower = n_lo;
      tr.newly_screened_upper = n_up;
      tr.eps = act.eps;
      tr.radius = act.radius;
      tr.step = eta;
      tr.certified_gap = cert_gap;
      tr.restarts = restarts_round;
      tr.momentum = mom_round;
    }
    if (converged) break;
    // a StepSizeTooLarge of a speculative step that stands is the next
    // round's (the reference raises it from that round's pg_step)
    if (c->spec_pending && c->hsc->err_spec)
      return fail(c, BX_ERR_STEP_TOO_LARGE, "objective rose from %.6e to %.6e", c->hsc->spec_v1, c->hsc->spec_v2);
    if (optimal) {
      // KKT-optimal active set: the certified gap alone decides (driver.py:246-252)
      TRY(certified<T>(c, alpha));
      TRY(sync_scalars<T>(c));
      TRY(check_dev_err(c));
      gap_out = c->hsc->cert.gap;
      c->theta_is_cert = true;
      const double tol_c = cfg->relative_gap ? tol * fmax(1.0, fabs(c->hsc->cert.primal)) : tol;
      converged = gap_out < tol_c;
      break;
    }
  }
  // a speculative step past the last round is dropped: x is the last round's
  TRY(spec_undo<T>(c, kind));
  // x_full <- current preserved iterate (ws.sync, driver.py:252)
  k_scatter_x<double><<<grid1d(c, c->k), RT, 0, c->stream>>>(c->k, c->idx[c->cur], (const double*)c->x[c->cur], (double*)c->xfull);
  LAUNCHED();
  CU(cudaStreamSynchronize(c->stream));
  if (out) {
    out->rounds = rounds;
    out->converged = converged ? 1 : 0;
    out->gap = gap_out;
    out->n_sat_lower = c->n_sat_lo;
    out->n_sat_upper = c->n_sat_up;
    out->iterations = iters;
    out->step = eta;
    out->sigma = sigma;
    out->kernel_launches = c->launches;
    out->restarts = last_restarts;
    out->spec_kept = spec_kept;
    out->spec_undone = spec_undone;
  }
  return BX_OK;
}

// ---- spec-level primitives (fine-grained C ABI) ------------------------------
template <typename T>
int set_state_typed(bx_ctx* c, const int64_t* pres, int64_t k, const double* xf, const double* z) {
  if (k < 0 || k > c->n) return fail(c, BX_ERR_DIMENSION, "preserved count %lld outside [0, n]", (long long)k);
  if (k > 0 && !pres) return fail(c, BX_ERR_INVALID_ARGUMENT, "preserved indices");
  if (!xf) return fail(c, BX_ERR_INVALID_ARGUMENT, "x_full");
  for (int64_t i = 0; i < k; ++i)
    if (pres[i] < 0 || pres[i] >= c->n || (i && pres[i] <= pres[i - 1]))
      return fail(c, BX_ERR_INVALID_ARGUMENT, "preserved indices must be ascending and in [0, n)");
  c->cur = 0;
  c->k = k;
  c->act_is_orig = true;
  c->dense = (k == c->n);  // ascending and k == n: the identity
  c->kphys = c->n;
  c->n_sat_lo = c->n_sat_up = 0;
  c->spec_pending = c->dot_done = c->dot_spec = c->g_valid = c->theta_is_cert = false;
  c->gram_dirty = true;
  c->as_dirty = true;
  if (k > 0) {
    CU(cudaMemcpyAsync(c->sat_lo, pres, k * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    k_gather_state<<<grid1d(c, k), RT, 0, c->stream>>>(
        k, c->sat_lo, c->idx[0], xf, (const double*)c->lofull, (const double*)c->hifull, (const double*)c->nrmfull,
        (const double*)c->attfull, (double*)c->x[0], (double*)c->lo[0], (double*)c->hi[0], (double*)c->nrm[0],
        (double*)c->att[0], (double*)c->xprev[0], (double*)c->gprev[0]);
    LAUNCHED();
  }
  CU(cudaMemcpyAsync(c->xfull, xf, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemsetAsync(c->z, 0, c->mp * sizeof(double), c->stream));
  if (z) CU(cudaMemcpyAsync(c->z, z, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  k_offsets<double><<<grid1d(c, c->m), RT, 0, c->stream>>>(c->m, (const double*)c->y, (const double*)c->z,
                                                           (double*)c->off, (double*)c->tgt);
  LAUNCHED();
  DevScalars h;
  memset(&h, 0, sizeof(h));
  const bool f32 = sizeof(T) == 4;
  h.mom_t = 1.0;
  h.P = INFINITY;
  h.rise_rel = f32 ? 1e-5 : 0.0;
  h.rs_f = f32 ? 1e-6 : 1e-12;
  h.rs_g = f32 ? 1e-5 : 1e-12;
  CU(cudaMemcpyAsync(c->sc, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  TRY(refresh_resid<T>(c));
  TRY(sync_scalars<T>(c));
  return check_dev_err(c);
}

template <typename T>
int gradient_typed(bx_ctx* c, double* resid, double* grad) {
  const int s = c->cur;
  if (c->k > 0) {
    int G = 1;
    TRY(run_pass<T>(c, act_view<T>(c), U_DOT, (const double*)c->r, nullptr, nullptr, nullptr, nullptr,
                    (const double*)c->hi[s], (double*)c->g, (const double*)c->att[s], nullptr, nullptr, 0, &G));
    c->g_valid = true;
  }
  if (resid) CU(cudaMemcpyAsync(resid, c->r, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if (grad && c->k > 0) CU(cudaMemcpyAsync(grad, c->g, c->k * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

template <typename T>
int apply_a_typed(bx_ctx* c, const int32_t* cols, int64_t k, const double* coef, const double* z_add, double* out) {
  if (!out) return fail(c, BX_ERR_INVALID_ARGUMENT, "out");
  if (!cols && k != c->n) return fail(c, BX_ERR_DIMENSION, "all columns: k must be n");
  if (k == 0) {
    if (z_add)
      CU(cudaMemcpyAsync(out, z_add, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    else
      CU(cudaMemsetAsync(out, 0, c->m * sizeof(double), c->stream));
  } else {
    if (!coef) return fail(c, BX_ERR_INVALID_ARGUMENT, "coef");
    View<T> vw{(const T*)c->A, c->lda, cols, k};
    int G = 1;
    const bool acc64 = sizeof(T) == 4 && c->m <= (int64_t)NT * 4 * 12;  // fp32 storage: fp64 sums (as certified())
    TRY(run_pass<T>(c, vw, U_AX, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, coef,
                    nullptr, 0, &G, nullptr, 0, -1, -1, acc64));
    if (acc64)
      TRY(run_reduce<double>(c, G, z_add, out, R_PLAIN, nullptr, 0, 0));
    else
      TRY(run_reduce<T>(c, G, z_add, out, R_PLAIN, nullptr, 0, 0));
  }
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

template <typename T>
int apply_at_typed(bx_ctx* c, const double* v, double* out) {
  if (!v || !out) return fail(c, BX_ERR_INVALID_ARGUMENT, "v / out");
  int G = 1;
  const bool acc64 = sizeof(T) == 4 && c->m <= (int64_t)NT * 4 * 12;
  TRY(run_pass<T>(c, full_view<T>(c), U_DOT, v, nullptr, nullptr, nullptr, nullptr, (const double*)c->hifull, out,
                  (const double*)c->attfull, nullptr, nullptr, 0, &G, nullptr, 0, -1, -1, acc64));
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

template <typename T>
int dual_point_typed(bx_ctx* c, const double* xf, double alpha, double* theta, double* atheta, double* out) {
  if (!xf) return fail(c, BX_ERR_INVALID_ARGUMENT, "x_full");
  CU(cudaMemcpyAsync(c->xfull, xf, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemsetAsync(&c->sc->err, 0, sizeof(int32_t), c->stream));
  TRY(certify_full<T>(c, alpha));
  if (theta) CU(cudaMemcpyAsync(theta, c->thetac, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if (atheta) CU(cudaMemcpyAsync(atheta, c->vfull, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  TRY(sync_scalars<T>(c));
  const int st = check_dev_err(c);
  if (out) {
    out[0] = c->hsc->cert.gap;
    out[1] = c->hsc->cert.primal;
    out[2] = c->hsc->cert.dual;
    out[3] = c->hsc->cert.eps;
  }
  return st;
}

template <typename T>
int eval_dual_typed(bx_ctx* c, const double* theta, const double* atheta, double* d) {
  if (!theta) return fail(c, BX_ERR_INVALID_ARGUMENT, "theta");
  // k_dual evaluates theta = -r and v = -g with no translation (eps = 0)
  k_neg<double><<<grid1d(c, c->m), RT, 0, c->stream>>>(c->m, theta, (double*)c->rc);
  LAUNCHED();
  if (atheta) {
    k_neg<double><<<grid1d(c, c->n), RT, 0, c->stream>>>(c->n, atheta, (double*)c->gfull);
    LAUNCHED();
  } else {
    int G = 1;
    const bool acc64 = sizeof(T) == 4 && c->m <= (int64_t)NT * 4 * 12;
    TRY(run_pass<T>(c, full_view<T>(c), U_DOT, (const double*)c->rc, nullptr, nullptr, nullptr, nullptr,
                    (const double*)c->hifull, (double*)c->gfull, (const double*)c->attfull, nullptr, nullptr, 0, &G,
                    nullptr, 0, -1, -1, acc64));
  }
  const double inf = INFINITY;  // no primal here: the weak-duality check cannot fire
  CU(cudaMemcpyAsync(&c->sc->cert_P, &inf, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int nb = grid1d(c, c->m > c->n ? c->m : c->n);
  k_dual<double><<<nb, RT, 0, c->stream>>>((const double*)c->rc, (const double*)c->t, (const double*)c->y,
                                           (double*)c->thetac, c->m, (const double*)c->gfull,
                                           (const double*)c->attfull, (const double*)c->lofull,
                                           (const double*)c->hifull, (double*)c->vfull, c->n, nullptr, 0, 0, c->sc, 1,
                                           c->bpart3, 0.0, 1.0, 5, nullptr);
  LAUNCHED();
  TRY(sync_scalars<T>(c));
  if (d) *d = c->hsc->cert.dual;
  return BX_OK;
}

__global__ void k_mask_io(int64_t k, const uint8_t* __restrict__ in, double* __restrict__ pmask,
                          uint8_t* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < k; p += (int64_t)gridDim.x * blockDim.x) {
    if (in) pmask[p] = in[p] ? 1.0 : 0.0;
    if (out) out[p] = pmask[p] != 0.0 ? 1 : 0;
  }
}

template <typename T>
int active_set_step_typed(bx_ctx* c, const uint8_t* pin, uint8_t* pout, int32_t* optimal) {
  if (!c->as) return fail(c, BX_ERR_WORKSPACE, "active-set scratch not attached (bx_ctx_set_active_set_workspace)");
  c->last_kind = BX_ACTIVE_SET;
  double* pmask = (double*)c->xprev[c->cur];
  if (pin && c->k > 0) {
    k_mask_io<<<grid1d(c, c->k), RT, 0, c->stream>>>(c->k, pin, pmask, nullptr);
    LAUNCHED();
    c->as_dirty = true;
  }
  bool opt = false;
  TRY(as_step<T>(c, &opt));
  if (pout && c->k > 0) {
    k_mask_io<<<grid1d(c, c->k), RT, 0, c->stream>>>(c->k, nullptr, pmask, pout);
    LAUNCHED();
  }
  CU(cudaStreamSynchronize(c->stream));
  if (optimal) *optimal = opt ? 1 : 0;
  return BX_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

size_t bx_workspace_bytes(int64_t m, int64_t n, int32_t dtype) {
  bx_ctx tmp;
  tmp.m = m;
  tmp.n = n;
  tmp.dtype = dtype;
  tmp.esz = dtype == BX_F32 ? 4 : 8;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0) tmp.nsm = nsm;
  }
  shape_params(&tmp);
  Carver w{nullptr, 0, 0, true};
  carve(&tmp, w);
  return w.off + kAlign;
}

int bx_ctx_create(bx_ctx** out, int64_t m, int64_t n, int32_t dtype, const void* a, int64_t lda, const void* y,
                  const void* lower, const void* upper, const void* t, void* workspace, size_t workspace_bytes,
                  void* cuda_stream) {
  if (!out) return BX_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  bx_ctx* c = new bx_ctx();
  *out = c;
  if (m < 1 || n < 1) return fail(c, BX_ERR_DIMENSION, "A must have at least one row and column");
  if (n > INT32_MAX) return fail(c, BX_ERR_UNSUPPORTED, "n too large");
  if (dtype != BX_F64 && dtype != BX_F32) return fail(c, BX_ERR_INVALID_ARGUMENT, "dtype");
  c->m = m;
  c->n = n;
  c->dtype = dtype;
  c->esz = dtype == BX_F32 ? 4 : 8;
  if (lda < m) return fail(c, BX_ERR_DIMENSION, "lda < m");
  if (((uintptr_t)a % 16) || ((lda * (int64_t)c->esz) % 16))
    return fail(c, BX_ERR_INVALID_ARGUMENT, "A base and column stride must be 16-byte aligned");
  c->A = a;
  c->lda = lda;
  c->stream = (cudaStream_t)cuda_stream;
  int dev = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev));
  int smem_optin = 0;
  CU(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  c->smem_cap = (size_t)smem_optin;
  shape_params(c);
  Carver dry{nullptr, 0, 0, true};
  carve(c, dry);
  if (!workspace || workspace_bytes < dry.off + kAlign)
    return fail(c, BX_ERR_WORKSPACE, "workspace of %zu bytes, need %zu", workspace_bytes, dry.off + kAlign);
  char* base = (char*)align_up((uintptr_t)workspace, kAlign);
  Carver w{base, 0, workspace_bytes, false};
  carve(c, w);
  c->hsc = (DevScalars*)pin_acquire(sizeof(DevScalars));
  if (!c->hsc) return fail(c, BX_ERR_CUDA, "pinned scalar mirror");
  memset(c->hsc, 0, sizeof(DevScalars));
  CU(cudaMemsetAsync(c->sc, 0, sizeof(DevScalars), c->stream));
  CU(cudaMemsetAsync(c->part, 0, (size_t)c->Gmax * c->ldp * 8, c->stream));
  CU(cudaMemsetAsync(c->bar, 0, 4 * kMaxRanks * 4, c->stream));
  c->small_ok = getenv("BX_NO_SMALL") == nullptr;
  {
    const char* e = getenv("BX_SPEC");
    c->spec_on = !(e && e[0] == '0');
    c->zskip_on = getenv("BX_NO_ZSKIP") == nullptr;
    const char* fz = getenv("BX_FUSE");
    c->fuse_on = !(fz && fz[0] == '0');
    const char* to = getenv("BX_PEER_TIMEOUT_S");
    if (to && atof(to) > 0) c->xtimeout_ns = (uint64_t)(atof(to) * 1e9);
  }
  if (dtype == BX_F64) return create_typed<double>(c, y, lower, upper, t);
  return create_typed<float>(c, y, lower, upper, t);
}

int bx_ctx_destroy(bx_ctx* c) {
  if (!c) return BX_OK;
  for (auto& e : c->ev) cudaEventDestroy(e);
  pin_release(c->hsc);
  pin_release(c->has);
  for (void* p : c->xopened) cudaIpcCloseMemHandle(p);
  if (c->xbuf) cudaFree(c->xbuf);
  if (c->comm_owned) delete c->comm;
  delete c;
  return BX_OK;
}

const char* bx_last_error(const bx_ctx* c) { return c ? c->err.c_str() : "null context"; }

int bx_col_norms(bx_ctx* c, void* out) {
  CU(cudaMemcpyAsync(out, c->nrmfull, c->n * 8, cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

int bx_att(bx_ctx* c, void* out) {
  CU(cudaMemcpyAsync(out, c->attfull, c->n * 8, cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

int bx_power_iter(bx_ctx* c, int32_t iters, const double* v0_host, double* sigma_out) {
  if (!sigma_out) return fail(c, BX_ERR_INVALID_ARGUMENT, "sigma_out");
  if (c->dtype == BX_F64) return power_iter<double>(c, iters, v0_host, sigma_out, c->k);
  return power_iter<float>(c, iters, v0_host, sigma_out, c->k);
}

int bx_reset(bx_ctx* c) {
  if (c->dtype == BX_F64) return reset_state<double>(c, BX_APG);
  return reset_state<float>(c, BX_APG);
}

int bx_primal_passes(bx_ctx* c, int32_t kind, double eta, int32_t passes) {
  CU(cudaMemcpyAsync(&c->sc->eta, &eta, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int s = (c->dtype == BX_F64) ? primal_passes<double>(c, kind, passes) : primal_passes<float>(c, kind, passes);
  if (s != BX_OK) return s;
  CU(cudaMemcpyAsync(c->hsc, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return check_dev_err(c);
}

int bx_dual_screen(bx_ctx* c, int32_t screening, double slack_scale, double alpha, double* o) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  if (!(alpha > 0)) return fail(c, BX_ERR_INVALID_ARGUMENT, "alpha must be positive");
  int s = (c->dtype == BX_F64) ? dual_screen<double>(c, screening, slack_scale, alpha)
                               : dual_screen<float>(c, screening, slack_scale, alpha);
  if (s != BX_OK) return s;
  CU(cudaMemcpyAsync(c->hsc, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  s = check_dev_err(c);
  if (o) {
    const DualOut& d = c->hsc->act;
    o[0] = d.primal;
    o[1] = d.dual;
    o[2] = d.gap;
    o[3] = d.eps;
    o[4] = d.radius;
    o[5] = d.slack;
    o[6] = (double)c->hsc->n_lo;
    o[7] = (double)c->hsc->n_up;
  }
  return s;
}

int bx_compact(bx_ctx* c) {
  const int64_t lo = c->hsc->n_lo, up = c->hsc->n_up, keep = c->hsc->n_keep;
  if (lo + up == 0) return BX_OK;
  const bool zu = ((c->bound_bits & 1) && lo > 0) || ((c->bound_bits & 2) && up > 0);
  int s = (c->dtype == BX_F64) ? compact<double>(c, lo, up, keep, c->last_kind, zu)
                               : compact<float>(c, lo, up, keep, c->last_kind, zu);
  if (s != BX_OK) return s;
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

int bx_certified_gap(bx_ctx* c, double alpha, double* o) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  if (!(alpha > 0)) return fail(c, BX_ERR_INVALID_ARGUMENT, "alpha must be positive");
  int s = (c->dtype == BX_F64) ? certified<double>(c, alpha) : certified<float>(c, alpha);
  if (s != BX_OK) return s;
  CU(cudaMemcpyAsync(c->hsc, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  s = check_dev_err(c);
  if (o) {
    o[0] = c->hsc->cert.gap;
    o[1] = c->hsc->cert.primal;
    o[2] = c->hsc->cert.dual;
    o[3] = c->hsc->cert.eps;
  }
  return s;
}

int64_t bx_preserved_count(const bx_ctx* c) { return c ? c->k : -1; }

int bx_set_state(bx_ctx* c, const int64_t* pres, int64_t k, const double* xf, const double* z) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  return c->dtype == BX_F64 ? set_state_typed<double>(c, pres, k, xf, z) : set_state_typed<float>(c, pres, k, xf, z);
}

int bx_get_prev_iterate(bx_ctx* c, double* x_prev) {
  if (!c || !x_prev) return BX_ERR_INVALID_ARGUMENT;
  // screened coordinates sit at their bound in x_prev too (the snap of
  // apply_screening applies to both iterates)
  CU(cudaMemcpyAsync(x_prev, c->xfull, c->n * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (c->k > 0) {
    const double* src = (const double*)(c->spec_pending ? c->xbak[c->cur] : c->xprev[c->cur]);
    k_scatter_x<double><<<grid1d(c, c->k), RT, 0, c->stream>>>(c->k, c->idx[c->cur], src, x_prev);
    LAUNCHED();
  }
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

int bx_active_set_step(bx_ctx* c, const uint8_t* passive_in, uint8_t* passive_out, int32_t* optimal) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  return c->dtype == BX_F64 ? active_set_step_typed<double>(c, passive_in, passive_out, optimal)
                            : active_set_step_typed<float>(c, passive_in, passive_out, optimal);
}

int bx_gradient(bx_ctx* c, double* resid, double* grad) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  return c->dtype == BX_F64 ? gradient_typed<double>(c, resid, grad) : gradient_typed<float>(c, resid, grad);
}

int bx_apply_a(bx_ctx* c, const int32_t* cols, int64_t k, const double* coef, const double* z_add, double* out) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  if (k < 0 || k > c->n) return fail(c, BX_ERR_DIMENSION, "column count %lld", (long long)k);
  return c->dtype == BX_F64 ? apply_a_typed<double>(c, cols, k, coef, z_add, out)
                            : apply_a_typed<float>(c, cols, k, coef, z_add, out);
}

int bx_apply_at(bx_ctx* c, const double* v, double* out) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  return c->dtype == BX_F64 ? apply_at_typed<double>(c, v, out) : apply_at_typed<float>(c, v, out);
}

int bx_dual_point(bx_ctx* c, const double* xf, double alpha, double* theta, double* atheta, double* out) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  if (!(alpha > 0)) return fail(c, BX_ERR_INVALID_ARGUMENT, "alpha must be positive");
  return c->dtype == BX_F64 ? dual_point_typed<double>(c, xf, alpha, theta, atheta, out)
                            : dual_point_typed<float>(c, xf, alpha, theta, atheta, out);
}

int bx_eval_dual(bx_ctx* c, const double* theta, const double* atheta, double* d) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  return c->dtype == BX_F64 ? eval_dual_typed<double>(c, theta, atheta, d)
                            : eval_dual_typed<float>(c, theta, atheta, d);
}

int bx_sphere_test(bx_ctx* c, const double* v, const int32_t* pres, int64_t k, double radius, double slack,
                   uint8_t* flags) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  if (k < 0 || k > c->n) return fail(c, BX_ERR_DIMENSION, "preserved count %lld", (long long)k);
  if (k == 0) return BX_OK;
  if (!v || !pres || !flags) return fail(c, BX_ERR_INVALID_ARGUMENT, "a_t_theta / preserved / flags");
  k_sphere_given<<<grid1d(c, k), RT, 0, c->stream>>>(v, (const double*)c->nrmfull, (const double*)c->hifull, pres, k,
                                                    radius, slack, flags);
  LAUNCHED();
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

int bx_solve(bx_ctx* c, const bx_solve_cfg* cfg, bx_start_vector_fn fn, void* user, bx_trace_rec* trace,
             int64_t cap, bx_solve_out* out) {
  if (!c || !cfg) return BX_ERR_INVALID_ARGUMENT;
  if (cfg->kind != BX_PG && cfg->kind != BX_CD && cfg->kind != BX_APG && cfg->kind != BX_ACTIVE_SET)
    return fail(c, BX_ERR_INVALID_ARGUMENT, "unknown solver kind %d", cfg->kind);
  if (!(cfg->gap_tol > 0)) return fail(c, BX_ERR_INVALID_ARGUMENT, "gap_tol must be positive");
  if (cfg->inner_passes < 1) return fail(c, BX_ERR_INVALID_ARGUMENT, "inner_passes must be >= 1");
  c->launches = 0;
  if (c->dtype == BX_F64) return solve_typed<double>(c, cfg, fn, user, trace, cap, out);
  return solve_typed<float>(c, cfg, fn, user, trace, cap, out);
}

int bx_get_state(bx_ctx* c, void* x, void* theta, int64_t* sat_lower, int64_t* sat_upper) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  if (x) {
    // x_full <- the current preserved iterate (screened entries are already
    // at their bounds): valid after any sequence of fine-grained calls
    if (c->k > 0) {
      k_scatter_x<double><<<grid1d(c, c->k), RT, 0, c->stream>>>(c->k, c->idx[c->cur], round_x(c), (double*)c->xfull);
      LAUNCHED();
    }
    CU(cudaMemcpyAsync(x, c->xfull, c->n * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (theta)
    CU(cudaMemcpyAsync(theta, c->theta_is_cert ? c->thetac : c->theta, c->m * 8, cudaMemcpyDeviceToDevice,
                       c->stream));
  if (sat_lower && c->n_sat_lo)
    CU(cudaMemcpyAsync(sat_lower, c->sat_lo, c->n_sat_lo * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (sat_upper && c->n_sat_up)
    CU(cudaMemcpyAsync(sat_upper, c->sat_up, c->n_sat_up * 8, cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BX_OK;
}

size_t bx_active_set_workspace_bytes(int64_t m, int64_t n) {
  const int64_t pcap = std::max<int64_t>(1, std::min(m, n));
  const int64_t mp = round_up(m, 32);
  Carver w{nullptr, 0, 0, true};
  w.take((size_t)pcap * pcap * 8);
  for (int i = 0; i < 3; ++i) w.take((size_t)(pcap + 1) * 4);
  for (int i = 0; i < 2; ++i) w.take((size_t)mp * 8);
  for (int i = 0; i < 4; ++i) w.take((size_t)(pcap + 1) * 8);
  w.take(sizeof(AsState));
  return w.off + kAlign;
}

int bx_ctx_set_active_set_workspace(bx_ctx* c, void* workspace, size_t bytes) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  const size_t need = bx_active_set_workspace_bytes(c->m, c->n);
  if (!workspace || bytes < need)
    return fail(c, BX_ERR_WORKSPACE, "active-set workspace of %zu bytes, need %zu", bytes, need);
  c->pcap = (int)std::max<int64_t>(1, std::min(c->m, c->n));
  const int64_t pcap = c->pcap;
  Carver w{(char*)align_up((uintptr_t)workspace, kAlign), 0, bytes, false};
  c->asR = (double*)w.take((size_t)pcap * pcap * 8);
  c->as_cslot = (int32_t*)w.take((size_t)(pcap + 1) * 4);
  c->as_plist = (int32_t*)w.take((size_t)(pcap + 1) * 4);
  c->as_hitf = (int32_t*)w.take((size_t)(pcap + 1) * 4);
  c->as_avec = (double*)w.take((size_t)c->mp * 8);
  c->as_rhs = (double*)w.take((size_t)c->mp * 8);
  c->as_c = (double*)w.take((size_t)(pcap + 1) * 8);
  c->as_b = (double*)w.take((size_t)(pcap + 1) * 8);
  c->as_s = (double*)w.take((size_t)(pcap + 1) * 8);
  c->as_frac = (double*)w.take((size_t)(pcap + 1) * 8);
  c->as = (AsState*)w.take(sizeof(AsState));
  if (!c->has) {
    c->has = (AsState*)pin_acquire(sizeof(AsState));
    if (!c->has) return fail(c, BX_ERR_CUDA, "pinned active-set mirror");
  }
  memset(c->has, 0, sizeof(AsState));
  c->as_dirty = true;
  return BX_OK;
}

int bx_peer_alloc(bx_ctx* c, unsigned char* handle_out) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  if (!c->sharded()) return fail(c, BX_ERR_INVALID_ARGUMENT, "attach a communicator before bx_peer_alloc");
  if (c->nranks > kXPeers) return fail(c, BX_ERR_UNSUPPORTED, "fused exchange: at most %d ranks", kXPeers);
  if (!c->xbuf) {
    const size_t bytes = xbuf_bytes(c->mp, c->nsm);
    CU(cudaMalloc(&c->xbuf, bytes));
    CU(cudaMemset(c->xbuf, 0, bytes));
    CU(cudaDeviceSynchronize());
  }
  if (handle_out) {
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, c->xbuf));
    memcpy(handle_out, &h, sizeof(h));
  }
  return BX_OK;
}

// CTAs of the fused reduction: row blocks of a multiple of XCH rows
static int x_fit_nb(const bx_ctx* c, int64_t cap) {
  const int64_t per = xrows_per_cta(c->m, (int)std::max<int64_t>(1, cap));
  return (int)std::max<int64_t>(1, (c->m + per - 1) / per);
}

int bx_peer_open(bx_ctx* c, const unsigned char* handles) {
  if (!c || !c->xbuf) return c ? fail(c, BX_ERR_INVALID_ARGUMENT, "bx_peer_alloc first") : BX_ERR_INVALID_ARGUMENT;
  auto fit_nb = [&](int64_t cap) { return x_fit_nb(c, cap); };
  if (!handles) {
    LocalComm* lc = dynamic_cast<LocalComm*>(c->comm);
    if (!lc) return fail(c, BX_ERR_INVALID_ARGUMENT, "NULL handles need the in-process group");
    lc->g->xbufs.resize(lc->g->n, nullptr);
    lc->g->xargs.resize(lc->g->n);
    lc->g->xbufs[c->rank] = c->xbuf;
    // every emulated rank's CTAs must be co-resident in one cooperative grid
    c->xnb = fit_nb(c->nsm / c->nranks);
    c->xmode = 2;
    return BX_OK;
  }
  for (int q = 0; q < c->nranks; ++q) {
    void* p = nullptr;
    if (q == c->rank) {
      p = c->xbuf;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, handles + 64 * q, sizeof(h));
      CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      c->xopened.push_back(p);
    }
    c->xpeer_recv[q] = static_cast<double*>(p);
    c->xpeer_flag[q] = reinterpret_cast<unsigned*>(static_cast<char*>(p) + xrecv_doubles(c->mp) * 8);
  }
  c->xnb = fit_nb(c->nsm);
  c->xmode = 1;
  return BX_OK;
}

int bx_peer_disable(bx_ctx* c) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  for (void* p : c->xopened) cudaIpcCloseMemHandle(p);
  c->xopened.clear();
  c->xmode = 0;
  return BX_OK;
}

int bx_nccl_unique_id(unsigned char* id_out) {
  if (!g_nccl.load()) return BX_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (g_nccl.get_id(&id) != 0) return BX_ERR_CUDA;
  memcpy(id_out, id.internal, 128);
  return BX_OK;
}

int bx_ctx_set_comm(bx_ctx* c, const unsigned char* id_host, int32_t rank, int32_t nranks, int64_t col_offset,
                    int64_t n_global) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return fail(c, BX_ERR_INVALID_ARGUMENT, "rank %d of %d", rank, nranks);
  if (!g_nccl.load()) return fail(c, BX_ERR_UNSUPPORTED, "libnccl.so.2 not found");
  ncclUniqueId id;
  memcpy(id.internal, id_host, 128);
  NcclComm* nc = new NcclComm();
  const int r = g_nccl.init_rank(&nc->comm, nranks, id, rank);
  if (r != 0) {
    delete nc;
    return fail(c, BX_ERR_CUDA, "ncclCommInitRank: %d", r);
  }
  if (c->comm_owned) delete c->comm;
  c->comm = nc;
  c->comm_owned = true;
  c->rank = rank;
  c->nranks = nranks;
  c->col_offset = col_offset;
  c->n_global = n_global;
  return BX_OK;
}

int bx_comm_create(bx_comm** out, const unsigned char* id_host, int32_t rank, int32_t nranks) {
  if (!out || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return BX_ERR_INVALID_ARGUMENT;
  if (!g_nccl.load()) return BX_ERR_UNSUPPORTED;
  ncclUniqueId id;
  memcpy(id.internal, id_host, 128);
  bx_comm* cm = new bx_comm();
  cm->nc = new NcclComm();
  if (g_nccl.init_rank(&cm->nc->comm, nranks, id, rank) != 0) {
    delete cm;
    return BX_ERR_CUDA;
  }
  cm->rank = rank;
  cm->nranks = nranks;
  *out = cm;
  return BX_OK;
}

int bx_comm_destroy(bx_comm* cm) {
  delete cm;
  return BX_OK;
}

int bx_comm_peer_alloc(bx_comm* cm, int64_t m, unsigned char* handle_out) {
  if (!cm || m < 1 || !handle_out) return BX_ERR_INVALID_ARGUMENT;
  if (cm->nranks > kXPeers) return BX_ERR_UNSUPPORTED;
  if (!cm->xbuf) {
    int dev = 0, nsm = 0;
    CUR(cudaGetDevice(&dev));
    CUR(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    cm->xmp = round_up(m, 32);
    cm->xnsm = nsm;
    const size_t bytes = xbuf_bytes(cm->xmp, nsm);
    CUR(cudaMalloc(&cm->xbuf, bytes));
    CUR(cudaMemset(cm->xbuf, 0, bytes));
    CUR(cudaDeviceSynchronize());
  }
  cudaIpcMemHandle_t h;
  CUR(cudaIpcGetMemHandle(&h, cm->xbuf));
  memcpy(handle_out, &h, sizeof(h));
  return BX_OK;
}

int bx_comm_peer_open(bx_comm* cm, const unsigned char* handles) {
  if (!cm || !cm->xbuf || !handles) return BX_ERR_INVALID_ARGUMENT;
  for (int q = 0; q < cm->nranks; ++q) {
    void* p = nullptr;
    if (q == cm->rank) {
      p = cm->xbuf;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, handles + 64 * q, sizeof(h));
      CUR(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      cm->xopened.push_back(p);
    }
    cm->xpeer_recv[q] = static_cast<double*>(p);
    cm->xpeer_flag[q] = reinterpret_cast<unsigned*>(static_cast<char*>(p) + xrecv_doubles(cm->xmp) * 8);
  }
  cm->xmode = 1;
  return BX_OK;
}

int bx_comm_peer_disable(bx_comm* cm) {
  if (!cm) return BX_ERR_INVALID_ARGUMENT;
  for (void* p : cm->xopened) cudaIpcCloseMemHandle(p);
  cm->xopened.clear();
  cm->xmode = 0;
  return BX_OK;
}

int bx_ctx_use_comm(bx_ctx* c, bx_comm* cm, int64_t col_offset, int64_t n_global) {
  if (!c || !cm || !cm->nc) return c ? fail(c, BX_ERR_INVALID_ARGUMENT, "null communicator") : BX_ERR_INVALID_ARGUMENT;
  if (cm->xmode == 1 && (c->mp > cm->xmp || c->nsm > cm->xnsm))
    return fail(c, BX_ERR_UNSUPPORTED, "communicator exchange buffer sized for m <= %lld", (long long)cm->xmp);
  if (c->comm_owned) delete c->comm;
  c->comm = cm->nc;
  c->comm_owned = false;
  c->rank = cm->rank;
  c->nranks = cm->nranks;
  c->col_offset = col_offset;
  c->n_global = n_global;
  c->xmode = cm->xmode;
  if (cm->xmode == 1) {
    for (int q = 0; q < cm->nranks; ++q) {
      c->xpeer_recv[q] = cm->xpeer_recv[q];
      c->xpeer_flag[q] = cm->xpeer_flag[q];
    }
    c->xnb = x_fit_nb(c, c->nsm);
    c->xepoch_p = &cm->xepoch;
  }
  return BX_OK;
}

int bx_group_create(bx_group** out, int32_t nranks) {
  if (!out || nranks < 1 || nranks > kMaxRanks) return BX_ERR_INVALID_ARGUMENT;
  bx_group* g = new bx_group();
  g->n = nranks;
  g->ptrs.assign(nranks, nullptr);
  {
    const char* e = getenv("BX_GROUP_XREDUCE");
    g->per_rank = e && strcmp(e, "rank") == 0;
  }
  *out = g;
  return BX_OK;
}

int bx_group_destroy(bx_group* g) {
  delete g;
  return BX_OK;
}

int bx_ctx_set_group(bx_ctx* c, bx_group* g, int32_t rank, int64_t col_offset, int64_t n_global) {
  if (!c || !g || rank < 0 || rank >= g->n) return BX_ERR_INVALID_ARGUMENT;
  LocalComm* lc = new LocalComm();
  lc->g = g;
  lc->rank = rank;
  lc->tmp = c->grp_tmp;
  lc->dptrs = c->grp_ptrs;
  if (c->comm_owned) delete c->comm;
  c->comm = lc;
  c->comm_owned = true;
  c->rank = rank;
  c->nranks = g->n;
  c->col_offset = col_offset;
  c->n_global = n_global;
  return BX_OK;
}

int bx_set_profiling(bx_ctx* c, int32_t on) {
  if (!c) return BX_ERR_INVALID_ARGUMENT;
  c->prof = on != 0;
  memset(c->pstat, 0, sizeof(c->pstat));
  c->pending.clear();
  return BX_OK;
}

int bx_get_profile(bx_ctx* c, bx_prof_entry* out, int32_t n) {
  if (!c || !out) return BX_ERR_INVALID_ARGUMENT;
  TRY(prof_drain(c));
  for (int i = 0; i < n && i < BX_PROF_SLOTS; ++i) out[i] = c->pstat[i];
  return BX_OK;
}

// ---------------------------------------------------------------------------
// batched many-RHS FISTA (config 5)
// ---------------------------------------------------------------------------
}  // extern "C"

struct bx_batch {
  BatchArgs a;
  int64_t K_user = 0;
  cudaStream_t stream = nullptr;
  double* t = nullptr;
  int* flags = nullptr;
  double* red = nullptr;   // [4] round summary
  double* hred = nullptr;  // pinned mirror
  int64_t launches = 0;
  int blocked_Gw = 0;  // row-blocked path: block count of the last k_colupdate partials
  std::string err;
  int nsm = 148;
  size_t smem = 0;
  int tile = 64;  // problems per CTA tile of k_batched_round
  int sched = 2;  // 2: warp-per-octet schedule over a TMA chunk ring (bx_batched2.cuh); 1: the first schedule
  size_t smem2 = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};  // around every round kernel (live duration for the roofline)
  cudaStream_t copy_stream = nullptr;      // result rows leaving for the host during the last round
  cudaEvent_t ev_wave = nullptr, ev_copy = nullptr;
  double round_ms = 0.0;
  bool pipe = true;  // software-pipelined chunk loop (BX_BT_PIPE=0: the A/B control)
  double last_max_gap = 0.0;
  int check_every = 1;  // rounds per launch between convergence checks (second schedule)
  int mtc = 0;    // compile-time row-tile count of the launched instantiation (0: run-time m)
};

namespace {
// rounds one launch of the second schedule may run (check_every is capped by it)
constexpr int kBatchRoundsPerLaunch = 16;
struct BatchLayout {
  int64_t Kp, ldx, ldy, nw;
  size_t bytes;
};
BatchLayout batch_layout(int64_t m, int64_t n, int64_t K, bx_batch* b, char* base) {
  BatchLayout L;
  L.Kp = round_up(K, BT_TILE);
  L.ldx = round_up(n, 16);
  L.ldy = round_up(m, 8);
  L.nw = (n + 31) / 32;
  Carver w{base, 0, 0, base == nullptr};
  double* Y = (double*)w.take(L.Kp * L.ldy * 8);
  double* X0 = (double*)w.take(L.Kp * L.ldx * 8);
  double* X1 = (double*)w.take(L.Kp * L.ldx * 8);
  double* R0 = (double*)w.take(L.Kp * L.ldy * 8);
  double* R1 = (double*)w.take(L.Kp * L.ldy * 8);
  uint32_t* mask = (uint32_t*)w.take(L.Kp * L.nw * 4);
  const int64_t n_pad = round_up(n, BT_CH), sa2 = round_up(m, 8) + 4;
  double* nrm = (double*)w.take(n_pad * 8);
  double* att = (double*)w.take(n_pad * 8);
  double* Ap = (double*)w.take(n_pad * sa2 * 8);
  double* t = (double*)w.take(L.ldy * 8);
  double* mom = (double*)w.take(L.Kp * 8);
  double* P = (double*)w.take(L.Kp * 8);
  double* stats = (double*)w.take(5 * L.Kp * 8);
  int* flags = (int*)w.take(64);
  double* red = (double*)w.take(4 * kBatchRoundsPerLaunch * 8);
  unsigned long long* sweeps2 = (unsigned long long*)w.take(64);
  unsigned* oct_round = (unsigned*)w.take((L.Kp / 8) * 4);
  double* osum = (double*)w.take((size_t)kBatchRoundsPerLaunch * (L.Kp / 8) * 4 * 8);
  L.bytes = w.off + kAlign;
  if (b) {
    b->a.Y = Y;
    b->a.X[0] = X0;
    b->a.X[1] = X1;
    b->a.R[0] = R0;
    b->a.R[1] = R1;
    b->a.mask = mask;
    b->a.nrm = nrm;
    b->a.att = att;
    b->a.Ap = Ap;
    b->a.sa2 = (int)sa2;
    b->a.nch = (int)(n_pad / BT_CH);
    b->a.sweeps2 = sweeps2;
    b->a.oct_round = oct_round;
    b->a.osum = osum;
    b->a.osum_rounds = kBatchRoundsPerLaunch;
    b->a.mom = mom;
    b->a.P = P;
    b->a.stats = stats;
    b->t = t;
    b->flags = flags;
    b->red = red;
  }
  return L;
}

__global__ void k_batched_summary(const double* __restrict__ stats, int64_t Kp, int64_t K, double gap_tol,
                                  double* __restrict__ out) {
  // out = {converged count, max gap, sum gap, sum preserved} over the first K problems (one block, fixed order)
  __shared__ double sh[4][32];
  double cnt = 0.0, mx = 0.0, sg = 0.0, sp = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const double gp = stats[2 * Kp + k];
    cnt += gp < gap_tol ? 1.0 : 0.0;
    mx = fmax(mx, gp);
    sg += gp;
    sp += stats[4 * Kp + k];
  }
  cnt = warp_sum<double>(cnt);
  sg = warp_sum<double>(sg);
  sp = warp_sum<double>(sp);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][warp] = cnt;
    sh[1][warp] = mx;
    sh[2][warp] = sg;
    sh[3][warp] = sp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double c = 0, m = 0, g = 0, p = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      c += sh[0][w];
      m = fmax(m, sh[1][w]);
      g += sh[2][w];
      p += sh[3][w];
    }
    out[0] = c;
    out[1] = m;
    out[2] = g;
    out[3] = p;
  }
}

__global__ void k_pad_copy(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                           double* __restrict__ dst, int64_t ldd, int64_t cols_pad) {
  const int64_t tot = ldd * cols_pad;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = q / ldd, r = q - c * ldd;
    dst[q] = (c < cols && r < rows) ? src[c * lds + r] : 0.0;
  }
}
}  // namespace

extern "C" {

size_t bx_batched_workspace_bytes(int64_t m, int64_t n, int64_t k_rhs) {
  return batch_layout(m, n, k_rhs, nullptr, nullptr).bytes;
}

#define BCU(call)                                                                            \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      b->err = std::string(#call) + ": " + cudaGetErrorString(e_);                           \
      return BX_ERR_CUDA;                                                                    \
    }                                                                                        \
  } while (0)

#define TRY_B(call)            \
  do {                         \
    const int st_ = (call);    \
    if (st_ != BX_OK) return st_; \
  } while (0)

int bx_batched_create(bx_batch** out, int64_t m, int64_t n, int64_t k_rhs, const double* a, int64_t lda,
                      const double* y, int64_t ldy, void* workspace, size_t workspace_bytes, void* stream) {
  if (!out) return BX_ERR_INVALID_ARGUMENT;
  bx_batch* b = new bx_batch();
  *out = b;
  if (m < 1 || n < 1 || k_rhs < 1) return BX_ERR_DIMENSION;
  if (m > 8 * BT_MT) {
    b->err = "batched solver: m must be <= 208";
    return BX_ERR_UNSUPPORTED;
  }
  if (((uintptr_t)a % 16) || (lda % 2) || lda < m) {
    b->err = "A must be 16-byte aligned with an even lda >= m";
    return BX_ERR_INVALID_ARGUMENT;
  }
  const BatchLayout L0 = batch_layout(m, n, k_rhs, nullptr, nullptr);
  if (!workspace || workspace_bytes < L0.bytes) {
    b->err = "workspace too small";
    return BX_ERR_WORKSPACE;
  }
  char* base = (char*)align_up((uintptr_t)workspace, kAlign);
  const BatchLayout L = batch_layout(m, n, k_rhs, b, base);
  b->K_user = k_rhs;
  b->stream = (cudaStream_t)stream;
  BatchArgs& A = b->a;
  A.A = a;
  A.lda = lda;
  A.m = (int)m;
  A.n = (int)n;
  A.K = (int)L.Kp;
  A.ldy = L.ldy;
  A.ldx = L.ldx;
  A.nw = (int)L.nw;
  const int m8 = (int)round_up(m, 8);
  A.sa = m8 + ((4 - (m8 % 16)) + 16) % 16;  // >= m8 and == 4 (mod 16)
  A.rs_f = 1e-12;
  A.rs_g = 1e-12;
  A.slack_scale = 1e-12;
  int dev = 0;
  BCU(cudaGetDevice(&dev));
  BCU(cudaDeviceGetAttribute(&b->nsm, cudaDevAttrMultiProcessorCount, dev));
  // problem tile: 64 (one CTA per SM) or 32 (two CTAs per SM); BX_BT_TILE overrides
  {
    const char* e = getenv("BX_BT_TILE");
    b->tile = (e && atoi(e) == 32) ? 32 : 64;
    const char* v1 = getenv("BX_BT_V1");
    b->sched = (v1 && atoi(v1) == 1) ? 1 : 2;
    if (b->sched == 2) b->tile = 64;
  }
  b->smem2 = ((size_t)(B2_NST * BT_CH + BT_TILE) * A.sa2) * 8 + B2_NST * 12 + 16;
  // the config-5 row count (25 row tiles) has its own fully unrolled instantiation
  b->mtc = (m8 / 8 == 25 && !getenv("BX_BT_GENERIC")) ? 25 : 0;
  b->pipe = !(getenv("BX_BT_PIPE") && atoi(getenv("BX_BT_PIPE")) == 0);
  if (b->mtc == 25 && !b->pipe)
    BCU(cudaFuncSetAttribute(k_batched_round2<25, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)b->smem2));
  else if (b->mtc == 25)
    BCU(cudaFuncSetAttribute(k_batched_round2<25>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->smem2));
  else
    BCU(cudaFuncSetAttribute(k_batched_round2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->smem2));
  const int nb = b->tile == 64 ? 2 : 1;
  b->smem = ((size_t)b->tile * A.sa + (size_t)nb * BT_CH * A.sa + (size_t)(2 * nb + 1) * b->tile * BT_SX +
             9 * (size_t)b->tile) * 8 + 2 * (size_t)b->tile * 4 + 64;
  if (b->tile == 64)
    BCU(cudaFuncSetAttribute(k_batched_round<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->smem));
  else
    BCU(cudaFuncSetAttribute(k_batched_round<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->smem));
  b->hred = (double*)pin_acquire(4 * kBatchRoundsPerLaunch * 8);
  if (!b->hred) return BX_ERR_CUDA;
  BCU(cudaEventCreate(&b->ev[0]));
  BCU(cudaEventCreate(&b->ev[1]));
  // padded copy of Y, t = -1, column norms and A't of the dictionary
  k_pad_copy<<<1024, 256, 0, b->stream>>>(y, ldy, m, k_rhs, const_cast<double*>(A.Y), L.ldy, L.Kp);
  k_fill<double><<<4, 256, 0, b->stream>>>(L.ldy, b->t, 0.0);
  k_fill<double><<<4, 256, 0, b->stream>>>(m, b->t, -1.0);
  BCU(cudaMemsetAsync(b->flags, 0, 64, b->stream));
  k_colstats<double><<<(int)((n * 32 + 255) / 256 < 2048 ? (n * 32 + 255) / 256 : 2048), 256, 0, b->stream>>>(
      a, lda, n, m, b->t, const_cast<double*>(A.nrm), const_cast<double*>(A.att), 1, b->flags);
  k_b2_pack<<<1024, 256, 0, b->stream>>>(a, lda, (int)m, (int)n, A.nrm, A.att, const_cast<double*>(A.Ap), A.sa2, A.nch);
  int fl = 0;
  BCU(cudaMemcpyAsync(&fl, b->flags, 4, cudaMemcpyDeviceToHost, b->stream));
  BCU(cudaStreamSynchronize(b->stream));
  if (fl & 2) {
    b->err = "neg-ones translation vector is not strictly interior (A must be entrywise nonnegative)";
    return BX_ERR_NO_INTERIOR;
  }
  if (fl & 1) {
    b->err = "zero column in A";
    return BX_ERR_ZERO_COLUMN;
  }
  {
    // constants of the sphere-test bound (second schedule)
    std::vector<double> hn(n), ha(n);
    BCU(cudaMemcpyAsync(hn.data(), A.nrm, n * 8, cudaMemcpyDeviceToHost, b->stream));
    BCU(cudaMemcpyAsync(ha.data(), A.att, n * 8, cudaMemcpyDeviceToHost, b->stream));
    BCU(cudaStreamSynchronize(b->stream));
    double amax = 0.0, nmin = hn[0];
    for (int64_t j = 0; j < n; ++j) {
      amax = std::max(amax, std::fabs(ha[j]));
      nmin = std::min(nmin, hn[j]);
    }
    A.att_max = amax;
    A.nrm_min = nmin;
    A.bound_skip = getenv("BX_BT_NOSKIP") ? 0 : 1;
  }
  return BX_OK;
}

}  // extern "C"

namespace {
// one round over tiles [t0, t1) with the selected schedule
int batched_launch(bx_batch* b, int t0, int t1, int round0, int nrl) {
  BatchArgs& A = b->a;
  const int per_sm = b->tile == 64 ? 1 : 2;
  const int64_t units = (int64_t)(t1 - t0) * nrl;
  const int grid = per_sm * b->nsm < units ? per_sm * b->nsm : (int)units;
  A.tile0 = t0;
  A.tile1 = t1;
  A.round0 = round0;
  A.nrl = nrl;
  if (b->sched == 2) {
    // several rounds per launch: CTAs wait on flags other CTAs of the launch
    // publish, so the grid must be co-resident -- a cooperative launch
    // guarantees it (or fails) instead of assuming idle SMs
    const void* fn = (b->mtc == 25 && !b->pipe) ? (const void*)k_batched_round2<25, false>
                     : b->mtc == 25             ? (const void*)k_batched_round2<25, true>
                                                : (const void*)k_batched_round2<0, true>;
    void* kargs[] = {(void*)&A};
    if (nrl > 1)
      BCU(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(B2_NT), kargs, b->smem2, b->stream));
    else
      BCU(cudaLaunchKernel(fn, dim3(grid), dim3(B2_NT), kargs, b->smem2, b->stream));
  } else if (b->tile == 64)
    k_batched_round<64><<<grid, 64 * 8, b->smem, b->stream>>>(A);
  else
    k_batched_round<32><<<grid, 32 * 8, b->smem, b->stream>>>(A);
  ++b->launches;
  BCU(cudaGetLastError());
  return BX_OK;
}

// x_host (optional, pinned, n x K column-major with stride ldx_host): the
// result on the host when the call returns.  In the last round of the budget
// the tiles are launched wave by wave and each wave's rows of X leave for the
// host while the next waves compute (the 4 GB of config 5 cross PCIe behind
// ~150 ms of tensor work instead of after it); a solve that converges earlier
// copies after its last round.
int batched_run(bx_batch* b, double eta, int32_t passes, int32_t rounds, int32_t screening, double gap_tol,
                double* trace_host, int64_t trace_cap, bx_batched_out* out, double* x_host, int64_t ldx_host) {
  if (!b) return BX_ERR_INVALID_ARGUMENT;
  BatchArgs& A = b->a;
  if (x_host && ldx_host < A.n) return BX_ERR_INVALID_ARGUMENT;
  A.eta = eta;
  A.passes = passes;
  A.screening = screening;
  A.par = 0;
  BCU(cudaMemsetAsync(A.sweeps2, 0, 8, b->stream));
  A.dbg = nullptr;
  if (getenv("BX_BT_DEBUG")) BCU(cudaMalloc(&A.dbg, 148 * 8 * 4 * 8));
  k_batched_init<<<1024, 256, 0, b->stream>>>(A);
  b->launches = 1;
  b->round_ms = 0.0;
  const int ntiles = A.K / b->tile;
  const int wave = (b->tile == 64 ? 1 : 2) * b->nsm;
  bool streamed = false;
  int64_t r = 0;
  int64_t conv = 0;
  A.K_user = b->K_user;
  A.gap_tol = gap_tol;
  BCU(cudaMemsetAsync(A.oct_round, 0, (A.K / 8) * 4, b->stream));
  const int noct = A.K / 8;
  const bool stream_last = x_host && b->sched == 2 && ntiles > wave;
  while (r < rounds) {
    // rounds of this launch: one, or (second schedule) up to check_every with
    // the tiles' rounds overlapping across the launch; the budget's last round
    // runs alone when its result streams out
    int nb = 1;
    const bool last_alone = stream_last && r == rounds - 1;
    if (b->sched == 2 && !last_alone) {
      nb = (int)std::min<int64_t>({(int64_t)b->check_every, (int64_t)kBatchRoundsPerLaunch,
                                   rounds - r - (stream_last ? 1 : 0)});
      if (nb < 1) nb = 1;
    }
    BCU(cudaEventRecord(b->ev[0], b->stream));
    if (last_alone) {
      if (!b->copy_stream) {
        BCU(cudaStreamCreateWithFlags(&b->copy_stream, cudaStreamNonBlocking));
        BCU(cudaEventCreateWithFlags(&b->ev_wave, cudaEventDisableTiming));
        BCU(cudaEventCreateWithFlags(&b->ev_copy, cudaEventDisableTiming));
      }
      const int par_after = (passes & 1) ? A.par ^ 1 : A.par;
      for (int t0 = 0; t0 < ntiles; t0 += wave) {
        const int t1 = t0 + wave < ntiles ? t0 + wave : ntiles;
        TRY_B(batched_launch(b, t0, t1, (int)r, 1));
        BCU(cudaEventRecord(b->ev_wave, b->stream));
        BCU(cudaStreamWaitEvent(b->copy_stream, b->ev_wave, 0));
        const int64_t k0 = (int64_t)t0 * b->tile;
        const int64_t k1 = std::min<int64_t>((int64_t)t1 * b->tile, b->K_user);
        if (k1 > k0)
          BCU(cudaMemcpy2DAsync(x_host + k0 * ldx_host, ldx_host * 8, A.X[par_after] + k0 * A.ldx, A.ldx * 8,
                                A.n * 8, k1 - k0, cudaMemcpyDeviceToHost, b->copy_stream));
      }
      BCU(cudaEventRecord(b->ev_copy, b->copy_stream));
      BCU(cudaStreamWaitEvent(b->stream, b->ev_copy, 0));
      streamed = true;
    } else {
      TRY_B(batched_launch(b, 0, ntiles, (int)r, nb));
    }
    BCU(cudaEventRecord(b->ev[1], b->stream));
    for (int q = 0; q < nb; ++q) {
      if (b->sched == 2)
        k_b2_summary<<<1, 1024, 0, b->stream>>>(
            A.osum + (size_t)((r + q) % kBatchRoundsPerLaunch) * noct * 4, noct, b->red + 4 * q);
      else
        k_batched_summary<<<1, 1024, 0, b->stream>>>(A.stats, A.K, b->K_user, gap_tol, b->red);
      ++b->launches;
    }
    BCU(cudaGetLastError());
    if ((nb * passes) & 1) A.par ^= 1;
    BCU(cudaMemcpyAsync(b->hred, b->red, 4 * nb * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
    BCU(cudaStreamSynchronize(b->stream));
    {
      float ms = 0.f;
      BCU(cudaEventElapsedTime(&ms, b->ev[0], b->ev[1]));
      b->round_ms += ms;
    }
    for (int q = 0; q < nb; ++q) {
      const double* h = b->hred + 4 * q;
      if (trace_host && r + q < trace_cap) {
        trace_host[4 * (r + q) + 0] = h[0];
        trace_host[4 * (r + q) + 1] = h[1];
        trace_host[4 * (r + q) + 2] = h[2] / (double)b->K_user;
        trace_host[4 * (r + q) + 3] = h[3] / (double)b->K_user;
      }
    }
    r += nb;
    conv = (int64_t)b->hred[4 * (nb - 1)];
    b->last_max_gap = b->hred[4 * (nb - 1) + 1];
    if (conv == b->K_user) break;
  }
  if (x_host && !streamed) {
    BCU(cudaMemcpy2DAsync(x_host, ldx_host * 8, A.X[A.par], A.ldx * 8, A.n * 8, b->K_user, cudaMemcpyDeviceToHost,
                          b->stream));
    BCU(cudaStreamSynchronize(b->stream));
  }
  if (A.dbg) {
    std::vector<unsigned long long> h(148 * 8 * 4);
    BCU(cudaMemcpy(h.data(), A.dbg, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int cta : {0, 1, 77, 147})
      for (int w = 0; w < 8; ++w) {
        const unsigned long long* o = &h[(size_t)(cta * 8 + w) * 4];
        fprintf(stderr, "cta %3d warp %d: wait %6.2f%% of %llu clk, long waits %llu of %llu chunks\n", cta, w,
                100.0 * (double)o[0] / (double)o[2], o[2], o[1], o[3]);
      }
    cudaFree(A.dbg);
    A.dbg = nullptr;
  }
  if (out) {
    out->rounds = r;
    out->converged = conv;
    out->iterations = r * passes;
    out->kernel_launches = b->launches;
    out->max_gap = b->last_max_gap;
    unsigned long long sw = 0;
    BCU(cudaMemcpy(&sw, A.sweeps2, 8, cudaMemcpyDeviceToHost));
    out->sphere_sweeps = b->sched == 2 ? (int64_t)sw : (screening ? r * (A.K / b->tile) : 0);
    out->tiles = A.K / b->tile;
    out->round_kernel_ms = b->round_ms;
  }
  return BX_OK;
}
}  // namespace

extern "C" {

int bx_batched_set_check_every(bx_batch* b, int32_t rounds_per_check) {
  if (!b || rounds_per_check < 1) return BX_ERR_INVALID_ARGUMENT;
  b->check_every = rounds_per_check < kBatchRoundsPerLaunch ? rounds_per_check : kBatchRoundsPerLaunch;
  return BX_OK;
}

int bx_batched_run(bx_batch* b, double eta, int32_t passes, int32_t rounds, int32_t screening, double gap_tol,
                   double* trace_host, int64_t trace_cap, bx_batched_out* out) {
  return batched_run(b, eta, passes, rounds, screening, gap_tol, trace_host, trace_cap, out, nullptr, 0);
}

int bx_batched_run_to_host(bx_batch* b, double eta, int32_t passes, int32_t rounds, int32_t screening, double gap_tol,
                           double* trace_host, int64_t trace_cap, bx_batched_out* out, double* x_host,
                           int64_t ldx_host) {
  if (!x_host) return BX_ERR_INVALID_ARGUMENT;
  return batched_run(b, eta, passes, rounds, screening, gap_tol, trace_host, trace_cap, out, x_host, ldx_host);
}

int bx_batched_get(bx_batch* b, double* x, int64_t ldx_out, double* stats) {
  BatchArgs& A = b->a;
  if (x)
    BCU(cudaMemcpy2DAsync(x, ldx_out * 8, A.X[A.par], A.ldx * 8, A.n * 8, b->K_user, cudaMemcpyDeviceToDevice,
                          b->stream));
  if (stats)
    for (int q = 0; q < 5; ++q)
      BCU(cudaMemcpyAsync(stats + q * b->K_user, A.stats + q * A.K, b->K_user * 8, cudaMemcpyDeviceToDevice,
                          b->stream));
  BCU(cudaStreamSynchronize(b->stream));
  return BX_OK;
}

const char* bx_batched_last_error(const bx_batch* b) { return b ? b->err.c_str() : "null"; }

int bx_batched_destroy(bx_batch* b) {
  if (!b) return BX_OK;
  pin_release(b->hred);
  for (cudaEvent_t e : {b->ev[0], b->ev[1], b->ev_wave, b->ev_copy})
    if (e) cudaEventDestroy(e);
  if (b->copy_stream) cudaStreamDestroy(b->copy_stream);
  delete b;
  return BX_OK;
}

}  // extern "C"
