// snp_comm.cu — transports of the multi-GPU exchange (snp_comm.h).
//
// NCCL is opened with dlopen at the first snp_dist_unique_id / snp_dist_init:
// when PyTorch already loaded its libnccl.so.2 the same copy is reused (one
// NCCL per process), otherwise the system's.  Every NCCL call is issued on
// the system's stream; the host then waits for the stream while polling
// ncclCommGetAsyncError, and aborts the communicator (SNP_E_NCCL) on an
// asynchronous error or after SNP_DIST_TIMEOUT_S seconds (default 600), so
// a peer that died never hangs the caller.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/snp.h"
#include "snp_comm.h"

namespace snp {
namespace {

double timeout_s() {
  const char* e = getenv("SNP_DIST_TIMEOUT_S");
  return e ? atof(e) : 600.0;
}

// ---------------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    bool all = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        a.why = std::string("NCCL symbol missing: ") + name;
      }
    };
    get(a.GetUniqueId, "ncclGetUniqueId");
    get(a.CommInitRank, "ncclCommInitRank");
    get(a.CommDestroy, "ncclCommDestroy");
    get(a.CommAbort, "ncclCommAbort");
    get(a.CommGetAsyncError, "ncclCommGetAsyncError");
    get(a.AllGather, "ncclAllGather");
    get(a.Send, "ncclSend");
    get(a.Recv, "ncclRecv");
    get(a.GroupStart, "ncclGroupStart");
    get(a.GroupEnd, "ncclGroupEnd");
    get(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    return a;
  }();
  return api;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  bool broken = false;
  int64_t* dscratch = nullptr;
  size_t dcap = 0;
  cudaEvent_t done = nullptr;

  ~NcclComm() override {
    if (done) cudaEventDestroy(done);
    if (dscratch) cudaFree(dscratch);
    if (comm) {
      if (broken) nccl().CommAbort(comm);
      else nccl().CommDestroy(comm);
    }
  }
  const char* kind() const override { return "nccl"; }

  int fail_nccl(ncclResult_t r, const char* what, std::string* err) {
    *err = std::string(what) + ": " + nccl().GetErrorString(r);
    broken = true;
    return SNP_E_NCCL;
  }
  // wait for the stream, watching for asynchronous NCCL errors and a timeout
  int wait(cudaStream_t st, const char* what, std::string* err) {
    if (cudaEventRecord(done, st) != cudaSuccess) {
      *err = std::string(what) + ": cudaEventRecord failed";
      return SNP_E_CUDA;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = timeout_s();
    for (;;) {
      cudaError_t q = cudaEventQuery(done);
      if (q == cudaSuccess) return SNP_OK;
      if (q != cudaErrorNotReady) {
        *err = std::string(what) + ": " + cudaGetErrorString(q);
        return SNP_E_CUDA;
      }
      ncclResult_t a = ncclSuccess;
      nccl().CommGetAsyncError(comm, &a);
      if (a != ncclSuccess && a != ncclInProgress) return fail_nccl(a, what, err);
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
        *err = std::string(what) + ": timed out (SNP_DIST_TIMEOUT_S); communicator aborted";
        broken = true;
        return SNP_E_NCCL;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  int allgather_i64(const int64_t* mine, int n, int64_t* out, cudaStream_t st, std::string* err) override {
    if (broken) { *err = "communicator aborted"; return SNP_E_NCCL; }
    const size_t need = (size_t)P * n * 8;
    if (need > dcap) {
      if (dscratch) cudaFree(dscratch);
      dscratch = nullptr;
      if (cudaMalloc(&dscratch, need) != cudaSuccess) { *err = "allgather scratch"; dcap = 0; return SNP_E_OOM; }
      dcap = need;
    }
    if (cudaMemcpyAsync(dscratch + (size_t)rank * n, mine, (size_t)n * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      *err = "allgather H2D";
      return SNP_E_CUDA;
    }
    ncclResult_t r = nccl().AllGather(dscratch + (size_t)rank * n, dscratch, (size_t)n, ncclInt64, comm, st);
    if (r != ncclSuccess) return fail_nccl(r, "ncclAllGather", err);
    if (cudaMemcpyAsync(out, dscratch, need, cudaMemcpyDeviceToHost, st) != cudaSuccess) {
      *err = "allgather D2H";
      return SNP_E_CUDA;
    }
    return wait(st, "allgather", err);
  }
  int alltoallv(const void* send, const int64_t* sc, void* recv, const int64_t* rc, size_t elem, cudaStream_t st,
                std::string* err) override {
    if (broken) { *err = "communicator aborted"; return SNP_E_NCCL; }
    ncclResult_t r = nccl().GroupStart();
    if (r != ncclSuccess) return fail_nccl(r, "ncclGroupStart", err);
    size_t so = 0, ro = 0;
    for (int q = 0; q < P; ++q) {
      if (sc[q] > 0) {
        r = nccl().Send(static_cast<const uint8_t*>(send) + so * elem, (size_t)sc[q] * elem, ncclUint8, q, comm, st);
        if (r != ncclSuccess) { nccl().GroupEnd(); return fail_nccl(r, "ncclSend", err); }
      }
      if (rc[q] > 0) {
        r = nccl().Recv(static_cast<uint8_t*>(recv) + ro * elem, (size_t)rc[q] * elem, ncclUint8, q, comm, st);
        if (r != ncclSuccess) { nccl().GroupEnd(); return fail_nccl(r, "ncclRecv", err); }
      }
      so += (size_t)sc[q];
      ro += (size_t)rc[q];
    }
    r = nccl().GroupEnd();
    if (r != ncclSuccess) return fail_nccl(r, "ncclGroupEnd", err);
    return wait(st, "alltoallv", err);
  }
};

}  // namespace

int nccl_unique_id(void* out, std::string* err) {
  if (!nccl().ok) { *err = nccl().why; return SNP_E_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) { *err = std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r); return SNP_E_NCCL; }
  static_assert(sizeof(ncclUniqueId) == DIST_ID_BYTES, "NCCL unique id size");
  memcpy(out, &id, sizeof id);
  return SNP_OK;
}

Comm* make_nccl_comm(const void* unique_id, int rank, int P, std::string* err, int* status) {
  *status = SNP_OK;
  if (!nccl().ok) { *err = nccl().why; *status = SNP_E_NCCL; return nullptr; }
  auto* c = new NcclComm();
  c->rank = rank;
  c->P = P;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof id);
  ncclResult_t r = nccl().CommInitRank(&c->comm, P, id, rank);
  if (r != ncclSuccess) {
    *err = std::string("ncclCommInitRank: ") + nccl().GetErrorString(r);
    *status = SNP_E_NCCL;
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  if (cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming) != cudaSuccess) {
    *err = "cudaEventCreate";
    *status = SNP_E_CUDA;
    delete c;
    return nullptr;
  }
  return c;
}

// ---------------------------------------------------------------------------
// in-process group: P ranks = P host threads of one process (one GPU)
// ---------------------------------------------------------------------------
struct LocalGroup {
  int P;
  std::atomic<int> refs{1};
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<std::vector<int64_t>> vals;
  std::vector<const void*> sendp;
  std::vector<std::vector<int64_t>> scounts;
  std::vector<cudaEvent_t> ready;
  explicit LocalGroup(int p) : P(p), vals(p), sendp(p), scounts(p), ready(p, nullptr) {
    for (auto& e : ready) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  ~LocalGroup() {
    for (auto& e : ready)
      if (e) cudaEventDestroy(e);
  }
  // false after SNP_DIST_TIMEOUT_S without every rank arriving
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::duration<double>(timeout_s()), [&] { return gen != g; });
  }
};

LocalGroup* local_group_create(int P) { return new LocalGroup(P); }
int local_group_size(const LocalGroup* g) { return g->P; }
void local_group_release(LocalGroup* g) {
  if (g && --g->refs == 0) delete g;
}

namespace {
struct LocalComm : Comm {
  LocalGroup* g;
  explicit LocalComm(LocalGroup* grp, int r) : g(grp) {
    rank = r;
    P = grp->P;
    g->refs++;
  }
  ~LocalComm() override { local_group_release(g); }
  const char* kind() const override { return "local"; }
  int allgather_i64(const int64_t* mine, int n, int64_t* out, cudaStream_t, std::string* err) override {
    g->vals[rank].assign(mine, mine + n);
    if (!g->barrier()) { *err = "local group: a peer did not arrive (allgather)"; return SNP_E_NCCL; }
    for (int r = 0; r < P; ++r)
      for (int i = 0; i < n; ++i) out[(size_t)r * n + i] = g->vals[r][i];
    if (!g->barrier()) { *err = "local group: a peer did not arrive (allgather)"; return SNP_E_NCCL; }
    return SNP_OK;
  }
  int alltoallv(const void* send, const int64_t* sc, void* recv, const int64_t* rc, size_t elem, cudaStream_t st,
                std::string* err) override {
    g->sendp[rank] = send;
    g->scounts[rank].assign(sc, sc + P);
    if (cudaEventRecord(g->ready[rank], st) != cudaSuccess) { *err = "cudaEventRecord"; return SNP_E_CUDA; }
    if (!g->barrier()) { *err = "local group: a peer did not arrive (alltoallv)"; return SNP_E_NCCL; }
    size_t ro = 0;
    int status = SNP_OK;
    for (int q = 0; q < P && status == SNP_OK; ++q) {
      size_t so = 0;
      for (int k = 0; k < rank; ++k) so += (size_t)g->scounts[q][k];
      if ((int64_t)g->scounts[q][rank] != rc[q]) { *err = "alltoallv: counts disagree"; status = SNP_E_ARG; break; }
      if (rc[q] > 0) {
        if (cudaStreamWaitEvent(st, g->ready[q], 0) != cudaSuccess ||
            cudaMemcpyAsync(static_cast<uint8_t*>(recv) + ro * elem, static_cast<const uint8_t*>(g->sendp[q]) + so * elem,
                            (size_t)rc[q] * elem, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
          *err = "alltoallv copy";
          status = SNP_E_CUDA;
        }
      }
      ro += (size_t)rc[q];
    }
    if (status == SNP_OK && cudaStreamSynchronize(st) != cudaSuccess) { *err = "alltoallv sync"; status = SNP_E_CUDA; }
    if (!g->barrier()) { *err = "local group: a peer did not arrive (alltoallv)"; return SNP_E_NCCL; }
    return status;
  }
};
}  // namespace

Comm* make_local_comm(LocalGroup* g, int rank) { return new LocalComm(g, rank); }

}  // namespace snp
