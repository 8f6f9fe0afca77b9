// snp_comm.h — the exchange layer of multi-GPU exploration:
// the few collectives one BFS level needs, issued by the library itself on the
// system's CUDA stream.  Two transports:
//   * NCCL (one process per GPU; libnccl.so.2 is opened at run time, so the
//     library loads without it) — the product path over NVLink / NVSwitch;
//   * an in-process group (P logical ranks, one host thread and one
//     snp_system each, device-to-device copies) — the same protocol on one
//     GPU, used by the tests and by logical-rank runs.
// Not part of the public ABI (include/snp.h).
#pragma once
#include <cstdint>
#include <cstddef>
#include <string>
#include <cuda_runtime.h>

namespace snp {

struct Comm {
  int rank = 0, P = 1;
  virtual ~Comm() = default;
  // small host values: out[r * n + i] = value i of rank r (every rank gets all)
  virtual int allgather_i64(const int64_t* mine, int n, int64_t* out, cudaStream_t st, std::string* err) = 0;
  // device buffers, counts in elements of `elem` bytes; rank r's rows
  // [Σ_{q<r} send_counts[q], +send_counts[r]) go to rank r and arrive at
  // [Σ_{q<src} recv_counts[q], ...) of recv.  Complete on return.
  virtual int alltoallv(const void* send, const int64_t* send_counts, void* recv, const int64_t* recv_counts,
                        size_t elem, cudaStream_t st, std::string* err) = 0;
  virtual const char* kind() const = 0;
};

// return codes of the Comm calls: 0 ok, else an snp_status (SNP_E_NCCL / SNP_E_CUDA)
Comm* make_nccl_comm(const void* unique_id, int rank, int P, std::string* err, int* status);
int nccl_unique_id(void* out, std::string* err);  // SNP_DIST_ID_BYTES bytes
constexpr int DIST_ID_BYTES = 128;

struct LocalGroup;
LocalGroup* local_group_create(int P);
void local_group_release(LocalGroup* g);     // refcounted: the creator and every rank comm hold one
int local_group_size(const LocalGroup* g);
Comm* make_local_comm(LocalGroup* g, int rank);

}  // namespace snp
