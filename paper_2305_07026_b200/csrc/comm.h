// comm.h — the two exchange steps of a DABA iteration across ranks.
//   halo exchange : boundary x^k to the neighbours that read it (Alg. 1);
//   allreduce     : one vector of rank-local sums (F(x^k), the E(x_acc|x^k) parts, ...) for the global
//                   restart test (reading D2; Lemma 1(a)).
// Backends: NCCL (one process per GPU; loaded with dlopen so single-GPU use needs no NCCL), and LOCAL (ranks are
// host threads of one process sharing a hub; no device-side waiting, used by tests to run several ranks on one
// GPU).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace daba {

struct PeerSeg {
  int rank;
  int64_t send_off, send_cnt;  // doubles in this rank's send buffer
  int64_t recv_off, recv_cnt;  // doubles in this rank's recv buffer
};

class Comm {
 public:
  virtual ~Comm() {}
  // sum n doubles across ranks (device pointers), result on every rank
  virtual std::string allreduce(const double* d_in, double* d_out, int n, cudaStream_t st) = 0;
  virtual std::string exchange(const double* d_send, double* d_recv, const std::vector<PeerSeg>& segs,
                               cudaStream_t st) = 0;
  // the allreduce and the exchange issued together (one NCCL group: the transfers overlap)
  virtual std::string allreduce_exchange(const double* d_in, double* d_out, int n, const double* d_send,
                                         double* d_recv, const std::vector<PeerSeg>& segs, cudaStream_t st) {
    std::string e = allreduce(d_in, d_out, n, st);
    if (!e.empty() || segs.empty()) return e;
    return exchange(d_send, d_recv, segs, st);
  }
  virtual bool capturable() const = 0;
};

// Create a communicator.  kind: 0 NCCL, 1 LOCAL, 2 NONE (measurement only: no peers; see include/daba.h).
// id: 128 bytes.  Returns nullptr and sets *err on failure.
Comm* make_comm(int kind, const void* id, int rank, int nranks, std::string* err);
// ncclGetUniqueId through the dynamically loaded library.
std::string nccl_unique_id(void* id_out);

}  // namespace daba
