// comm.cu — the collectives of the row-partitioned path.
//
// The Krylov path needs three exchanges ("transparently on one or more GPU accelerators"):
//   * the halo of every SpMM: owners send the rows of y that other ranks' nonzeros reference
//     (grouped point-to-point, comm_sendrecv);
//   * the allreduce of every Gram pass, so H and every coefficient are bit-identical on all ranks
//     (comm_allreduce);
//   * small host exchanges while the operator is built: row ranges, halo request counts and ids
//     (comm_allgather_host, comm_alltoallv_host).
// Two transports implement them behind the same calls:
//   * NCCL, one process per GPU (wl_comm_create): ncclSend/ncclRecv in a group, ncclAllReduce;
//   * loopback (wl_loopback_create + wl_comm_create_loopback): P ranks in ONE process on one
//     device, one host thread per rank.  Each collective is a two-barrier rendezvous: ranks publish
//     their buffers and a "ready" event, then every receiver enqueues waits on the senders' events
//     and device-to-device copies (or the fixed-order sum of the P buffers for the allreduce) on
//     its own stream, and records a "done" event that every rank waits on before it may overwrite
//     a published buffer.  The stream semantics are NCCL's: the call is stream-ordered and returns
//     before the data moved.  This drives the multi-rank code path (pack_rows, the HALO SpMM
//     instantiations, the halo id plan, replicated coefficients) on a single GPU for testing.
#include "walklap.h"
#include "wl_internal.cuh"

#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

struct wl_loopback {
  int P = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  int refs = 0;                                  // comms attached
  std::vector<wl_comm*> ranks;                   // rank -> comm (events, scratch)
  std::vector<const void*> send_ptr;             // [src * P + dst]
  std::vector<size_t> send_bytes;                // [src * P + dst]
  std::vector<const double*> red_ptr;            // [rank] allreduce input
  std::vector<const int64_t*> host_ptr;          // [src * P + dst] host payloads
  std::vector<size_t> host_cnt;                  // [src * P + dst]
  double timeout_s = 600.0;

  // generation barrier; a timeout (a rank died or skipped a collective) breaks the group for good
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) throw wl::Error(WL_ENCCL, "loopback group broken by an earlier timeout");
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      throw wl::Error(WL_ENCCL, "loopback collective timed out (a rank did not join)");
    }
  }
};

#define WL_NCCL(x)                                                                                     \
  do {                                                                                                 \
    ncclResult_t r_ = (x);                                                                             \
    if (r_ != ncclSuccess) throw ::wl::Error(WL_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

namespace wl {
namespace {

inline ncclComm_t nc(const wl_comm* c) { return reinterpret_cast<ncclComm_t>(c->nccl); }

// device scratch of a loopback rank (allreduce sums), grown on demand
double* scratch(wl_comm* c, size_t count) {
  if (c->scratch_n < count) {
    if (c->scratch) cudaFree(c->scratch);
    c->scratch = nullptr;
    c->scratch_n = 0;
    WL_CUDA(cudaMalloc(&c->scratch, sizeof(double) * count));
    c->scratch_n = count;
  }
  return c->scratch;
}

}  // namespace

void comm_allreduce(wl_comm* c, double* buf, size_t count, cudaStream_t s) {
  if (!c || c->nranks <= 1 || count == 0) return;
  if (!c->lb) {
    WL_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, nc(c), s));
    return;
  }
  wl_loopback* g = c->lb;
  const int P = g->P, me = c->rank;
  double* tmp = scratch(c, count);
  WL_CUDA(cudaEventRecord(c->ev_ready, s));
  g->red_ptr[me] = buf;
  g->barrier();  // every rank's buffer and ready event are published
  SumSrc src{};
  for (int p = 0; p < P; ++p) {
    WL_CUDA(cudaStreamWaitEvent(s, g->ranks[p]->ev_ready, 0));
    src.p[p] = g->red_ptr[p];
  }
  sum_ranks(src, P, (int64_t)count, tmp, s);  // fixed rank order: identical bits on every rank
  WL_CUDA(cudaEventRecord(c->ev_done, s));
  g->barrier();  // every rank has enqueued its reads of the published buffers
  for (int p = 0; p < P; ++p) WL_CUDA(cudaStreamWaitEvent(s, g->ranks[p]->ev_done, 0));
  WL_CUDA(cudaMemcpyAsync(buf, tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
}

void comm_sendrecv(wl_comm* c, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) {
  if (!c || c->nranks <= 1) return;
  if (!c->lb) {
    WL_NCCL(ncclGroupStart());
    for (const Xfer& x : sends)
      if (x.bytes) WL_NCCL(ncclSend(x.ptr, x.bytes, ncclUint8, x.peer, nc(c), s));
    for (const Xfer& x : recvs)
      if (x.bytes) WL_NCCL(ncclRecv(x.ptr, x.bytes, ncclUint8, x.peer, nc(c), s));
    WL_NCCL(ncclGroupEnd());
    return;
  }
  wl_loopback* g = c->lb;
  const int P = g->P, me = c->rank;
  WL_CUDA(cudaEventRecord(c->ev_ready, s));
  for (int p = 0; p < P; ++p) {
    g->send_ptr[(size_t)me * P + p] = nullptr;
    g->send_bytes[(size_t)me * P + p] = 0;
  }
  for (const Xfer& x : sends) {
    g->send_ptr[(size_t)me * P + x.peer] = x.ptr;
    g->send_bytes[(size_t)me * P + x.peer] = x.bytes;
  }
  g->barrier();
  for (const Xfer& x : recvs) {
    if (!x.bytes) continue;
    const size_t k = (size_t)x.peer * P + me;
    if (g->send_bytes[k] != x.bytes) throw Error(WL_ENCCL, "loopback send/recv size mismatch");
    WL_CUDA(cudaStreamWaitEvent(s, g->ranks[x.peer]->ev_ready, 0));
    WL_CUDA(cudaMemcpyAsync(x.ptr, g->send_ptr[k], x.bytes, cudaMemcpyDeviceToDevice, s));
  }
  WL_CUDA(cudaEventRecord(c->ev_done, s));
  g->barrier();
  for (int p = 0; p < P; ++p) WL_CUDA(cudaStreamWaitEvent(s, g->ranks[p]->ev_done, 0));
}

// host int64 exchanges (operator build time; synchronous)
void comm_alltoallv_host(wl_comm* c, const std::vector<std::vector<int64_t>>& send,
                         std::vector<std::vector<int64_t>>& recv, cudaStream_t s) {
  const int P = c->nranks, me = c->rank;
  recv.assign(P, {});
  if (c->lb) {
    wl_loopback* g = c->lb;
    for (int p = 0; p < P; ++p) {
      g->host_ptr[(size_t)me * P + p] = send[p].data();
      g->host_cnt[(size_t)me * P + p] = send[p].size();
    }
    g->barrier();
    for (int p = 0; p < P; ++p) {
      const size_t k = (size_t)p * P + me;
      recv[p].assign(g->host_ptr[k], g->host_ptr[k] + g->host_cnt[k]);
    }
    g->barrier();  // senders' vectors stay alive until every rank copied
    return;
  }
  // NCCL: counts first, then the payloads, staged through device memory
  std::vector<int64_t> cnt_s(P), cnt_r(P);
  for (int p = 0; p < P; ++p) cnt_s[p] = (int64_t)send[p].size();
  int64_t *dcs = nullptr, *dcr = nullptr;
  WL_CUDA(cudaMalloc(&dcs, sizeof(int64_t) * P));
  WL_CUDA(cudaMalloc(&dcr, sizeof(int64_t) * P));
  std::unique_ptr<int64_t, decltype(&cudaFree)> g1(dcs, cudaFree), g2(dcr, cudaFree);
  WL_CUDA(cudaMemcpy(dcs, cnt_s.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice));
  WL_NCCL(ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    WL_NCCL(ncclSend(dcs + p, 1, ncclInt64, p, nc(c), s));
    WL_NCCL(ncclRecv(dcr + p, 1, ncclInt64, p, nc(c), s));
  }
  WL_NCCL(ncclGroupEnd());
  WL_CUDA(cudaStreamSynchronize(s));
  WL_CUDA(cudaMemcpy(cnt_r.data(), dcr, sizeof(int64_t) * P, cudaMemcpyDeviceToHost));
  int64_t ns = 0, nr = 0;
  std::vector<int64_t> ds(P), dr(P);
  for (int p = 0; p < P; ++p) {
    ds[p] = ns;
    dr[p] = nr;
    ns += cnt_s[p];
    nr += cnt_r[p];
  }
  int64_t *bs = nullptr, *br = nullptr;
  WL_CUDA(cudaMalloc(&bs, sizeof(int64_t) * std::max<int64_t>(1, ns)));
  WL_CUDA(cudaMalloc(&br, sizeof(int64_t) * std::max<int64_t>(1, nr)));
  std::unique_ptr<int64_t, decltype(&cudaFree)> g3(bs, cudaFree), g4(br, cudaFree);
  for (int p = 0; p < P; ++p)
    if (cnt_s[p]) WL_CUDA(cudaMemcpy(bs + ds[p], send[p].data(), sizeof(int64_t) * cnt_s[p], cudaMemcpyHostToDevice));
  WL_NCCL(ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    if (cnt_s[p]) WL_NCCL(ncclSend(bs + ds[p], (size_t)cnt_s[p], ncclInt64, p, nc(c), s));
    if (cnt_r[p]) WL_NCCL(ncclRecv(br + dr[p], (size_t)cnt_r[p], ncclInt64, p, nc(c), s));
  }
  WL_NCCL(ncclGroupEnd());
  WL_CUDA(cudaStreamSynchronize(s));
  for (int p = 0; p < P; ++p) {
    recv[p].resize((size_t)cnt_r[p]);
    if (cnt_r[p]) WL_CUDA(cudaMemcpy(recv[p].data(), br + dr[p], sizeof(int64_t) * cnt_r[p], cudaMemcpyDeviceToHost));
  }
}

void comm_allgather_host(wl_comm* c, const std::vector<int64_t>& mine, std::vector<std::vector<int64_t>>& all,
                         cudaStream_t s) {
  std::vector<std::vector<int64_t>> send(c->nranks, mine);
  comm_alltoallv_host(c, send, all, s);
}

void comm_barrier_host(wl_comm* c) {
  if (c && c->lb) c->lb->barrier();
}

}  // namespace wl

using namespace wl;

extern "C" {

wl_status wl_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) throw Error(WL_EINVAL, "out128 is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    WL_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, 128);
  });
}

wl_status wl_comm_create(int32_t nranks, int32_t rank, const void* id128, int32_t device, wl_comm** out) {
  return guarded([&] {
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) throw Error(WL_EINVAL, "bad comm args");
    WL_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<wl_comm>();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t nccl = nullptr;
    WL_NCCL(ncclCommInitRank(&nccl, nranks, id, rank));
    c->nccl = nccl;
    *out = c.release();
  });
}

wl_status wl_loopback_create(int32_t nranks, wl_loopback** out) {
  return guarded([&] {
    if (!out || nranks < 1 || nranks > kMaxRanks) throw Error(WL_EINVAL, "nranks must be in [1, 64]");
    auto g = std::make_unique<wl_loopback>();
    g->P = nranks;
    g->ranks.assign(nranks, nullptr);
    g->send_ptr.assign((size_t)nranks * nranks, nullptr);
    g->send_bytes.assign((size_t)nranks * nranks, 0);
    g->red_ptr.assign(nranks, nullptr);
    g->host_ptr.assign((size_t)nranks * nranks, nullptr);
    g->host_cnt.assign((size_t)nranks * nranks, 0);
    *out = g.release();
  });
}

wl_status wl_loopback_set_timeout(wl_loopback* g, double seconds) {
  return guarded([&] {
    if (!g || !(seconds > 0.0)) throw Error(WL_EINVAL, "bad timeout");
    std::lock_guard<std::mutex> lk(g->m);
    g->timeout_s = seconds;
  });
}

void wl_loopback_destroy(wl_loopback* g) { delete g; }

wl_status wl_comm_create_loopback(wl_loopback* g, int32_t rank, int32_t device, wl_comm** out) {
  return guarded([&] {
    if (!g || !out || rank < 0 || rank >= g->P) throw Error(WL_EINVAL, "bad loopback comm args");
    WL_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<wl_comm>();
    c->nranks = g->P;
    c->rank = rank;
    c->device = device;
    c->lb = g;
    WL_CUDA(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
    WL_CUDA(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    {
      std::lock_guard<std::mutex> lk(g->m);
      if (g->ranks[rank]) throw Error(WL_EINVAL, "loopback rank already attached");
      g->ranks[rank] = c.get();
      g->refs++;
    }
    *out = c.release();
  });
}

void wl_comm_destroy(wl_comm* c) {
  if (!c) return;
  if (c->nccl) ncclCommDestroy(reinterpret_cast<ncclComm_t>(c->nccl));
  if (c->lb) {
    std::lock_guard<std::mutex> lk(c->lb->m);
    c->lb->ranks[c->rank] = nullptr;
    c->lb->refs--;
  }
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->scratch) cudaFree(c->scratch);
  delete c;
}

}  // extern "C"
