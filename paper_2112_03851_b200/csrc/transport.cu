// Transport implementations (see transport.h): NCCL across processes, and the in-process hub.
#include <chrono>
#include <cstring>

#include "ctx.h"
#include "transport.h"

#define OSM_NCCL(call)                                                                         \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess) ::osm::fail(OSM_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// ================================================================== in-process hub (C ABI object)
struct osm_hub {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int64_t gen = 0;
  int count = 0;
  bool poisoned = false;
  std::vector<int> joined;  // 1 once rank r has attached a context
  struct Slot {
    std::map<std::pair<int, int>, const double*> out;  // (iface, which) -> outbox of that side
    cudaEvent_t ev_send = nullptr;  // the rank's outboxes / Phi are complete
    cudaEvent_t ev_recv = nullptr;  // the rank's copies out of its peers' buffers are complete
    std::vector<double> host;       // allgather contribution
    double* phi = nullptr;
    int device = -1;
  };
  std::vector<Slot> slot;

  void barrier() {
    std::unique_lock<std::mutex> l(m);
    if (poisoned) osm::fail(OSM_ERR_STATE, "osm_hub: another rank failed");
    const int64_t g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    const bool ok = cv.wait_for(l, std::chrono::seconds(600), [&] { return gen != g || poisoned; });
    if (gen != g) return;
    poisoned = true;
    cv.notify_all();
    osm::fail(OSM_ERR_STATE, ok ? "osm_hub: another rank failed" : "osm_hub: barrier timeout (600 s)");
  }
};

namespace osm {

static thread_local osm_hub* t_cur_hub = nullptr;

void hub_set_current(osm_hub* hub) { t_cur_hub = hub; }

void hub_poison_current() {
  if (!t_cur_hub) return;
  std::lock_guard<std::mutex> l(t_cur_hub->m);
  t_cur_hub->poisoned = true;
  t_cur_hub->cv.notify_all();
}

// ------------------------------------------------------------------ NCCL
struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  bool loopback = false;           // OSM_FORCE_REMOTE: every side talks to its own rank (1-rank comm)
  double* gather_buf = nullptr;    // persistent allgather buffer (device)
  int64_t gather_cap = 0;
  std::vector<double> gather_host;

  ~NcclTransport() override {
    if (gather_buf) cudaFree(gather_buf);
    if (comm) ncclCommDestroy(comm);
  }
  const char* name() const override { return "nccl"; }

  void exchange(Ctx& c, int part) override {
    const int64_t nG = c.nG;
    OSM_NCCL(ncclGroupStart());
    if (loopback) {
      // NCCL matches the j-th send with the j-th receive on the same peer, so each receive is posted
      // into the partner of the j-th sender
      for (const Side& sd : c.sides) {
        if (part == 1) OSM_NCCL(ncclSend(sd.out, 2 * nG, ncclDouble, c.rank, comm, c.stream));
        else if (sd.which == 1) OSM_NCCL(ncclSend(sd.out + 2 * nG, nG, ncclDouble, c.rank, comm, c.stream));
      }
      for (const Side& sd : c.sides) {
        const Side& dst = c.sides[sd.partner];
        if (part == 1) OSM_NCCL(ncclRecv(dst.inbuf, 2 * nG, ncclDouble, c.rank, comm, c.stream));
        else if (sd.which == 1) OSM_NCCL(ncclRecv(dst.inbuf + 2 * nG, nG, ncclDouble, c.rank, comm, c.stream));
      }
    } else {
      for (const Side& sd : c.sides) {
        if (!sd.remote) continue;
        if (part == 1) {
          OSM_NCCL(ncclSend(sd.out, 2 * nG, ncclDouble, sd.peer, comm, c.stream));
          OSM_NCCL(ncclRecv(sd.inbuf, 2 * nG, ncclDouble, sd.peer, comm, c.stream));
        } else if (sd.which == 1) {
          OSM_NCCL(ncclSend(sd.out + 2 * nG, nG, ncclDouble, sd.peer, comm, c.stream));
        } else {
          OSM_NCCL(ncclRecv(sd.inbuf + 2 * nG, nG, ncclDouble, sd.peer, comm, c.stream));
        }
      }
    }
    OSM_NCCL(ncclGroupEnd());
  }

  std::vector<double> allgather_host(Ctx& c, const std::vector<double>& local, int width) override {
    const int nloc = c.s_end - c.s_begin;
    const int64_t total = (int64_t)c.nsub * width;
    if (total > gather_cap) {
      if (gather_buf) OSM_CUDA(cudaFree(gather_buf));
      gather_buf = nullptr;
      OSM_CUDA(cudaMalloc((void**)&gather_buf, sizeof(double) * total));
      gather_cap = total;
    }
    double* d = gather_buf;
    OSM_CUDA(cudaMemcpyAsync(d + (int64_t)c.s_begin * width, local.data(), sizeof(double) * nloc * width,
                             cudaMemcpyHostToDevice, c.stream));
    OSM_NCCL(ncclAllGather(d + (int64_t)c.s_begin * width, d, (size_t)nloc * width, ncclDouble, comm, c.stream));
    std::vector<double> all((size_t)total);
    OSM_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(double) * total, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    return all;
  }

  void reduce_phi(Ctx& c, double* phi, int64_t n) override {
    if (c.nranks > 1) OSM_NCCL(ncclReduce(phi, phi, n, ncclDouble, ncclSum, 0, comm, c.stream));
  }
};

Transport* make_nccl_transport(Ctx& c, const void* uid128, bool loopback) {
  auto* t = new NcclTransport();
  try {
    ncclUniqueId id;
    if (uid128) std::memcpy(&id, uid128, sizeof(id));
    else OSM_NCCL(ncclGetUniqueId(&id));
    OSM_NCCL(ncclCommInitRank(&t->comm, loopback ? 1 : c.nranks, id, loopback ? 0 : c.rank));
    t->loopback = loopback;
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

// ------------------------------------------------------------------ hub
__global__ void k_add_into(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

struct HubTransport : Transport {
  osm_hub* hub = nullptr;
  int rank = 0;
  double* stage = nullptr;  // rank 0: staging buffer for the Phi reduce
  int64_t stage_cap = 0;

  ~HubTransport() override {
    if (stage) cudaFree(stage);
    if (hub) {
      std::lock_guard<std::mutex> l(hub->m);
      auto& s = hub->slot[rank];
      if (s.ev_send) cudaEventDestroy(s.ev_send);
      if (s.ev_recv) cudaEventDestroy(s.ev_recv);
      s.ev_send = s.ev_recv = nullptr;
      hub->joined[rank] = 0;
    }
  }
  const char* name() const override { return "hub"; }

  void exchange(Ctx& c, int part) override {
    const int64_t nG = c.nG;
    osm_hub::Slot& me = hub->slot[rank];
    me.out.clear();
    for (const Side& sd : c.sides)
      if (sd.remote) me.out[{sd.iface, sd.which}] = sd.out;
    OSM_CUDA(cudaEventRecord(me.ev_send, c.stream));
    hub->barrier();  // every rank's outboxes are published (pointers) and recorded (events)
    std::vector<int> peers;
    for (const Side& sd : c.sides) {
      if (!sd.remote) continue;
      osm_hub::Slot& ps = hub->slot[sd.peer];
      auto it = ps.out.find({sd.iface, 1 - sd.which});
      if (it == ps.out.end()) fail(OSM_ERR_STATE, "osm_hub: partner side not found on the peer rank");
      OSM_CUDA(cudaStreamWaitEvent(c.stream, ps.ev_send, 0));
      if (part == 1) {
        OSM_CUDA(cudaMemcpyAsync(sd.inbuf, it->second, sizeof(double) * 2 * nG, cudaMemcpyDefault, c.stream));
      } else if (sd.which == 0) {
        OSM_CUDA(cudaMemcpyAsync(sd.inbuf + 2 * nG, it->second + 2 * nG, sizeof(double) * nG, cudaMemcpyDefault,
                                 c.stream));
      }
      peers.push_back(sd.peer);
    }
    OSM_CUDA(cudaEventRecord(me.ev_recv, c.stream));
    hub->barrier();  // every rank has enqueued its copies
    // a rank may overwrite its outboxes only after its peers' copies out of them are done
    for (int p : peers) OSM_CUDA(cudaStreamWaitEvent(c.stream, hub->slot[p].ev_recv, 0));
  }

  std::vector<double> allgather_host(Ctx& c, const std::vector<double>& local, int width) override {
    hub->slot[rank].host = local;
    hub->barrier();
    std::vector<double> all;
    all.reserve((size_t)c.nsub * width);
    for (int r = 0; r < hub->n; ++r) all.insert(all.end(), hub->slot[r].host.begin(), hub->slot[r].host.end());
    hub->barrier();  // nobody rewrites its contribution before everyone has read it
    if ((int64_t)all.size() != (int64_t)c.nsub * width) fail(OSM_ERR_STATE, "osm_hub: allgather size mismatch");
    return all;
  }

  void reduce_phi(Ctx& c, double* phi, int64_t n) override {
    osm_hub::Slot& me = hub->slot[rank];
    me.phi = phi;
    OSM_CUDA(cudaEventRecord(me.ev_send, c.stream));
    hub->barrier();
    if (rank == 0) {
      if (n > stage_cap) {
        if (stage) OSM_CUDA(cudaFree(stage));
        stage = nullptr;
        OSM_CUDA(cudaMalloc((void**)&stage, sizeof(double) * n));
        stage_cap = n;
      }
      for (int r = 1; r < hub->n; ++r) {  // rank order; every point has one nonzero contribution
        OSM_CUDA(cudaStreamWaitEvent(c.stream, hub->slot[r].ev_send, 0));
        OSM_CUDA(cudaMemcpyAsync(stage, hub->slot[r].phi, sizeof(double) * n, cudaMemcpyDefault, c.stream));
        k_add_into<<<4 * 148, 256, 0, c.stream>>>(phi, stage, n);
        OSM_CHECK_LAUNCH();
      }
    }
    OSM_CUDA(cudaEventRecord(me.ev_recv, c.stream));
    hub->barrier();
    if (rank != 0) OSM_CUDA(cudaStreamWaitEvent(c.stream, hub->slot[0].ev_recv, 0));
  }
};

Transport* make_hub_transport(Ctx& c, osm_hub* hub) {
  if (hub->n != c.nranks) fail(OSM_ERR_INVALID_ARG, "osm_hub created for a different rank count");
  {
    std::lock_guard<std::mutex> l(hub->m);
    if (hub->joined[c.rank]) fail(OSM_ERR_INVALID_ARG, "osm_hub: rank already attached");
    hub->joined[c.rank] = 1;
  }
  auto* t = new HubTransport();
  t->hub = hub;
  t->rank = c.rank;
  osm_hub::Slot& s = hub->slot[c.rank];
  s.device = c.device;
  OSM_CUDA(cudaEventCreateWithFlags(&s.ev_send, cudaEventDisableTiming));
  OSM_CUDA(cudaEventCreateWithFlags(&s.ev_recv, cudaEventDisableTiming));
  return t;
}

}  // namespace osm

// ================================================================== C ABI of the hub
namespace osm {
extern thread_local std::string g_last_error;
}
using osm::g_last_error;

extern "C" {

osm_status osm_hub_create(int nranks, osm_hub** out) {
  if (!out || nranks < 1) {
    g_last_error = "osm_hub_create: bad arguments";
    return OSM_ERR_INVALID_ARG;
  }
  auto* h = new osm_hub();
  h->n = nranks;
  h->slot.resize(nranks);
  h->joined.assign(nranks, 0);
  *out = h;
  return OSM_OK;
}

void osm_hub_destroy(osm_hub* h) { delete h; }

}  // extern "C"
