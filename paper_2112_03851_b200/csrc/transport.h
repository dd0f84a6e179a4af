// Transport seam of libosm: the three inter-rank steps of the Schwarz iteration (
// PAPER.md:157-158 one subdomain block per processor, "inter-subdomain communications").
//
//   exchange(part)   part 1: the [g | u] outbox of every remote side to the partner side's inbox
//                    (2 nG doubles each way); part 2: the right slab's interface-row
//                    residual w (nG doubles) to the owning left slab (a6).
//   allgather_host   per-subdomain values of every rank, in subdomain order (a6's residual partials
//                    and the inner counts; summed in a fixed order on every rank, so h(n) is bitwise
//                    independent of the rank count).
//   reduce_phi       the glued Phi to rank 0 (each lattice point is written by exactly one rank, the
//                    others hold 0: the sum is exact).
//
// Two implementations:
//   NcclTransport  one process per GPU, grouped ncclSend/ncclRecv, ncclAllGather, ncclReduce on the
//                  library stream (the production path across GPUs over NVLink / NVSwitch);
//   HubTransport   ranks are host threads of ONE process (osm_hub): device-to-device copies on the
//                  ranks' streams ordered by CUDA events, host barriers between the phases.  No kernel
//                  ever waits on another rank's kernel (only stream/event dependencies), so several
//                  ranks may share one GPU.  It runs every nranks > 1 branch of the library (plan
//                  offsets, remote sides, allgather offsets, the Phi reduce) without NCCL.
#pragma once
#include <condition_variable>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.h"

namespace osm {

struct Ctx;

struct Transport {
  virtual ~Transport() = default;
  virtual void exchange(Ctx& c, int part) = 0;
  virtual std::vector<double> allgather_host(Ctx& c, const std::vector<double>& local, int width) = 0;
  virtual void reduce_phi(Ctx& c, double* phi, int64_t n) = 0;
  virtual const char* name() const = 0;
};

Transport* make_nccl_transport(Ctx& c, const void* uid128, bool loopback);
Transport* make_hub_transport(Ctx& c, osm_hub* hub);
// Marks the hub of the context whose API call is failing, so that ranks blocked in a hub barrier
// return an error instead of waiting for the failed rank.
void hub_poison_current();
void hub_set_current(osm_hub* hub);

}  // namespace osm
