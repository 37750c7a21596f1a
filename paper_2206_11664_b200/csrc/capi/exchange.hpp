// Qubit-remap exchanges between the shards of a state (exchange.cpp).
#pragma once

#include <vector>

#include "../internal.hpp"
#include "../plan/planner.hpp"

namespace sdb {

void nccl_unique_id(unsigned char out[128]);
void nccl_attach(StateImpl& s, const unsigned char id[128]);
void nccl_detach(StateImpl& s);
// stream-ordered barrier over the communicator (a 1-element all-reduce)
void nccl_barrier(StateImpl& s);
// sum of v over all ranks of the state's communicator
double nccl_sum(StateImpl& s, double v);
// all-gather of a small host vector: result[r * size + i] = rank r's local[i]
std::vector<double> nccl_gather(StateImpl& s, const std::vector<double>& local);
// whole-shard copy of rank `partner` into s.xbuf (every rank calls it with its
// own partner; partner(partner(r)) == r), stream-ordered
void nccl_copy_partner(StateImpl& s, int partner);
// Chunk routing of one exchange for `rank` (offsets and counts in amplitudes):
// send B[send_off, +count) to `peer`, receive into A[recv_off, +count);
// peer == rank is a local copy. Both transports use exactly this.
struct Route {
    int peer;
    uint64_t send_off, recv_off, count;
};
std::vector<Route> exchange_routes(int n_local, int n, int rank, const ExchangeSpec& ex);
// B = s.xbuf (already stored through sigma) -> A = s.amps, stream-ordered
void exchange_nccl(StateImpl& s, const ExchangeSpec& ex);
// same routing for shards driven by one process (shards[r] = rank r)
void exchange_local(const std::vector<StateImpl*>& shards, const ExchangeSpec& ex);

}  // namespace sdb
