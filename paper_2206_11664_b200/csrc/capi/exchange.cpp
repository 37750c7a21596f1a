// Qubit-remap exchanges of a sharded state (planner.hpp
// ExchangeSpec). The pass in front of an exchange has already stored this
// rank's shard through sigma into the exchange buffer B (s.xbuf), so the top
// g' local bits T hold the qubits that leave. Rank r then, for every chunk
// index c of those bits, sends B[c] to the peer whose swapped global bits are
// c and receives that peer's chunk into A[c] (A = s.amps); c == own bits is a
// device-local copy. Two transports share this routing:
//   * NCCL (one process per GPU): grouped ncclSend/ncclRecv on the state's
//     stream. libnccl.so.2 is resolved at run time (dlopen, reusing the copy
//     torch has already loaded) so the library has no link-time NCCL
//     dependency and single-GPU users never need it;
//   * local (several shards driven by one process, e.g. virtual shards on one
//     GPU for tests): cudaMemcpyPeerAsync between the shards' buffers.
#include <cuda_runtime_api.h>
#include <dlfcn.h>
#include <nccl.h>

#include <bit>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "exchange.hpp"

namespace sdb {

namespace {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) err = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(api.getUniqueId, "ncclGetUniqueId");
        sym(api.commInitRank, "ncclCommInitRank");
        sym(api.commDestroy, "ncclCommDestroy");
        sym(api.groupStart, "ncclGroupStart");
        sym(api.groupEnd, "ncclGroupEnd");
        sym(api.send, "ncclSend");
        sym(api.recv, "ncclRecv");
        sym(api.allReduce, "ncclAllReduce");
        sym(api.allGather, "ncclAllGather");
        sym(api.errorString, "ncclGetErrorString");
    });
    if (!err.empty()) throw NcclError(err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const NcclApi& a = nccl();
        throw NcclError(std::string(what) + ": " + a.errorString(r));
    }
}

uint64_t with_bits(uint64_t r, int n_local, const ExchangeSpec& ex, uint32_t c) {
    for (size_t i = 0; i < ex.swaps.size(); ++i) {
        const uint64_t b = 1ull << (ex.swaps[i].first - n_local);
        r = ((c >> i) & 1u) ? (r | b) : (r & ~b);
    }
    return r;
}

void check_spec(int n_local, int n, const ExchangeSpec& ex) {
    const int gp = static_cast<int>(ex.swaps.size());
    if (gp < 1 || gp > n - n_local) throw std::invalid_argument("exchange: bad number of swapped bits");
    for (int i = 0; i < gp; ++i) {
        if (ex.swaps[i].second != n_local - gp + i || ex.swaps[i].first < n_local || ex.swaps[i].first >= n) {
            throw std::invalid_argument("exchange: swaps must pair global bits with the top local bits");
        }
    }
}

}  // namespace

std::vector<Route> exchange_routes(int n_local, int n, int rank, const ExchangeSpec& ex) {
    check_spec(n_local, n, ex);
    const int gp = static_cast<int>(ex.swaps.size());
    const uint64_t chunk = uint64_t(1) << (n_local - gp);
    std::vector<Route> out;
    for (uint32_t c = 0; c < (1u << gp); ++c) {
        const int peer = static_cast<int>(with_bits(static_cast<uint64_t>(rank), n_local, ex, c));
        // the peer holds our chunk c after the swap at our swapped bits; we
        // receive its chunk (its swapped bits = c) into A[c]
        out.push_back({peer, chunk * c, chunk * c, chunk});
    }
    return out;
}

void nccl_unique_id(unsigned char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

void nccl_attach(StateImpl& s, const unsigned char id[128]) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    SDB_CUDA(cudaSetDevice(s.device));
    ncclComm_t comm = nullptr;
    nccl_check(nccl().commInitRank(&comm, s.world, uid, s.rank), "ncclCommInitRank");
    if (s.nccl) nccl().commDestroy(static_cast<ncclComm_t>(s.nccl));
    s.nccl = comm;
    if (!s.reduce_buf) SDB_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.reduce_buf), 148 * 16 * 16));
}

void nccl_detach(StateImpl& s) {
    if (s.nccl) {
        nccl().commDestroy(static_cast<ncclComm_t>(s.nccl));
        s.nccl = nullptr;
    }
}

void nccl_barrier(StateImpl& s) {
    if (!s.nccl) throw std::runtime_error("sharded state has no communicator (sd_state_attach_comm)");
    nccl_check(nccl().allReduce(s.reduce_buf, s.reduce_buf, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(s.nccl),
                                s.stream),
               "ncclAllReduce");
}

double nccl_sum(StateImpl& s, double v) {
    if (!s.nccl) throw std::runtime_error("sharded state has no communicator (sd_state_attach_comm)");
    double* d = s.reduce_buf;
    SDB_CUDA(cudaMemcpyAsync(d, &v, sizeof(double), cudaMemcpyHostToDevice, s.stream));
    nccl_check(nccl().allReduce(d, d, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(s.nccl), s.stream),
               "ncclAllReduce");
    SDB_CUDA(cudaMemcpyAsync(&v, d, sizeof(double), cudaMemcpyDeviceToHost, s.stream));
    SDB_CUDA(cudaStreamSynchronize(s.stream));
    return v;
}

std::vector<double> nccl_gather(StateImpl& s, const std::vector<double>& local) {
    if (!s.nccl) throw std::runtime_error("sharded state has no communicator (sd_state_attach_comm)");
    const size_t m = local.size();
    std::vector<double> out(m * static_cast<size_t>(s.world));
    if (m == 0) return out;
    double* d = nullptr;
    SDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(double) * m * (1 + s.world), s.stream));
    SDB_CUDA(cudaMemcpyAsync(d, local.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s.stream));
    nccl_check(nccl().allGather(d, d + m, m, ncclDouble, static_cast<ncclComm_t>(s.nccl), s.stream), "ncclAllGather");
    SDB_CUDA(cudaMemcpyAsync(out.data(), d + m, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, s.stream));
    SDB_CUDA(cudaFreeAsync(d, s.stream));
    SDB_CUDA(cudaStreamSynchronize(s.stream));
    return out;
}

void nccl_copy_partner(StateImpl& s, int partner) {
    if (!s.nccl) throw std::runtime_error("sharded state has no communicator (sd_state_attach_comm)");
    if (!s.xbuf) throw std::logic_error("partner copy needs the exchange buffer");
    const NcclApi& a = nccl();
    auto comm = static_cast<ncclComm_t>(s.nccl);
    const size_t count = 2 * s.amps_count();
    nccl_check(a.groupStart(), "ncclGroupStart");
    nccl_check(a.send(s.amps, count, ncclDouble, partner, comm, s.stream), "ncclSend");
    nccl_check(a.recv(s.xbuf, count, ncclDouble, partner, comm, s.stream), "ncclRecv");
    nccl_check(a.groupEnd(), "ncclGroupEnd");
}

void exchange_nccl(StateImpl& s, const ExchangeSpec& ex) {
    if (!s.nccl) throw std::runtime_error("sharded state has no communicator (sd_state_attach_comm)");
    const std::vector<Route> routes = exchange_routes(s.n_local, s.n, s.rank, ex);
    const NcclApi& a = nccl();
    auto comm = static_cast<ncclComm_t>(s.nccl);
    nccl_check(a.groupStart(), "ncclGroupStart");
    for (const Route& rt : routes) {
        if (rt.peer == s.rank) continue;
        nccl_check(a.send(s.xbuf + 2 * rt.send_off, 2 * rt.count, ncclDouble, rt.peer, comm, s.stream), "ncclSend");
        nccl_check(a.recv(s.amps + 2 * rt.recv_off, 2 * rt.count, ncclDouble, rt.peer, comm, s.stream), "ncclRecv");
    }
    nccl_check(a.groupEnd(), "ncclGroupEnd");
    for (const Route& rt : routes) {
        if (rt.peer != s.rank) continue;
        SDB_CUDA(cudaMemcpyAsync(s.amps + 2 * rt.recv_off, s.xbuf + 2 * rt.send_off, 16 * rt.count,
                                 cudaMemcpyDeviceToDevice, s.stream));
    }
}

void exchange_local(const std::vector<StateImpl*>& shards, const ExchangeSpec& ex) {
    const int world = static_cast<int>(shards.size());
    for (StateImpl* s : shards) {
        SDB_CUDA(cudaSetDevice(s->device));
        SDB_CUDA(cudaStreamSynchronize(s->stream));
    }
    for (int r = 0; r < world; ++r) {
        StateImpl& dst = *shards[r];
        // rank r receives, for each route, the peer's chunk destined for it
        for (const Route& rt : exchange_routes(dst.n_local, dst.n, r, ex)) {
            StateImpl& src = *shards[rt.peer];
            // the peer's matching route towards r names the chunk it sends
            uint64_t peer_send = 0;
            for (const Route& pr : exchange_routes(src.n_local, src.n, rt.peer, ex)) {
                if (pr.peer == r) peer_send = pr.send_off;
            }
            SDB_CUDA(cudaSetDevice(dst.device));
            SDB_CUDA(cudaMemcpyPeerAsync(dst.amps + 2 * rt.recv_off, dst.device, src.xbuf + 2 * peer_send, src.device,
                                         16 * rt.count, dst.stream));
        }
    }
    for (StateImpl* s : shards) {
        SDB_CUDA(cudaSetDevice(s->device));
        SDB_CUDA(cudaStreamSynchronize(s->stream));
    }
}

}  // namespace sdb
