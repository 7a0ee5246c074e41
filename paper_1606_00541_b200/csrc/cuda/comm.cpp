// Comm backends (see comm.hpp).

#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "device_runtime.hpp"

namespace hec::dev {

namespace {

// libnccl entry points, resolved at first use. If the process already holds a
// libnccl.so.2 (torch loads its own), dlopen returns that copy.
struct NcclApi {
    ncclResult_t (*GetVersion)(int*) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("cannot open libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            if (!f) api.why = std::string("libnccl lacks ") + name;
            return f != nullptr;
        };
        api.ok = sym(api.GetVersion, "ncclGetVersion") && sym(api.GetUniqueId, "ncclGetUniqueId") &&
                 sym(api.CommInitRank, "ncclCommInitRank") && sym(api.CommDestroy, "ncclCommDestroy") &&
                 sym(api.AllReduce, "ncclAllReduce") && sym(api.Send, "ncclSend") && sym(api.Recv, "ncclRecv") &&
                 sym(api.GroupStart, "ncclGroupStart") && sym(api.GroupEnd, "ncclGroupEnd") &&
                 sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!api.ok) throw std::runtime_error("hecsolve-b200: NCCL unavailable (" + api.why + ")");
    return api;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
}

}  // namespace

int nccl_version() {
    try {
        int v = 0;
        check(nccl().GetVersion(&v), "ncclGetVersion");
        return v;
    } catch (const std::exception&) {
        return 0;
    }
}

void nccl_unique_id(unsigned char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

NcclComm::NcclComm(const unsigned char* unique_id, int rank, int world) : rank_(rank), world_(world) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("NcclComm: bad rank / world");
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t c = nullptr;
    check(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank");
    comm_ = c;
}

NcclComm::~NcclComm() {
    if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::allreduce_sum(double* dev, int count, cudaStream_t st) {
    if (count == 0) return;  // (a one-rank communicator still runs the collective: tests the plumbing)
    ++allreduces;
    check(nccl().AllReduce(dev, dev, static_cast<size_t>(count), ncclDouble, ncclSum,
                           static_cast<ncclComm_t>(comm_), st),
          "ncclAllReduce");
}

void NcclComm::exchange(const double* send_dev, const std::vector<int>& send_off, double* recv_dev,
                        const std::vector<int>& recv_off, cudaStream_t st) {
    ++exchanges;
    const NcclApi& N = nccl();
    check(N.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < world_; ++p) {
        if (p == rank_) continue;
        const int ns = send_off[p + 1] - send_off[p], nr = recv_off[p + 1] - recv_off[p];
        if (ns) check(N.Send(send_dev + send_off[p], ns, ncclDouble, p, static_cast<ncclComm_t>(comm_), st), "ncclSend");
        if (nr) check(N.Recv(recv_dev + recv_off[p], nr, ncclDouble, p, static_cast<ncclComm_t>(comm_), st), "ncclRecv");
    }
    check(N.GroupEnd(), "ncclGroupEnd");
}

void CallbackComm::allreduce_sum(double* dev, int count, cudaStream_t st) {
    if (world_ == 1 || count == 0) return;
    ++allreduces;
    hs_.resize(static_cast<size_t>(count));
    HEC_CUDA(cudaMemcpyAsync(hs_.data(), dev, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    HEC_CUDA(cudaStreamSynchronize(st));
    if (cb_.allreduce_sum(cb_.ctx, hs_.data(), count) != 0) throw std::runtime_error("comm callback: allreduce failed");
    HEC_CUDA(cudaMemcpyAsync(dev, hs_.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
    HEC_CUDA(cudaStreamSynchronize(st));
}

void CallbackComm::exchange(const double* send_dev, const std::vector<int>& send_off, double* recv_dev,
                            const std::vector<int>& recv_off, cudaStream_t st) {
    if (world_ == 1) return;
    ++exchanges;
    const int ns = send_off.back(), nr = recv_off.back();
    hs_.resize(static_cast<size_t>(std::max(ns, 1)));
    hr_.resize(static_cast<size_t>(std::max(nr, 1)));
    if (ns) HEC_CUDA(cudaMemcpyAsync(hs_.data(), send_dev, sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
    HEC_CUDA(cudaStreamSynchronize(st));
    if (cb_.exchange(cb_.ctx, hs_.data(), ns, hr_.data(), nr) != 0) throw std::runtime_error("comm callback: exchange failed");
    if (nr) HEC_CUDA(cudaMemcpyAsync(recv_dev, hr_.data(), sizeof(double) * nr, cudaMemcpyHostToDevice, st));
    HEC_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hec::dev
