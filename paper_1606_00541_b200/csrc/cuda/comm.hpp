#pragma once
// Communication between the ranks of a distributed (RAS) solve, one process
// per GPU. The GMRES engine needs two collectives:
//   * the halo exchange of a local [own | halo] vector before the local
//     preconditioner apply and the local SpMV (point-to-point, each peer sends
//     the rows the other's halo holds);
//   * a sum all-reduce of a few doubles (the Gram-Schmidt dots and norms).
// Backends: none (one rank), NCCL over NVLink / NVSwitch (device buffers, on
// the solve's stream; libnccl is opened at first use so the library shares the
// copy a host application -- e.g. torch -- already loaded), and host callbacks
// (the caller moves host buffers: MPI, gloo, ...).

#include <cuda_runtime.h>

#include <memory>
#include <vector>

namespace hec::dev {

class Comm {
public:
    virtual ~Comm() = default;
    virtual int world() const = 0;
    virtual int rank() const = 0;
    // in place, over all ranks, on `st`
    virtual void allreduce_sum(double* dev, int count, cudaStream_t st) = 0;
    // send_dev[send_off[p] .. send_off[p+1]) goes to peer p, which stores it in its
    // recv segment for this rank; recv_dev[recv_off[p] .. recv_off[p+1]) comes from p
    virtual void exchange(const double* send_dev, const std::vector<int>& send_off, double* recv_dev,
                          const std::vector<int>& recv_off, cudaStream_t st) = 0;
    virtual const char* name() const = 0;
    long long allreduces = 0, exchanges = 0;
};

// One rank: nothing to exchange.
class NullComm final : public Comm {
public:
    int world() const override { return 1; }
    int rank() const override { return 0; }
    void allreduce_sum(double*, int, cudaStream_t) override {}
    void exchange(const double*, const std::vector<int>&, double*, const std::vector<int>&, cudaStream_t) override {}
    const char* name() const override { return "none"; }
};

// NCCL: grouped ncclSend / ncclRecv for the halo, ncclAllReduce for the dots.
class NcclComm final : public Comm {
public:
    // unique_id: the 128 bytes of an ncclUniqueId made by nccl_unique_id() on one
    // rank and shared with the others by the caller.
    NcclComm(const unsigned char* unique_id, int rank, int world);
    ~NcclComm() override;
    int world() const override { return world_; }
    int rank() const override { return rank_; }
    void allreduce_sum(double* dev, int count, cudaStream_t st) override;
    void exchange(const double* send_dev, const std::vector<int>& send_off, double* recv_dev,
                  const std::vector<int>& recv_off, cudaStream_t st) override;
    const char* name() const override { return "nccl"; }

private:
    void* comm_ = nullptr;  // ncclComm_t
    int rank_ = 0, world_ = 1;
};
void nccl_unique_id(unsigned char out[128]);
int nccl_version();  // 0 when libnccl cannot be opened

// Host callbacks (return 0 on success): the engine synchronises its stream and
// stages through host buffers.
struct CommCallbacks {
    void* ctx = nullptr;
    int (*allreduce_sum)(void* ctx, double* buf, int count) = nullptr;
    // send[send_off[p]..) -> peer p; recv[recv_off[p]..) <- peer p (offsets as given to the plan)
    int (*exchange)(void* ctx, const double* send, int send_count, double* recv, int recv_count) = nullptr;
};
class CallbackComm final : public Comm {
public:
    CallbackComm(const CommCallbacks& cb, int rank, int world) : cb_(cb), rank_(rank), world_(world) {}
    int world() const override { return world_; }
    int rank() const override { return rank_; }
    void allreduce_sum(double* dev, int count, cudaStream_t st) override;
    void exchange(const double* send_dev, const std::vector<int>& send_off, double* recv_dev,
                  const std::vector<int>& recv_off, cudaStream_t st) override;
    const char* name() const override { return "callbacks"; }

private:
    CommCallbacks cb_;
    int rank_ = 0, world_ = 1;
    std::vector<double> hs_, hr_;
};

}  // namespace hec::dev
