// peer.h -- CUDA VMM allocations shared between neighbouring ranks and the
// stream memory operations that order sweeps across them (peer.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace lbm {
namespace peer {

struct Alloc {
    unsigned long long handle = 0;  // CUmemGenericAllocationHandle
    void* va = nullptr;             // mapped device address (read/write on this device)
    size_t size = 0, gran = 0;
};

bool available();
// physical memory on `device`, exportable as a POSIX fd, mapped here
bool alloc(int device, size_t bytes, Alloc* out, std::string* err);
void release(Alloc* m);
int export_fd(const Alloc& m, std::string* err);
// map another allocation (exported descriptor) for `device`
bool import_fd(int device, int fd, size_t size, size_t gran, Alloc* out, std::string* err);
// descriptor rendezvous over abstract Unix sockets "lbm-b200-<key>-<rank>":
// every rank serves my_fds and fetches those of each rank in `peers`
bool exchange_fds(const std::string& key, int rank, const std::vector<int>& peers, const std::vector<int>& my_fds,
                  std::vector<std::vector<int>>* peer_fds, double timeout_s, std::string* err);
bool can_flush_remote_writes(int device);
cudaError_t stream_write(cudaStream_t s, void* addr, uint32_t value);
cudaError_t stream_wait_geq(cudaStream_t s, void* addr, uint32_t value, bool flush);

}  // namespace peer
}  // namespace lbm
