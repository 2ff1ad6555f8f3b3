// peer.cu -- the cross-GPU fused halo (the paper's
// "we only synchronize at the intersection layers every two time steps",
// PAPER.md:747-749): each rank's lattice buffers live in CUDA virtual-memory
// allocations exported as POSIX file descriptors; the descriptors travel to
// the neighbouring ranks over a Unix domain socket (SCM_RIGHTS) and are
// mapped into their address spaces, so a K2 sweep stores the ghost planes
// its neighbours read straight into their next-sweep buffers over NVLink --
// no NCCL kernels, no exchange launches.  Sweeps are ordered across ranks by
// stream memory operations (a done-counter the neighbour's stream writes
// into this rank's flag page, and a stream wait on it), not by kernels that
// spin on one another.  Host-only code; the protocol itself is in api.cu.
#include "peer.h"

#include <cuda.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace lbm {
namespace peer {

namespace {

struct Api {
    bool ok = false;
    decltype(&cuMemCreate) MemCreate = nullptr;
    decltype(&cuMemRelease) MemRelease = nullptr;
    decltype(&cuMemAddressReserve) AddressReserve = nullptr;
    decltype(&cuMemAddressFree) AddressFree = nullptr;
    decltype(&cuMemMap) Map = nullptr;
    decltype(&cuMemUnmap) Unmap = nullptr;
    decltype(&cuMemSetAccess) SetAccess = nullptr;
    decltype(&cuMemGetAllocationGranularity) Granularity = nullptr;
    decltype(&cuMemExportToShareableHandle) Export = nullptr;
    decltype(&cuMemImportFromShareableHandle) Import = nullptr;
    decltype(&cuStreamWriteValue32_v2) WriteValue32 = nullptr;
    decltype(&cuStreamWaitValue32_v2) WaitValue32 = nullptr;
    decltype(&cuDeviceGetAttribute) DeviceGetAttribute = nullptr;
};

Api g_api;
std::once_flag g_once;

template <typename F>
void sym(F& f, const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        f = reinterpret_cast<F>(p);
    else
        cudaGetLastError();
}

const Api& api() {
    std::call_once(g_once, [] {
        Api& a = g_api;
        sym(a.MemCreate, "cuMemCreate");
        sym(a.MemRelease, "cuMemRelease");
        sym(a.AddressReserve, "cuMemAddressReserve");
        sym(a.AddressFree, "cuMemAddressFree");
        sym(a.Map, "cuMemMap");
        sym(a.Unmap, "cuMemUnmap");
        sym(a.SetAccess, "cuMemSetAccess");
        sym(a.Granularity, "cuMemGetAllocationGranularity");
        sym(a.Export, "cuMemExportToShareableHandle");
        sym(a.Import, "cuMemImportFromShareableHandle");
        sym(a.WriteValue32, "cuStreamWriteValue32");
        sym(a.WaitValue32, "cuStreamWaitValue32");
        sym(a.DeviceGetAttribute, "cuDeviceGetAttribute");
        a.ok = a.MemCreate && a.MemRelease && a.AddressReserve && a.AddressFree && a.Map && a.Unmap &&
               a.SetAccess && a.Granularity && a.Export && a.Import && a.WriteValue32 && a.WaitValue32 &&
               a.DeviceGetAttribute;
    });
    return g_api;
}

CUmemAllocationProp prop_for(int device) {
    CUmemAllocationProp p;
    memset(&p, 0, sizeof p);
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return p;
}

std::string errstr(const char* what, CUresult r) {
    char b[160];
    snprintf(b, sizeof b, "%s failed (CUresult %d)", what, int(r));
    return b;
}

// map the physical allocation h at a fresh address range, read/write for device
bool map_handle(int device, CUmemGenericAllocationHandle h, size_t size, size_t gran, Alloc* out, std::string* err) {
    const Api& a = api();
    CUdeviceptr va = 0;
    CUresult r = a.AddressReserve(&va, size, gran, 0, 0);
    if (r != CUDA_SUCCESS) return *err = errstr("cuMemAddressReserve", r), false;
    r = a.Map(va, size, 0, h, 0);
    if (r != CUDA_SUCCESS) {
        a.AddressFree(va, size);
        return *err = errstr("cuMemMap", r), false;
    }
    CUmemAccessDesc acc;
    memset(&acc, 0, sizeof acc);
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = a.SetAccess(va, size, &acc, 1);
    if (r != CUDA_SUCCESS) {
        a.Unmap(va, size);
        a.AddressFree(va, size);
        return *err = errstr("cuMemSetAccess", r), false;
    }
    out->handle = h;
    out->va = reinterpret_cast<void*>(va);
    out->size = size;
    return true;
}

// ---- Unix-domain-socket rendezvous (abstract namespace: nothing on disk) ----
socklen_t sock_addr(const std::string& key, int rank, sockaddr_un* a) {
    memset(a, 0, sizeof *a);
    a->sun_family = AF_UNIX;
    const std::string name = "lbm-b200-" + key + "-" + std::to_string(rank);
    const size_t n = std::min(name.size(), sizeof(a->sun_path) - 2);
    memcpy(a->sun_path + 1, name.data(), n);  // sun_path[0] = 0: abstract
    return socklen_t(offsetof(sockaddr_un, sun_path) + 1 + n);
}

bool send_fds(int sock, int my_rank, const std::vector<int>& fds) {
    msghdr m;
    memset(&m, 0, sizeof m);
    iovec io{&my_rank, sizeof my_rank};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    std::vector<char> ctl(CMSG_SPACE(sizeof(int) * fds.size()));
    m.msg_control = ctl.data();
    m.msg_controllen = ctl.size();
    cmsghdr* c = CMSG_FIRSTHDR(&m);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int) * fds.size());
    memcpy(CMSG_DATA(c), fds.data(), sizeof(int) * fds.size());
    return sendmsg(sock, &m, 0) == ssize_t(sizeof my_rank);
}

bool recv_fds(int sock, int* peer_rank, std::vector<int>* fds, size_t n) {
    msghdr m;
    memset(&m, 0, sizeof m);
    iovec io{peer_rank, sizeof *peer_rank};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    std::vector<char> ctl(CMSG_SPACE(sizeof(int) * n));
    m.msg_control = ctl.data();
    m.msg_controllen = ctl.size();
    if (recvmsg(sock, &m, 0) != ssize_t(sizeof *peer_rank)) return false;
    cmsghdr* c = CMSG_FIRSTHDR(&m);
    if (!c || c->cmsg_type != SCM_RIGHTS || c->cmsg_len != CMSG_LEN(sizeof(int) * n)) return false;
    fds->resize(n);
    memcpy(fds->data(), CMSG_DATA(c), sizeof(int) * n);
    return true;
}

bool wait_fd(int fd, short ev, double timeout_s) {
    pollfd p{fd, ev, 0};
    return poll(&p, 1, int(timeout_s * 1000)) == 1 && (p.revents & ev);
}

}  // namespace

bool available() { return api().ok; }

bool alloc(int device, size_t bytes, Alloc* out, std::string* err) {
    const Api& a = api();
    if (!a.ok) return *err = "CUDA virtual memory management entry points unavailable", false;
    int posix = 0;
    a.DeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, device);
    if (!posix) return *err = "device cannot export memory as POSIX file descriptors", false;
    const CUmemAllocationProp p = prop_for(device);
    size_t gran = 0;
    CUresult r = a.Granularity(&gran, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS || !gran) return *err = errstr("cuMemGetAllocationGranularity", r), false;
    const size_t size = (bytes + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h;
    r = a.MemCreate(&h, size, &p, 0);
    if (r != CUDA_SUCCESS) return *err = errstr("cuMemCreate", r), false;
    if (!map_handle(device, h, size, gran, out, err)) {
        a.MemRelease(h);
        return false;
    }
    out->gran = gran;
    return true;
}

void release(Alloc* m) {
    if (!m || !m->va) return;
    const Api& a = api();
    a.Unmap(reinterpret_cast<CUdeviceptr>(m->va), m->size);
    a.AddressFree(reinterpret_cast<CUdeviceptr>(m->va), m->size);
    a.MemRelease(m->handle);
    m->va = nullptr;
}

int export_fd(const Alloc& m, std::string* err) {
    int fd = -1;
    CUresult r = api().Export(&fd, m.handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) {
        *err = errstr("cuMemExportToShareableHandle", r);
        return -1;
    }
    return fd;
}

bool import_fd(int device, int fd, size_t size, size_t gran, Alloc* out, std::string* err) {
    const Api& a = api();
    CUmemGenericAllocationHandle h;
    CUresult r = a.Import(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) return *err = errstr("cuMemImportFromShareableHandle", r), false;
    if (!map_handle(device, h, size, gran, out, err)) {
        a.MemRelease(h);
        return false;
    }
    out->gran = gran;
    return true;
}

bool exchange_fds(const std::string& key, int rank, const std::vector<int>& peers, const std::vector<int>& my_fds,
                  std::vector<std::vector<int>>* peer_fds, double timeout_s, std::string* err) {
    // distinct peers; each connects once to every other's socket (itself too:
    // a periodic single rank maps its own buffers as its neighbour)
    std::vector<int> uniq = peers;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    const int lsock = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (lsock < 0) return *err = "socket() failed", false;
    sockaddr_un addr;
    socklen_t alen = sock_addr(key, rank, &addr);
    if (bind(lsock, reinterpret_cast<sockaddr*>(&addr), alen) != 0 || listen(lsock, int(uniq.size()) + 4) != 0) {
        close(lsock);
        return *err = "bind/listen on the rendezvous socket failed (another context with the same id?)", false;
    }
    // server: hand my descriptors to every peer that connects
    bool serve_ok = true;
    std::thread server([&] {
        for (size_t i = 0; i < uniq.size(); ++i) {
            if (!wait_fd(lsock, POLLIN, timeout_s)) {
                serve_ok = false;
                return;
            }
            const int cs = accept4(lsock, nullptr, nullptr, SOCK_CLOEXEC);
            if (cs < 0 || !send_fds(cs, rank, my_fds)) serve_ok = false;
            if (cs >= 0) {
                char b;
                wait_fd(cs, POLLIN, timeout_s);  // the peer closes after receiving
                (void)!read(cs, &b, 1);
                close(cs);
            }
        }
    });
    // client: fetch every peer's descriptors (retry until its socket exists)
    bool ok = true;
    peer_fds->assign(peers.size(), {});
    std::vector<std::vector<int>> got(uniq.size());
    const auto t0 = std::chrono::steady_clock::now();
    for (size_t i = 0; i < uniq.size() && ok; ++i) {
        sockaddr_un pa;
        const socklen_t plen = sock_addr(key, uniq[i], &pa);
        int s = -1;
        for (;;) {
            s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
            if (s >= 0 && connect(s, reinterpret_cast<sockaddr*>(&pa), plen) == 0) break;
            if (s >= 0) close(s);
            s = -1;
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) break;
            usleep(2000);
        }
        int who = -1;
        if (s < 0 || !wait_fd(s, POLLIN, timeout_s) || !recv_fds(s, &who, &got[i], my_fds.size()) || who != uniq[i]) {
            ok = false;
            *err = "receiving a neighbour's buffer descriptors failed (peer lost or timed out)";
        }
        if (s >= 0) close(s);
    }
    server.join();
    close(lsock);
    if (ok && !serve_ok) {
        ok = false;
        *err = "serving this rank's buffer descriptors failed";
    }
    if (!ok) {
        for (auto& v : got)
            for (int fd : v) close(fd);
        return false;
    }
    // one copy of the descriptors per listed peer (duplicates share them)
    for (size_t j = 0; j < peers.size(); ++j) {
        const size_t i = size_t(std::lower_bound(uniq.begin(), uniq.end(), peers[j]) - uniq.begin());
        for (int fd : got[i]) (*peer_fds)[j].push_back(dup(fd));
    }
    for (auto& v : got)
        for (int fd : v) close(fd);
    return true;
}

bool can_flush_remote_writes(int device) {
    int v = 0;
    return api().DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, device) == CUDA_SUCCESS && v;
}

cudaError_t stream_write(cudaStream_t s, void* addr, uint32_t value) {
    // default flags: a system-scope fence precedes the write, ordering the
    // sweep's (remote) stores before the counter the neighbour waits on
    return api().WriteValue32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value, 0) ==
                   CUDA_SUCCESS
               ? cudaSuccess
               : cudaErrorUnknown;
}

cudaError_t stream_wait_geq(cudaStream_t s, void* addr, uint32_t value, bool flush) {
    unsigned flags = CU_STREAM_WAIT_VALUE_GEQ | (flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
    return api().WaitValue32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value, flags) ==
                   CUDA_SUCCESS
               ? cudaSuccess
               : cudaErrorUnknown;
}

}  // namespace peer
}  // namespace lbm

// Test hook (not part of include/lbm.h): the descriptor rendezvous alone, on
// plain file descriptors, so the socket protocol is testable on a CPU
// (tests/test_peer_fds.py).  Returns 0 on success; out_fds[j * nfd + m] is
// descriptor m of peers[j].
extern "C" int lbm_internal_exchange_fds(const char* key, int rank, const int* peers, int npeers, const int* fds,
                                         int nfd, int* out_fds, double timeout_s) {
    std::vector<std::vector<int>> got;
    std::string err;
    if (!lbm::peer::exchange_fds(key, rank, std::vector<int>(peers, peers + npeers), std::vector<int>(fds, fds + nfd),
                                 &got, timeout_s, &err))
        return 1;
    for (int j = 0; j < npeers; ++j)
        for (int m = 0; m < nfd; ++m) out_fds[j * nfd + m] = got[size_t(j)][size_t(m)];
    return 0;
}
