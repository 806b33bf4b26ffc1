// TEST INFRASTRUCTURE ONLY -- a stand-in for libnccl.so.2 that lets several
// ranks share ONE GPU in the tests (real NCCL rejects two ranks on a device).
// It implements the NCCL entry points libhegmm_b200.so binds (csrc/comm.cpp)
// over TCP on 127.0.0.1 in a star around rank 0, staging through host memory
// after synchronising the stream.  Rank 0 must be a party of every Send/Recv
// (the library only gathers to its root).  Selected with HGM_NCCL_LIB.
#include <arpa/inet.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

struct ncclComm {
    int rank = 0, world = 1;
    std::vector<int> fd;  // rank 0: fd[r] to rank r; others: fd[0] to rank 0
};

namespace {

bool io_all(int fd, void* p, size_t n, bool wr) {
    char* c = static_cast<char*>(p);
    while (n) {
        const ssize_t k = wr ? ::send(fd, c, n, MSG_NOSIGNAL) : ::recv(fd, c, n, 0);
        if (k <= 0) return false;
        c += k;
        n -= (size_t)k;
    }
    return true;
}
int port_of(const ncclUniqueId& id) {
    uint16_t p;
    std::memcpy(&p, id.internal, 2);
    return 20000 + p % 20000;
}
size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}
ncclResult_t sync(cudaStream_t s) { return cudaStreamSynchronize(s) == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError; }
// copies ordered on the communicator's stream and complete on return (a plain
// cudaMemcpy from pageable memory may return before its DMA lands)
bool copy(void* dst, const void* src, size_t n, cudaMemcpyKind k, cudaStream_t s) {
    return cudaMemcpyAsync(dst, src, n, k, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetVersion(int* v) {
    *v = 99999;
    return ncclSuccess;
}
const char* ncclGetErrorString(ncclResult_t) { return "nccl tcp shim error"; }
const char* ncclGetLastError(ncclComm_t) { return "nccl tcp shim"; }
ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::random_device rd;
    for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) id->internal[i] = (char)(rd() & 0xff);
    return ncclSuccess;
}
ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
    auto* c = new ncclComm;
    c->rank = rank;
    c->world = nranks;
    c->fd.assign(nranks, -1);
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_port = htons((uint16_t)port_of(id));
    a.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
    int one = 1;
    if (rank == 0) {
        const int ls = socket(AF_INET, SOCK_STREAM, 0);
        setsockopt(ls, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
        if (bind(ls, (sockaddr*)&a, sizeof(a)) || listen(ls, nranks)) return ncclSystemError;
        for (int k = 1; k < nranks; ++k) {
            const int f = accept(ls, nullptr, nullptr);
            int r = -1;
            if (f < 0 || !io_all(f, &r, sizeof(r), false) || r <= 0 || r >= nranks) return ncclSystemError;
            setsockopt(f, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
            c->fd[r] = f;
        }
        close(ls);
    } else {
        int f = -1;
        for (int tries = 0; tries < 600; ++tries) {  // rank 0 may not listen yet
            f = socket(AF_INET, SOCK_STREAM, 0);
            if (connect(f, (sockaddr*)&a, sizeof(a)) == 0) break;
            close(f);
            f = -1;
            usleep(100000);
        }
        if (f < 0 || !io_all(f, &rank, sizeof(rank), true)) return ncclSystemError;
        setsockopt(f, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
        c->fd[0] = f;
    }
    *out = c;
    return ncclSuccess;
}
ncclResult_t ncclCommDestroy(ncclComm_t c) {
    for (int f : c->fd)
        if (f >= 0) close(f);
    delete c;
    return ncclSuccess;
}
ncclResult_t ncclCommCount(const ncclComm_t c, int* n) {
    *n = c->world;
    return ncclSuccess;
}
ncclResult_t ncclGroupStart() { return ncclSuccess; }
ncclResult_t ncclGroupEnd() { return ncclSuccess; }

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s) {
    if (c->rank != 0 && peer != 0) return ncclInvalidUsage;
    if (sync(s) != ncclSuccess) return ncclUnhandledCudaError;
    std::vector<char> h(count * type_size(t));
    if (!copy(h.data(), buf, h.size(), cudaMemcpyDeviceToHost, s)) return ncclUnhandledCudaError;
    return io_all(c->fd[peer], h.data(), h.size(), true) ? ncclSuccess : ncclSystemError;
}
ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s) {
    if (c->rank != 0 && peer != 0) return ncclInvalidUsage;
    if (sync(s) != ncclSuccess) return ncclUnhandledCudaError;
    std::vector<char> h(count * type_size(t));
    if (!io_all(c->fd[peer], h.data(), h.size(), false)) return ncclSystemError;
    return copy(buf, h.data(), h.size(), cudaMemcpyHostToDevice, s) ? ncclSuccess : ncclUnhandledCudaError;
}
// all-gather / all-reduce(max) through rank 0
ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t t, ncclComm_t c,
                           cudaStream_t s) {
    if (sync(s) != ncclSuccess) return ncclUnhandledCudaError;
    const size_t b = count * type_size(t);
    std::vector<char> all(b * c->world);
    if (!copy(all.data() + b * c->rank, send, b, cudaMemcpyDeviceToHost, s)) return ncclUnhandledCudaError;
    if (c->rank == 0) {
        for (int r = 1; r < c->world; ++r)
            if (!io_all(c->fd[r], all.data() + b * r, b, false)) return ncclSystemError;
        for (int r = 1; r < c->world; ++r)
            if (!io_all(c->fd[r], all.data(), all.size(), true)) return ncclSystemError;
    } else {
        if (!io_all(c->fd[0], all.data() + b * c->rank, b, true) || !io_all(c->fd[0], all.data(), all.size(), false))
            return ncclSystemError;
    }
    return copy(recv, all.data(), all.size(), cudaMemcpyHostToDevice, s) ? ncclSuccess : ncclUnhandledCudaError;
}
ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t c, cudaStream_t s) {
    if (t != ncclFloat64 || op != ncclMax || count != 1) return ncclInvalidUsage;
    std::vector<double> all(c->world);
    double* tmp = nullptr;
    if (cudaMalloc(&tmp, sizeof(double) * c->world) != cudaSuccess) return ncclUnhandledCudaError;
    const ncclResult_t r = ncclAllGather(send, tmp, 1, ncclFloat64, c, s);
    const bool ok = copy(all.data(), tmp, sizeof(double) * c->world, cudaMemcpyDeviceToHost, s);
    cudaFree(tmp);
    double m = all[0];
    for (double v : all) m = v > m ? v : m;
    if (!ok || !copy(recv, &m, sizeof(m), cudaMemcpyHostToDevice, s)) return ncclUnhandledCudaError;
    return r;
}

}  // extern "C"
