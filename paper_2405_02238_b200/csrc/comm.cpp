// comm.cpp -- the library's multi-GPU plumbing: one process per
// GPU, one NCCL communicator per session over NVLink / NVSwitch.
//
// HEGMM's work shards by independent products (config 4) or output row blocks
// (config 5); every rank holds the keys replicated and runs its shard with no
// data-path collective.  The communicator exists only to MOVE results (a
// gather of result ciphertexts to the decrypting rank: NCCL reductions wrap
// mod 2^64, not mod q, so ciphertexts are never reduced in transit) and for
// control (barrier, max over ranks of a timing).  Everything is stream-ordered
// on the session's stream, after the work that produced the buffers.
//
// Reference analogue: the std::async pool over independent cases,
// /root/reference/proj/src/costmodel.cpp:273-296 (one backend session per case).
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hegmm_b200.h"
#include "capi_internal.hpp"

using namespace hgm;

struct hgm_comm {
    hgm_ctx* owner = nullptr;
    int rank = 0, world = 1;
    ncclComm_t nc = nullptr;
    u64* scratch = nullptr;  // device: world words (count exchange, control values)
};

namespace {

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// NCCL is bound at first use (dlopen), not at load time: single-GPU users never
// load it, and a process that also loads another NCCL build (e.g. torch's
// wheel) shares that one instead of pinning an older soname first.  Order:
// $HGM_NCCL_LIB, an already-loaded libnccl.so.2, then the system library.
struct Nccl {
    decltype(&::ncclGetUniqueId) GetUniqueId;
    decltype(&::ncclCommInitRank) CommInitRank;
    decltype(&::ncclCommDestroy) CommDestroy;
    decltype(&::ncclCommCount) CommCount;
    decltype(&::ncclGetVersion) GetVersion;
    decltype(&::ncclAllGather) AllGather;
    decltype(&::ncclAllReduce) AllReduce;
    decltype(&::ncclSend) Send;
    decltype(&::ncclRecv) Recv;
    decltype(&::ncclGroupStart) GroupStart;
    decltype(&::ncclGroupEnd) GroupEnd;
    decltype(&::ncclGetErrorString) GetErrorString;
    decltype(&::ncclGetLastError) GetLastError;
    std::string path;
};

const Nccl& nccl() {
    static const Nccl* api = [] {
        void* h = nullptr;
        std::string from;
        if (const char* e = std::getenv("HGM_NCCL_LIB"); e && *e) {
            h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
            from = e;
        }
        if (!h && (h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD))) from = "libnccl.so.2 (already loaded)";
        if (!h && (h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL))) from = "libnccl.so.2";
        if (!h) throw std::runtime_error(std::string("cannot load NCCL: ") + dlerror());
        auto* n = new Nccl;
        auto sym = [&](const char* name) {
            void* f = dlsym(h, name);
            if (!f) throw std::runtime_error(std::string("NCCL symbol missing: ") + name);
            return f;
        };
#define HGM_NCCL_SYM(field, name) n->field = reinterpret_cast<decltype(n->field)>(sym(name))
        HGM_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
        HGM_NCCL_SYM(CommInitRank, "ncclCommInitRank");
        HGM_NCCL_SYM(CommDestroy, "ncclCommDestroy");
        HGM_NCCL_SYM(CommCount, "ncclCommCount");
        HGM_NCCL_SYM(GetVersion, "ncclGetVersion");
        HGM_NCCL_SYM(AllGather, "ncclAllGather");
        HGM_NCCL_SYM(AllReduce, "ncclAllReduce");
        HGM_NCCL_SYM(Send, "ncclSend");
        HGM_NCCL_SYM(Recv, "ncclRecv");
        HGM_NCCL_SYM(GroupStart, "ncclGroupStart");
        HGM_NCCL_SYM(GroupEnd, "ncclGroupEnd");
        HGM_NCCL_SYM(GetErrorString, "ncclGetErrorString");
        HGM_NCCL_SYM(GetLastError, "ncclGetLastError");
#undef HGM_NCCL_SYM
        n->path = from;
        return n;
    }();
    return *api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw NcclError(std::string(what) + ": " + nccl().GetErrorString(r) + " (" + nccl().GetLastError(nullptr) +
                        ")");
}
#define HGM_NCCL(x) nccl_check((x), #x)

template <typename F>
int comm_guarded(F&& f) {
    try {
        f();
        return HGM_OK;
    } catch (const CudaError& e) {
        return set_error(HGM_ECUDA, e.what());
    } catch (const std::invalid_argument& e) {
        return set_error(HGM_EARG, e.what());
    } catch (const std::exception& e) {
        return set_error(HGM_EINTERNAL, e.what());
    }
}

// all-gather of one u64 per rank (host in, host out), on the session stream
std::vector<u64> allgather_u64(hgm_comm* cm, u64 mine) {
    Context& ctx = session_context(cm->owner);
    std::vector<u64> all(cm->world, 0);
    HGM_CUDA(cudaMemcpyAsync(cm->scratch + cm->rank, &mine, 8, cudaMemcpyHostToDevice, ctx.stream()));
    HGM_NCCL(nccl().AllGather(cm->scratch + cm->rank, cm->scratch, 1, ncclUint64, cm->nc, ctx.stream()));
    HGM_CUDA(cudaMemcpyAsync(all.data(), cm->scratch, 8 * all.size(), cudaMemcpyDeviceToHost, ctx.stream()));
    HGM_CUDA(cudaStreamSynchronize(ctx.stream()));
    return all;
}

void write_id_file(const std::string& path, const ncclUniqueId& id) {
    const std::string tmp = path + ".tmp." + std::to_string(getpid());
    const int fd = open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0600);
    if (fd < 0) throw std::invalid_argument("cannot create " + tmp);
    const ssize_t w = write(fd, &id, sizeof(id));
    close(fd);
    if (w != (ssize_t)sizeof(id) || rename(tmp.c_str(), path.c_str()) != 0)
        throw std::invalid_argument("cannot publish the NCCL id at " + path);
}

ncclUniqueId read_id_file(const std::string& path, double timeout_s) {
    ncclUniqueId id;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {  // rank 0 publishes by rename(), so a visible file is complete
        const int fd = open(path.c_str(), O_RDONLY);
        if (fd >= 0) {
            const ssize_t r = read(fd, &id, sizeof(id));
            close(fd);
            if (r == (ssize_t)sizeof(id)) return id;
        }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
            throw std::invalid_argument("timed out waiting for the NCCL id at " + path);
        std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
}

hgm_comm* make_comm(hgm_ctx* c, int rank, int world, const ncclUniqueId& id) {
    auto* cm = new hgm_comm;
    cm->owner = c;
    cm->rank = rank;
    cm->world = world;
    try {
        Context& ctx = session_context(c);
        HGM_NCCL(nccl().CommInitRank(&cm->nc, world, id, rank));
        cm->scratch = ctx.alloc((size_t)world + 2);
        int n = 0, ver = 0;
        nccl().CommCount(cm->nc, &n);
        nccl().GetVersion(&ver);
        std::fprintf(stderr, "hgm_comm: rank %d of %d on device %d, NCCL %d (%s), comm nranks %d\n", rank, world,
                     session_device(c), ver, nccl().path.c_str(), n);
    } catch (...) {
        if (cm->nc) nccl().CommDestroy(cm->nc);
        delete cm;
        throw;
    }
    session_retain(c);
    return cm;
}

}  // namespace

extern "C" {

int hgm_comm_unique_id(uint8_t* id) {
    return comm_guarded([&] {
        if (!id) throw std::invalid_argument("null id buffer");
        static_assert(sizeof(ncclUniqueId) == HGM_COMM_ID_BYTES, "NCCL unique id size");
        ncclUniqueId u;
        HGM_NCCL(nccl().GetUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
    });
}

int hgm_comm_init(hgm_ctx* c, int rank, int world, const uint8_t* id, hgm_comm** out) {
    if (!c || !out || !id) return set_error(HGM_EARG, "null argument");
    std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(c));
    DeviceGuard dev(session_device(c));
    return comm_guarded([&] {
        if (world < 1 || rank < 0 || rank >= world)
            throw std::invalid_argument("bad rank " + std::to_string(rank) + " of " + std::to_string(world));
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        *out = make_comm(c, rank, world, u);
    });
}

int hgm_comm_init_file(hgm_ctx* c, int rank, int world, const char* path, double timeout_s, hgm_comm** out) {
    if (!c || !out || !path) return set_error(HGM_EARG, "null argument");
    std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(c));
    DeviceGuard dev(session_device(c));
    return comm_guarded([&] {
        if (world < 1 || rank < 0 || rank >= world)
            throw std::invalid_argument("bad rank " + std::to_string(rank) + " of " + std::to_string(world));
        ncclUniqueId u;
        if (rank == 0) {
            HGM_NCCL(nccl().GetUniqueId(&u));
            write_id_file(path, u);
        } else {
            u = read_id_file(path, timeout_s > 0 ? timeout_s : 120.0);
        }
        hgm_comm* cm = make_comm(c, rank, world, u);
        // every rank has joined once this returns: the id file can go
        try {
            allgather_u64(cm, 0);
        } catch (...) {
            hgm_comm_destroy(cm);
            throw;
        }
        if (rank == 0) unlink(path);
        *out = cm;
    });
}

void hgm_comm_destroy(hgm_comm* cm) {
    if (!cm) return;
    hgm_ctx* c = cm->owner;
    {
        std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(c));
        DeviceGuard dev(session_device(c));
        try {
            Context& ctx = session_context(c);
            ctx.sync();
            if (cm->nc) nccl().CommDestroy(cm->nc);
            if (cm->scratch) ctx.release(cm->scratch);
            ctx.sync();
        } catch (const std::exception& e) {
            set_error(HGM_EINTERNAL, e.what());
        }
        delete cm;
    }
    session_release(c);
}

int hgm_comm_rank(const hgm_comm* cm) { return cm ? cm->rank : -1; }
int hgm_comm_size(const hgm_comm* cm) { return cm ? cm->world : 0; }

int hgm_comm_barrier(hgm_comm* cm) {
    if (!cm) return set_error(HGM_EARG, "null communicator");
    std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(cm->owner));
    DeviceGuard dev(session_device(cm->owner));
    return comm_guarded([&] {
        session_context(cm->owner).sync();  // the rank's queued work is part of what the barrier waits for
        allgather_u64(cm, 0);
    });
}

int hgm_comm_max(hgm_comm* cm, double* value) {
    if (!cm || !value) return set_error(HGM_EARG, "null argument");
    std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(cm->owner));
    DeviceGuard dev(session_device(cm->owner));
    return comm_guarded([&] {
        Context& ctx = session_context(cm->owner);
        double v = *value;
        double* d = reinterpret_cast<double*>(cm->scratch + cm->world);
        HGM_CUDA(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, ctx.stream()));
        HGM_NCCL(nccl().AllReduce(d, d, 1, ncclFloat64, ncclMax, cm->nc, ctx.stream()));
        HGM_CUDA(cudaMemcpyAsync(&v, d, 8, cudaMemcpyDeviceToHost, ctx.stream()));
        HGM_CUDA(cudaStreamSynchronize(ctx.stream()));
        *value = v;
    });
}

int hgm_comm_gather(hgm_comm* cm, const uint64_t* send, size_t send_words, uint64_t* recv, size_t recv_cap_words,
                    int root, size_t* recv_words) {
    if (!cm) return set_error(HGM_EARG, "null communicator");
    std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(cm->owner));
    DeviceGuard dev(session_device(cm->owner));
    return comm_guarded([&] {
        if (root < 0 || root >= cm->world) throw std::invalid_argument("bad root rank");
        if (send_words && !send) throw std::invalid_argument("null send buffer");
        Context& ctx = session_context(cm->owner);
        // host buffers are staged through device memory (NCCL moves device memory only)
        u64* st_send = nullptr;
        u64* st_recv = nullptr;
        uint64_t* host_recv = nullptr;
        struct Staging {
            Context& ctx;
            u64*& a;
            u64*& b;
            ~Staging() {
                try {
                    ctx.sync();
                    if (a) ctx.release(a);
                    if (b) ctx.release(b);
                    ctx.sync();
                } catch (...) {
                }
            }
        } staging{ctx, st_send, st_recv};
        if (send_words && !is_device_pointer(send)) {
            st_send = ctx.alloc(send_words);
            HGM_CUDA(cudaMemcpyAsync(st_send, send, send_words * 8, cudaMemcpyHostToDevice, ctx.stream()));
            send = st_send;
        }
        if (cm->rank == root && recv && recv_cap_words && !is_device_pointer(recv)) {
            st_recv = ctx.alloc(recv_cap_words);
            host_recv = recv;
            recv = st_recv;
        }
        const std::vector<u64> cnt = allgather_u64(cm, send_words);  // also orders after the producing work
        size_t total = 0;
        for (u64 x : cnt) total += x;
        // every rank checks the root's capacity, so no rank enqueues a transfer the root will refuse
        const std::vector<u64> caps = allgather_u64(cm, cm->rank == root ? (u64)recv_cap_words : 0);
        if (cm->rank == root && total && !recv) throw std::invalid_argument("null receive buffer on the root");
        static const bool trace = [] {
            const char* e = std::getenv("HGM_TRACE");
            return e && e[0] == '1';
        }();
        if (trace) {
            std::fprintf(stderr, "hgm_comm_gather rank %d: send %zu words, counts", cm->rank, send_words);
            for (u64 x : cnt) std::fprintf(stderr, " %llu", (unsigned long long)x);
            std::fprintf(stderr, ", root cap %llu\n", (unsigned long long)caps[root]);
        }
        if (total > caps[root])
            throw std::invalid_argument("gather of " + std::to_string(total) + " words exceeds the root's buffer of " +
                                        std::to_string(caps[root]));
        if (cm->rank == root) {
            size_t off = 0;
            HGM_NCCL(nccl().GroupStart());
            for (int r = 0; r < cm->world; ++r) {
                if (cnt[r] == 0) continue;
                if (r == root) {
                    if (recv + off != send)
                        HGM_CUDA(cudaMemcpyAsync(recv + off, send, cnt[r] * 8, cudaMemcpyDeviceToDevice, ctx.stream()));
                } else {
                    HGM_NCCL(nccl().Recv(recv + off, cnt[r], ncclUint64, r, cm->nc, ctx.stream()));
                }
                off += cnt[r];
            }
            HGM_NCCL(nccl().GroupEnd());
        } else if (send_words) {
            HGM_NCCL(nccl().Send(send, send_words, ncclUint64, root, cm->nc, ctx.stream()));
        }
        if (host_recv && total)
            HGM_CUDA(cudaMemcpyAsync(host_recv, recv, total * 8, cudaMemcpyDeviceToHost, ctx.stream()));
        HGM_CUDA(cudaStreamSynchronize(ctx.stream()));
        if (recv_words) *recv_words = cm->rank == root ? total : 0;
    });
}

int hgm_comm_gather_batch(hgm_comm* cm, hgm_batch* b, int root, uint64_t** dev_out, size_t* total_count) {
    if (!cm || !dev_out || !total_count) return set_error(HGM_EARG, "null argument");
    if (b && batch_session(b) != cm->owner) return set_error(HGM_EARG, "batch belongs to another session");
    std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(cm->owner));
    DeviceGuard dev(session_device(cm->owner));
    return comm_guarded([&] {
        if (root < 0 || root >= cm->world) throw std::invalid_argument("bad root rank");
        Context& ctx = session_context(cm->owner);
        const size_t W = ctx.ct_words();
        size_t count = 0;
        const u64* mine = batch_results(b, &count);
        const std::vector<u64> cnt = allgather_u64(cm, count);
        size_t total = 0;
        for (u64 x : cnt) total += x;
        u64* recv = nullptr;
        if (cm->rank == root && total) recv = ctx.alloc(total * W);
        size_t got = 0;
        const int rc = hgm_comm_gather(cm, mine, count * W, recv, total * W, root, &got);
        if (rc != HGM_OK) {
            if (recv) ctx.release(recv);
            throw std::runtime_error(hgm_last_error());
        }
        *dev_out = recv;
        *total_count = cm->rank == root ? total : 0;
    });
}

int hgm_comm_buffer_free(hgm_comm* cm, uint64_t* p) {
    if (!cm) return set_error(HGM_EARG, "null communicator");
    if (!p) return HGM_OK;
    std::lock_guard<std::recursive_mutex> lk(session_exec_mutex(cm->owner));
    DeviceGuard dev(session_device(cm->owner));
    return comm_guarded([&] {
        Context& ctx = session_context(cm->owner);
        ctx.release(p);
        ctx.sync();
    });
}

}  // extern "C"
