// Halo exchange of an element-partitioned mesh: the cut-face pack
// kernel and the run-time binding of NCCL's point-to-point API.
//
// The RHS reads across elements only through the exterior trace
// (solver.hpp:263-264: proj[nbr](nq + perm)), so once per RK stage a rank ships
// the projected traces of its cut faces: 3 fields x npf nodes per face.  The wire
// format packs three faces per [3][nf] pseudo-element (face i of a message at
// pseudo-element i/3, face position i%3), which is exactly the layout of the
// receiver's halo slots in the trace buffer — a received message needs no unpack.
// The SBP scheme reads the neighbours' face-node STATES instead (solver.hpp:405-407):
// its pseudo-elements are [3][nq] state blocks holding three faces' node values at the
// volume nodes face_index[position npf + node], the halo slots of the state buffers.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace swedg {

// One thread per (sent face, field, node): buf[dst[i]] = base[src[i]].  Modal: base is
// the face-trace buffer ([K][3][nf]); SBP: the stage's input state ([K][3][nq], face
// node values, solver.hpp:405-407).  The index lists are built once by swedg_set_halo.
struct HaloPackParams {
    const double* base;
    const long long* src;  // [n] offsets into base
    const long long* dst;  // [n] offsets into buf (wire format)
    double* buf;
    long long n;
};

__global__ void halo_pack_kernel(HaloPackParams p) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < p.n) p.buf[p.dst[i]] = p.base[p.src[i]];
}

// Peer-memory variant: the entry goes straight to the destination rank's halo slot,
// rbase[rpeer[i]] + rdst[i] (the peer's buffer, mapped into this process).
struct HaloPackP2PParams {
    const double* base;
    const long long* src;    // [n] offsets into base
    const long long* rdst;   // [n] offsets into the destination buffer
    const int* rpeer;        // [n] index into rbase
    double* const* rbase;    // destination buffers (peer memory)
    long long n;
};

__global__ void halo_pack_p2p_kernel(HaloPackP2PParams p) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < p.n) p.rbase[p.rpeer[i]][p.rdst[i]] = p.base[p.src[i]];
}

// Stream memory operations (driver API, resolved through the runtime: no libcuda link).
struct StreamMemOps {
    int (*wait32)(cudaStream_t, unsigned long long, unsigned int, unsigned int) = nullptr;
    int (*write32)(cudaStream_t, unsigned long long, unsigned int, unsigned int) = nullptr;
    bool ok = false;
};
constexpr unsigned kWaitEq = 0x1;     // CU_STREAM_WAIT_VALUE_EQ
constexpr unsigned kWaitFlush = 1u << 30;  // CU_STREAM_WAIT_VALUE_FLUSH

inline StreamMemOps& stream_mem_ops() {
    static StreamMemOps ops;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q1, q2;
        void* w = nullptr;
        void* x = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWriteValue32", &x, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && x) {
            ops.wait32 = reinterpret_cast<int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int)>(w);
            ops.write32 = reinterpret_cast<int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int)>(x);
            ops.ok = true;
        }
    });
    return ops;
}

// This rank's descriptor for the peer-memory transport (swedg_p2p_export): the halo
// slots' buffers (modal: the trace buffer; SBP: the three state buffers) and the flag
// array by IPC handle and by address, and the receive table (message pairing).
constexpr int kP2pMaxRanks = 1024;  // flags: [0, R) ready from rank r, [R, 2R) free from rank r
constexpr int kP2pMaxMsgs = 64;
struct P2pBlob {
    uint32_t magic, version;
    int rank, pid, device, nbuf;
    cudaIpcMemHandle_t buf_ipc[3];
    unsigned long long buf_ptr[3];
    long long halo_off;  // doubles from a buffer's base to its halo slots
    cudaIpcMemHandle_t flag_ipc;
    unsigned long long flag_ptr;
    int n_recv;
    int recv_peer[kP2pMaxMsgs];
    long long recv_off[kP2pMaxMsgs], recv_len[kP2pMaxMsgs];  // doubles from the halo slots
};
constexpr uint32_t kP2pMagic = 0x50325053u;  // "SP2P"

// ---- NCCL, resolved at run time ---------------------------------------------
// The library does not link libnccl: it binds the symbols of the libnccl.so.2 the
// process already has (torch's, when called from Python) or loads it, so the
// communicator a caller passes and the calls made here come from one NCCL.
struct NcclUid {
    char internal[128];
};
struct NcclApi {
    int (*GetUniqueId)(NcclUid*) = nullptr;
    int (*CommInitRank)(void**, int, NcclUid, int) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool ok = false;
    std::string error;
};
constexpr int kNcclFloat64 = 8;  // ncclDataType_t ncclFloat64 (nccl.h)

inline NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("SWEDG_NCCL_LIB");
        void* lib = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            api.error = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(lib, n); };
        api.GetUniqueId = reinterpret_cast<int (*)(NcclUid*)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<int (*)(void**, int, NcclUid, int)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<int (*)(void*)>(sym("ncclCommDestroy"));
        api.Send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<int (*)()>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<int (*)()>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<const char* (*)(int)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
                 api.GroupEnd && api.GetErrorString;
        if (!api.ok) api.error = "libnccl.so.2 lacks the point-to-point API";
    });
    return api;
}

}  // namespace swedg
