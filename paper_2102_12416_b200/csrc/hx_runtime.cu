// libhx runtime plumbing: devices, streams, events, pinned memory, peer
// access and the CUDA-IPC handle cache used by persistent channels.
//
// Replaces the reference's simulated device registry and in-process wire
// copies (cl/devicesim.py:121-224, cl/transport.py:284-289, 430-432,
// 459-463) with real HBM allocations and NVLink P2P mappings. The driver
// API is reached through cudaGetDriverEntryPoint so the library links only
// the static CUDA runtime (it loads on machines without a GPU driver, where
// only symbol presence is checked).
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "hx_internal.cuh"

namespace {

std::mutex g_mu;
std::map<std::string, void *> g_driver_syms;

struct IpcEntry {
    void *base;
    int refs;
};
std::map<std::string, IpcEntry> g_ipc;  // handle bytes -> mapping

}  // namespace

void *hx_internal_driver_sym(const char *name) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_driver_syms.find(name);
    if (it != g_driver_syms.end()) return it->second;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        fn = nullptr;
    g_driver_syms[name] = fn;
    return fn;
}

int hx_internal_driver_init() {
    return hx_internal_driver_sym("cuGetErrorString") ? 0 : HX_E_NODRIVER;
}

extern "C" {

int hx_abi_version(void) { return HX_ABI_VERSION; }

const char *hx_error_string(int code) {
    switch (code) {
        case 0: return "ok";
        case HX_E_INVALID: return "hx: invalid argument";
        case HX_E_TIMEOUT: return "hx: device flag wait timed out";
        case HX_E_NODRIVER: return "hx: CUDA driver entry point unavailable";
        case HX_E_TMA: return "hx: tensor map encoding failed";
        default: return code > 0 ? cudaGetErrorString((cudaError_t)code) : "hx: unknown error";
    }
}

int hx_device_count(int *n) {
    if (!n) return HX_E_INVALID;
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        *n = 0;
        cudaGetLastError();
        return (int)e;
    }
    return 0;
}

int hx_set_device(int dev) { return (int)cudaSetDevice(dev); }
int hx_get_device(int *dev) { return dev ? (int)cudaGetDevice(dev) : HX_E_INVALID; }

int hx_sm_count(int dev, int *n) {
    if (!n) return HX_E_INVALID;
    return (int)cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, dev);
}

int hx_device_synchronize(void) { return (int)cudaDeviceSynchronize(); }

int hx_stream_create(void **stream) {
    if (!stream) return HX_E_INVALID;
    cudaStream_t s;
    HX_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = (void *)s;
    return 0;
}

int hx_stream_destroy(void *stream) { return (int)cudaStreamDestroy((cudaStream_t)stream); }
int hx_stream_synchronize(void *stream) { return (int)cudaStreamSynchronize((cudaStream_t)stream); }

int hx_event_create(void **ev, int timing) {
    if (!ev) return HX_E_INVALID;
    cudaEvent_t e;
    HX_TRY(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    *ev = (void *)e;
    return 0;
}

int hx_event_destroy(void *ev) { return (int)cudaEventDestroy((cudaEvent_t)ev); }

int hx_event_record(void *ev, void *stream) {
    return (int)cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream);
}

int hx_event_query(void *ev) {
    cudaError_t e = cudaEventQuery((cudaEvent_t)ev);
    if (e == cudaSuccess) return 0;
    if (e == cudaErrorNotReady) {
        cudaGetLastError();  // NotReady is sticky-free but clear it anyway
        return 1;
    }
    return (int)e;
}

int hx_event_synchronize(void *ev) { return (int)cudaEventSynchronize((cudaEvent_t)ev); }

int hx_event_elapsed_ms(void *start, void *stop, float *ms) {
    if (!ms) return HX_E_INVALID;
    return (int)cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop);
}

int hx_stream_wait_event(void *stream, void *ev) {
    return (int)cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0);
}

int hx_malloc(void **ptr, size_t bytes) {
    if (!ptr) return HX_E_INVALID;
    return (int)cudaMalloc(ptr, bytes ? bytes : 1);
}

int hx_free(void *ptr) { return (int)cudaFree(ptr); }

int hx_malloc_host(void **ptr, size_t bytes) {
    if (!ptr) return HX_E_INVALID;
    return (int)cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable);
}

int hx_free_host(void *ptr) { return (int)cudaFreeHost(ptr); }

// ------------------------------------------------------------------ peers

int hx_can_access_peer(int dev, int peer, int *ok) {
    if (!ok) return HX_E_INVALID;
    if (dev == peer) {
        *ok = 1;
        return 0;
    }
    return (int)cudaDeviceCanAccessPeer(ok, dev, peer);
}

int hx_enable_peer(int dev, int peer) {
    if (dev == peer) return 0;
    int prev;
    HX_TRY(cudaGetDevice(&prev));
    HX_TRY(cudaSetDevice(dev));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        e = cudaSuccess;
    }
    cudaSetDevice(prev);
    return (int)e;
}

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

int hx_ipc_get(void *ptr, void *handle_out, size_t *offset_out) {
    if (!ptr || !handle_out || !offset_out) return HX_E_INVALID;
    auto range = (PFN_getAddressRange)hx_internal_driver_sym("cuMemGetAddressRange");
    if (!range) return HX_E_NODRIVER;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return HX_E_INVALID;
    cudaIpcMemHandle_t h;
    HX_TRY(cudaIpcGetMemHandle(&h, (void *)base));
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (size_t)((CUdeviceptr)ptr - base);
    return 0;
}

int hx_alloc_range(const void *ptr, void **base_out, size_t *size_out) {
    if (!ptr || !base_out || !size_out) return HX_E_INVALID;
    auto range = (PFN_getAddressRange)hx_internal_driver_sym("cuMemGetAddressRange");
    if (!range) return HX_E_NODRIVER;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return HX_E_INVALID;
    *base_out = (void *)base;
    *size_out = size;
    return 0;
}

int hx_ipc_open(const void *handle, void **base_out) {
    if (!handle || !base_out) return HX_E_INVALID;
    std::string key((const char *)handle, sizeof(cudaIpcMemHandle_t));
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_ipc.find(key);
    if (it != g_ipc.end()) {
        it->second.refs++;
        *base_out = it->second.base;
        return 0;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    HX_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    g_ipc[key] = IpcEntry{base, 1};
    *base_out = base;
    return 0;
}

int hx_ipc_close(void *base) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_ipc.begin(); it != g_ipc.end(); ++it) {
        if (it->second.base == base) {
            if (--it->second.refs == 0) {
                cudaError_t e = cudaIpcCloseMemHandle(base);
                g_ipc.erase(it);
                return (int)e;
            }
            return 0;
        }
    }
    return HX_E_INVALID;
}

// ------------------------------------------------------------------ copies

int hx_memcpy(void *dst, const void *src, size_t bytes, void *stream) {
    if (bytes == 0) return 0;
    return (int)cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream);
}

int hx_memcpy_peer(void *dst, int dst_dev, const void *src, int src_dev, size_t bytes,
                   void *stream) {
    if (bytes == 0) return 0;
    return (int)cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, bytes, (cudaStream_t)stream);
}

int hx_read_u64(const unsigned long long *dev_ptr, unsigned long long *host_out) {
    if (!dev_ptr || !host_out) return HX_E_INVALID;
    return (int)cudaMemcpy(host_out, dev_ptr, sizeof(*host_out), cudaMemcpyDefault);
}

}  // extern "C"
