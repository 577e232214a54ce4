// C ABI of the device layer: streams, events, stream-ordered memory.
// Replaces the simulated device backend (p/core/src/device.cpp:45-348):
// the command DAG of dependency callbacks becomes CUDA stream order plus
// cudaStreamWaitEvent, worker threads become the GPU, Buffer storage becomes
// a stream-ordered pool allocation.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../../include/ndx.h"

extern "C" {

const char* ndx_error_string(int code) {
  switch (code) {
    case 0: return "success";
    case NDX_E_INVALID: return "ndx: invalid argument";
    case NDX_E_TOO_LARGE: return "ndx: input exceeds the u32 index format (n >= 2^31)";
    case NDX_E_NO_DEVICE: return "ndx: no CUDA device";
    default: return cudaGetErrorString(static_cast<cudaError_t>(code));
  }
}

int ndx_abi_version(void) { return 1; }

int ndx_device_count(int* count) {
  if (!count) return NDX_E_INVALID;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    *count = 0;
    return 0;
  }
  return e;
}

int ndx_device_open(int ordinal) {
  int count = 0;
  int rc = ndx_device_count(&count);
  if (rc) return rc;
  if (count == 0) return NDX_E_NO_DEVICE;
  if (ordinal < 0 || ordinal >= count) return NDX_E_INVALID;
  cudaError_t e = cudaSetDevice(ordinal);
  if (e) return e;
  // Keep freed blocks in the pool: buffers churn every build.
  cudaMemPool_t pool;
  if ((e = cudaDeviceGetDefaultMemPool(&pool, ordinal))) return e;
  uint64_t keep = UINT64_MAX;
  return cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
}

int ndx_device_bind(int ordinal) { return cudaSetDevice(ordinal); }

int ndx_malloc_shared(void** p, size_t bytes) {
  if (!p) return NDX_E_INVALID;
  return cudaMalloc(p, bytes ? bytes : 1);
}
int ndx_free_shared(void* p) { return cudaFree(p); }
int ndx_ipc_handle(const void* p, void* handle64) {
  if (!p || !handle64) return NDX_E_INVALID;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(p));
  if (!e) memcpy(handle64, &h, sizeof h);
  return e;
}
int ndx_ipc_open(const void* handle64, void** p) {
  if (!handle64 || !p) return NDX_E_INVALID;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  return cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess);
}
int ndx_ipc_close(void* p) { return cudaIpcCloseMemHandle(p); }

int ndx_device_sm_count(int ordinal, int* sms) {
  if (!sms) return NDX_E_INVALID;
  return cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, ordinal);
}

int ndx_device_synchronize(void) { return cudaDeviceSynchronize(); }

int ndx_stream_create(void** stream) {
  if (!stream) return NDX_E_INVALID;
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  *stream = e ? nullptr : s;
  return e;
}
int ndx_stream_destroy(void* stream) {
  return cudaStreamDestroy(static_cast<cudaStream_t>(stream));
}
int ndx_stream_synchronize(void* stream) {
  return cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
}
int ndx_stream_query(void* stream) {
  cudaError_t e = cudaStreamQuery(static_cast<cudaStream_t>(stream));
  return e == cudaErrorNotReady ? 1 : int(e);
}

int ndx_event_create(void** event, int timing) {
  if (!event) return NDX_E_INVALID;
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, timing ? cudaEventDefault : cudaEventDisableTiming);
  *event = e ? nullptr : ev;
  return e;
}
int ndx_event_destroy(void* event) { return cudaEventDestroy(static_cast<cudaEvent_t>(event)); }
int ndx_event_record(void* event, void* stream) {
  return cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream));
}
int ndx_event_query(void* event) {
  cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
  return e == cudaErrorNotReady ? 1 : int(e);
}
int ndx_event_synchronize(void* event) {
  return cudaEventSynchronize(static_cast<cudaEvent_t>(event));
}
int ndx_stream_wait_event(void* stream, void* event) {
  return cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0);
}
int ndx_event_elapsed_ms(void* start, void* stop, float* ms) {
  if (!ms) return NDX_E_INVALID;
  return cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(stop));
}

int ndx_malloc_async(void** d_ptr, size_t bytes, void* stream) {
  if (!d_ptr) return NDX_E_INVALID;
  if (bytes == 0) bytes = 256;  // every buffer gets a distinct address
  return cudaMallocAsync(d_ptr, bytes, static_cast<cudaStream_t>(stream));
}
int ndx_free_async(void* d_ptr, void* stream) {
  if (!d_ptr) return 0;
  return cudaFreeAsync(d_ptr, static_cast<cudaStream_t>(stream));
}
int ndx_memset_async(void* d_ptr, int value, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  return cudaMemsetAsync(d_ptr, value, bytes, static_cast<cudaStream_t>(stream));
}
int ndx_host_alloc(void** h_ptr, size_t bytes) {
  if (!h_ptr) return NDX_E_INVALID;
  return cudaMallocHost(h_ptr, bytes ? bytes : 1);
}
int ndx_host_free(void* h_ptr) { return h_ptr ? cudaFreeHost(h_ptr) : 0; }

int ndx_memcpy_h2d_async(void* d_dst, const void* h_src, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  return cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice,
                         static_cast<cudaStream_t>(stream));
}
int ndx_memcpy_d2h_async(void* h_dst, const void* d_src, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  return cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost,
                         static_cast<cudaStream_t>(stream));
}
int ndx_memcpy_d2d_async(void* d_dst, const void* d_src, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  return cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDeviceToDevice,
                         static_cast<cudaStream_t>(stream));
}

}  // extern "C"
