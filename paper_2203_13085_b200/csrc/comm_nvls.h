// NVLink SHARP (in-switch reduction) support of the communicator: multicast setup
// through the driver API and the tolerance-mode mean kernel (comm_nvls.cu).
#ifndef LASGD_COMM_NVLS_H
#define LASGD_COMM_NVLS_H

#include "comm_launch.cuh"

namespace lasgd {

struct NvlsState;
// 1 if `device` supports multicast objects exportable as POSIX file descriptors.
int nvls_supported(int device);
// Granularity-rounded multicast object for `world` devices of payload_bytes each.  With
// fd_out the object is created and exported (the creating rank); without, the state only
// records the size and waits for nvls_import.
int nvls_create(NvlsState** out, int device, int world, size_t payload_bytes, int* fd_out);
int nvls_import(NvlsState* s, int fd);
int nvls_add_device(NvlsState* s);
// Allocate this rank's physical memory, bind it and map the unicast and multicast views.
int nvls_bind(NvlsState* s, void** uc, void** mc);
void nvls_destroy(NvlsState* s);
int launch_nvls_mean(int P, const CommArgs& a, const void* mc_src, void* mc_dst, int nblocks, cudaStream_t s);

}  // namespace lasgd

#endif  // LASGD_COMM_NVLS_H
