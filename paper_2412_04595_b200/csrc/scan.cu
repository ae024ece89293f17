// Device-wide exclusive prefix sums for the counting sorts of S1 (CUB decoupled look-back
// scan: library plumbing for the bucket offsets, not part of the method's arithmetic).
#include <cub/device/device_scan.cuh>

#include "launch.h"

namespace sog {

// in[0..n] with in[n] == 0  ->  out[0..n], out[n] = sum in[0..n)
size_t scan_temp_bytes(int n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int*)nullptr, (int*)nullptr, n + 1);
    return bytes;
}

int launch_exclusive_scan(const int* in, int* out, int n, void* temp, size_t temp_bytes, cudaStream_t st) {
    size_t bytes = temp_bytes;
    if (cub::DeviceScan::ExclusiveSum(temp, bytes, in, out, n + 1, st) != cudaSuccess) return 2;
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace sog

#include <cub/device/device_select.cuh>

namespace sog {

// stable compaction of the flagged particles (x-slab halos)
size_t select_temp_bytes(int n) {
    size_t bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, bytes, (const d4*)nullptr, (const int*)nullptr, (d4*)nullptr, (int*)nullptr, n);
    return bytes;
}

int launch_select_flagged(const d4* in, const int* flags, d4* out, int* nsel, int n, void* temp, size_t temp_bytes,
                          cudaStream_t st) {
    size_t bytes = temp_bytes;
    if (cub::DeviceSelect::Flagged(temp, bytes, in, flags, out, nsel, n, st) != cudaSuccess) return 2;
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace sog
