// Minimal NCCL binding resolved at run time with dlopen/dlsym.
//
// libluffy does not link NCCL: it binds to the libnccl.so.2 already loaded in the process (the one
// PyTorch's ProcessGroupNCCL uses), else loads it by soname.  That keeps the library loadable on a
// machine without NCCL/GPU (the CPU test suite) and guarantees one NCCL version per process.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace luffy {
namespace nccl {

typedef int Result;  // ncclResult_t, 0 = ncclSuccess
typedef struct Comm* CommPtr;
typedef struct { char internal[128]; } UniqueId;
enum DataType { kUint8 = 1, kInt32 = 2 };

struct Api {
  Result (*GetUniqueId)(UniqueId*);
  Result (*CommInitRank)(CommPtr*, int, UniqueId, int);
  Result (*CommDestroy)(CommPtr);
  Result (*AllGather)(const void*, void*, size_t, int, CommPtr, cudaStream_t);
  Result (*Send)(const void*, size_t, int, int, CommPtr, cudaStream_t);
  Result (*Recv)(void*, size_t, int, int, CommPtr, cudaStream_t);
  Result (*GroupStart)();
  Result (*GroupEnd)();
  const char* (*GetErrorString)(Result);
};

// nullptr if NCCL cannot be loaded (luffy_last_error explains).
const Api* api();

}  // namespace nccl
}  // namespace luffy
