// tmap.cuh — host access to the driver's cuTensorMapEncodeTiled (TMA descriptors),
// resolved once through the runtime (no -lcuda link dependency).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

namespace dmpq {
PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn();   // null if the driver does not provide it
}
