// SPDX-License-Identifier: Apache-2.0
// Kernel launch with the programmatic-stream-serialization attribute (PDL), see pipeline.cuh.
#pragma once

#include <cuda_runtime.h>
#include <cstdlib>

namespace trg {

inline bool pdl_enabled() {
    static const bool on = getenv("TRG_NO_PDL") == nullptr;
    return on;
}

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace trg
