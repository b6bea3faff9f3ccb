// GPUs the drop-in spreads its work over: XYZ_GPU_DEVICES="0,1,2,3" (a
// comma-separated list of CUDA ordinals), default every visible device. A
// search replicates X on each and shards its repetitions over them
// (xyzb_problem.devices) — the GPU replacement of run_pass's thread waves
// (search.cpp:59-111); SearchConfig::threads stays accepted and unused.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "xyzb.h"

namespace xyz {

inline std::vector<int32_t> gpu_devices() {
    std::vector<int32_t> out;
    if (const char* e = std::getenv("XYZ_GPU_DEVICES")) {
        std::string s = e;
        size_t at = 0;
        while (at < s.size()) {
            const size_t comma = s.find(',', at);
            const std::string tok = s.substr(at, comma == std::string::npos ? std::string::npos : comma - at);
            if (!tok.empty()) out.push_back(static_cast<int32_t>(std::strtol(tok.c_str(), nullptr, 10)));
            if (comma == std::string::npos) break;
            at = comma + 1;
        }
    }
    if (out.empty()) {
        const int n = xyzb_device_count();
        for (int d = 0; d < n; ++d) out.push_back(d);
    }
    if (out.empty()) out.push_back(0);  // no device: dataset creation reports the CUDA error
    return out;
}

} // namespace xyz
