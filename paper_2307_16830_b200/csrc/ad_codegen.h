// Pattern compiler interface (ad_codegen.cpp): tape -> CUDA source -> NVRTC.
#pragma once

#include <string>
#include <vector>

#include "internal.h"

namespace gn {

constexpr int kPatternThreads = 128;

// CUDA source with one device function per distinct pattern and a fused
// record kernel `gn_ad_patterns`; pattern_of[b] = pattern id of block b
std::string pattern_source(const Model &M, std::vector<int> &pattern_of);
// compiled kernel (a CUfunction), cached process-wide by source; nullptr
// with `err` set when NVRTC or the driver API is unavailable
void *compile_patterns(const std::string &src, std::string &err);
bool launch_patterns(void *fn, unsigned grid, void *stream, void **args, unsigned batch = 1);

}  // namespace gn
