// tnsr.hpp -- TNSR tensor files (tensor_io.hpp:9-11) on the host and straight into HBM.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace lmra_host {

struct TnsrHeader {
  std::vector<uint64_t> dims;
  size_t data_offset = 0;  // bytes before the values
  size_t count = 0;        // number of values
};

TnsrHeader tnsr_read_header(const std::string& path);
void tnsr_load_host(const std::string& path, double* out);
// values -> device memory dst (count doubles), chunked through pinned staging on stream st
void tnsr_load_device(const std::string& path, double* dst, cudaStream_t st);
void tnsr_save(const std::string& path, const std::vector<uint64_t>& dims, const double* values, bool device,
               cudaStream_t st);

}  // namespace lmra_host
