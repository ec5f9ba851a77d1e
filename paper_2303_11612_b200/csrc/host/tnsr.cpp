// tnsr.cpp -- the reference's binary tensor format "TNSR" (tensor_io.hpp:9-11,
// tensor_io.cpp:27-69), read straight into device memory.
//
// Format: magic "TNSR", u32 version (= 1), u32 order N, N u64 dimensions, then the values as
// little-endian IEEE-754 float64 in storage order (first index fastest).  Round trips are
// bit-exact.  Error messages are the reference's (std::runtime_error texts).
//
// Device load: the values are read with pread() in chunks into two pinned staging buffers
// and copied to the device on a stream, so the file read of chunk k+1 overlaps the H2D copy
// of chunk k (an 8 GB tensor never needs a pageable 8 GB host copy).
#include "tnsr.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace lmra_host {

namespace {

constexpr char kMagic[4] = {'T', 'N', 'S', 'R'};
constexpr uint32_t kVersion = 1;
constexpr size_t kChunkBytes = size_t(64) << 20;  // staging chunk (two in flight)

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// pread until n bytes or EOF; returns bytes read
size_t pread_full(int fd, void* buf, size_t n, off_t off) {
  size_t got = 0;
  while (got < n) {
    const ssize_t r = ::pread(fd, static_cast<char*>(buf) + got, n - got, off + (off_t)got);
    if (r < 0) {
      if (errno == EINTR) continue;
      throw std::runtime_error(std::string("read failure on tensor file: ") + std::strerror(errno));
    }
    if (r == 0) break;
    got += (size_t)r;
  }
  return got;
}

void read_exact(int fd, void* buf, size_t n, off_t off, const char* what) {
  if (pread_full(fd, buf, n, off) != n)
    throw std::runtime_error(std::string("tensor file truncated while reading ") + what);
}

}  // namespace

TnsrHeader tnsr_read_header(const std::string& path) {  // tensor_io.cpp:50-66
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  if (f.fd < 0) throw std::runtime_error("cannot open tensor file: " + path);
  char magic[4];
  read_exact(f.fd, magic, 4, 0, "magic");
  if (std::memcmp(magic, kMagic, 4) != 0) throw std::runtime_error("bad magic in tensor file: " + path);
  uint32_t version = 0, order = 0;
  read_exact(f.fd, &version, 4, 4, "version");
  if (version != kVersion) throw std::runtime_error("unsupported tensor file version " + std::to_string(version));
  read_exact(f.fd, &order, 4, 8, "order");
  TnsrHeader h;
  h.dims.resize(order);
  for (uint32_t k = 0; k < order; ++k) {
    uint64_t v = 0;
    read_exact(f.fd, &v, 8, 12 + 8 * (off_t)k, "dimensions");
    h.dims[k] = v;
  }
  h.data_offset = 12 + 8 * (size_t)order;
  h.count = 1;
  for (uint64_t d : h.dims) h.count *= d;
  return h;
}

void tnsr_load_host(const std::string& path, double* out) {
  const TnsrHeader h = tnsr_read_header(path);
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  if (f.fd < 0) throw std::runtime_error("cannot open tensor file: " + path);
  read_exact(f.fd, out, h.count * sizeof(double), (off_t)h.data_offset, "values");
}

void tnsr_load_device(const std::string& path, double* dst, cudaStream_t st) {
  const TnsrHeader h = tnsr_read_header(path);
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  if (f.fd < 0) throw std::runtime_error("cannot open tensor file: " + path);
  const size_t total = h.count * sizeof(double);
  if (total == 0) return;
  const size_t chunk = std::min(kChunkBytes, total);
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  struct Cleanup {
    void** stage;
    cudaEvent_t* done;
    ~Cleanup() {
      for (int i = 0; i < 2; ++i) {
        if (done[i]) {
          cudaEventSynchronize(done[i]);
          cudaEventDestroy(done[i]);
        }
        if (stage[i]) cudaFreeHost(stage[i]);
      }
    }
  } cleanup{stage, done};
  for (int i = 0; i < 2; ++i) {
    if (cudaMallocHost(&stage[i], chunk) != cudaSuccess) throw std::runtime_error("cudaMallocHost failed");
    if (cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess)
      throw std::runtime_error("cudaEventCreate failed");
  }
  size_t off = 0;
  for (int k = 0; off < total; ++k, off += chunk) {
    const int b = k & 1;
    const size_t n = std::min(chunk, total - off);
    if (cudaEventSynchronize(done[b]) != cudaSuccess)  // the copy that last used this buffer
      throw std::runtime_error("cudaEventSynchronize failed");
    read_exact(f.fd, stage[b], n, (off_t)(h.data_offset + off), "values");
    if (cudaMemcpyAsync(reinterpret_cast<char*>(dst) + off, stage[b], n, cudaMemcpyHostToDevice, st) != cudaSuccess)
      throw std::runtime_error("H2D copy of tensor file failed");
    if (cudaEventRecord(done[b], st) != cudaSuccess) throw std::runtime_error("cudaEventRecord failed");
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("H2D copy of tensor file failed");
}

void tnsr_save(const std::string& path, const std::vector<uint64_t>& dims, const double* values,
               bool device, cudaStream_t st) {  // tensor_io.cpp:27-47
  Fd f;
  f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (f.fd < 0) throw std::runtime_error("cannot open tensor file for writing: " + path);
  std::vector<char> head(12 + 8 * dims.size());
  std::memcpy(head.data(), kMagic, 4);
  const uint32_t version = kVersion, order = (uint32_t)dims.size();
  std::memcpy(head.data() + 4, &version, 4);
  std::memcpy(head.data() + 8, &order, 4);
  size_t count = 1;
  for (size_t k = 0; k < dims.size(); ++k) {
    std::memcpy(head.data() + 12 + 8 * k, &dims[k], 8);
    count *= dims[k];
  }
  auto write_all = [&](const void* p, size_t n) {
    size_t put = 0;
    while (put < n) {
      const ssize_t r = ::write(f.fd, static_cast<const char*>(p) + put, n - put);
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) throw std::runtime_error("write failure on tensor file: " + path);
      put += (size_t)r;
    }
  };
  write_all(head.data(), head.size());
  const size_t total = count * sizeof(double);
  if (!device) {
    write_all(values, total);
    return;
  }
  const size_t chunk = std::min(kChunkBytes, std::max<size_t>(total, 1));
  void* stage = nullptr;
  if (cudaMallocHost(&stage, chunk) != cudaSuccess) throw std::runtime_error("cudaMallocHost failed");
  struct Free {
    void* p;
    ~Free() { cudaFreeHost(p); }
  } fr{stage};
  for (size_t off = 0; off < total; off += chunk) {
    const size_t n = std::min(chunk, total - off);
    if (cudaMemcpyAsync(stage, reinterpret_cast<const char*>(values) + off, n, cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      throw std::runtime_error("D2H copy for tensor file failed");
    write_all(stage, n);
  }
}

}  // namespace lmra_host
