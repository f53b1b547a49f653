// grkan_host.cu -- the reference's host-array calls (forward_tensor / backward_blocked on
// NumPy buffers, pkg/src/grkan/rational.py:325-345, backward.py:275-372) as one native
// pipeline per call: pageable host memory in, pageable host memory out.
//
// A drop-in caller holds plain host arrays, so every call pays PCIe both ways.  A call
// walks the rows in chunks through S = 3 slots:
//
//   host threads   memcpy x[, dy] chunk i  -> pinned in-slot      (T threads in parallel)
//   h2d stream     pinned in-slot           -> device in-slot
//   compute stream grkan_fwd / grkan_bwd_partials on the slot
//   d2h stream     device out-slot          -> pinned out-slot
//   host threads   memcpy pinned out-slot   -> y / dx chunk i - 2
//
// A caller buffer that is already page-locked (a torch pinned tensor behind the NumPy
// array -- what the shim allocates its outputs in, from torch's caching host
// allocator) skips its staging copy: the DMA reads or writes it in place.
//
// so the host copies of chunk i and i-2 overlap the PCIe transfers and kernels of
// chunk i-1 (PCIe is full duplex).  The backward writes per-row-block partials (the
// deterministic family, grkan_bwd_partials) and folds them once at the end with
// grkan_reduce_partials: chunks are cut on row-block boundaries, so da / db are
// bitwise those of grkan_bwd(..., GRKAN_FLAG_DETERMINISTIC) on the whole tensor,
// whatever the chunk size.  y / dx are elementwise, so EXACT stays bitwise.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/grkan_b200.h"
#include "grkan_types.h"

namespace {

// Messages land in the library's per-thread buffer (grkan_last_error()).
int hfail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return grkan::set_error(code, buf);
}
int hcuda(cudaError_t e, const char* where) {
  return hfail(GRKAN_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}
int passthrough(int rc) { return rc; }  // the callee already set the message

size_t elem_bytes(int32_t dtype) {
  return dtype == GRKAN_F32 ? 4 : dtype == GRKAN_F64 ? 8 : dtype == GRKAN_BF16 ? 2 : 0;
}
size_t coeff_bytes(int32_t dtype) { return dtype == GRKAN_F64 ? 8 : 4; }

// Fixed pool of host threads for parallel memcpy (one job at a time, caller waits).
class CopyPool {
 public:
  explicit CopyPool(int n) : n_(n < 1 ? 1 : n) {
    for (int t = 1; t < n_; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return n_; }

  // dst[0:n) = src[0:n), split into page-aligned pieces over the pool (the caller is
  // thread 0).  Pieces of >= 1 MiB: below that one thread is as fast.
  void memcpy_par(void* dst, const void* src, size_t n) {
    const size_t kMin = 1 << 20;
    int parts = static_cast<int>(std::min<size_t>(n_, (n + kMin - 1) / kMin));
    if (parts <= 1) {
      std::memcpy(dst, src, n);
      return;
    }
    size_t piece = (n + parts - 1) / parts;
    piece = (piece + 4095) & ~static_cast<size_t>(4095);
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    run(parts, [=](int k) {
      const size_t lo = static_cast<size_t>(k) * piece;
      if (lo >= n) return;
      const size_t hi = std::min(n, lo + piece);
      std::memcpy(d + lo, s + lo, hi - lo);
    });
  }

 private:
  void run(int parts, std::function<void(int)> fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = std::move(fn);
      parts_ = parts;
      pending_ = parts - 1;  // part 0 runs on the caller
      ++gen_;
    }
    cv_.notify_all();
    job_(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      std::function<void(int)> fn;
      int parts;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = job_;
        parts = parts_;
      }
      if (t < parts) {
        fn(t);
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_all();
      }
    }
  }
  int n_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(int)> job_;
  int parts_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

constexpr int kSlots = 3;

}  // namespace

struct grkan_host_ctx {
  int device = 0;
  size_t chunk_bytes = 0;  // requested staging per tensor per slot
  size_t slot_bytes = 0;   // allocated per tensor per slot (>= one row / one row block)
  CopyPool* pool = nullptr;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  void* pin_in[2][kSlots] = {};
  void* pin_out[kSlots] = {};
  void* dev_in[2][kSlots] = {};
  void* dev_out[kSlots] = {};
  cudaEvent_t ev_h2d[kSlots] = {}, ev_comp[kSlots] = {}, ev_d2h[kSlots] = {};
  // grown on demand: per-chunk status blocks, per-block partials, coefficients, da/db
  void* dev_scratch = nullptr;
  size_t scratch_bytes = 0;
  void* pin_small = nullptr;  // coefficients in, da/db and status words out
  size_t pin_small_bytes = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int grow(grkan_host_ctx* c, size_t dev_need, size_t pin_need) {
  cudaError_t e;
  if (dev_need > c->scratch_bytes) {
    if (c->dev_scratch) {
      cudaStreamSynchronize(c->comp);
      cudaFree(c->dev_scratch);
      c->dev_scratch = nullptr;
      c->scratch_bytes = 0;
    }
    e = cudaMalloc(&c->dev_scratch, dev_need);
    if (e != cudaSuccess) return hcuda(e, "cudaMalloc(scratch)");
    c->scratch_bytes = dev_need;
  }
  if (pin_need > c->pin_small_bytes) {
    if (c->pin_small) {
      cudaFreeHost(c->pin_small);
      c->pin_small = nullptr;
      c->pin_small_bytes = 0;
    }
    e = cudaHostAlloc(&c->pin_small, pin_need, cudaHostAllocDefault);
    if (e != cudaSuccess) return hcuda(e, "cudaHostAlloc(small)");
    c->pin_small_bytes = pin_need;
  }
  return GRKAN_OK;
}

// After a failed call: let every enqueued copy and kernel finish before the slots
// are reused or the caller's buffers are released.
void drain(grkan_host_ctx* c) {
  cudaStreamSynchronize(c->h2d);
  cudaStreamSynchronize(c->comp);
  cudaStreamSynchronize(c->d2h);
}

size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

int status_to_code(const grkan_device_status& s) {
  if (s.nonfinite_input) return hfail(GRKAN_ERR_NONFINITE_INPUT, "non-finite input");
  if (s.accum_overflow) return hfail(GRKAN_ERR_ACCUM_OVERFLOW, "accumulation overflow");
  return GRKAN_OK;
}

void free_slots(grkan_host_ctx* c) {
  for (int s = 0; s < kSlots; ++s) {
    for (int t = 0; t < 2; ++t) {
      if (c->pin_in[t][s]) cudaFreeHost(c->pin_in[t][s]);
      if (c->dev_in[t][s]) cudaFree(c->dev_in[t][s]);
      c->pin_in[t][s] = c->dev_in[t][s] = nullptr;
    }
    if (c->pin_out[s]) cudaFreeHost(c->pin_out[s]);
    if (c->dev_out[s]) cudaFree(c->dev_out[s]);
    c->pin_out[s] = c->dev_out[s] = nullptr;
  }
  c->slot_bytes = 0;
}

// Slots of at least `bytes` per tensor (a call whose row or row block is larger than
// the requested chunk grows them; the context is idle between calls).
int ensure_slots(grkan_host_ctx* c, size_t bytes) {
  if (bytes <= c->slot_bytes) return GRKAN_OK;
  bytes = align256(bytes);
  free_slots(c);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t r) { return (e = r) == cudaSuccess; };
  bool good = true;
  for (int s = 0; good && s < kSlots; ++s) {
    for (int t = 0; good && t < 2; ++t)
      good = ok(cudaHostAlloc(&c->pin_in[t][s], bytes, cudaHostAllocDefault)) &&
             ok(cudaMalloc(&c->dev_in[t][s], bytes));
    good = good && ok(cudaHostAlloc(&c->pin_out[s], bytes, cudaHostAllocDefault)) &&
           ok(cudaMalloc(&c->dev_out[s], bytes));
  }
  if (!good) {
    free_slots(c);
    return hcuda(e, "staging slots");
  }
  c->slot_bytes = bytes;
  return GRKAN_OK;
}

// Page-locked host memory (cudaHostAlloc / cudaHostRegister, e.g. a torch pinned
// tensor behind a NumPy array): the DMA engines can read or write it in place, so its
// chunks skip the staging copy.
bool is_pinned(const void* p, size_t n) {
  if (!p || n == 0) return false;
  cudaPointerAttributes a{}, b{};
  const char* last = static_cast<const char*>(p) + (n - 1);
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess || cudaPointerGetAttributes(&b, last) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unknown pointer
    return false;
  }
  return a.type == cudaMemoryTypeHost && b.type == cudaMemoryTypeHost;
}

// One pipelined pass.  n_in input tensors (1 forward, 2 backward), one output tensor.
// `launch(i, r0, nr, ins, out)` enqueues chunk i's kernels on c->comp.
int pipeline(grkan_host_ctx* c, int n_in, const void* const* host_in, void* host_out, int64_t rows,
             size_t row_bytes, int64_t chunk_rows,
             const std::function<int(int64_t, int64_t, int64_t, void* const*, void*)>& launch) {
  const int64_t n_chunks = (rows + chunk_rows - 1) / chunk_rows;
  const size_t total = static_cast<size_t>(rows) * row_bytes;
  bool in_pinned[2] = {false, false};
  for (int t = 0; t < n_in; ++t) in_pinned[t] = is_pinned(host_in[t], total);
  const bool out_pinned = is_pinned(host_out, total);
  cudaError_t e;
  for (int64_t i = 0; i < n_chunks + kSlots - 1; ++i) {
    if (i < n_chunks) {
      const int s = static_cast<int>(i % kSlots);
      const int64_t r0 = i * chunk_rows;
      const int64_t nr = std::min(chunk_rows, rows - r0);
      const size_t off = static_cast<size_t>(r0) * row_bytes, nb = static_cast<size_t>(nr) * row_bytes;
      if (i >= kSlots && !(in_pinned[0] && (n_in < 2 || in_pinned[1])) &&
          (e = cudaEventSynchronize(c->ev_h2d[s])) != cudaSuccess)
        return hcuda(e, "wait h2d");  // the pinned in-slot has been read by the DMA
      const void* src[2] = {nullptr, nullptr};
      for (int t = 0; t < n_in; ++t) {
        const char* h = static_cast<const char*>(host_in[t]) + off;
        if (in_pinned[t]) {
          src[t] = h;  // DMA straight from the caller's page-locked buffer
        } else {
          c->pool->memcpy_par(c->pin_in[t][s], h, nb);
          src[t] = c->pin_in[t][s];
        }
      }
      if ((e = cudaStreamWaitEvent(c->h2d, c->ev_comp[s], 0)) != cudaSuccess) return hcuda(e, "h2d wait");
      for (int t = 0; t < n_in; ++t)
        if ((e = cudaMemcpyAsync(c->dev_in[t][s], src[t], nb, cudaMemcpyHostToDevice, c->h2d)) != cudaSuccess)
          return hcuda(e, "cudaMemcpyAsync(h2d)");
      cudaEventRecord(c->ev_h2d[s], c->h2d);
      cudaStreamWaitEvent(c->comp, c->ev_h2d[s], 0);
      cudaStreamWaitEvent(c->comp, c->ev_d2h[s], 0);  // the device out-slot has been drained
      void* ins[2] = {c->dev_in[0][s], c->dev_in[1][s]};
      int rc = launch(i, r0, nr, ins, c->dev_out[s]);
      if (rc != GRKAN_OK) return passthrough(rc);
      cudaEventRecord(c->ev_comp[s], c->comp);
      cudaStreamWaitEvent(c->d2h, c->ev_comp[s], 0);
      void* dst = out_pinned ? static_cast<void*>(static_cast<char*>(host_out) + off) : c->pin_out[s];
      if ((e = cudaMemcpyAsync(dst, c->dev_out[s], nb, cudaMemcpyDeviceToHost, c->d2h)) != cudaSuccess)
        return hcuda(e, "cudaMemcpyAsync(d2h)");
      cudaEventRecord(c->ev_d2h[s], c->d2h);
    }
    const int64_t j = i - (kSlots - 1);
    if (!out_pinned && j >= 0 && j < n_chunks) {
      const int s = static_cast<int>(j % kSlots);
      const int64_t r0 = j * chunk_rows;
      const int64_t nr = std::min(chunk_rows, rows - r0);
      if ((e = cudaEventSynchronize(c->ev_d2h[s])) != cudaSuccess) return hcuda(e, "wait d2h");
      c->pool->memcpy_par(static_cast<char*>(host_out) + static_cast<size_t>(r0) * row_bytes, c->pin_out[s],
                          static_cast<size_t>(nr) * row_bytes);
    }
  }
  return GRKAN_OK;
}

int check_args(grkan_host_ctx* c, int64_t rows, int32_t d, int32_t ng, int32_t m1, int32_t n, int32_t dtype) {
  if (!c) return hfail(GRKAN_ERR_INVALID, "null host context");
  int64_t plan[6];
  int rc = grkan_plan(rows, d, ng, m1, n, dtype, plan);  // layout / degree / dtype checks
  if (rc != GRKAN_OK) return passthrough(rc);
  return GRKAN_OK;
}

}  // namespace

extern "C" {

const char* grkan_host_last_error(void) { return grkan_last_error(); }

int grkan_host_create(int32_t device, size_t chunk_bytes, int32_t threads, grkan_host_ctx** out) {
  if (!out) return hfail(GRKAN_ERR_INVALID, "null output");
  *out = nullptr;
  if (chunk_bytes == 0) chunk_bytes = 32u << 20;
  chunk_bytes = align256(chunk_bytes);
  if (threads <= 0) {
    const unsigned hc = std::thread::hardware_concurrency();
    threads = hc ? static_cast<int32_t>(std::min(hc, 16u)) : 8;
  }
  grkan_host_ctx* c = new (std::nothrow) grkan_host_ctx();
  if (!c) return hfail(GRKAN_ERR_INVALID, "out of host memory");
  c->device = device;
  c->chunk_bytes = chunk_bytes;
  DeviceGuard g(device);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t r) { return (e = r) == cudaSuccess; };
  bool good = ok(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking)) &&
              ok(cudaStreamCreateWithFlags(&c->comp, cudaStreamNonBlocking)) &&
              ok(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  for (int s = 0; good && s < kSlots; ++s)
    good = ok(cudaEventCreateWithFlags(&c->ev_h2d[s], cudaEventDisableTiming)) &&
           ok(cudaEventCreateWithFlags(&c->ev_comp[s], cudaEventDisableTiming)) &&
           ok(cudaEventCreateWithFlags(&c->ev_d2h[s], cudaEventDisableTiming));
  if (!good) {
    int rc = hcuda(e, "grkan_host_create");
    grkan_host_destroy(c);
    return rc;
  }
  int rc = ensure_slots(c, chunk_bytes);
  if (rc != GRKAN_OK) {
    grkan_host_destroy(c);
    return rc;
  }
  c->pool = new CopyPool(threads);
  *out = c;
  return GRKAN_OK;
}

int grkan_host_destroy(grkan_host_ctx* c) {
  if (!c) return GRKAN_OK;
  DeviceGuard g(c->device);
  if (c->comp) cudaStreamSynchronize(c->comp);
  if (c->h2d) cudaStreamSynchronize(c->h2d);
  if (c->d2h) cudaStreamSynchronize(c->d2h);
  free_slots(c);
  for (int s = 0; s < kSlots; ++s) {
    if (c->ev_h2d[s]) cudaEventDestroy(c->ev_h2d[s]);
    if (c->ev_comp[s]) cudaEventDestroy(c->ev_comp[s]);
    if (c->ev_d2h[s]) cudaEventDestroy(c->ev_d2h[s]);
  }
  if (c->dev_scratch) cudaFree(c->dev_scratch);
  if (c->pin_small) cudaFreeHost(c->pin_small);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->comp) cudaStreamDestroy(c->comp);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  delete c->pool;
  delete c;
  return GRKAN_OK;
}

int grkan_host_threads(const grkan_host_ctx* c) { return c && c->pool ? c->pool->size() : 0; }

int grkan_host_fwd(grkan_host_ctx* c, const void* x, void* y, const void* a, const void* b, int64_t rows,
                   int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype, uint32_t flags) {
  int rc = check_args(c, rows, d, n_groups, m1, n, dtype);
  if (rc) return rc;
  if (flags & GRKAN_FLAG_DETERMINISTIC) return hfail(GRKAN_ERR_INVALID, "DETERMINISTIC is a backward flag");
  if (rows == 0) return GRKAN_OK;
  if (!x || !y || !a || (n > 0 && !b)) return hfail(GRKAN_ERR_INVALID, "null host pointer");
  DeviceGuard g(c->device);
  const size_t es = elem_bytes(dtype), cs = coeff_bytes(dtype);
  const size_t row_bytes = static_cast<size_t>(d) * es;
  const int64_t chunk_rows = std::max<int64_t>(1, static_cast<int64_t>(c->chunk_bytes / row_bytes));
  if ((rc = ensure_slots(c, static_cast<size_t>(chunk_rows) * row_bytes)) != GRKAN_OK) return rc;
  const int64_t n_chunks = (rows + chunk_rows - 1) / chunk_rows;
  const size_t na = static_cast<size_t>(n_groups) * m1 * cs, nb = static_cast<size_t>(n_groups) * n * cs;
  const size_t st_off = align256(na) + align256(nb);
  const size_t st_bytes = static_cast<size_t>(n_chunks) * sizeof(grkan_device_status);
  if ((rc = grow(c, st_off + align256(st_bytes), std::max(st_off, st_bytes))) != GRKAN_OK) return rc;
  char* dev = static_cast<char*>(c->dev_scratch);
  char* pin = static_cast<char*>(c->pin_small);
  const bool check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
  cudaStreamSynchronize(c->comp);  // pin_small / scratch are free (a previous call may have failed midway)
  std::memcpy(pin, a, na);
  if (n > 0) std::memcpy(pin + align256(na), b, nb);
  cudaError_t e = cudaMemcpyAsync(dev, pin, st_off, cudaMemcpyHostToDevice, c->comp);
  if (e != cudaSuccess) return hcuda(e, "coefficients h2d");
  grkan_device_status* st = reinterpret_cast<grkan_device_status*>(dev + st_off);
  const void* in[1] = {x};
  rc = pipeline(c, 1, in, y, rows, row_bytes, chunk_rows,
                [&](int64_t i, int64_t, int64_t nr, void* const* ins, void* out) {
                  return grkan_fwd(ins[0], out, dev, dev + align256(na), nr, d, n_groups, m1, n, dtype, flags,
                                   check ? st + i : nullptr, c->comp);
                });
  if (rc != GRKAN_OK) {
    drain(c);
    return rc;
  }
  if (check) {
    if ((e = cudaMemcpyAsync(pin, st, st_bytes, cudaMemcpyDeviceToHost, c->comp)) != cudaSuccess)
      return hcuda(e, "status d2h");
  }
  if ((e = cudaStreamSynchronize(c->comp)) != cudaSuccess) return hcuda(e, "grkan_host_fwd");
  if ((e = cudaStreamSynchronize(c->d2h)) != cudaSuccess) return hcuda(e, "grkan_host_fwd");
  if (check) {
    grkan_device_status acc{};
    for (int64_t i = 0; i < n_chunks; ++i) acc.nonfinite_input |= reinterpret_cast<grkan_device_status*>(pin)[i].nonfinite_input;
    return status_to_code(acc);
  }
  return GRKAN_OK;
}

int grkan_host_bwd(grkan_host_ctx* c, const void* x, const void* dy, const void* a, const void* b, void* dx,
                   void* da, void* db, int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n,
                   int32_t dtype, uint32_t flags) {
  int rc = check_args(c, rows, d, n_groups, m1, n, dtype);
  if (rc) return rc;
  if (!da || (n > 0 && !db)) return hfail(GRKAN_ERR_INVALID, "null gradient pointer");
  const size_t es = elem_bytes(dtype), cs = coeff_bytes(dtype);
  const size_t na = static_cast<size_t>(n_groups) * m1 * cs, nb = static_cast<size_t>(n_groups) * n * cs;
  if (rows == 0) {  // the reference's gradients of an empty tensor: exact zeros
    std::memset(da, 0, na);
    if (n > 0) std::memset(db, 0, nb);
    return GRKAN_OK;
  }
  if (!x || !dy || !dx || !a || (n > 0 && !b)) return hfail(GRKAN_ERR_INVALID, "null host pointer");
  DeviceGuard g(c->device);
  const size_t row_bytes = static_cast<size_t>(d) * es;
  const int64_t rb = grkan_det_block_rows(d, n_groups, dtype);
  if (rb <= 0) return hfail(GRKAN_ERR_LAYOUT, "layout mismatch");
  // chunks on row-block boundaries (at least one block): the fold is chunk-size invariant
  const int64_t chunk_rows = std::max<int64_t>(1, static_cast<int64_t>(c->chunk_bytes / row_bytes) / rb) * rb;
  if ((rc = ensure_slots(c, static_cast<size_t>(chunk_rows) * row_bytes)) != GRKAN_OK) return rc;
  const int64_t n_chunks = (rows + chunk_rows - 1) / chunk_rows;
  const int64_t n_blocks = (rows + rb - 1) / rb;
  const size_t blk_bytes = static_cast<size_t>(n_groups) * (m1 + n) * cs;
  // scratch: a | b | da | db | status[n_chunks + 1] | partials[n_blocks]
  const size_t o_b = align256(na), o_da = o_b + align256(nb), o_db = o_da + align256(na);
  const size_t o_st = o_db + align256(nb);
  const size_t st_bytes = static_cast<size_t>(n_chunks + 1) * sizeof(grkan_device_status);
  const size_t o_part = o_st + align256(st_bytes);
  const size_t part_bytes = static_cast<size_t>(n_blocks) * blk_bytes;
  const size_t small = o_part;  // pinned mirror of everything but the partials
  if ((rc = grow(c, o_part + part_bytes, small)) != GRKAN_OK) return rc;
  char* dev = static_cast<char*>(c->dev_scratch);
  char* pin = static_cast<char*>(c->pin_small);
  cudaStreamSynchronize(c->comp);
  std::memcpy(pin, a, na);
  if (n > 0) std::memcpy(pin + o_b, b, nb);
  cudaError_t e = cudaMemcpyAsync(dev, pin, o_da, cudaMemcpyHostToDevice, c->comp);
  if (e != cudaSuccess) return hcuda(e, "coefficients h2d");
  grkan_device_status* st = reinterpret_cast<grkan_device_status*>(dev + o_st);
  const bool check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
  const uint32_t kflags = (flags & ~GRKAN_FLAG_DETERMINISTIC);
  const void* in[2] = {x, dy};
  rc = pipeline(c, 2, in, dx, rows, row_bytes, chunk_rows,
                [&](int64_t i, int64_t r0, int64_t nr, void* const* ins, void* out) {
                  char* part = dev + o_part + static_cast<size_t>(r0 / rb) * blk_bytes;
                  const size_t pb = static_cast<size_t>((nr + rb - 1) / rb) * blk_bytes;
                  return grkan_bwd_partials(ins[0], ins[1], dev, dev + o_b, out, part, pb, nr, d, n_groups, m1, n,
                                            dtype, kflags, check ? st + 1 + i : nullptr, c->comp);
                });
  if (rc != GRKAN_OK) {
    drain(c);
    return rc;
  }
  rc = grkan_reduce_partials(dev + o_part, n_blocks, n_groups, m1, n, dev + o_da, dev + o_db, dtype, st, c->comp);
  if (rc != GRKAN_OK) return passthrough(rc);
  if ((e = cudaMemcpyAsync(pin + o_da, dev + o_da, o_part - o_da, cudaMemcpyDeviceToHost, c->comp)) != cudaSuccess)
    return hcuda(e, "da/db d2h");
  if ((e = cudaStreamSynchronize(c->comp)) != cudaSuccess) return hcuda(e, "grkan_host_bwd");
  if ((e = cudaStreamSynchronize(c->d2h)) != cudaSuccess) return hcuda(e, "grkan_host_bwd");
  const grkan_device_status* hs = reinterpret_cast<const grkan_device_status*>(pin + o_st);
  grkan_device_status acc{};
  acc.accum_overflow = hs[0].accum_overflow;
  if (check)
    for (int64_t i = 0; i < n_chunks; ++i) acc.nonfinite_input |= hs[1 + i].nonfinite_input;
  if ((rc = status_to_code(acc)) != GRKAN_OK) return rc;
  std::memcpy(da, pin + o_da, na);
  if (n > 0) std::memcpy(db, pin + o_db, nb);
  return GRKAN_OK;
}

}  // extern "C"
