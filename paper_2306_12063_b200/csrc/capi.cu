// capi.cu -- the extern "C" boundary of libqcb200.so (declared in include/qcb200.h).
//
// Validation mirrors the reference's decoder._check_block / decode_block
// (/root/reference/pkg/src/qcldpc/decoder.py:179-186, 217-258): errors are
// reported before any work is queued, the kernels themselves never fail on
// data.  Outputs are caller-owned, exactly like the reference kernel boundary
// (_kernels.py:17-19: hard/iters/conv are written in place).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <immintrin.h>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <condition_variable>
#include <thread>
#include <vector>

#include "../../include/qcb200.h"
#include "common.cuh"
#include "kernels.h"

using namespace qcb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail((int)e, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

struct DeviceTables {
  int32_t* d = nullptr;  // tier_start (mb+1) | ent_j (ne) | ent_e (ne)
};

}  // namespace

struct qc_code_s {
  int32_t mb = 0, nb = 0, kb = 0, z = 0, n = 0, ne = 0, max_deg = 0;
  int32_t structure = -1;            // index into kStructureMasks, -1 = generic only
  bool native = false;               // structure's own Z0 and SHIFT0 (compile-time shift kernels)
  bool scaled = false;               // WiMAX structure with the standard scaled shifts at z
  std::vector<int32_t> shifts;       // mb x nb
  std::vector<int32_t> tier_start, ent_j, ent_e;
  int32_t enc_y = -1, enc_hb = -1;   // encoder plan (find_y, encoder.py:39-46), -1 if malformed
  std::mutex mu;
  std::map<int, DeviceTables> dev;   // generic decoder tables per device

  std::vector<int32_t> host_tables;  // tier_start | ent_j | ent_e (the upload source, kept alive)

  // Generic-kernel tables on `device`: uploaded once (qc_code_create does it
  // eagerly for the current device), stream ordered on `stream` otherwise.
  // Refused inside a CUDA graph capture: cudaMalloc is not capturable.
  const int32_t* tables(int device, cudaStream_t stream, cudaError_t* err, bool* capturing) {
    std::lock_guard<std::mutex> lk(mu);
    *capturing = false;
    auto it = dev.find(device);
    if (it != dev.end()) return it->second.d;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    *err = cudaStreamIsCapturing(stream, &cs);
    if (*err != cudaSuccess) return nullptr;
    if (cs != cudaStreamCaptureStatusNone) { *capturing = true; return nullptr; }
    if (host_tables.empty()) {
      host_tables = tier_start;
      host_tables.insert(host_tables.end(), ent_j.begin(), ent_j.end());
      host_tables.insert(host_tables.end(), ent_e.begin(), ent_e.end());
    }
    int32_t* d = nullptr;
    *err = cudaMalloc(&d, host_tables.size() * sizeof(int32_t));
    if (*err != cudaSuccess) return nullptr;
    *err = cudaMemcpyAsync(d, host_tables.data(), host_tables.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                           stream);
    if (*err != cudaSuccess) { cudaFree(d); return nullptr; }
    dev[device].d = d;
    return d;
  }
};

namespace {

int build_code(int32_t mb, int32_t nb, int32_t z, const int32_t* shifts, qc_code_t* out) {
  if (!out) return fail(QC_EINVAL, "out is NULL");
  *out = nullptr;
  if (!shifts || mb < 1 || nb <= mb || z < 1) return fail(QC_EINVAL, "bad code shape mb=%d nb=%d z=%d", mb, nb, z);
  if ((int64_t)nb * z > (1 << 30)) return fail(QC_EINVAL, "code too long");
  std::unique_ptr<qc_code_s> c(new (std::nothrow) qc_code_s());
  if (!c) return fail(QC_ENOMEM, "out of host memory");
  c->mb = mb; c->nb = nb; c->kb = nb - mb; c->z = z; c->n = nb * z;
  c->shifts.assign(shifts, shifts + (size_t)mb * nb);
  c->tier_start.push_back(0);
  for (int i = 0; i < mb; ++i) {
    int deg = 0;
    for (int j = 0; j < nb; ++j) {
      const int e = shifts[i * nb + j];
      if (e < -1 || e >= z) return fail(QC_EINVAL, "shift %d at (%d,%d) outside [-1, %d)", e, i, j, z);
      if (e >= 0) { c->ent_j.push_back(j); c->ent_e.push_back(e); ++deg; }
    }
    if (deg > kMaxDeg) return fail(QC_EUNSUPPORTED, "row degree %d > 32 (sign bitmap width)", deg);
    c->max_deg = std::max(c->max_deg, deg);
    c->tier_start.push_back((int32_t)c->ent_j.size());
  }
  c->ne = (int32_t)c->ent_j.size();
  // specialised structure?
  for (int s = 0; s < kNumStructures; ++s) {
    const StructureMask& m = kStructureMasks[s];
    if (m.mb != mb || m.nb != nb) continue;
    bool same = true;
    for (int i = 0; i < mb && same; ++i) {
      unsigned row = 0;
      for (int j = 0; j < nb; ++j) row |= (shifts[i * nb + j] >= 0 ? 1u : 0u) << j;
      same = row == m.rows[i];
    }
    if (same && z * 1 <= 384) { c->structure = s; break; }
  }
  if (c->structure >= 0) c->native = spec_is_native(c->structure, z, c->ent_e.data(), c->ne);
  if (c->structure >= 0) c->scaled = spec_is_scaled(c->structure, z, c->ent_e.data(), c->ne);
  // encoder plan: the single interior non-negative entry of the h_b column
  if (mb >= 3) {
    int y = -1, cnt = 0;
    for (int i = 1; i < mb - 1; ++i)
      if (shifts[i * nb + c->kb] >= 0) { y = i; ++cnt; }
    if (cnt == 1) { c->enc_y = y; c->enc_hb = shifts[y * nb + c->kb]; }
  }
  *out = c.release();
  return QC_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Codewords per CTA of the generic kernel, 0 if one codeword does not fit in shared memory.
int generic_cw_per_cta(const qc_code_s* c, int elem) {
  int g = std::max(1, std::min(64, 256 / std::max(1, c->z)));
  const size_t limit = 160 * 1024;
  while (g > 1 && generic_smem_bytes(g, c->n, c->mb * c->z, elem) > limit) --g;
  return generic_smem_bytes(g, c->n, c->mb * c->z, elem) > 227 * 1024 ? 0 : g;
}

template <typename T>
int decode_device(qc_code_t c, const T* llr, int64_t w, int32_t max_iters, int32_t early_term,
                  uint8_t* hard, int32_t hard_packed, int32_t* iters, uint8_t* conv, T* post,
                  cudaStream_t stream) {
  if (!c) return fail(QC_EINVAL, "code is NULL");
  if (w < 0 || max_iters < 0) return fail(QC_EINVAL, "w=%lld max_iters=%d", (long long)w, max_iters);
  if (w == 0) return QC_OK;
  if (!llr || !hard || !iters || !conv) return fail(QC_EINVAL, "NULL buffer");
  if (w > (int64_t)1 << 40) return fail(QC_EINVAL, "batch too large");
  const int elem = (int)sizeof(T);
  cudaError_t e;
  if (c->structure >= 0) {
    SpecArgs a;
    memset(&a, 0, sizeof a);
    a.llr = llr; a.hard = hard; a.iters = iters; a.conv = conv; a.post = post;
    a.w = w; a.n = c->n; a.z = c->z; a.max_iters = max_iters; a.early_term = early_term ? 1 : 0;
    a.hard_packed = hard_packed ? 1 : 0;
    a.native = c->native ? 1 : 0;
    a.scaled = (!c->native && c->scaled) ? 1 : 0;
#if QCB_DEBUG_CHECKS
    static const int inject = getenv("QCB_DEBUG_INJECT") ? 1 : 0;   // negative control of debug_checks.cuh
    a.dbg_inject = inject;
#endif
    spec_plan(c->structure, elem, c->z, (a.native || a.scaled) ? 1 : 0, w, &a.pairs, &a.tmem_cols, &a.pair16);
    const int cell = a.pair16 ? 4 : elem;                  // int16 pairs share one 4-byte cell
    a.k_one = 1u; a.k_sign = 0x80000000u; a.k_shr = 0x80000001u; a.k_neg1 = 0xFFFFFFFFu; a.k_lane1 = 0x00010001u;
    for (int i = 0; i < c->ne; ++i) {
      a.off[i] = (c->ent_j[i] * c->z + c->ent_e[i]) * cell;   // cell (c = r + e, j) at 4 (j Z + c)
      a.thr[i] = c->z - c->ent_e[i];                      // row r wraps when r >= Z - e
    }
    e = launch_spec(c->structure, elem, a, stream);
    if (e != cudaSuccess) return cuda_fail(e, "decode (specialised kernel)");
    return QC_OK;
  }
  int device = 0;
  e = cudaGetDevice(&device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  bool capturing = false;
  const int32_t* tab = c->tables(device, stream, &e, &capturing);
  if (capturing)
    return fail(QC_EINVAL, "first use of a generic code on device %d inside a CUDA graph capture: decode once "
                "before capturing (qc_code_create uploads the tables for the current device)", device);
  if (!tab) return cuda_fail(e, "uploading code tables");
  GenericArgs a;
  memset(&a, 0, sizeof a);
  a.llr = llr; a.hard = hard; a.iters = iters; a.conv = conv; a.post = post;
  a.w = w; a.n = c->n; a.z = c->z; a.mb = c->mb; a.max_iters = max_iters;
  a.early_term = early_term ? 1 : 0; a.hard_packed = hard_packed ? 1 : 0;
  a.tier_start = tab; a.ent_j = tab + c->mb + 1; a.ent_e = tab + c->mb + 1 + c->ne;
  const int g = generic_cw_per_cta(c, elem);
  if (g < 1) return fail(QC_EUNSUPPORTED, "one codeword (N=%d) does not fit in shared memory", c->n);
  a.cw_per_cta = g;
  e = launch_generic(a, elem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "decode (generic kernel)");
  return QC_OK;
}

// ---- host-buffer path: cached codes, device workspace, pinned staging ----------

// Staging copies with non-temporal (streaming) stores: the destination is not
// read back by this process soon (the DMA engine reads the pinned slot; the
// caller reads its output array later), and a regular store first reads the
// line for ownership -- 4 memory passes per byte instead of 3.  AVX-512 / AVX2
// selected at run time; plain memcpy otherwise.  QCB_NT_COPY=0 turns it off.
__attribute__((target("avx512f"))) static void copy_nt512(char* d, const char* s, size_t n) {
  while (n && (reinterpret_cast<uintptr_t>(d) & 63)) { *d++ = *s++; --n; }
  for (; n >= 256; n -= 256, d += 256, s += 256) {
    const __m512i a = _mm512_loadu_si512(s), b = _mm512_loadu_si512(s + 64);
    const __m512i c = _mm512_loadu_si512(s + 128), e = _mm512_loadu_si512(s + 192);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d), a);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + 64), b);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + 128), c);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + 192), e);
  }
  _mm_sfence();
  if (n) memcpy(d, s, n);
}
__attribute__((target("avx2"))) static void copy_nt256(char* d, const char* s, size_t n) {
  while (n && (reinterpret_cast<uintptr_t>(d) & 31)) { *d++ = *s++; --n; }
  for (; n >= 128; n -= 128, d += 128, s += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 96), e);
  }
  _mm_sfence();
  if (n) memcpy(d, s, n);
}
static void stage_copy(void* dst, const void* src, size_t n) {
  static const int mode = [] {
    const char* e = getenv("QCB_NT_COPY");
    if (e && e[0] == '0') return 0;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") ? 2 : (__builtin_cpu_supports("avx2") ? 1 : 0);
  }();
  if (mode == 2 && n >= 4096) copy_nt512(static_cast<char*>(dst), static_cast<const char*>(src), n);
  else if (mode == 1 && n >= 4096) copy_nt256(static_cast<char*>(dst), static_cast<const char*>(src), n);
  else memcpy(dst, src, n);
}

// A small persistent pool of host threads for the staging copies between the
// caller's (pageable) arrays and the pinned slots: one memcpy thread moves
// ~6-10 GB/s, a PCIe 5 x16 link ~50 GB/s per direction.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();   // never destroyed: threads outlive static teardown
    return *p;
  }
  struct Task { void* dst; const void* src; size_t n; };
  // Run every task split into ~equal pieces over the pool; returns when all are done.
  void run(const std::vector<Task>& tasks) {
    size_t total = 0;
    for (const Task& t : tasks) total += t.n;
    if (total == 0) return;
    std::vector<Task> pieces;
    const size_t piece = std::max<size_t>(1 << 20, (total + 4 * nthreads_ - 1) / (4 * nthreads_));
    for (const Task& t : tasks)
      for (size_t o = 0; o < t.n; o += piece)
        pieces.push_back({static_cast<char*>(t.dst) + o, static_cast<const char*>(t.src) + o,
                          std::min(piece, t.n - o)});
    if (nthreads_ <= 1 || pieces.size() == 1) {
      for (const Task& p : pieces) stage_copy(p.dst, p.src, p.n);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    work_ = &pieces;
    next_ = 0;
    left_ = pieces.size();
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    drain();                                  // the caller works too
    lk.lock();
    done_cv_.wait(lk, [&] { return left_ == 0; });
    work_ = nullptr;
  }

 private:
  CopyPool() {
    // every hardware thread of this process's share of the host (the caller is
    // blocked in the call anyway): measured on C5's pageable e2e (16 threads on
    // the GPU box): 4 / 8 / 12 / 16 copy threads 9.4 / 14.3 / 17.7 / 19.0 Gbit/s;
    // torchrun's LOCAL_WORLD_SIZE ranks on one host split the threads
    const char* v = getenv("QCB_COPY_THREADS");
    const char* lw = getenv("LOCAL_WORLD_SIZE");
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned ranks = lw ? (unsigned)std::max(1, atoi(lw)) : 1u;
    nthreads_ = v ? std::max(1, atoi(v)) : (int)std::min(64u, std::max(1u, hw / ranks));
    for (int i = 1; i < nthreads_; ++i) std::thread([this] { loop(); }).detach();
  }
  void drain() {
    for (;;) {
      size_t i;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!work_ || next_ >= work_->size()) return;
        i = next_++;
      }
      const Task& p = (*work_)[i];
      stage_copy(p.dst, p.src, p.n);
      std::lock_guard<std::mutex> lk(mu_);
      if (--left_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
      }
      drain();
    }
  }
  int nthreads_ = 1;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::vector<Task>* work_ = nullptr;
  size_t next_ = 0, left_ = 0;
  uint64_t gen_ = 0;
};

constexpr int kHostSlots = 3;

struct HostSlot {
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  void* dev = nullptr;  size_t dev_cap = 0;    // llr | hard | iters | conv
  void* pin = nullptr;  size_t pin_cap = 0;    // pinned staging: llr | hard | iters | conv
};

struct HostCtx {
  std::mutex mu;
  HostSlot slot[kHostSlots];
  std::map<std::vector<int32_t>, qc_code_t> codes;
};

HostCtx& host_ctx(int device) {
  static std::mutex m;
  static std::map<int, std::unique_ptr<HostCtx>> ctxs;
  std::lock_guard<std::mutex> lk(m);
  auto& p = ctxs[device];
  if (!p) p.reset(new HostCtx());
  return *p;
}

// true when [p, p+n) is page-locked (cudaHostAlloc / cudaHostRegister / torch pin_memory)
bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeHost;
}

int csr_to_shifts(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx, int64_t n_edges,
                  int32_t mb, int32_t z, int32_t n, std::vector<int32_t>& tab) {
  if (!row_ptr || !col_idx || mb < 1 || z < 1 || n < 1 || n % z)
    return fail(QC_EINVAL, "bad CSR shape (mb=%d z=%d n=%d)", mb, z, n);
  if (row_ptr_len != (int64_t)mb * z + 1) return fail(QC_EINVAL, "row_ptr length %lld != mb*z+1", (long long)row_ptr_len);
  const int nb = n / z;
  tab.assign((size_t)mb * nb, -1);
  for (int i = 0; i < mb; ++i) {
    const int64_t lo = row_ptr[(int64_t)i * z], hi = row_ptr[(int64_t)i * z + 1];
    if (lo < 0 || hi < lo || hi > n_edges) return fail(QC_EINVAL, "row_ptr out of range");
    int prev = -1;
    for (int64_t p = lo; p < hi; ++p) {
      const int col = col_idx[p];
      if (col < 0 || col >= n) return fail(QC_EINVAL, "column %d out of range", col);
      const int j = col / z;
      if (j <= prev) return fail(QC_EUNSUPPORTED, "tier %d: block columns not ascending", i);
      prev = j;
      tab[(size_t)i * nb + j] = col % z;
    }
    // every row of the tier must be the cyclic shift of row i*z
    for (int r = 0; r < z; ++r) {
      const int64_t a0 = row_ptr[(int64_t)i * z + r], a1 = row_ptr[(int64_t)i * z + r + 1];
      if (a1 - a0 != hi - lo) return fail(QC_EUNSUPPORTED, "tier %d: rows differ in degree (not QC)", i);
      int64_t p = a0;
      for (int j = 0; j < nb; ++j) {
        const int e = tab[(size_t)i * nb + j];
        if (e < 0) continue;
        if (p >= n_edges || col_idx[p] != j * z + (r + e) % z)
          return fail(QC_EUNSUPPORTED, "tier %d row %d: CSR is not a quasi-cyclic expansion", i, r);
        ++p;
      }
    }
  }
  return QC_OK;
}

template <typename T>
int decode_host(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx, int64_t n_edges,
                int32_t mb, int32_t z, const T* llrs, int64_t w, int64_t n, int32_t max_iters,
                int32_t early_term, uint8_t* hard, int32_t* iters, uint8_t* conv) {
  if (w < 0 || n < 1 || n > (1 << 30)) return fail(QC_EINVAL, "bad w/n");
  std::vector<int32_t> tab;
  int rc = csr_to_shifts(row_ptr, row_ptr_len, col_idx, n_edges, mb, z, (int32_t)n, tab);
  if (rc) return rc;
  if (w == 0) return QC_OK;
  if (!llrs || !hard || !iters || !conv) return fail(QC_EINVAL, "NULL buffer");
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  HostCtx& ctx = host_ctx(device);
  std::lock_guard<std::mutex> lk(ctx.mu);
  std::vector<int32_t> key(tab);
  key.push_back(mb); key.push_back(z); key.push_back((int32_t)n);
  qc_code_t code;
  auto it = ctx.codes.find(key);
  if (it == ctx.codes.end()) {
    rc = build_code(mb, (int32_t)(n / z), z, tab.data(), &code);
    if (rc) return rc;
    ctx.codes[key] = code;
  } else {
    code = it->second;
  }
  // Caller buffers that are already page-locked are copied by the DMA engines
  // directly; pageable ones (numpy, as decode_block passes them,
  // decoder.py:235-246) go through pinned staging slots filled and drained by
  // a host copy pool, so the copies of chunk i+1 / i-2 overlap chunk i's
  // transfer and decode.
  const bool direct = is_pinned(llrs) && is_pinned(hard) && is_pinned(iters) && is_pinned(conv);
  static const int64_t chunk_bytes = [] {
    const char* v = getenv("QCB_HOST_CHUNK_MB");
    return (int64_t)(v ? atoi(v) : 32) << 20;   // tools/exp/e2e_chunk.sh: 16-32 MB best
  }();
  const int64_t chunk = std::min<int64_t>(w, std::max<int64_t>(512, chunk_bytes / (n * (int64_t)sizeof(T))));
  const size_t llr_b = (size_t)chunk * n * sizeof(T), hard_b = (size_t)chunk * n;
  const size_t it_off = (llr_b + hard_b + 127) & ~(size_t)127;
  const size_t need = it_off + (size_t)chunk * 5 + 256;
  const size_t pin_it = (hard_b + 127) & ~(size_t)127, pin_need = llr_b + pin_it + (size_t)chunk * 5 + 256;
  for (HostSlot& s : ctx.slot) {
    if (!s.st) {
      e = cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "host path streams");
    }
    if (s.dev_cap < need) {
      if (s.dev) cudaFree(s.dev);
      s.dev = nullptr; s.dev_cap = 0;
      e = cudaMalloc(&s.dev, need);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc workspace");
      s.dev_cap = need;
    }
    if (!direct && s.pin_cap < pin_need) {
      if (s.pin) cudaFreeHost(s.pin);
      s.pin = nullptr; s.pin_cap = 0;
      e = cudaHostAlloc(&s.pin, pin_need, cudaHostAllocDefault);
      if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc staging");
      s.pin_cap = pin_need;
    }
  }
  CopyPool& pool = CopyPool::get();
  int64_t pending[kHostSlots] = {-1, -1, -1};   // first codeword of the chunk a slot holds (staged path)
  auto copy_out = [&](int b, std::vector<CopyPool::Task>& tasks) {
    const int64_t c0 = pending[b];
    if (c0 < 0) return;
    const int64_t cw = std::min(chunk, w - c0);
    char* p = static_cast<char*>(ctx.slot[b].pin);
    tasks.push_back({hard + c0 * n, p + llr_b, (size_t)cw * n});
    tasks.push_back({iters + c0, p + llr_b + pin_it, (size_t)cw * 4});
    tasks.push_back({conv + c0, p + llr_b + pin_it + (size_t)chunk * 4, (size_t)cw});
    pending[b] = -1;
  };
  for (int64_t c0 = 0, ci = 0; c0 < w; c0 += chunk, ++ci) {
    const int b = (int)(ci % kHostSlots);
    HostSlot& s = ctx.slot[b];
    const int64_t cw = std::min(chunk, w - c0);
    char* base = static_cast<char*>(s.dev);
    T* d_llr = reinterpret_cast<T*>(base);
    uint8_t* d_hard = reinterpret_cast<uint8_t*>(base + llr_b);
    int32_t* d_it = reinterpret_cast<int32_t*>(base + it_off);
    uint8_t* d_conv = reinterpret_cast<uint8_t*>(d_it + chunk);
    const T* src = llrs + c0 * n;
    uint8_t* o_hard = hard + c0 * n;
    int32_t* o_it = iters + c0;
    uint8_t* o_conv = conv + c0;
    if (!direct) {
      // the slot's previous chunk (c0 - 3 chunks) must have landed before its
      // staging buffer is reused; drain it and stage this chunk in one pass
      e = cudaEventSynchronize(s.done);
      if (e != cudaSuccess) return cuda_fail(e, "decode (host path)");
      std::vector<CopyPool::Task> tasks;
      copy_out(b, tasks);
      char* p = static_cast<char*>(s.pin);
      tasks.push_back({p, src, (size_t)cw * n * sizeof(T)});
      pool.run(tasks);
      src = reinterpret_cast<const T*>(p);
      o_hard = reinterpret_cast<uint8_t*>(p + llr_b);
      o_it = reinterpret_cast<int32_t*>(p + llr_b + pin_it);
      o_conv = reinterpret_cast<uint8_t*>(p + llr_b + pin_it + (size_t)chunk * 4);
      pending[b] = c0;
    }
    e = cudaMemcpyAsync(d_llr, src, (size_t)cw * n * sizeof(T), cudaMemcpyHostToDevice, s.st);
    if (e != cudaSuccess) return cuda_fail(e, "H2D llr");
    rc = decode_device<T>(code, d_llr, cw, max_iters, early_term, d_hard, 0, d_it, d_conv, nullptr, s.st);
    if (rc) return rc;
    e = cudaMemcpyAsync(o_hard, d_hard, (size_t)cw * n, cudaMemcpyDeviceToHost, s.st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(o_it, d_it, (size_t)cw * 4, cudaMemcpyDeviceToHost, s.st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(o_conv, d_conv, (size_t)cw, cudaMemcpyDeviceToHost, s.st);
    if (e == cudaSuccess) e = cudaEventRecord(s.done, s.st);
    if (e != cudaSuccess) return cuda_fail(e, "D2H outputs");
  }
  // drain the slots in chunk order
  const int64_t nchunks = (w + chunk - 1) / chunk;
  for (int64_t ci = std::max<int64_t>(0, nchunks - kHostSlots); ci < nchunks; ++ci) {
    const int b = (int)(ci % kHostSlots);
    e = cudaEventSynchronize(ctx.slot[b].done);
    if (e != cudaSuccess) return cuda_fail(e, "decode (host path)");
    if (!direct) {
      std::vector<CopyPool::Task> tasks;
      copy_out(b, tasks);
      pool.run(tasks);
    }
  }
  return QC_OK;
}

}  // namespace

extern "C" {

int qc_version(void) { return 110; }
const char* qc_last_error(void) { return g_err.c_str(); }

int qc_code_create(int32_t mb, int32_t nb, int32_t z, const int32_t* shifts, qc_code_t* out) {
  const int rc = build_code(mb, nb, z, shifts, out);
  if (rc || (*out)->structure >= 0) return rc;
  // generic code: upload its tables for the current device now, so the first
  // decode is free of allocations (and capturable).  No device: skip quietly.
  int device = 0, count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0 || cudaGetDevice(&device) != cudaSuccess) {
    cudaGetLastError();
    return rc;
  }
  cudaError_t e = cudaSuccess;
  bool capturing = false;
  if ((*out)->tables(device, nullptr, &e, &capturing) && e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
  if (e != cudaSuccess) cudaGetLastError();   // decode retries (and reports) the upload
  return rc;
}

int qc_code_from_csr(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx,
                     int64_t n_edges, int32_t mb, int32_t z, int32_t n, qc_code_t* out) {
  std::vector<int32_t> tab;
  int rc = csr_to_shifts(row_ptr, row_ptr_len, col_idx, n_edges, mb, z, n, tab);
  if (rc) return rc;
  return build_code(mb, n / z, z, tab.data(), out);
}

int qc_code_destroy(qc_code_t code) {
  if (!code) return QC_OK;
  for (auto& kv : code->dev) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(kv.first);
    cudaFree(kv.second.d);
    cudaSetDevice(cur);
  }
  delete code;
  return QC_OK;
}

int qc_code_info(qc_code_t c, int32_t* mb, int32_t* nb, int32_t* z, int32_t* n_edges,
                 int32_t* max_row_degree, int32_t* kernel) {
  if (!c) return fail(QC_EINVAL, "code is NULL");
  if (mb) *mb = c->mb;
  if (nb) *nb = c->nb;
  if (z) *z = c->z;
  if (n_edges) *n_edges = c->ne * c->z;
  if (max_row_degree) *max_row_degree = c->max_deg;
  if (kernel) *kernel = c->structure >= 0 ? 1 : 0;
  return QC_OK;
}

int qc_decode_f32(qc_code_t code, const float* llr, int64_t w, int32_t max_iters, int32_t early_term,
                  uint8_t* hard, int32_t hard_packed, int32_t* iters, uint8_t* conv, float* post_out,
                  void* stream) {
  return decode_device<float>(code, llr, w, max_iters, early_term, hard, hard_packed, iters, conv,
                              post_out, as_stream(stream));
}

int qc_decode_i16(qc_code_t code, const int16_t* llr, int64_t w, int32_t max_iters, int32_t early_term,
                  uint8_t* hard, int32_t hard_packed, int32_t* iters, uint8_t* conv, int16_t* post_out,
                  void* stream) {
  return decode_device<int16_t>(code, llr, w, max_iters, early_term, hard, hard_packed, iters, conv,
                                post_out, as_stream(stream));
}

}  // extern "C"

namespace {

// Per-device side streams for the grouped launch (created once, never freed).
#ifndef QCB_GROUP_STREAMS
#define QCB_GROUP_STREAMS 8
#endif
constexpr int kGroupStreams = QCB_GROUP_STREAMS;
cudaStream_t* group_streams(int device, cudaError_t* err) {
  static std::mutex m;
  static std::map<int, std::vector<cudaStream_t>> all;
  std::lock_guard<std::mutex> lk(m);
  auto& v = all[device];
  if (v.empty()) {
    for (int i = 0; i < kGroupStreams; ++i) {
      cudaStream_t s = nullptr;
      *err = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (*err != cudaSuccess) return nullptr;
      v.push_back(s);
    }
  }
  *err = cudaSuccess;
  return v.data();
}

template <typename T>
int validate_job(const qc_decode_job_t& j, int32_t max_iters) {
  if (!j.code) return fail(QC_EINVAL, "code is NULL");
  if (j.w < 0 || max_iters < 0) return fail(QC_EINVAL, "w=%lld max_iters=%d", (long long)j.w, max_iters);
  if (j.w > 0 && (!j.llr || !j.hard || !j.iters || !j.conv)) return fail(QC_EINVAL, "NULL buffer");
  if (j.w > (int64_t)1 << 40) return fail(QC_EINVAL, "batch too large");
  // the one data-independent failure decode_device can report, checked before any job is queued
  if (j.code->structure < 0 && generic_cw_per_cta(j.code, (int)sizeof(T)) < 1)
    return fail(QC_EUNSUPPORTED, "one codeword (N=%d) does not fit in shared memory", j.code->n);
  return QC_OK;
}

// Mixed-code batch.  Every job is validated before any work is queued (argument
// checks and the generic kernel's shared-memory fit; a CUDA launch failure can
// still stop the call part-way, and then the outputs are unspecified); the
// jobs then fork from the caller's stream onto per-device side streams
// (event record / wait, so the call stays stream-ordered and can be captured
// into a CUDA graph) and join back, so the codes' kernels run concurrently:
// the tail wave of one code's grid overlaps the next code's CTAs.
template <typename T>
int grouped(const qc_decode_job_t* jobs, int32_t n_jobs, int32_t max_iters, int32_t early_term,
            int32_t hard_packed, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return fail(QC_EINVAL, "bad job list");
  for (int i = 0; i < n_jobs; ++i) {
    const int rc = validate_job<T>(jobs[i], max_iters);
    if (rc) return rc;
  }
  auto run = [&](const qc_decode_job_t& j, cudaStream_t s) {
    return decode_device<T>(j.code, (const T*)j.llr, j.w, max_iters, early_term, j.hard, hard_packed, j.iters,
                            j.conv, (T*)j.post_out, s);
  };
  const cudaStream_t origin = as_stream(stream);
  if (n_jobs <= 1 || std::getenv("QCB_GROUPED_SERIAL")) {
    for (int i = 0; i < n_jobs; ++i) {
      const int rc = run(jobs[i], origin);
      if (rc) return rc;
    }
    return QC_OK;
  }
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  cudaStream_t* side = group_streams(device, &e);
  if (!side) return cuda_fail(e, "side streams");
  const int ns = std::min<int>(n_jobs, kGroupStreams);
  cudaEvent_t ev[kGroupStreams + 1];
  int made = 0, rc = QC_OK;
  for (; made < ns + 1; ++made) {
    e = cudaEventCreateWithFlags(&ev[made], cudaEventDisableTiming);
    if (e != cudaSuccess) { rc = cuda_fail(e, "cudaEventCreate"); break; }
  }
  if (!rc) {
    e = cudaEventRecord(ev[ns], origin);
    for (int k = 0; k < ns && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(side[k], ev[ns], 0);
    if (e != cudaSuccess) rc = cuda_fail(e, "fork");
  }
  // largest jobs first, round-robin over the side streams
  std::vector<int> order(n_jobs);
  for (int i = 0; i < n_jobs; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return jobs[a].w * (int64_t)jobs[a].code->ne * jobs[a].code->z > jobs[b].w * (int64_t)jobs[b].code->ne * jobs[b].code->z;
  });
  for (int q = 0; q < n_jobs && !rc; ++q) rc = run(jobs[order[q]], side[q % ns]);
  // join (also after a failure, so no side stream is left ahead of the caller)
  for (int k = 0; k < ns && made == ns + 1; ++k) {
    e = cudaEventRecord(ev[k], side[k]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(origin, ev[k], 0);
    if (e != cudaSuccess && !rc) rc = cuda_fail(e, "join");
  }
  for (int k = 0; k < made; ++k) cudaEventDestroy(ev[k]);
  return rc;
}

}  // namespace

extern "C" {

int qc_decode_grouped_f32(const qc_decode_job_t* jobs, int32_t n_jobs, int32_t max_iters, int32_t early_term,
                          int32_t hard_packed, void* stream) {
  return grouped<float>(jobs, n_jobs, max_iters, early_term, hard_packed, stream);
}

int qc_decode_grouped_i16(const qc_decode_job_t* jobs, int32_t n_jobs, int32_t max_iters, int32_t early_term,
                          int32_t hard_packed, void* stream) {
  return grouped<int16_t>(jobs, n_jobs, max_iters, early_term, hard_packed, stream);
}

int qc_decode_batch_f32_host(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx,
                             int64_t n_edges, int32_t mb, int32_t z, const float* llrs, int64_t w, int64_t n,
                             int32_t max_iters, int32_t early_term, uint8_t* hard, int32_t* iters,
                             uint8_t* conv) {
  return decode_host<float>(row_ptr, row_ptr_len, col_idx, n_edges, mb, z, llrs, w, n, max_iters,
                            early_term, hard, iters, conv);
}

int qc_decode_batch_i16_host(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx,
                             int64_t n_edges, int32_t mb, int32_t z, const int16_t* llrs, int64_t w, int64_t n,
                             int32_t max_iters, int32_t early_term, uint8_t* hard, int32_t* iters,
                             uint8_t* conv) {
  return decode_host<int16_t>(row_ptr, row_ptr_len, col_idx, n_edges, mb, z, llrs, w, n, max_iters,
                              early_term, hard, iters, conv);
}

int qc_encode_packed(qc_code_t c, const uint8_t* info, int64_t w, uint8_t* cw, void* stream) {
  if (!c) return fail(QC_EINVAL, "code is NULL");
  if (c->z % 8) return fail(QC_EUNALIGNED, "packed encoder needs z %% 8 == 0, got z=%d", c->z);
  if (c->enc_y < 0) return fail(QC_EMALFORMED, "h_b column lacks a single interior entry");
  if (c->mb > 12 || c->nb > 24 || c->z > 128) return fail(QC_EUNSUPPORTED, "encoder supports mb<=12, nb<=24, z<=128");
  if (w < 0) return fail(QC_EINVAL, "w < 0");
  if (w == 0) return QC_OK;
  if (!info || !cw) return fail(QC_EINVAL, "NULL buffer");
  EncodeArgs a;
  memset(&a, 0, sizeof a);
  a.info = info; a.cw = cw; a.w = w; a.mb = c->mb; a.nb = c->nb; a.z = c->z; a.hb_shift = c->enc_hb;
  a.native = c->native ? 1 : 0;
  a.scaled = c->scaled ? 1 : 0;
  for (int i = 0; i < c->mb * c->nb; ++i) a.shifts[i] = c->shifts[i];
  cudaError_t e = launch_encode_packed(a, c->structure, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "encode_packed");
  return QC_OK;
}

int qc_encode_bits(qc_code_t c, const uint8_t* info, int64_t w, uint8_t* cw, void* stream) {
  if (!c) return fail(QC_EINVAL, "code is NULL");
  if (c->z % 8 == 0) return qc_encode_packed(c, info, w, cw, stream);   // the same byte layout
  if (c->enc_y < 0) return fail(QC_EMALFORMED, "h_b column lacks a single interior entry");
  if (c->mb > 12 || c->nb > 24 || c->mb < 2 || c->z > 97)
    return fail(QC_EUNSUPPORTED, "bit-granular encoder supports 2<=mb<=12, nb<=24, z<=97");
  if (w < 0) return fail(QC_EINVAL, "w < 0");
  if (w == 0) return QC_OK;
  if (!info || !cw) return fail(QC_EINVAL, "NULL buffer");
  EncodeArgs a;
  memset(&a, 0, sizeof a);
  a.info = info; a.cw = cw; a.w = w; a.mb = c->mb; a.nb = c->nb; a.z = c->z; a.hb_shift = c->enc_hb;
  for (int i = 0; i < c->mb * c->nb; ++i) a.shifts[i] = c->shifts[i];
  a.native = c->native ? 1 : 0;
  a.scaled = c->scaled ? 1 : 0;
  cudaError_t e = launch_encode_packed(a, c->structure, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "encode_bits");
  return QC_OK;
}

int qc_encode_packed_host(qc_code_t c, const uint8_t* info, int64_t w, uint8_t* cw) {
  if (!c) return fail(QC_EINVAL, "code is NULL");
  if (w < 0) return fail(QC_EINVAL, "w < 0");
  if (w == 0) return QC_OK;
  if (!info || !cw) return fail(QC_EINVAL, "NULL buffer");
  const size_t kb = (size_t)(c->kb * c->z / 8), nbt = (size_t)(c->n / 8);
  uint8_t *d_in = nullptr, *d_out = nullptr;
  cudaError_t e = cudaMalloc(&d_in, (size_t)w * kb);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, (size_t)w * nbt);
  if (e == cudaSuccess) e = cudaMemcpy(d_in, info, (size_t)w * kb, cudaMemcpyHostToDevice);
  int rc = QC_OK;
  if (e == cudaSuccess) {
    rc = qc_encode_packed(c, d_in, w, d_out, nullptr);
    if (rc == QC_OK) e = cudaMemcpy(cw, d_out, (size_t)w * nbt, cudaMemcpyDeviceToHost);
  }
  cudaFree(d_in);
  cudaFree(d_out);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "encode_packed (host path)");
  return QC_OK;
}

// ---- channel, waterfall counters, records --------------------------

int qc_encode_array(qc_code_t c, const uint8_t* info_bits, int64_t w, uint8_t* cw_bits, void* stream) {
  if (!c) return fail(QC_EINVAL, "code is NULL");
  if (c->enc_y < 0) return fail(QC_EMALFORMED, "h_b column lacks a single interior entry");
  if (c->mb > 12 || c->nb > 24 || c->mb < 2) return fail(QC_EUNSUPPORTED, "encoder supports 2<=mb<=12, nb<=24");
  if (w < 0) return fail(QC_EINVAL, "w < 0");
  if (w == 0) return QC_OK;
  if (!info_bits || !cw_bits) return fail(QC_EINVAL, "NULL buffer");
  EncodeArgs a;
  memset(&a, 0, sizeof a);
  a.info = info_bits; a.cw = cw_bits; a.w = w; a.mb = c->mb; a.nb = c->nb; a.z = c->z; a.hb_shift = c->enc_hb;
  for (int i = 0; i < c->mb * c->nb; ++i) a.shifts[i] = c->shifts[i];
  cudaError_t e = launch_encode_array(a, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "encode_array");
  return QC_OK;
}

int qc_frames_info(uint64_t seed, uint32_t point, int64_t frame0, int64_t w, int32_t k, uint8_t* info_bits,
                   void* stream) {
  if (w < 0 || k < 0 || frame0 < 0) return fail(QC_EINVAL, "negative size");
  if (w == 0 || k == 0) return QC_OK;
  if (!info_bits) return fail(QC_EINVAL, "NULL buffer");
  cudaError_t e = launch_frames_info(seed, point, frame0, w, k, info_bits, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "frames_info");
  return QC_OK;
}

int qc_channel_llr(const uint8_t* cw_bits, int64_t w, int32_t n, double sigma2, const double* noise,
                   uint64_t seed, uint32_t point, int64_t frame0, int32_t q_b, double l_clip, void* llr,
                   void* stream) {
  if (!(sigma2 > 0.0)) return fail(QC_EINVAL, "sigma2 = %g (must be > 0, chansim.py:59-60)", sigma2);
  if (w < 0 || n < 0 || (n & 1) || frame0 < 0) return fail(QC_EINVAL, "bad shape w=%lld n=%d", (long long)w, n);
  if (q_b < 0 || q_b > 14) return fail(QC_EINVAL, "q_b must stay in [1, 14] (0 = float32 out)");
  if (q_b > 0 && !(l_clip > 0.0)) return fail(QC_EINVAL, "l_clip must be > 0");
  if (w == 0 || n == 0) return QC_OK;
  if (!cw_bits || !llr) return fail(QC_EINVAL, "NULL buffer");
  ChannelArgs a;
  memset(&a, 0, sizeof a);
  a.bits = cw_bits; a.noise = noise; a.llr = llr; a.w = w; a.n = n;
  a.seed = seed; a.point = point; a.frame0 = frame0;
  a.sqrt_sigma2 = std::sqrt(sigma2);
  a.two_over_sigma2 = 2.0 / sigma2;
  if (q_b > 0) {
    const double lim = (double)((1 << q_b) - 1);
    a.q_lim = lim;
    a.q_scale = lim / l_clip;
  }
  cudaError_t e = launch_channel(a, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "channel_llr");
  return QC_OK;
}

int qc_quantize_llr(const float* x, int64_t count, int32_t q_b, double l_clip, int16_t* out, void* stream) {
  if (q_b < 1 || q_b > 14) return fail(QC_EINVAL, "q_b must stay in [1, 14] (decoder.py:167-168)");
  if (!(l_clip > 0.0)) return fail(QC_EINVAL, "l_clip must be > 0");
  if (count < 0) return fail(QC_EINVAL, "count < 0");
  if (count == 0) return QC_OK;
  if (!x || !out) return fail(QC_EINVAL, "NULL buffer");
  const double lim = (double)((1 << q_b) - 1);
  cudaError_t e = launch_quantize(x, count, lim / l_clip, lim, out, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "quantize_llr");
  return QC_OK;
}

int qc_count_errors(const uint8_t* hard, int32_t hard_packed, const uint8_t* info_bits, const int32_t* iters,
                    int64_t w, int32_t n, int32_t k, int32_t batch, uint64_t* batch_sums, void* stream) {
  if (w < 0 || n <= 0 || k < 0 || k > n || batch < 1) return fail(QC_EINVAL, "bad shape");
  if (!hard || !info_bits || !iters || !batch_sums) return fail(QC_EINVAL, "NULL buffer");
  cudaError_t e = launch_count_errors(hard, hard_packed ? 1 : 0, info_bits, iters, w, n, k, batch,
                                      reinterpret_cast<unsigned long long*>(batch_sums), as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "count_errors");
  return QC_OK;
}

int qc_pack_records(const uint8_t* hard_packed, const int32_t* iters, const uint8_t* conv, int64_t w, int32_t n,
                    uint8_t* records, void* stream) {
  if (w < 0 || n <= 0) return fail(QC_EINVAL, "bad shape");
  if (w == 0) return QC_OK;
  if (!hard_packed || !iters || !conv || !records) return fail(QC_EINVAL, "NULL buffer");
  cudaError_t e = launch_pack_records(hard_packed, iters, conv, w, (n + 7) / 8, records, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pack_records");
  return QC_OK;
}

}  // extern "C"
