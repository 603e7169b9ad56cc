// corpus_io.cpp -- host-side formats either side of the sampler hot path
// (include/samelda_io.h).
//
// load_uci_bow (corpus.cpp:62-183) is the reference's two-iostream-pass
// parser: ~60 s for a NYTimes-sized docword file, longer than a whole
// training run on the GPU.  Here the file is mmap'ed and tokenised by all
// host threads, in three parallel passes over byte ranges cut at whitespace:
//   A  count the integer tokens of each range (a range stops at its first
//      token that is not an integer, exactly where `in >> x` would fail);
//   B  parse again, storing token g as field g % 3 of triplet g / 3 and
//      recording the first range violation of each byte range;
//   C  CSR: per-document row sizes, scatter, per-row sort + duplicate merge
//      (the merged row is independent of the scatter order), empty-row
//      compaction.
// The first error in the reference's sequential order is reconstructed from
// the per-range records, so malformed input fails with the same IoError
// message (test_corpus.cpp cases, tests/test_corpus_io.py).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <charconv>
#include <chrono>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/samelda_io.h"

// uninitialised POD array: pages are first touched by the parallel writers
// (std::vector would zero-fill gigabytes on one thread first)
template <class T>
struct Pod {
  std::unique_ptr<T[]> p;
  size_t n = 0;
  void alloc(size_t k) {
    p.reset(k ? new T[k] : nullptr);
    n = k;
  }
  T* data() { return p.get(); }
  const T* data() const { return p.get(); }
  size_t size() const { return n; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
};

struct samelda_io_corpus {
  std::vector<int64_t> offsets;
  Pod<int32_t> words;
  Pod<int32_t> counts;
  int64_t n_docs = 0;
  int64_t n_words = 0;
  int64_t n_tokens = 0;
  int64_t dropped = 0;
  std::string vocab;  // n_words lines, each '\n'-terminated
};

namespace {

thread_local std::string g_err;

struct IoFail {
  int code;
  std::string msg;
};

[[noreturn]] void io_fail(const std::string& msg) { throw IoFail{SAMELDA_CU_IO, msg}; }

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return SAMELDA_CU_OK;
  } catch (const IoFail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return SAMELDA_CU_IO;
  }
}

int threads_for(int n_threads) {
  if (n_threads > 0) return n_threads;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(h) : 1;
}

// fn(part, begin, end) over n items in `parts` contiguous ranges
template <class F>
void parallel_ranges(int64_t n, int parts, F&& fn) {
  if (parts <= 1 || n < 2) {
    fn(0, int64_t{0}, n);
    return;
  }
  parts = static_cast<int>(std::min<int64_t>(parts, n));
  std::vector<std::thread> pool;
  pool.reserve(parts);
  for (int p = 0; p < parts; ++p) {
    const int64_t b = n * p / parts, e = n * (p + 1) / parts;
    pool.emplace_back([&fn, p, b, e] { fn(p, b, e); });
  }
  for (auto& t : pool) t.join();
}

struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  void* base = nullptr;
  ~Mapped() {
    if (base) munmap(base, n);
  }
};

bool map_file(const char* path, Mapped& m) {
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return false;
  struct stat st;
  if (fstat(fd, &st) != 0 || S_ISDIR(st.st_mode)) {
    close(fd);
    return false;
  }
  m.n = static_cast<size_t>(st.st_size);
  if (m.n == 0) {
    m.p = "";
    close(fd);
    return true;
  }
  m.base = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
  close(fd);
  if (m.base == MAP_FAILED) {
    m.base = nullptr;
    return false;
  }
  madvise(m.base, m.n, MADV_SEQUENTIAL);
  m.p = static_cast<const char*>(m.base);
  return true;
}

inline bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// `in >> int64_t` (C locale): skip whitespace, optional sign, one or more
// decimal digits; out-of-range values fail.  False at end of input or on a
// token that is not an integer (s is then left anywhere).
inline bool next_int(const char*& s, const char* e, int64_t& v) {
  while (s < e && is_ws(*s)) ++s;
  if (s == e) return false;
  const char* q = s;
  bool neg = false;
  if (*q == '+' || *q == '-') {
    neg = *q == '-';
    ++q;
  }
  if (q == e || static_cast<unsigned>(*q - '0') > 9u) return false;
  const uint64_t lim = neg ? (uint64_t{1} << 63) : (uint64_t{1} << 63) - 1;
  uint64_t acc = 0;
  bool over = false;
  for (; q < e && static_cast<unsigned>(*q - '0') <= 9u; ++q) {
    const unsigned d = static_cast<unsigned>(*q - '0');
    if (acc > (lim - d) / 10) over = true;
    else acc = acc * 10 + d;
  }
  if (over) return false;
  v = neg ? static_cast<int64_t>(0 - acc) : static_cast<int64_t>(acc);
  s = q;
  return true;
}

// getline semantics (corpus.cpp:168-175): '\n'-separated lines, a final line
// without '\n' counts, one trailing '\r' stripped per line
int64_t read_vocab_lines(const Mapped& m, std::string& out) {
  out.clear();
  out.reserve(m.n + 1);
  int64_t lines = 0;
  size_t i = 0;
  while (i < m.n) {
    const char* nl = static_cast<const char*>(memchr(m.p + i, '\n', m.n - i));
    size_t end = nl ? static_cast<size_t>(nl - m.p) : m.n;
    size_t len = end - i;
    if (len > 0 && m.p[i + len - 1] == '\r') --len;
    out.append(m.p + i, len);
    out.push_back('\n');
    ++lines;
    i = end + 1;
  }
  return lines;
}

// range violation of triplet j, field f (0 doc, 1 word, 2 count); value v
struct RangeErr {
  int64_t j = std::numeric_limits<int64_t>::max();
  int f = 0;
  int64_t v = 0;
  int64_t doc = 0;
};

struct PhaseTimer {
  bool on = std::getenv("SAMELDA_IO_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[io] %-10s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

void load_uci(const char* docword_path, const char* vocab_path, int n_threads,
              samelda_io_corpus& c) {
  PhaseTimer pt;
  Mapped m;
  if (!map_file(docword_path, m)) io_fail(std::string("cannot open docword file: ") + docword_path);
  const char* s = m.p;
  const char* e = m.p + m.n;
  int64_t D = 0, W = 0, NNZ = 0;
  if (!next_int(s, e, D)) io_fail("malformed docword header: missing document count");
  if (!next_int(s, e, W)) io_fail("malformed docword header: missing vocabulary size");
  if (!next_int(s, e, NNZ)) io_fail("malformed docword header: missing nonzero count");
  if (D < 1 || W < 1 || NNZ < 0) io_fail("malformed docword header: nonpositive dimension");

  // byte ranges cut at whitespace: no token straddles two ranges
  const int T = threads_for(n_threads);
  const int64_t len = e - s;
  const int parts = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(T * 4, len / 65536 + 1)));
  std::vector<const char*> cut(parts + 1);
  cut[0] = s;
  cut[parts] = e;
  for (int p = 1; p < parts; ++p) {
    const char* b = s + len * p / parts;
    while (b < e && !is_ws(*b)) ++b;
    cut[p] = std::max(b, cut[p - 1]);
  }
  // pass A: integer tokens per range, and whether the range hit a non-integer
  std::vector<int64_t> ntok(parts, 0);
  std::vector<char> stopped(parts, 0);
  std::atomic<int> next{0};
  auto worker_pool = [&](auto&& body) {
    next = 0;
    std::vector<std::thread> pool;
    const int nt = std::min(T, parts);
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&] {
        for (int p; (p = next.fetch_add(1)) < parts;) body(p);
      });
    for (auto& th : pool) th.join();
  };
  worker_pool([&](int p) {
    const char* q = cut[p];
    const char* qe = cut[p + 1];
    int64_t v, n = 0;
    for (;;) {
      const char* before = q;
      if (!next_int(q, qe, v)) {
        while (before < qe && is_ws(*before)) ++before;
        stopped[p] = before < qe;  // a non-integer token (not just the end)
        break;
      }
      ++n;
    }
    ntok[p] = n;
  });
  pt.mark("count");
  // the sequential reader stops at the first non-integer token
  std::vector<int64_t> gbase(parts + 1, 0);
  int last = parts - 1;
  for (int p = 0; p < parts; ++p) {
    gbase[p + 1] = gbase[p] + ntok[p];
    if (stopped[p]) {
      last = p;
      break;
    }
  }
  const int64_t total = gbase[last + 1];
  const int64_t J = total / 3;  // complete triplets
  const int64_t rem = total % 3;
  // pass B: store triplets 0..NNZ (one past the declared count, whose range
  // checks precede the "more triplets" error) and record range violations
  const int64_t keep = std::min(J, NNZ + 1);
  Pod<int32_t> tdoc, tword, tcnt;
  tdoc.alloc(static_cast<size_t>(keep));
  tword.alloc(static_cast<size_t>(keep));
  tcnt.alloc(static_cast<size_t>(keep));
  std::vector<RangeErr> rerr(parts);
  worker_pool([&](int p) {
    if (p > last) return;
    const char* q = cut[p];
    const char* qe = cut[p + 1];
    int64_t g = gbase[p];
    const int64_t gend = gbase[p + 1];
    RangeErr& re = rerr[p];
    int64_t v;
    while (g < gend && next_int(q, qe, v)) {
      const int64_t j = g / 3;
      const int f = static_cast<int>(g % 3);
      ++g;
      if (j >= keep) break;
      if (f == 0) {
        tdoc[j] = static_cast<int32_t>(v - 1);
        if ((v < 1 || v > D) && j < re.j) re = RangeErr{j, 0, v, v};
      } else if (f == 1) {
        tword[j] = static_cast<int32_t>(v - 1);
        if ((v < 1 || v > W) && j < re.j) re = RangeErr{j, 1, v, 0};
      } else {
        tcnt[j] = static_cast<int32_t>(v);
        if (v < 1 && j < re.j) re = RangeErr{j, 2, v, 0};
      }
    }
  });
  pt.mark("parse");
  // first error in the reference's order (corpus.cpp:76-97)
  RangeErr first;
  for (const auto& r : rerr)
    if (r.j < first.j || (r.j == first.j && r.f < first.f)) first = r;
  const int64_t more_at = J > NNZ ? NNZ : std::numeric_limits<int64_t>::max();
  const int64_t incomplete_at = rem > 0 ? J : std::numeric_limits<int64_t>::max();
  const int64_t err_at = std::min({first.j, more_at, incomplete_at});
  if (err_at != std::numeric_limits<int64_t>::max()) {
    if (first.j == err_at) {
      if (first.f == 0)
        io_fail("docword entry out of declared range: docID " + std::to_string(first.v));
      if (first.f == 1)
        io_fail("docword entry out of declared range: wordID " + std::to_string(first.v));
      io_fail("docword entry with count <= 0 at docID " +
              std::to_string(static_cast<int64_t>(tdoc[first.j]) + 1));
    }
    if (incomplete_at == err_at && incomplete_at < more_at)
      io_fail("malformed docword entry: incomplete triplet");
    io_fail("docword file has more triplets than the declared NNZ");
  }
  if (J != NNZ)
    io_fail("docword file declares NNZ=" + std::to_string(NNZ) + " but has " + std::to_string(J) +
            " triplets");

  // pass C: CSR rows (corpus.cpp:99-160).  Fast paths for the usual UCI
  // layout (triplets grouped by document, rows sorted by word id): no
  // scatter, no sort, no copy; the general path scatters with atomics and
  // sorts each row.  The merged row is the same either way.
  std::vector<char> part_sorted(static_cast<size_t>(T), 1);
  parallel_ranges(NNZ, T, [&](int part, int64_t b, int64_t en) {
    for (int64_t j = std::max<int64_t>(b, 1); j < en; ++j)
      if (tdoc[j] < tdoc[j - 1]) {
        part_sorted[part] = 0;
        break;
      }
  });
  bool doc_sorted = true;
  for (char v : part_sorted) doc_sorted = doc_sorted && v;
  std::vector<int64_t> row(static_cast<size_t>(D) + 1, 0);
  Pod<int32_t> rw, rc;  // rows, grouped by document
  if (doc_sorted) {
    // row starts from the (non-decreasing) document column: row[d] = first
    // j with tdoc[j] >= d, each entry written once, in parallel
    parallel_ranges(NNZ, T, [&](int, int64_t b, int64_t en) {
      for (int64_t j = b; j < en; ++j) {
        const int64_t prev = j ? tdoc[j - 1] : -1;
        for (int64_t d = prev + 1; d <= tdoc[j]; ++d) row[d] = j;
      }
    });
    for (int64_t d = (NNZ ? tdoc[NNZ - 1] + 1 : 0); d <= D; ++d) row[d] = NNZ;
    rw = std::move(tword);
    rc = std::move(tcnt);
  } else {
    std::vector<std::atomic<int64_t>> pos(static_cast<size_t>(D));
    parallel_ranges(D, T, [&](int, int64_t b, int64_t en) {
      for (int64_t d = b; d < en; ++d) pos[d].store(0, std::memory_order_relaxed);
    });
    parallel_ranges(NNZ, T, [&](int, int64_t b, int64_t en) {
      for (int64_t j = b; j < en; ++j) pos[tdoc[j]].fetch_add(1, std::memory_order_relaxed);
    });
    for (int64_t d = 0; d < D; ++d) row[d + 1] = row[d] + pos[d].load(std::memory_order_relaxed);
    for (int64_t d = 0; d < D; ++d) pos[d].store(row[d], std::memory_order_relaxed);
    rw.alloc(static_cast<size_t>(NNZ));
    rc.alloc(static_cast<size_t>(NNZ));
    parallel_ranges(NNZ, T, [&](int, int64_t b, int64_t en) {
      for (int64_t j = b; j < en; ++j) {
        const int64_t at = pos[tdoc[j]].fetch_add(1, std::memory_order_relaxed);
        rw[at] = tword[j];
        rc[at] = tcnt[j];
      }
    });
  }
  tdoc = Pod<int32_t>();
  tword = Pod<int32_t>();
  tcnt = Pod<int32_t>();
  pt.mark("rows");
  // per-row sort (skipped when already increasing) + merge, in place
  std::vector<int64_t> msize(static_cast<size_t>(D), 0);
  std::vector<int64_t> mtok(static_cast<size_t>(T), 0);
  std::vector<int64_t> overflow_doc(static_cast<size_t>(T), std::numeric_limits<int64_t>::max());
  std::vector<char> part_changed(static_cast<size_t>(T), 0);
  parallel_ranges(D, T, [&](int part, int64_t b, int64_t en) {
    int64_t tok = 0;
    std::vector<uint64_t> key;
    for (int64_t d = b; d < en; ++d) {
      int32_t* w = rw.data() + row[d];
      int32_t* cn = rc.data() + row[d];
      const int64_t n = row[d + 1] - row[d];
      if (n == 0) continue;
      bool increasing = true;
      for (int64_t i = 1; i < n && increasing; ++i) increasing = w[i] > w[i - 1];
      if (increasing) {
        for (int64_t i = 0; i < n; ++i) tok += cn[i];  // counts >= 1 (validated)
        msize[d] = n;
        continue;
      }
      part_changed[part] = 1;
      key.resize(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i)
        key[i] = (static_cast<uint64_t>(static_cast<uint32_t>(w[i])) << 32) |
                 static_cast<uint32_t>(cn[i]);
      std::sort(key.begin(), key.end());
      int64_t out = 0, i = 0;
      while (i < n) {
        const uint32_t wd = static_cast<uint32_t>(key[i] >> 32);
        int64_t sum = 0;
        for (; i < n && static_cast<uint32_t>(key[i] >> 32) == wd; ++i)
          sum += static_cast<int32_t>(static_cast<uint32_t>(key[i]));
        if (sum > std::numeric_limits<int32_t>::max() && d < overflow_doc[part])
          overflow_doc[part] = d;
        w[out] = static_cast<int32_t>(wd);
        cn[out] = static_cast<int32_t>(sum);
        tok += sum;
        ++out;
      }
      msize[d] = out;
    }
    mtok[part] = tok;
  });
  pt.mark("sort");
  const int64_t od = *std::min_element(overflow_doc.begin(), overflow_doc.end());
  if (od != std::numeric_limits<int64_t>::max())
    io_fail("merged count overflows at docID " + std::to_string(od + 1));
  // compact: drop empty documents (corpus.cpp:137-140), close merged gaps
  std::vector<int64_t> src;
  src.reserve(static_cast<size_t>(D));
  c.offsets.assign(1, 0);
  for (int64_t d = 0; d < D; ++d) {
    if (msize[d] == 0) {
      ++c.dropped;
      continue;
    }
    src.push_back(d);
    c.offsets.push_back(c.offsets.back() + msize[d]);
  }
  c.n_docs = static_cast<int64_t>(src.size());
  const int64_t nnz = c.offsets.back();
  bool changed = false;
  for (char v : part_changed) changed = changed || v;
  if (!changed) {  // no merges: rows are already contiguous (empty rows take no space)
    c.words = std::move(rw);
    c.counts = std::move(rc);
  } else {
    c.words.alloc(static_cast<size_t>(nnz));
    c.counts.alloc(static_cast<size_t>(nnz));
    parallel_ranges(c.n_docs, T, [&](int, int64_t b, int64_t en) {
      for (int64_t i = b; i < en; ++i) {
        const int64_t d = src[i];
        const int64_t n = c.offsets[i + 1] - c.offsets[i];
        std::memcpy(c.words.data() + c.offsets[i], rw.data() + row[d], n * sizeof(int32_t));
        std::memcpy(c.counts.data() + c.offsets[i], rc.data() + row[d], n * sizeof(int32_t));
      }
    });
  }
  c.words.n = static_cast<size_t>(nnz);
  c.counts.n = static_cast<size_t>(nnz);
  c.n_tokens = 0;
  for (auto t : mtok) c.n_tokens += t;
  pt.mark("compact");
  c.n_words = W;
  if (c.dropped > 0)
    std::fprintf(stderr, "load_uci_bow: dropped %lld empty document(s)\n",
                 static_cast<long long>(c.dropped));
  if (c.n_docs == 0) io_fail("docword file contains no non-empty documents");

  Mapped vm;
  if (!map_file(vocab_path, vm)) io_fail(std::string("cannot open vocab file: ") + vocab_path);
  const int64_t lines = read_vocab_lines(vm, c.vocab);
  if (lines != W)
    io_fail("vocab length mismatch: docword declares W=" + std::to_string(W) +
            " but vocab file has " + std::to_string(lines) + " lines");
}

// ----------------------------------------------------------- binary cache

constexpr char kCsrMagic[8] = {'S', 'A', 'M', 'E', 'C', 'S', 'R', '1'};

struct CsrHeader {
  char magic[8];
  uint32_t version;
  uint32_t reserved;
  int64_t n_docs, n_words, nnz, n_tokens, vocab_bytes;
};

void write_all(FILE* f, const void* p, size_t n, const std::string& path) {
  if (n && std::fwrite(p, 1, n, f) != n) io_fail("write failed: " + path);
}

void read_at(int fd, void* dst, size_t n, off_t off, int T, const std::string& path) {
  if (n == 0) return;
  std::atomic<bool> bad{false};
  const int64_t blocks = static_cast<int64_t>((n + (8u << 20) - 1) / (8u << 20));
  parallel_ranges(blocks, T, [&](int, int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      size_t lo = static_cast<size_t>(i) * (8u << 20), hi = std::min(n, lo + (8u << 20));
      while (lo < hi) {
        const ssize_t r = pread(fd, static_cast<char*>(dst) + lo, hi - lo, off + static_cast<off_t>(lo));
        if (r <= 0) {
          bad = true;
          return;
        }
        lo += static_cast<size_t>(r);
      }
    }
  });
  if (bad) io_fail("truncated corpus cache: " + path);
}

void load_csr(const char* path, int n_threads, samelda_io_corpus& c) {
  const int T = threads_for(n_threads);
  const std::string p(path);
  const int fd = open(path, O_RDONLY);
  if (fd < 0) io_fail("cannot open corpus cache: " + p);
  struct Closer {
    int fd;
    ~Closer() { close(fd); }
  } closer{fd};
  struct stat st;
  if (fstat(fd, &st) != 0) io_fail("cannot open corpus cache: " + p);
  CsrHeader h;
  if (pread(fd, &h, sizeof h, 0) != static_cast<ssize_t>(sizeof h) ||
      std::memcmp(h.magic, kCsrMagic, 8) != 0)
    io_fail("not a corpus cache: " + p);
  if (h.version != 1) io_fail("unsupported corpus cache version in " + p);
  if (h.n_docs < 1 || h.n_words < 1 || h.nnz < 0 || h.vocab_bytes < 0 ||
      h.n_words > (int64_t{1} << 31))
    io_fail("implausible corpus cache header in " + p);
  const int64_t want = static_cast<int64_t>(sizeof h) + (h.n_docs + 1) * 8 + h.nnz * 8 + h.vocab_bytes;
  if (st.st_size != want) io_fail("corpus cache size disagrees with its header: " + p);
  c.n_docs = h.n_docs;
  c.n_words = h.n_words;
  c.n_tokens = h.n_tokens;
  c.offsets.resize(static_cast<size_t>(h.n_docs) + 1);
  c.words.alloc(static_cast<size_t>(h.nnz));
  c.counts.alloc(static_cast<size_t>(h.nnz));
  c.vocab.resize(static_cast<size_t>(h.vocab_bytes));
  off_t off = sizeof h;
  read_at(fd, c.offsets.data(), c.offsets.size() * 8, off, T, p);
  off += static_cast<off_t>(c.offsets.size() * 8);
  read_at(fd, c.words.data(), c.words.size() * 4, off, T, p);
  off += static_cast<off_t>(c.words.size() * 4);
  read_at(fd, c.counts.data(), c.counts.size() * 4, off, T, p);
  off += static_cast<off_t>(c.counts.size() * 4);
  read_at(fd, c.vocab.data(), c.vocab.size(), off, T, p);
  // CSR invariants (corpus.hpp:12-15) and totals
  if (c.offsets[0] != 0 || c.offsets[h.n_docs] != h.nnz) io_fail("corrupt corpus cache: " + p);
  std::vector<int64_t> tok(static_cast<size_t>(T), 0);
  std::vector<char> bad(static_cast<size_t>(T), 0);
  parallel_ranges(h.n_docs, T, [&](int part, int64_t b, int64_t e) {
    int64_t t = 0;
    for (int64_t d = b; d < e && !bad[part]; ++d) {
      const int64_t lo = c.offsets[d], hi = c.offsets[d + 1];
      if (hi < lo || hi > h.nnz) {
        bad[part] = 1;
        break;
      }
      for (int64_t i = lo; i < hi; ++i) {
        if (c.words[i] < 0 || c.words[i] >= h.n_words || c.counts[i] < 1 ||
            (i > lo && c.words[i] <= c.words[i - 1])) {
          bad[part] = 1;
          break;
        }
        t += c.counts[i];
      }
    }
    tok[part] = t;
  });
  int64_t sum = 0;
  for (int i = 0; i < T; ++i) {
    if (bad[i]) io_fail("corrupt corpus cache: " + p);
    sum += tok[i];
  }
  if (sum != h.n_tokens) io_fail("corrupt corpus cache (token total): " + p);
  int64_t lines = 0;
  for (char ch : c.vocab) lines += ch == '\n';
  if (lines != h.n_words || (!c.vocab.empty() && c.vocab.back() != '\n'))
    io_fail("corrupt corpus cache (vocabulary): " + p);
}

int64_t vocab_lines(const char* vocab, int64_t bytes) {
  int64_t n = 0;
  for (int64_t i = 0; i < bytes; ++i) n += vocab[i] == '\n';
  return n;
}

void check_view(const samelda_cu_corpus* c) {
  if (!c || !c->doc_offsets || c->n_docs < 0 || c->n_words < 1)
    throw IoFail{SAMELDA_CU_CONFIG, "corpus view is malformed"};
}

}  // namespace

extern "C" {

const char* samelda_io_last_error(void) { return g_err.c_str(); }

int samelda_io_load_uci(const char* docword_path, const char* vocab_path, int n_threads,
                        samelda_io_corpus** out) {
  if (!out || !docword_path || !vocab_path) {
    g_err = "samelda_io_load_uci: null argument";
    return SAMELDA_CU_CONFIG;
  }
  *out = nullptr;
  auto* c = new samelda_io_corpus;
  const int rc = guarded([&] { load_uci(docword_path, vocab_path, n_threads, *c); });
  if (rc != SAMELDA_CU_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return rc;
}

int samelda_io_save_csr(const char* path, const samelda_cu_corpus* corpus, const char* vocab,
                        int64_t vocab_bytes) {
  return guarded([&] {
    check_view(corpus);
    if (vocab_bytes < 0 || (vocab_bytes > 0 && !vocab) ||
        vocab_lines(vocab, vocab_bytes) != corpus->n_words ||
        (vocab_bytes > 0 && vocab[vocab_bytes - 1] != '\n'))
      throw IoFail{SAMELDA_CU_CONFIG, "corpus cache: vocabulary must hold n_words '\\n'-terminated lines"};
    const std::string p(path);
    FILE* f = std::fopen(path, "wb");
    if (!f) io_fail("cannot write corpus cache: " + p);
    struct Closer {
      FILE* f;
      ~Closer() {
        if (f) std::fclose(f);
      }
    } closer{f};
    const int64_t nnz = corpus->doc_offsets[corpus->n_docs];
    int64_t tokens = 0;
    for (int64_t i = 0; i < nnz; ++i) tokens += corpus->counts[i];
    CsrHeader h{};
    std::memcpy(h.magic, kCsrMagic, 8);
    h.version = 1;
    h.n_docs = corpus->n_docs;
    h.n_words = corpus->n_words;
    h.nnz = nnz;
    h.n_tokens = tokens;
    h.vocab_bytes = vocab_bytes;
    write_all(f, &h, sizeof h, p);
    write_all(f, corpus->doc_offsets, static_cast<size_t>(corpus->n_docs + 1) * 8, p);
    write_all(f, corpus->word_ids, static_cast<size_t>(nnz) * 4, p);
    write_all(f, corpus->counts, static_cast<size_t>(nnz) * 4, p);
    write_all(f, vocab, static_cast<size_t>(vocab_bytes), p);
    const int rc = std::fclose(f);
    closer.f = nullptr;
    if (rc != 0) io_fail("write failed: " + p);
  });
}

int samelda_io_load_csr(const char* path, int n_threads, samelda_io_corpus** out) {
  if (!out || !path) {
    g_err = "samelda_io_load_csr: null argument";
    return SAMELDA_CU_CONFIG;
  }
  *out = nullptr;
  auto* c = new samelda_io_corpus;
  const int rc = guarded([&] { load_csr(path, n_threads, *c); });
  if (rc != SAMELDA_CU_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return rc;
}

void samelda_io_corpus_dims(const samelda_io_corpus* c, int64_t* n_docs, int64_t* n_words,
                            int64_t* nnz, int64_t* n_tokens, int64_t* vocab_bytes,
                            int64_t* dropped_docs) {
  if (n_docs) *n_docs = c->n_docs;
  if (n_words) *n_words = c->n_words;
  if (nnz) *nnz = static_cast<int64_t>(c->words.size());
  if (n_tokens) *n_tokens = c->n_tokens;
  if (vocab_bytes) *vocab_bytes = static_cast<int64_t>(c->vocab.size());
  if (dropped_docs) *dropped_docs = c->dropped;
}

void samelda_io_corpus_view(const samelda_io_corpus* c, samelda_cu_corpus* view,
                            const char** vocab) {
  if (view) {
    view->doc_offsets = c->offsets.data();
    view->word_ids = c->words.data();
    view->counts = c->counts.data();
    view->n_docs = c->n_docs;
    view->n_words = c->n_words;
  }
  if (vocab) *vocab = c->vocab.data();
}

void samelda_io_corpus_free(samelda_io_corpus* c) { delete c; }

int samelda_io_save_uci(const samelda_cu_corpus* corpus, const char* vocab, int64_t vocab_bytes,
                        const char* docword_path, const char* vocab_path) {
  return guarded([&] {
    check_view(corpus);
    const std::string dp(docword_path), vp(vocab_path);
    FILE* f = std::fopen(docword_path, "w");
    if (!f) io_fail("cannot write docword file: " + dp);
    const int64_t D = corpus->n_docs;
    const int64_t nnz = corpus->doc_offsets[D];
    // corpus.cpp:192-199: header, then "d+1 w+1 c" per cell in row order;
    // rows formatted in parallel, written in order
    std::string head = std::to_string(D) + "\n" + std::to_string(corpus->n_words) + "\n" +
                       std::to_string(nnz) + "\n";
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    const int T = threads_for(0);
    const int64_t step = 1 << 16;
    for (int64_t d0 = 0; d0 < D && ok; d0 += step * T) {
      std::vector<std::string> bufs(static_cast<size_t>(T));
      parallel_ranges(T, T, [&](int, int64_t b, int64_t e) {
        for (int64_t t = b; t < e; ++t) {
          std::string& s = bufs[t];
          const int64_t lo = d0 + t * step, hi = std::min(D, lo + step);
          // "d w c\n": three integers of <= 20 digits each
          char num[24];
          auto put = [&](int64_t v, char sep) {
            const auto r = std::to_chars(num, num + sizeof num, v);
            s.append(num, static_cast<size_t>(r.ptr - num));
            s.push_back(sep);
          };
          for (int64_t d = lo; d < hi; ++d)
            for (int64_t i = corpus->doc_offsets[d]; i < corpus->doc_offsets[d + 1]; ++i) {
              put(d + 1, ' ');
              put(static_cast<int64_t>(corpus->word_ids[i]) + 1, ' ');
              put(corpus->counts[i], '\n');
            }
        }
      });
      for (auto& s : bufs) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) io_fail("write failed: " + dp);
    FILE* v = std::fopen(vocab_path, "w");
    if (!v) io_fail("cannot write vocab file: " + vp);
    bool vok = vocab_bytes == 0 || std::fwrite(vocab, 1, static_cast<size_t>(vocab_bytes), v) ==
                                       static_cast<size_t>(vocab_bytes);
    vok = (std::fclose(v) == 0) && vok;
    if (!vok) io_fail("write failed: " + vp);
  });
}

// ------------------------------------------------------------- checkpoint

int samelda_io_save_checkpoint(const char* path, int64_t n_topics, int64_t n_words, double alpha,
                               double beta, const double* phi_kw) {
  return guarded([&] {
    const std::string p(path);
    FILE* f = std::fopen(path, "wb");
    if (!f) io_fail("cannot write checkpoint: " + p);
    // model.cpp:59-66: magic, u32 version, u64 K, u64 W, f64 alpha, f64 beta, phi
    static const char magic[8] = {'S', 'A', 'M', 'E', 'L', 'D', 'A', '1'};
    const uint32_t version = 1;
    const uint64_t k = static_cast<uint64_t>(n_topics), w = static_cast<uint64_t>(n_words);
    bool ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(&version, 4, 1, f) == 1 &&
              std::fwrite(&k, 8, 1, f) == 1 && std::fwrite(&w, 8, 1, f) == 1 &&
              std::fwrite(&alpha, 8, 1, f) == 1 && std::fwrite(&beta, 8, 1, f) == 1;
    const size_t n = static_cast<size_t>(n_topics * n_words);
    ok = ok && (n == 0 || std::fwrite(phi_kw, 8, n, f) == n);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) io_fail("write failed: " + p);
  });
}

namespace {
struct CkptHeader {
  int64_t k, w;
  double alpha, beta;
};

// model.cpp:71-96 checks, in order
CkptHeader read_ckpt_header(FILE* f, const std::string& p) {
  char magic[8];
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, "SAMELDA1", 8) != 0)
    io_fail("not a model checkpoint: " + p);
  uint32_t version = 0;
  if (std::fread(&version, 4, 1, f) != 1) io_fail("truncated checkpoint: " + p);
  if (version != 1) io_fail("unsupported checkpoint version in " + p);
  uint64_t k = 0, w = 0;
  if (std::fread(&k, 8, 1, f) != 1) io_fail("truncated checkpoint: " + p);
  if (std::fread(&w, 8, 1, f) != 1) io_fail("truncated checkpoint: " + p);
  CkptHeader h{static_cast<int64_t>(k), static_cast<int64_t>(w), 0.0, 0.0};
  if (h.k < 1 || h.w < 1 || h.k > (1 << 20) || h.w > (int64_t{1} << 32))
    io_fail("implausible checkpoint header in " + p);
  if (std::fread(&h.alpha, 8, 1, f) != 1) io_fail("truncated checkpoint: " + p);
  if (std::fread(&h.beta, 8, 1, f) != 1) io_fail("truncated checkpoint: " + p);
  return h;
}
}  // namespace

int samelda_io_checkpoint_header(const char* path, int64_t* n_topics, int64_t* n_words,
                                 double* alpha, double* beta) {
  return guarded([&] {
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) io_fail("cannot open checkpoint: " + p);
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    const CkptHeader h = read_ckpt_header(f, p);
    *n_topics = h.k;
    *n_words = h.w;
    *alpha = h.alpha;
    *beta = h.beta;
  });
}

int samelda_io_load_checkpoint(const char* path, double* phi_kw, int64_t cap_elems) {
  return guarded([&] {
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) io_fail("cannot open checkpoint: " + p);
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    const CkptHeader h = read_ckpt_header(f, p);
    const int64_t n = h.k * h.w;
    if (n > cap_elems) throw IoFail{SAMELDA_CU_CONFIG, "checkpoint phi does not fit the buffer"};
    if (std::fread(phi_kw, 8, static_cast<size_t>(n), f) != static_cast<size_t>(n))
      io_fail("truncated checkpoint: " + p);
    char extra;
    if (std::fread(&extra, 1, 1, f) == 1) io_fail("trailing bytes in checkpoint: " + p);
  });
}

// ---------------------------------------------------------------- metrics

int samelda_io_write_metrics_csv(const char* path, const samelda_cu_trace_row* rows, int64_t n) {
  return guarded([&] {
    const std::string p(path);
    FILE* f = std::fopen(path, "w");
    if (!f) io_fail("cannot write metrics csv: " + p);
    bool ok = std::fputs("t,passes,samples_per_word,ll,wall_seconds,m_t\n", f) >= 0;
    char line[256];
    for (int64_t i = 0; i < n && ok; ++i) {
      const auto& r = rows[i];
      const int len = std::snprintf(line, sizeof line, "%lld,%.17g,%.17g,%.17g,%.17g,%.17g\n",
                                    static_cast<long long>(r.t), r.passes, r.samples_per_word,
                                    r.ll, r.wall_seconds, r.m_t);
      ok = std::fwrite(line, 1, static_cast<size_t>(len), f) == static_cast<size_t>(len);
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) io_fail("write failed: " + p);
  });
}

int samelda_io_read_metrics_csv(const char* path, samelda_cu_trace_row* rows, int64_t cap,
                                int64_t* n) {
  return guarded([&] {
    const std::string p(path);
    Mapped m;
    if (!map_file(path, m)) io_fail("cannot open metrics csv: " + p);
    std::string text(m.p, m.n);
    size_t pos = 0;
    auto getline = [&](std::string& line) {
      if (pos >= text.size()) return false;
      const size_t nl = text.find('\n', pos);
      const size_t end = nl == std::string::npos ? text.size() : nl;
      line.assign(text, pos, end - pos);
      pos = end + 1;
      return true;
    };
    std::string line;
    if (!getline(line) || line != "t,passes,samples_per_word,ll,wall_seconds,m_t")
      io_fail("unexpected metrics csv header in " + p);
    int64_t count = 0;
    while (getline(line)) {
      if (line.empty()) continue;
      samelda_cu_trace_row r{};
      char* cursor = line.data();
      char* end = nullptr;
      r.t = std::strtoll(cursor, &end, 10);
      double* fields[] = {&r.passes, &r.samples_per_word, &r.ll, &r.wall_seconds, &r.m_t};
      for (double* field : fields) {
        if (*end != ',') io_fail("malformed metrics csv row in " + p);
        cursor = end + 1;
        *field = std::strtod(cursor, &end);
      }
      if (count < cap && rows) rows[count] = r;
      ++count;
    }
    *n = count;
  });
}

}  // extern "C"
