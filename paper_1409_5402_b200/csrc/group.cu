// group.cu -- one process, several GPUs: the document-sharded train() of
// SURVEY.md 8(e) behind the C ABI (include/samelda_cu.h, samelda_cu_group_*),
// so the reference's own C++ callers (samelda::train, sampler.cpp:269-353,
// via shim/sampler_cuda.cpp) shard across the GPUs of a box without Python.
//
//   * documents are split into contiguous ranges balanced by nonzeros; device
//     i holds its range's CSR rows, theta rows and theta counts (a context of
//     its own, doc base = the range start, so every Philox key uses the
//     GLOBAL document id and each device draws exactly what one GPU would);
//   * one host MinibatchStream over the global corpus (corpus.cpp:252-285);
//     each device samples the batch documents it owns, in batch order;
//   * the one exchange per period: the W x K topic-word counts of the last
//     inner sweep (sampler.cpp:320-332), summed over devices in place with
//     ncclAllReduce on a communicator over the group's devices
//     (ncclCommInitAll, NVLink / NVSwitch), then the M-step runs replicated
//     -- integer counts, so phi is bit-identical to a single GPU in the
//     parity and throughput modes;
//   * evaluation on device 0 (every device holds the same phi).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the one torch already
// mapped in a Python process, else the system library).  A group whose
// device list repeats a device (tests on a one-GPU box) cannot form an NCCL
// communicator; its exchange sums the count buffers with a device kernel
// instead -- the same integer sum.
#include <cuda_runtime.h>
#include <cstdlib>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/samelda_cu.h"

namespace {

struct Nccl {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static const Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      r.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return r;
    }
    r.init_all = reinterpret_cast<decltype(r.init_all)>(dlsym(h, "ncclCommInitAll"));
    r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(dlsym(h, "ncclAllReduce"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "ncclCommDestroy"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    r.version = reinterpret_cast<decltype(r.version)>(dlsym(h, "ncclGetVersion"));
    r.ok = r.init_all && r.all_reduce && r.group_start && r.group_end && r.destroy && r.error_string;
    if (!r.ok) r.why = "libnccl.so.2 lacks a required symbol";
    return r;
  }();
  return n;
}

struct GroupFail {
  int code;
  std::string msg;
};

[[noreturn]] void gfail(int code, const std::string& msg) { throw GroupFail{code, msg}; }

void gck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) gfail(SAMELDA_CU_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// same-device exchange (a repeated device in the list): dst += src
__global__ void k_add_u64(unsigned long long* __restrict__ dst,
                          const unsigned long long* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}
__global__ void k_add_f64(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

}  // namespace

struct samelda_cu_group {
  std::vector<int> devices;
  std::vector<samelda_cu_ctx*> ctx;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> sampled;  // per member: its sampling is enqueued
  cudaEvent_t reduced = nullptr;     // same-device exchange finished (member 0's stream)
  std::vector<ncclComm_t> comms;     // empty when devices repeat
  // the int32 count exchange: per member a packed W x K buffer and its
  // over-bound cell count (device), and the counts read back (pinned)
  std::vector<void*> lo32, over_dev;
  unsigned long long* over_host = nullptr;
  bool local_exchange = false;
  std::string error;
  int64_t launches_nccl = 0;

  // resident training state
  bool ready = false;
  samelda_cu_config cfg{};
  int64_t D = 0, W = 0;
  std::vector<int64_t> lo, hi;           // member i owns global docs [lo[i], hi[i])
  std::vector<std::vector<int64_t>> offs;  // rebased CSR offsets per member
  std::vector<int32_t> owner;            // global doc -> member
  std::vector<double> doc_tokens;        // global
  double corpus_tokens = 0.0;
  std::vector<std::vector<int32_t>> ids;  // per-period owned local ids per member

  void check(int member, int rc, const char* what) {
    if (rc == SAMELDA_CU_OK) return;
    gfail(rc, std::string(what) + " (device " + std::to_string(devices[static_cast<size_t>(member)]) +
                  "): " + samelda_cu_last_error(ctx[static_cast<size_t>(member)]));
  }

  ~samelda_cu_group() {
    for (size_t i = 0; i < ctx.size(); ++i) {
      cudaSetDevice(devices[i]);
      if (ctx[i]) samelda_cu_destroy(ctx[i]);
      if (sampled.size() > i && sampled[i]) cudaEventDestroy(sampled[i]);
      if (streams.size() > i && streams[i]) cudaStreamDestroy(streams[i]);
    }
    if (reduced) {
      cudaSetDevice(devices[0]);
      cudaEventDestroy(reduced);
    }
    for (size_t i = 0; i < lo32.size(); ++i) {
      cudaSetDevice(devices[i]);
      if (lo32[i]) cudaFree(lo32[i]);
      if (over_dev[i]) cudaFree(over_dev[i]);
    }
    if (over_host) cudaFreeHost(over_host);
    if (!comms.empty() && nccl().ok)
      for (auto c : comms) nccl().destroy(c);
  }

  // integer counts over NCCL in int32 words (half the bytes): every member
  // packs its cells below (2^31 - 1) / n and counts the others; when no
  // member has such a cell the int32 sum is exact and is unpacked in place.
  // Returns false (nothing exchanged) when the u64 all-reduce is needed.
  bool exchange32(int64_t elems) {
    const size_t n = ctx.size();
    if (lo32.size() != n) {
      lo32.assign(n, nullptr);
      over_dev.assign(n, nullptr);
      gck(cudaMallocHost(reinterpret_cast<void**>(&over_host), sizeof(unsigned long long) * n), "pinned");
    }
    for (size_t i = 0; i < n; ++i) {
      gck(cudaSetDevice(devices[i]), "cudaSetDevice");
      if (!lo32[i]) {
        gck(cudaMalloc(&lo32[i], sizeof(int32_t) * static_cast<size_t>(elems)), "cudaMalloc");
        gck(cudaMalloc(&over_dev[i], sizeof(unsigned long long)), "cudaMalloc");
      }
      check(static_cast<int>(i),
            samelda_cu_phi_counts_pack32(ctx[i], lo32[i], elems, static_cast<int32_t>(n), over_dev[i]), "pack32");
      gck(cudaMemcpyAsync(over_host + i, over_dev[i], sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          streams[i]), "over count");
    }
    unsigned long long over = 0;
    for (size_t i = 0; i < n; ++i) {
      gck(cudaStreamSynchronize(streams[i]), "over count");  // the exchange's one host wait
      over += over_host[i];
    }
    if (over) return false;
    const Nccl& N = nccl();
    N.group_start();
    for (size_t i = 0; i < n; ++i) {
      gck(cudaSetDevice(devices[i]), "cudaSetDevice");
      const ncclResult_t r = N.all_reduce(lo32[i], lo32[i], static_cast<size_t>(elems), ncclInt32, ncclSum,
                                          comms[i], streams[i]);
      if (r != ncclSuccess) {
        N.group_end();
        gfail(SAMELDA_CU_CUDA, std::string("ncclAllReduce: ") + N.error_string(r));
      }
    }
    const ncclResult_t r = N.group_end();
    if (r != ncclSuccess) gfail(SAMELDA_CU_CUDA, std::string("ncclGroupEnd: ") + N.error_string(r));
    ++launches_nccl;
    for (size_t i = 0; i < n; ++i) {
      gck(cudaSetDevice(devices[i]), "cudaSetDevice");
      check(static_cast<int>(i), samelda_cu_phi_counts_unpack32(ctx[i], lo32[i], elems), "unpack32");
    }
    return true;
  }

  // the W x K phi-count exchange of one period (after every member's sample)
  void exchange() {
    const size_t n = ctx.size();
    if (n == 1 && comms.empty()) return;
    std::vector<void*> buf(n);
    int64_t elems = 0;
    int32_t eb = 0, is_f = 0;
    for (size_t i = 0; i < n; ++i)
      check(static_cast<int>(i), samelda_cu_phi_counts_device(ctx[i], &buf[i], &elems, &eb, &is_f),
            "phi counts");
    if (!local_exchange) {
      const char* ex = std::getenv("SAMELDA_EXCHANGE");  // "u64": keep the u64 all-reduce
      if (!is_f && !(ex && std::strcmp(ex, "u64") == 0) && exchange32(elems)) return;
      const Nccl& N = nccl();
      N.group_start();
      for (size_t i = 0; i < n; ++i) {
        gck(cudaSetDevice(devices[i]), "cudaSetDevice");
        const ncclResult_t r = N.all_reduce(buf[i], buf[i], static_cast<size_t>(elems),
                                            is_f ? ncclFloat64 : ncclUint64, ncclSum, comms[i],
                                            streams[i]);
        if (r != ncclSuccess) {
          N.group_end();
          gfail(SAMELDA_CU_CUDA, std::string("ncclAllReduce: ") + N.error_string(r));
        }
      }
      const ncclResult_t r = N.group_end();
      if (r != ncclSuccess) gfail(SAMELDA_CU_CUDA, std::string("ncclGroupEnd: ") + N.error_string(r));
      ++launches_nccl;
      return;
    }
    // one device: member 0 sums everyone's buffer, the others copy the sum back
    gck(cudaSetDevice(devices[0]), "cudaSetDevice");
    for (size_t i = 0; i < n; ++i) gck(cudaEventRecord(sampled[i], streams[i]), "event");
    for (size_t i = 1; i < n; ++i) {
      gck(cudaStreamWaitEvent(streams[0], sampled[i], 0), "wait");
      if (is_f)
        k_add_f64<<<148 * 4, 256, 0, streams[0]>>>(static_cast<double*>(buf[0]),
                                                   static_cast<const double*>(buf[i]), elems);
      else
        k_add_u64<<<148 * 4, 256, 0, streams[0]>>>(static_cast<unsigned long long*>(buf[0]),
                                                   static_cast<const unsigned long long*>(buf[i]),
                                                   elems);
    }
    gck(cudaEventRecord(reduced, streams[0]), "event");
    for (size_t i = 1; i < n; ++i) {
      gck(cudaStreamWaitEvent(streams[i], reduced, 0), "wait");
      gck(cudaMemcpyAsync(buf[i], buf[0], static_cast<size_t>(elems) * eb, cudaMemcpyDeviceToDevice,
                          streams[i]),
          "broadcast counts");
    }
    gck(cudaGetLastError(), "exchange");
  }
};

namespace {

template <class F>
int gguarded(samelda_cu_group* g, F&& fn) {
  if (g == nullptr) return SAMELDA_CU_CONFIG;
  try {
    fn();
    g->error.clear();
    return SAMELDA_CU_OK;
  } catch (const GroupFail& f) {
    g->error = f.msg;
    cudaGetLastError();
    return f.code;
  } catch (const std::exception& e) {
    g->error = e.what();
    return SAMELDA_CU_CUDA;
  }
}

// sampler.cpp:231-267 through the single-GPU ABI (the same host math)
double rho_at(int64_t t, const samelda_cu_config& c) {
  double v = 0.0;
  if (samelda_cu_rho_schedule(t, c.tau0, c.gamma, &v)) gfail(SAMELDA_CU_CONFIG, "rho_schedule");
  return v;
}
double m_at(int64_t t, const samelda_cu_config& c) {
  double v = 0.0;
  if (samelda_cu_anneal_m(c.schedule, t, c.t_max, c.m, &v)) gfail(SAMELDA_CU_CONFIG, "anneal_m");
  return v;
}

}  // namespace

extern "C" {

int samelda_cu_group_create(const int* devices, int n, samelda_cu_group** out) {
  if (out == nullptr || devices == nullptr || n < 1) return SAMELDA_CU_CONFIG;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return SAMELDA_CU_CUDA;
  }
  auto* g = new samelda_cu_group();
  const int rc = gguarded(g, [&] {
    g->devices.assign(devices, devices + n);
    for (int d : g->devices)
      if (d < 0 || d >= count) gfail(SAMELDA_CU_CONFIG, "group: device " + std::to_string(d) + " not present");
    std::vector<int> sorted = g->devices;
    std::sort(sorted.begin(), sorted.end());
    g->local_exchange = std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end();
    if (g->local_exchange && sorted.front() != sorted.back())
      gfail(SAMELDA_CU_CONFIG, "group: a device list either names distinct devices (NCCL) or one "
                               "device repeated (test mode)");
    g->ctx.assign(static_cast<size_t>(n), nullptr);
    g->streams.assign(static_cast<size_t>(n), nullptr);
    g->sampled.assign(static_cast<size_t>(n), nullptr);
    for (int i = 0; i < n; ++i) {
      if (samelda_cu_create(g->devices[static_cast<size_t>(i)], &g->ctx[static_cast<size_t>(i)]) !=
          SAMELDA_CU_OK)
        gfail(SAMELDA_CU_CUDA, "group: cannot create a context on device " +
                                   std::to_string(g->devices[static_cast<size_t>(i)]));
      gck(cudaSetDevice(g->devices[static_cast<size_t>(i)]), "cudaSetDevice");
      gck(cudaStreamCreateWithFlags(&g->streams[static_cast<size_t>(i)], cudaStreamNonBlocking), "stream");
      gck(cudaEventCreateWithFlags(&g->sampled[static_cast<size_t>(i)], cudaEventDisableTiming), "event");
      g->check(i, samelda_cu_set_stream(g->ctx[static_cast<size_t>(i)], g->streams[static_cast<size_t>(i)]),
               "set stream");
    }
    gck(cudaSetDevice(g->devices[0]), "cudaSetDevice");
    gck(cudaEventCreateWithFlags(&g->reduced, cudaEventDisableTiming), "event");
    if (!g->local_exchange) {
      const Nccl& N = nccl();
      if (!N.ok) gfail(SAMELDA_CU_CUDA, "group: " + N.why);
      g->comms.assign(static_cast<size_t>(n), nullptr);
      const ncclResult_t r = N.init_all(g->comms.data(), n, g->devices.data());
      if (r != ncclSuccess) {
        g->comms.clear();
        gfail(SAMELDA_CU_CUDA, std::string("ncclCommInitAll: ") + N.error_string(r));
      }
    }
  });
  if (rc != SAMELDA_CU_OK) {
    delete g;
    return rc;
  }
  *out = g;
  return SAMELDA_CU_OK;
}

void samelda_cu_group_destroy(samelda_cu_group* g) {
  if (g == nullptr) return;
  for (size_t i = 0; i < g->ctx.size(); ++i)
    if (g->ctx[i]) samelda_cu_synchronize(g->ctx[i]);
  delete g;
}

const char* samelda_cu_group_last_error(const samelda_cu_group* g) {
  return g ? g->error.c_str() : "null group";
}

int samelda_cu_group_size(const samelda_cu_group* g) { return g ? static_cast<int>(g->ctx.size()) : 0; }

int samelda_cu_group_uses_nccl(const samelda_cu_group* g) { return g && !g->comms.empty() ? 1 : 0; }

int samelda_cu_group_train_begin(samelda_cu_group* g, const samelda_cu_corpus* corpus,
                                 const samelda_cu_config* config) {
  return gguarded(g, [&] {
    if (corpus == nullptr || config == nullptr || corpus->doc_offsets == nullptr)
      gfail(SAMELDA_CU_CONFIG, "train: corpus / config is null");
    if (corpus->n_docs < 1) gfail(SAMELDA_CU_CONFIG, "train: corpus is empty");
    const size_t n = g->ctx.size();
    const int64_t D = corpus->n_docs;
    const int64_t* o = corpus->doc_offsets;
    const int64_t nnz = o[D];
    g->cfg = *config;
    g->D = D;
    g->W = corpus->n_words;
    // contiguous ranges balanced by nonzeros (parallel.hpp:29-43's idea);
    // every member gets at least one document when D >= n
    g->lo.assign(n, 0);
    g->hi.assign(n, 0);
    int64_t prev = 0;
    for (size_t i = 0; i < n; ++i) {
      int64_t b = D;
      if (i + 1 < n) {
        const int64_t target = nnz * static_cast<int64_t>(i + 1) / static_cast<int64_t>(n);
        b = std::lower_bound(o, o + D, target) - o;
        const int64_t left = static_cast<int64_t>(n - i - 1);
        b = std::max(b, std::min(prev + 1, D));  // non-empty when possible
        b = std::min(b, std::max(prev, D - left));
      }
      g->lo[i] = prev;
      g->hi[i] = b;
      prev = b;
    }
    g->owner.assign(static_cast<size_t>(D), 0);
    g->doc_tokens.assign(static_cast<size_t>(D), 0.0);
    g->corpus_tokens = 0.0;
    for (int64_t d = 0; d < D; ++d) {
      int64_t tok = 0;
      for (int64_t p = o[d]; p < o[d + 1]; ++p) tok += corpus->counts[p];
      g->doc_tokens[static_cast<size_t>(d)] = static_cast<double>(tok);
      g->corpus_tokens += static_cast<double>(tok);
    }
    g->offs.assign(n, {});
    g->ids.assign(n, {});
    for (size_t i = 0; i < n; ++i) {
      for (int64_t d = g->lo[i]; d < g->hi[i]; ++d) g->owner[static_cast<size_t>(d)] = static_cast<int32_t>(i);
      auto& off = g->offs[i];
      off.resize(static_cast<size_t>(g->hi[i] - g->lo[i] + 1));
      for (int64_t d = g->lo[i]; d <= g->hi[i]; ++d) off[static_cast<size_t>(d - g->lo[i])] = o[d] - o[g->lo[i]];
      // a member with no documents still holds phi (one empty document keeps
      // the corpus well-formed; it is never in a batch)
      const int64_t nd = std::max<int64_t>(g->hi[i] - g->lo[i], 1);
      if (g->hi[i] == g->lo[i]) off.assign(2, 0);
      static const int32_t zero = 0;
      const samelda_cu_corpus part{off.data(), nnz ? corpus->word_ids + o[g->lo[i]] : &zero,
                                   nnz ? corpus->counts + o[g->lo[i]] : &zero, nd, corpus->n_words};
      g->check(static_cast<int>(i), samelda_cu_train_begin(g->ctx[i], &part, config), "train_begin");
      g->check(static_cast<int>(i), samelda_cu_set_doc_base(g->ctx[i], g->lo[i]), "doc base");
    }
    g->ready = true;
  });
}

int samelda_cu_group_heldout(samelda_cu_group* g, const samelda_cu_corpus* test, uint64_t seed) {
  return gguarded(g, [&] { g->check(0, samelda_cu_heldout(g->ctx[0], test, seed), "heldout"); });
}

int samelda_cu_group_period(samelda_cu_group* g, const int32_t* doc_ids, int64_t B, int64_t t,
                            double m_t, double rho_t) {
  return gguarded(g, [&] {
    if (!g->ready) gfail(SAMELDA_CU_CONFIG, "period: call samelda_cu_group_train_begin first");
    const size_t n = g->ctx.size();
    for (auto& v : g->ids) v.clear();
    for (int64_t b = 0; b < B; ++b) {
      const int32_t d = doc_ids[b];
      if (d < 0 || d >= g->D) gfail(SAMELDA_CU_CONFIG, "batch doc id " + std::to_string(d) + " out of range");
      const size_t i = static_cast<size_t>(g->owner[static_cast<size_t>(d)]);
      g->ids[i].push_back(static_cast<int32_t>(d - g->lo[i]));
    }
    for (size_t i = 0; i < n; ++i)
      g->check(static_cast<int>(i),
               samelda_cu_period_sample(g->ctx[i], g->ids[i].data(), static_cast<int64_t>(g->ids[i].size()), t, m_t),
               "period sample");
    g->exchange();
    for (size_t i = 0; i < n; ++i)
      g->check(static_cast<int>(i), samelda_cu_period_update(g->ctx[i], rho_t), "period update");
  });
}

int samelda_cu_group_synchronize(samelda_cu_group* g) {
  return gguarded(g, [&] {
    for (size_t i = 0; i < g->ctx.size(); ++i)
      g->check(static_cast<int>(i), samelda_cu_synchronize(g->ctx[i]), "synchronize");
  });
}

int samelda_cu_group_evaluate(samelda_cu_group* g, double* ll_out) {
  return gguarded(g, [&] { g->check(0, samelda_cu_evaluate(g->ctx[0], ll_out), "evaluate"); });
}

int samelda_cu_group_model_download(samelda_cu_group* g, double* phi, double* theta) {
  return gguarded(g, [&] {
    if (!g->ready) gfail(SAMELDA_CU_CONFIG, "no model");
    if (phi) g->check(0, samelda_cu_model_download(g->ctx[0], phi, nullptr), "model download");
    if (theta)
      for (size_t i = 0; i < g->ctx.size(); ++i)
        if (g->hi[i] > g->lo[i])
          g->check(static_cast<int>(i),
                   samelda_cu_model_download(g->ctx[i], nullptr, theta + g->lo[i] * g->cfg.n_topics),
                   "model download");
  });
}

int samelda_cu_group_train(samelda_cu_group* g, const samelda_cu_corpus* corpus,
                           const samelda_cu_config* config, const samelda_cu_corpus* heldout,
                           int64_t eval_every, double* phi_out, double* theta_out,
                           samelda_cu_trace_row* trace, int64_t trace_cap, int64_t* n_trace) {
  // sampler.cpp:269-353 over the group (samelda_cu_train's loop, sharded)
  int rc = samelda_cu_group_train_begin(g, corpus, config);
  if (rc) return rc;
  *n_trace = 0;
  const bool do_eval = heldout != nullptr && eval_every > 0;
  if (do_eval && config->t_max > 0) {
    rc = samelda_cu_group_heldout(g, heldout, config->seed);
    if (rc) return rc;
  }
  return gguarded(g, [&] {
    if (config->t_max > 0) {
      samelda_cu_batches* bs = nullptr;
      if (samelda_cu_batches_create(corpus->n_docs, config->batch_fraction, config->seed, &bs))
        gfail(SAMELDA_CU_CONFIG, "minibatch_stream: batch_fraction must be in (0,1]");
      std::vector<int32_t> batch(static_cast<size_t>(samelda_cu_batches_size(bs)));
      const auto t_start = std::chrono::steady_clock::now();
      double tokens_seen = 0.0, samples_per_word = 0.0;
      try {
        for (int64_t t = 0; t < config->t_max; ++t) {
          const int64_t B = samelda_cu_batches_next(bs, batch.data());
          const double m_t = m_at(t + 1, *config);
          const double rho_t = rho_at(t, *config);
          int r = samelda_cu_group_period(g, batch.data(), B, t, m_t, rho_t);
          if (r) gfail(r, g->error);
          double batch_tokens = 0.0;
          for (int64_t b = 0; b < B; ++b) batch_tokens += g->doc_tokens[static_cast<size_t>(batch[b])];
          tokens_seen += batch_tokens;
          samples_per_word += m_t * batch_tokens / g->corpus_tokens;
          if (do_eval && ((t + 1) % eval_every == 0 || t + 1 == config->t_max)) {
            double ll = 0.0;
            r = samelda_cu_group_evaluate(g, &ll);
            if (r) gfail(r, g->error);
            const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t_start;
            if (*n_trace >= trace_cap) gfail(SAMELDA_CU_CONFIG, "trace buffer too small");
            trace[(*n_trace)++] = {t, tokens_seen / g->corpus_tokens, samples_per_word, ll, el.count(), m_t};
          }
        }
      } catch (...) {
        samelda_cu_batches_destroy(bs);
        throw;
      }
      samelda_cu_batches_destroy(bs);
    }
    const int r = samelda_cu_group_model_download(g, phi_out, theta_out);
    if (r) gfail(r, g->error);
  });
}

}  // extern "C"
