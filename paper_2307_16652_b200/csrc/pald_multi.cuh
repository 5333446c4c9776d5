// pald_multi.cuh -- several GPUs in ONE call of the C ABI (one process,
// one host thread per listed device): the B200 counterpart of
// parallel_pairwise / parallel_triplet (parallel.hpp:159-222, :257-320),
// whose ParallelPlan.workers becomes pald_gpu_opts.devices.
//
// Included by pald_gpu.cu inside its internal namespace (it uses the plan
// internals). Decomposition, every device holding the full D:
//   upload    device i copies row band i of D from the host, then pulls the
//             other bands from their devices (cudaMemcpyPeerAsync: NVLink
//             P2P where enabled, staged by the driver otherwise);
//   load      validation / range check / layout / rank codes on every device
//             (identical, O(n^2));
//   pass 1    device i computes share i of the pass-1 work units into its own
//             count buffer (RED: into every device's);
//   exchange  PEER: fused reduce + finish + all-gather (focus_finish_kernel
//             <PEERS>, each device a 1/N range of tiles, P2P loads of the
//             counts, P2P stores of U and W = 1/U); NCCL: ncclAllReduce of
//             the counts + local finish; RED: local finish;
//   pass 2    pair kernel: share i of the tile pairs, each finished tile
//             stored into every device's C (PEER) or into a zeroed C summed
//             by ncclAllReduce (NCCL); one-sided kernel (tie-heavy input,
//             InclusiveSplit, exact path): device i computes tile-row band
//             i -- no exchange at all;
//   download  device i copies row band i of U and C to the host.
// Every C entry is one in-order fp32 sum on one device, so U and C are
// bit-identical to one device for any device list. The host threads meet
// at a barrier between the phases (each after synchronizing its stream); no
// kernel ever waits on another device.
#pragma once
// (system headers <dlfcn.h>, <condition_variable>, <thread>, <atomic> are
// included at the top of pald_gpu.cu: this file is included inside a namespace)

// ---------------------------------------------------------------------------
// NCCL, loaded on first use (the library is not a link dependency: the PEER
// transport needs none, and torch may already have loaded its own copy).
struct NcclApi {
  bool tried = false;
  bool ok = false;
  std::string why;
  int (*CommInitAll)(void** comms, int ndev, const int* devlist) = nullptr;
  int (*CommDestroy)(void* comm) = nullptr;
  int (*AllReduce)(const void* send, void* recv, size_t count, int dtype, int op, void* comm,
                   cudaStream_t s) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
constexpr int kNcclFloat32 = 7, kNcclSum = 0;  // nccl.h: ncclFloat32, ncclSum

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.CommInitAll && api.CommDestroy && api.AllReduce && api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks the collective entry points";
  });
  return api;
}

// ---------------------------------------------------------------------------
// Pass-1 exchange by peer pull (see focus_finish_kernel<PEERS>): this plan
// finishes share `part` of `parts` of the upper-triangular tiles from the
// counts in every attached W, storing W = 1/U into every W and U into every
// attached U (u_all) or only its own.
int plan_focus_finish_peers_impl(pald_gpu_plan* p, uint64_t part, uint64_t parts, int u_mode, cudaStream_t s) {
  if (!p->loaded) return set_error(PALD_GPU_ERR_VALIDATION, "plan has no distances loaded");
  if (p->peer_rank < 0) return set_error(PALD_GPU_ERR_VALIDATION, "no peers attached");
  if (u_mode < 0 || u_mode > 2) return set_error(PALD_GPU_ERR_VALIDATION, "unknown U mode %d", u_mode);
  if (u_mode && p->peer_u.count != p->peer_w.count)
    return set_error(PALD_GPU_ERR_VALIDATION, "peer U buffers not attached");
  if (parts < 1 || part >= parts)
    return set_error(PALD_GPU_ERR_VALIDATION, "invalid share %llu of %llu", (unsigned long long)part,
                     (unsigned long long)parts);
  const uint64_t tiles = p->nb * (p->nb + 1) / 2;
  const uint64_t t0 = tiles * part / parts, t1 = tiles * (part + 1) / parts;
  if (t1 <= t0) return PALD_GPU_OK;
  FinishPeers fp{};
  fp.count = p->peer_w.count;
  fp.u_mode = u_mode;
  for (int q = 0; q < fp.count; ++q) {
    fp.w[q] = p->peer_w.ptr[q];
    fp.u[q] = reinterpret_cast<int32_t*>(u_mode ? p->peer_u.ptr[q] : nullptr);
  }
  focus_finish_kernel<true><<<(unsigned)((t1 - t0) * 4), 256, 0, s>>>(p->u, p->w, (int)p->n, (int)p->ld,
                                                                       (int)p->nb, (int)t0, fp);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}

// ---------------------------------------------------------------------------
class HostBarrier {
 public:
  explicit HostBarrier(int count) : count_(count) {}
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    const int gen = gen_;
    if (++waiting_ == count_) {
      waiting_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen != gen_; });
    }
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  int count_, waiting_ = 0, gen_ = 0;
};

// One plan, two streams and the band events per listed device, cached
// across calls with the same n and device list.
struct MultiCtx {
  int num = 0;
  int devs[PALD_GPU_MAX_DEVICES] = {};
  uint64_t n = 0;
  std::unique_ptr<pald_gpu_plan> plan[PALD_GPU_MAX_DEVICES];
  cudaStream_t s[PALD_GPU_MAX_DEVICES] = {}, sc[PALD_GPU_MAX_DEVICES] = {};
  cudaEvent_t ev_band[PALD_GPU_MAX_DEVICES] = {};
  bool peer_ok = false;  // every pair of listed devices has P2P access
  void* comms[PALD_GPU_MAX_DEVICES] = {};
  bool nccl_ready = false;

  ~MultiCtx() {
    for (int i = 0; i < num; ++i) {
      cudaSetDevice(devs[i]);
      if (s[i]) cudaStreamDestroy(s[i]);
      if (sc[i]) cudaStreamDestroy(sc[i]);
      if (ev_band[i]) cudaEventDestroy(ev_band[i]);
      if (comms[i] && nccl().ok) nccl().CommDestroy(comms[i]);
      if (plan[i]) {
        plan[i]->peer_w = PeerBufs{};  // not IPC mappings: nothing to close
        plan[i]->peer_c = PeerBufs{};
        plan[i]->peer_u = PeerBufs{};
        plan[i]->peer_rank = -1;
      }
      plan[i].reset();
    }
  }
};

std::unique_ptr<MultiCtx>& multi_slot() {
  static std::unique_ptr<MultiCtx> m;
  return m;
}

int get_multi(const pald_gpu_opts* o, uint64_t n, MultiCtx** out) {
  auto& slot = multi_slot();
  const int N = o->num_devices;
  bool same = slot && slot->n == n && slot->num == N;
  for (int i = 0; same && i < N; ++i) same = slot->devs[i] == o->devices[i];
  if (!same) {
    slot.reset();
    std::unique_ptr<MultiCtx> m(new MultiCtx());
    m->num = N;
    m->n = n;
    for (int i = 0; i < N; ++i) m->devs[i] = o->devices[i];
    for (int i = 0; i < N; ++i) {
      pald_gpu_opts oi = *o;
      oi.device = o->devices[i];
      oi.num_devices = 0;
      pald_gpu_plan* p = nullptr;
      int rc = pald_gpu_plan_create(n, &oi, &p);
      if (rc) return rc;
      m->plan[i].reset(p);
      DeviceGuard g(m->devs[i]);
      PALD_CUDA(cudaStreamCreateWithFlags(&m->s[i], cudaStreamNonBlocking));
      PALD_CUDA(cudaStreamCreateWithFlags(&m->sc[i], cudaStreamNonBlocking));
      PALD_CUDA(cudaEventCreateWithFlags(&m->ev_band[i], cudaEventDisableTiming));
    }
    // P2P access between every pair of distinct listed devices (a repeated
    // device reaches its own memory directly).
    m->peer_ok = true;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        const int a = m->devs[i], b = m->devs[j];
        if (a == b) continue;
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) {
          m->peer_ok = false;
          continue;
        }
        DeviceGuard g(a);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) m->peer_ok = false;
        cudaGetLastError();  // clear cudaErrorPeerAccessAlreadyEnabled
      }
    // Every plan sees every device's U, W and C (UVA pointers, no IPC).
    for (int i = 0; i < N; ++i) {
      pald_gpu_plan* p = m->plan[i].get();
      for (int q = 0; q < N; ++q) {
        p->peer_w.ptr[q] = m->plan[q]->w;
        p->peer_c.ptr[q] = m->plan[q]->c;
        p->peer_u.ptr[q] = reinterpret_cast<float*>(m->plan[q]->u);
      }
      p->peer_w.count = p->peer_c.count = p->peer_u.count = N;
      p->peer_rank = i;
    }
    slot = std::move(m);
  }
  for (int i = 0; i < N; ++i) {
    pald_gpu_plan* p = slot->plan[i].get();
    p->algorithm = o->algorithm;
    p->policy = o->policy;
    p->flags = o->flags;
    p->loaded = false;
  }
  *out = slot.get();
  return PALD_GPU_OK;
}

int ensure_nccl(MultiCtx* m) {
  if (m->nccl_ready) return PALD_GPU_OK;
  NcclApi& api = nccl();
  if (!api.ok) return set_error(PALD_GPU_ERR_COMM, "NCCL exchange unavailable: %s", api.why.c_str());
  for (int i = 0; i < m->num; ++i)
    for (int j = i + 1; j < m->num; ++j)
      if (m->devs[i] == m->devs[j])
        return set_error(PALD_GPU_ERR_COMM,
                         "NCCL exchange needs distinct devices (device %d is listed twice); use the PEER exchange",
                         m->devs[i]);
  const int r = api.CommInitAll(m->comms, m->num, m->devs);
  if (r != 0) return set_error(PALD_GPU_ERR_COMM, "ncclCommInitAll: %s", api.GetErrorString(r));
  m->nccl_ready = true;
  return PALD_GPU_OK;
}

int nccl_sum(MultiCtx* m, int i, float* buf, size_t count) {
  NcclApi& api = nccl();
  const int r = api.AllReduce(buf, buf, count, kNcclFloat32, kNcclSum, m->comms[i], m->s[i]);
  if (r != 0) return set_error(PALD_GPU_ERR_COMM, "ncclAllReduce: %s", api.GetErrorString(r));
  return PALD_GPU_OK;
}

// Multi-device one-shot call (pald_gpu_cohesion_f32 with num_devices > 1).
int run_multi(const float* D, uint64_t n, const pald_gpu_opts* o, int32_t* U_out, float* C_out,
              pald_gpu_phase_times* times) {
  const auto t_start = std::chrono::steady_clock::now();
  MultiCtx* m = nullptr;
  int rc = get_multi(o, n, &m);
  if (rc) return rc;
  const int N = m->num;
  int xf = o->exchange_focus, xc = o->exchange_cohesion;
  if (xf == PALD_GPU_EXCHANGE_AUTO) xf = m->peer_ok ? PALD_GPU_EXCHANGE_PEER : PALD_GPU_EXCHANGE_NCCL;
  if (xc == PALD_GPU_EXCHANGE_AUTO) xc = m->peer_ok ? PALD_GPU_EXCHANGE_PEER : PALD_GPU_EXCHANGE_NCCL;
  if (!m->peer_ok && (xf == PALD_GPU_EXCHANGE_PEER || xf == PALD_GPU_EXCHANGE_RED || xc == PALD_GPU_EXCHANGE_PEER))
    return set_error(PALD_GPU_ERR_COMM, "peer exchange requested but the listed devices lack P2P access");
  if ((xf == PALD_GPU_EXCHANGE_NCCL || xc == PALD_GPU_EXCHANGE_NCCL) && (rc = ensure_nccl(m))) return rc;

  // tile-aligned row bands: upload, one-sided pass 2 and download
  const uint64_t nb = m->plan[0]->nb, ld = m->plan[0]->ld;
  auto band = [&](int i, uint64_t& r0, uint64_t& r1) {
    r0 = std::min(n, nb * i / N * kTile);
    r1 = std::min(n, nb * (i + 1) / N * kTile);
  };
  HostBarrier bar(N);
  std::vector<int> status(N, PALD_GPU_OK);
  std::vector<std::string> msg(N);
  std::atomic<bool> failed{false};
  bool use_pairs = false;          // decided by slot 0 after the load (same D everywhere)
  double t_marks[4] = {0, 0, 0, 0};  // focus begin, focus end, cohesion end, download end
  auto now = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count(); };

  auto worker = [&](int i) {
    pald_gpu_plan* p = m->plan[i].get();
    const cudaStream_t s = m->s[i], sc = m->sc[i];
    uint64_t r0, r1;
    band(i, r0, r1);
    auto step = [&](auto&& fn) {  // run a phase unless a device failed, then meet the others
      if (!failed.load()) {
        const int r = fn();
        if (r) {
          status[i] = r;
          msg[i] = g_last_error;
          failed = true;
        }
      }
      bar.wait();
    };
    cudaSetDevice(m->devs[i]);
    // upload: own band from the host
    step([&]() -> int {
      if (r1 > r0)
        PALD_CUDA(cudaMemcpy2DAsync(p->c + r0 * ld, ld * 4, D + r0 * n, n * 4, n * 4, r1 - r0,
                                    cudaMemcpyHostToDevice, sc));
      PALD_CUDA(cudaEventRecord(m->ev_band[i], sc));
      return PALD_GPU_OK;
    });
    // the other bands from their devices, then the load
    step([&]() -> int {
      for (int j = 0; j < N; ++j) {
        PALD_CUDA(cudaStreamWaitEvent(s, m->ev_band[j], 0));
        uint64_t a0, a1;
        band(j, a0, a1);
        if (j == i || a1 <= a0) continue;
        pald_gpu_plan* q = m->plan[j].get();
        PALD_CUDA(cudaMemcpyPeerAsync(p->c + a0 * ld, m->devs[i], q->c + a0 * ld, m->devs[j], (a1 - a0) * ld * 4, s));
      }
      int r = plan_load_impl(p, p->c, ld, s);
      if (r) return r;
      PALD_CUDA(cudaStreamSynchronize(s));
      if (i == 0) {
        use_pairs = p->sym_ready && sym_preferred(p);
        t_marks[0] = now();
      }
      return PALD_GPU_OK;
    });
    // pass 1: share i of the work units
    step([&]() -> int {
      int r = plan_focus_counts_impl(p, i, N, s, xf == PALD_GPU_EXCHANGE_RED);
      if (r) return r;
      if (xf == PALD_GPU_EXCHANGE_NCCL && (r = nccl_sum(m, i, p->w, n * ld))) return r;
      PALD_CUDA(cudaStreamSynchronize(s));
      return PALD_GPU_OK;
    });
    // exchange + finish: U and W = 1/U complete on every device
    step([&]() -> int {
      // U only to the device that downloads its row (u_mode 2)
      int r = xf == PALD_GPU_EXCHANGE_PEER ? plan_focus_finish_peers_impl(p, i, N, 2, s)
                                           : plan_focus_finish_impl(p, s);
      if (r) return r;
      PALD_CUDA(cudaStreamSynchronize(s));
      if (i == 0) t_marks[1] = now();
      return PALD_GPU_OK;
    });
    // pass 2
    step([&]() -> int {
      int r;
      if (use_pairs && xc == PALD_GPU_EXCHANGE_PEER) {
        r = plan_cohesion_share_peers_impl(p, i, N, s);
      } else if (use_pairs) {  // NCCL: shares into zeroed C buffers, then their SUM
        if ((r = plan_cohesion_share_impl(p, i, N, s))) return r;
        r = nccl_sum(m, i, p->c, n * ld);
      } else {  // one-sided kernel: this device's row band, no exchange
        r = plan_cohesion_impl(p, r0, r1, s);
      }
      if (r) return r;
      PALD_CUDA(cudaStreamSynchronize(s));
      if (i == 0) t_marks[2] = now();
      return PALD_GPU_OK;
    });
    // download: row band i of U and C
    step([&]() -> int {
      if (r1 > r0) {
        if (U_out)
          PALD_CUDA(cudaMemcpy2DAsync(U_out + r0 * n, n * 4, p->u + r0 * ld, ld * 4, n * 4, r1 - r0,
                                      cudaMemcpyDeviceToHost, s));
        PALD_CUDA(cudaMemcpy2DAsync(C_out + r0 * n, n * 4, p->c + r0 * ld, ld * 4, n * 4, r1 - r0,
                                    cudaMemcpyDeviceToHost, s));
      }
      PALD_CUDA(cudaStreamSynchronize(s));
      return PALD_GPU_OK;
    });
  };
  std::vector<std::thread> threads;
  for (int i = 1; i < N; ++i) threads.emplace_back(worker, i);
  worker(0);
  for (auto& t : threads) t.join();
  t_marks[3] = now();
  for (int i = 0; i < N; ++i) {
    if (status[i]) {
      g_last_error = msg[i];
      for (int j = 0; j < N; ++j) {  // leave no work behind
        DeviceGuard g(m->devs[j]);
        cudaStreamSynchronize(m->s[j]);
        cudaStreamSynchronize(m->sc[j]);
      }
      return status[i];
    }
  }
  for (int i = 0; i < N; ++i) m->plan[i]->last_kernel = use_pairs ? PALD_GPU_KERNEL_PAIRS : m->plan[i]->last_kernel;
  if (times) {
    times->focus_seconds += t_marks[1] - t_marks[0];
    times->cohesion_seconds += t_marks[2] - t_marks[1];
    times->overhead_seconds += std::max(0.0, t_marks[3] - (t_marks[2] - t_marks[0]));
    times->total_seconds = t_marks[3];
  }
  return PALD_GPU_OK;
}
