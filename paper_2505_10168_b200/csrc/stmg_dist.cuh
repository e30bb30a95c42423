// Time-slab multi-GPU STMG; included by stmg_hierarchy.cu.
//
// Partition.  Level l of the hierarchy is *distributed* when its n_t steps split
// into `world` equal slabs of >= min_slab levels (even-sized when the next step
// coarsens in time, so causal restriction 2N, 2N+1 -> N and prolongation
// floor(n/2) stay rank-local).  Rank g owns rows [g n_t/W, (g+1) n_t/W); the
// last rank also owns level n_t.  The first non-distributed level Lg and all
// coarser ones (incl. the coarsest exact march, which is sequential in time)
// are *gathered*: their right-hand side is gathered to rank 0, which runs that
// tail of the V-cycle as an ordinary single-GPU hierarchy and broadcasts the
// correction back.
//
// Storage.  Every rank allocates only its slab rows plus kSlabMargin levels on
// each side of every distributed level vector (SlabBuf), addressed through a
// globally indexed base pointer, so both HBM traffic and capacity scale as 1/W
// while indexing and layout stay those of the single-GPU path.  Before every
// stencil pass the ghost levels of the input vector are exchanged with the
// neighbours (J reads level n-1, J^T level n+1; both ghosts are exchanged), the
// norms are all-reduced.  All operations are pointwise-identical to the
// single-GPU path, so the iterate after k cycles is bit-identical; only the
// norm summation order changes.
//
// Transport.  `Comm` has two implementations: NCCL (one rank per process,
// NVLink/NVSwitch; libnccl.so.2 is dlopen'ed, reusing an already-loaded copy
// such as PyTorch's) and Loopback (this process hosts all `world` ranks on one
// GPU and exchanges by device-to-device copies — the single-GPU validation of
// the exact slab code path).  Every transport call is stream-ordered and is
// captured into the V-cycle graph.

#include <dlfcn.h>
#include <nccl.h>

namespace stmgb {
namespace {

// ---------------------------------------------------------------------------
// Partition (shared with the CPU gloo tests through stmg_dist_partition)
// ---------------------------------------------------------------------------
struct SlabPlan {
  int world = 1;
  int Lg = 0;                                // levels [0, Lg) distributed
  std::vector<std::vector<int64_t>> bounds;  // [l][g], g = 0..world; bounds[l][world] = n_t+1
};

SlabPlan plan_slabs(const std::vector<int64_t>& nts, const std::vector<int32_t>& dirs, int world,
                    int64_t min_slab) {
  if (world < 1) throw std::invalid_argument("dist: world size must be >= 1");
  if (min_slab < 8) min_slab = 8;
  SlabPlan p;
  p.world = world;
  const int L = static_cast<int>(nts.size());
  for (int l = 0; l + 1 < L; ++l) {
    const int64_t nt = nts[l];
    if (nt % world != 0) break;
    const int64_t slab = nt / world;
    if (slab < min_slab) break;
    if (dirs[l] == STMG_DIR_T && slab % 2 != 0) break;
    std::vector<int64_t> b(static_cast<size_t>(world) + 1);
    for (int g = 0; g < world; ++g) b[g] = g * slab;
    b[world] = nt + 1;
    p.bounds.push_back(std::move(b));
    p.Lg = l + 1;
  }
  return p;
}

// Rows of the first gathered level that rank g produces when restricting from
// its slab of level Lg - 1.
std::pair<int64_t, int64_t> gathered_rows(const SlabPlan& p, int dir_into, int g, int64_t nt_coarse) {
  const auto& b = p.bounds[p.Lg - 1];
  if (dir_into == STMG_DIR_T) {
    const int64_t lo = b[g] / 2;
    const int64_t hi = (g == p.world - 1) ? nt_coarse + 1 : b[g + 1] / 2;
    return {lo, hi};
  }
  return {b[g], b[g + 1]};
}

// ---------------------------------------------------------------------------
// Transport
// ---------------------------------------------------------------------------
__global__ void k_sum_scalars(const double* const* in, int n, double* const* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s = s + *in[k];  // fixed rank order
    for (int k = 0; k < n; ++k) *out[k] = s;
  }
}

struct Comm {
  int world = 1;
  int n_local = 1;
  int rank0 = 0;  // global rank of local slot 0
  virtual ~Comm() = default;
  virtual const char* name() const = 0;
  // ghost exchange of one vector per local rank (rows of level partition b, nn doubles per
  // row): `depth` levels on each side of every slab boundary
  virtual void exchange(const std::vector<double*>& v, const std::vector<int64_t>& b, int64_t nn,
                        int depth, cudaStream_t s) = 0;
  virtual void allreduce_sum(const std::vector<double*>& in, const std::vector<double*>& out,
                             cudaStream_t s) = 0;
  // rows [lo_g, hi_g) of every rank's src (full-size, nn per row) -> dst on rank 0
  virtual void gather_rows(const std::vector<double*>& src, double* dst,
                           const std::vector<std::pair<int64_t, int64_t>>& rows, int64_t nn,
                           cudaStream_t s) = 0;
  // count doubles from rank 0's root buffer to every local rank's dst
  virtual void broadcast(const double* root, const std::vector<double*>& dst, int64_t count,
                         cudaStream_t s) = 0;
  bool is_root() const { return rank0 == 0; }
};

struct LoopbackComm : Comm {
  std::unique_ptr<DeviceBuf> ptrs;  // 2 * n_local device pointers for allreduce
  std::vector<const double*> last_in;
  std::vector<double*> last_out;
  explicit LoopbackComm(int w) {
    world = w;
    n_local = w;
    rank0 = 0;
  }
  const char* name() const override { return "loopback"; }
  void exchange(const std::vector<double*>& v, const std::vector<int64_t>& b, int64_t nn, int depth,
                cudaStream_t s) override {
    const size_t bytes = sizeof(double) * static_cast<size_t>(nn * depth);
    for (int g = 1; g < world; ++g) {
      // last rows of g-1 -> leading ghosts of g ; first rows of g -> trailing ghosts of g-1
      cuda_check(cudaMemcpyAsync(v[g] + (b[g] - depth) * nn, v[g - 1] + (b[g] - depth) * nn, bytes,
                                 cudaMemcpyDeviceToDevice, s), "ghost copy");
      cuda_check(cudaMemcpyAsync(v[g - 1] + b[g] * nn, v[g] + b[g] * nn, bytes,
                                 cudaMemcpyDeviceToDevice, s), "ghost copy");
    }
  }
  void allreduce_sum(const std::vector<double*>& in, const std::vector<double*>& out,
                     cudaStream_t s) override {
    if (!ptrs) ptrs = std::make_unique<DeviceBuf>(2 * static_cast<int64_t>(world));
    if (last_out != out || last_in.size() != in.size() ||
        !std::equal(in.begin(), in.end(), last_in.begin())) {
      std::vector<const void*> hp;
      for (double* p : in) hp.push_back(p);
      for (double* p : out) hp.push_back(p);
      cuda_check(cudaMemcpy(ptrs->p, hp.data(), hp.size() * sizeof(void*), cudaMemcpyHostToDevice),
                 "ptr upload");
      last_in.assign(in.begin(), in.end());
      last_out = out;
    }
    const double* const* pin = reinterpret_cast<const double* const*>(ptrs->p);
    double* const* pout = reinterpret_cast<double* const*>(reinterpret_cast<void**>(ptrs->p) + world);
    k_sum_scalars<<<1, 32, 0, s>>>(pin, world, pout);
    launch_check(static_cast<int>(cudaGetLastError()), "sum scalars");
  }
  void gather_rows(const std::vector<double*>& src, double* dst,
                   const std::vector<std::pair<int64_t, int64_t>>& rows, int64_t nn,
                   cudaStream_t s) override {
    for (int g = 0; g < world; ++g) {
      const auto [lo, hi] = rows[g];
      if (hi > lo)
        cuda_check(cudaMemcpyAsync(dst + lo * nn, src[g] + lo * nn,
                                   sizeof(double) * static_cast<size_t>((hi - lo) * nn),
                                   cudaMemcpyDeviceToDevice, s), "gather copy");
    }
  }
  void broadcast(const double* root, const std::vector<double*>& dst, int64_t count,
                 cudaStream_t s) override {
    for (int g = 0; g < world; ++g)
      cuda_check(cudaMemcpyAsync(dst[g], root, sizeof(double) * static_cast<size_t>(count),
                                 cudaMemcpyDeviceToDevice, s), "broadcast copy");
  }
};

// NCCL entry points resolved at run time from libnccl.so.2.
struct NcclApi {
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) throw std::runtime_error("dist: libnccl.so.2 not found");
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) throw std::runtime_error(std::string("dist: NCCL symbol missing: ") + n);
      return p;
    };
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(int w, int rank, const ncclUniqueId& id) {
    world = w;
    n_local = 1;
    rank0 = rank;
    nccl_check(nccl().CommInitRank(&comm, w, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  const char* name() const override { return "nccl"; }
  void exchange(const std::vector<double*>& v, const std::vector<int64_t>& b, int64_t nn, int depth,
                cudaStream_t s) override {
    const int g = rank0;
    double* x = v[0];
    const auto& A = nccl();
    const size_t cnt = static_cast<size_t>(nn * depth);
    nccl_check(A.GroupStart(), "group");
    if (g > 0) {
      nccl_check(A.Send(x + b[g] * nn, cnt, ncclDouble, g - 1, comm, s), "send");
      nccl_check(A.Recv(x + (b[g] - depth) * nn, cnt, ncclDouble, g - 1, comm, s), "recv");
    }
    if (g < world - 1) {
      nccl_check(A.Send(x + (b[g + 1] - depth) * nn, cnt, ncclDouble, g + 1, comm, s), "send");
      nccl_check(A.Recv(x + b[g + 1] * nn, cnt, ncclDouble, g + 1, comm, s), "recv");
    }
    nccl_check(A.GroupEnd(), "group");
  }
  void allreduce_sum(const std::vector<double*>& in, const std::vector<double*>& out,
                     cudaStream_t s) override {
    nccl_check(nccl().AllReduce(in[0], out[0], 1, ncclDouble, ncclSum, comm, s), "allreduce");
  }
  void gather_rows(const std::vector<double*>& src, double* dst,
                   const std::vector<std::pair<int64_t, int64_t>>& rows, int64_t nn,
                   cudaStream_t s) override {
    const auto& A = nccl();
    nccl_check(A.GroupStart(), "group");
    if (rank0 == 0) {
      for (int g = 1; g < world; ++g) {
        const auto [lo, hi] = rows[g];
        if (hi > lo) nccl_check(A.Recv(dst + lo * nn, (hi - lo) * nn, ncclDouble, g, comm, s), "recv");
      }
    } else {
      const auto [lo, hi] = rows[rank0];
      if (hi > lo) nccl_check(A.Send(src[0] + lo * nn, (hi - lo) * nn, ncclDouble, 0, comm, s), "send");
    }
    nccl_check(A.GroupEnd(), "group");
    if (rank0 == 0) {
      const auto [lo, hi] = rows[0];
      if (hi > lo)
        cuda_check(cudaMemcpyAsync(dst + lo * nn, src[0] + lo * nn,
                                   sizeof(double) * static_cast<size_t>((hi - lo) * nn),
                                   cudaMemcpyDeviceToDevice, s), "gather copy");
    }
  }
  void broadcast(const double* root, const std::vector<double*>& dst, int64_t count,
                 cudaStream_t s) override {
    nccl_check(nccl().Broadcast(rank0 == 0 ? root : dst[0], dst[0], count, ncclDouble, 0, comm, s),
               "broadcast");
  }
};

// ---------------------------------------------------------------------------
// Peer-memory ghost exchange (STMG_DIST_P2P=1): each rank PULLS its ghost levels
// straight out of the neighbours' level vectors over NVLink (CUDA IPC
// mappings; in loopback the neighbours' buffers are local), ordered by a
// neighbour-only epoch barrier instead of NCCL send/recv:
//   exchange e = (own completed epoch) + 1.  One kernel per exchange,
//   k_p2p_pull<POST = true>: block 0 first posts e into its slot of each
//   neighbour's flag words (fence.sys + release store, system scope) -- stream
//   order puts that after every kernel that wrote the vector, so the rows a
//   neighbour pulls are final -- then every block waits (acquire) until both
//   neighbours posted >= e and copies depth levels from each; the last block
//   to finish records e as completed.
//   Loopback (all ranks in this process, one stream) posts every rank's e
//   with k_p2p_signal before any rank's k_p2p_pull<false>, so its waits are
//   satisfied when they run; the wait, copy and epoch logic is the same kernel.
// A neighbour overwrites a pulled vector only after a LATER barrier, which
// needs this rank's next post, issued after its pull completed (ping-pong
// buffers: a vector is rewritten two exchanges after it was pulled), so no
// second handshake is needed.  All ranks issue the same exchange sequence.
// A world of one has no neighbours and no exchange.  A wait over 20 s traps instead
// of hanging the device.  allreduce / gather / broadcast are delegated to the
// wrapped transport (NCCL or loopback).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// flags: [0] own epoch (exchanges completed), [1] posted by the left neighbour,
// [2] by the right one, [3] block ticket of the running pull kernel, [4] set
// when a wait timed out (checked by the host after the solve)
constexpr int kP2pFlagWords = 8;
constexpr unsigned long long kP2pTimeoutNs = 20000000000ull;  // 20 s of neighbour skew
__device__ __forceinline__ void p2p_post(const unsigned long long* mine, unsigned long long* left_slot,
                                         unsigned long long* right_slot) {
  const unsigned long long e = mine[0] + 1;
  __threadfence_system();
  if (left_slot) st_release_sys(left_slot, e);
  if (right_slot) st_release_sys(right_slot, e);
}
// Loopback only: every local rank posts before any rank pulls.
__global__ void k_p2p_signal(const unsigned long long* mine, unsigned long long* left_slot,
                             unsigned long long* right_slot) {
  if (threadIdx.x == 0) p2p_post(mine, left_slot, right_slot);
}
// One rank's exchange e = mine[0] + 1, run by the `nblk` blocks of that rank (this
// block is `blk`): block 0 posts e to both neighbours (POST), every block waits for
// both neighbours' posts, the blocks copy the ghost levels out of the neighbours'
// vectors, and the last block to finish records epoch e.
template <bool POST>
__device__ __forceinline__ void p2p_rank_exchange(unsigned long long* mine, unsigned long long* left_slot,
                                                  unsigned long long* right_slot, double* x,
                                                  const double* __restrict__ left,
                                                  const double* __restrict__ right, int64_t lo, int64_t hi,
                                                  int64_t depth, int64_t nn, unsigned blk, unsigned nblk) {
  const unsigned long long e = mine[0] + 1;  // mine[0] changes only after every block is done
  if (threadIdx.x == 0) {
    if (POST && blk == 0) p2p_post(mine, left_slot, right_slot);
    // A neighbour later than the timeout (a stopped process, a replayed launch)
    // does not trap the context: the wait gives up, flags the failure in
    // mine[4] and the host turns it into STMG_ERUNTIME after the solve.
    const unsigned long long t0 = globaltimer_ns();
    for (int side = 1; side <= 2; ++side) {
      if ((side == 1 ? left : right) == nullptr) continue;
      while (ld_acquire_sys(mine + side) < e) {
        if (globaltimer_ns() - t0 > kP2pTimeoutNs) {
          atomicExch(mine + 4, 1ull);
          break;
        }
      }
    }
  }
  __syncthreads();
  const int64_t cnt = depth * nn;
  // leading ghosts [lo - depth, lo) from the left rank, trailing [hi, hi + depth) from the right
  for (int64_t k = (int64_t)blk * blockDim.x + threadIdx.x; k < 2 * cnt; k += (int64_t)nblk * blockDim.x) {
    const bool lead = k < cnt;
    const double* src = lead ? left : right;
    if (src == nullptr) continue;
    const int64_t off = (lead ? (lo - depth) * nn : hi * nn) + (lead ? k : k - cnt);
    x[off] = __ldcv(src + off);
  }
  if (threadIdx.x == 0) {
    // every block has read e (it did so before its ticket), so the last one may advance the epoch
    if (atomicAdd(mine + 3, 1ull) == nblk - 1) {
      mine[3] = 0;
      mine[0] = e;
    }
  }
}

// One rank per process: the kernel of that rank (the neighbours' run in their processes).
template <bool POST>
__global__ void __launch_bounds__(256) k_p2p_pull(unsigned long long* mine, unsigned long long* left_slot,
                                                  unsigned long long* right_slot, double* x,
                                                  const double* __restrict__ left,
                                                  const double* __restrict__ right, int64_t lo,
                                                  int64_t hi, int64_t depth, int64_t nn) {
  p2p_rank_exchange<POST>(mine, left_slot, right_slot, x, left, right, lo, hi, depth, nn, blockIdx.x, gridDim.x);
}

// Loopback (every rank in this process, on this GPU): ALL ranks' exchanges as one
// COOPERATIVE grid, `bpr` blocks per rank, each rank running the cross-process
// protocol unchanged -- its block 0 posts, its blocks spin on the neighbours'
// posts.  The blocks of different ranks wait on one another, so they must be
// co-resident: a cooperative launch guarantees that (separate launches or streams
// do not, B200_PROFILING.md).  This is the posting / waiting / epoch code path of
// a multi-GPU run, exercised with real races between ranks on one GPU.
constexpr int kP2pMaxLocal = 16;
struct P2pRankArgs {
  unsigned long long *mine, *left_slot, *right_slot;
  double* x;
  const double *left, *right;
  int64_t lo, hi;
};
struct P2pMultiArgs {
  P2pRankArgs r[kP2pMaxLocal];
};
__global__ void __launch_bounds__(256) k_p2p_pull_multi(const P2pMultiArgs a, int bpr, int64_t depth, int64_t nn) {
  const P2pRankArgs& r = a.r[blockIdx.x / bpr];
  p2p_rank_exchange<true>(r.mine, r.left_slot, r.right_slot, r.x, r.left, r.right, r.lo, r.hi, depth, nn,
                          blockIdx.x % bpr, (unsigned)bpr);
}

struct P2pComm : Comm {
  std::unique_ptr<Comm> base;
  struct Local {
    double* flags = nullptr;                   // own flag words (4 x u64)
    double* left_flags = nullptr;              // neighbours' flag words (peer-mapped or local)
    double* right_flags = nullptr;
    std::vector<double*> bufs, left, right;    // globally indexed bases: own / neighbours'
  };
  std::vector<Local> loc;
  std::vector<std::unique_ptr<DeviceBuf>> flag_mem;
  std::vector<void*> opened;  // IPC mappings to close
  // STMG_DIST_P2P=2: loopback with the pre-posted (signal, then pull) launches
  // instead of the cooperative all-ranks grid
  bool legacy_loopback = false;
  explicit P2pComm(std::unique_ptr<Comm> b) : base(std::move(b)) {
    world = base->world;
    n_local = base->n_local;
    rank0 = base->rank0;
    loc.resize(static_cast<size_t>(n_local));
    for (int k = 0; k < n_local; ++k) {
      flag_mem.push_back(std::make_unique<DeviceBuf>(kP2pFlagWords));
      cuda_check(cudaMemset(flag_mem.back()->p, 0, kP2pFlagWords * sizeof(double)), "memset");
      loc[k].flags = flag_mem.back()->p;
    }
  }
  ~P2pComm() override { close_peers(); }
  // Unmaps the neighbours' buffers (before this process frees its own).
  void close_peers() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    opened.clear();
  }
  // Any neighbour wait of this process timed out since the last call?
  bool timed_out(cudaStream_t s) {
    bool any = false;
    for (auto& L : loc) {
      unsigned long long f = 0;
      cuda_check(cudaMemcpyAsync(&f, reinterpret_cast<unsigned long long*>(L.flags) + 4, sizeof(f),
                                 cudaMemcpyDeviceToHost, s),
                 "p2p flag d2h");
      cuda_check(cudaStreamSynchronize(s), "sync");
      any = any || f != 0;
    }
    return any;
  }
  const char* name() const override { return "p2p"; }
  void exchange(const std::vector<double*>& v, const std::vector<int64_t>& b, int64_t nn, int depth,
                cudaStream_t s) override {
    using u64 = unsigned long long;
    if (world == 1) return;  // no neighbours
    auto slots = [&](int k, u64** ls, u64** rs) {
      const int g = rank0 + k;
      *ls = g > 0 ? reinterpret_cast<u64*>(loc[k].left_flags) + 2 : nullptr;
      *rs = g < world - 1 ? reinterpret_cast<u64*>(loc[k].right_flags) + 1 : nullptr;
    };
    const bool loopback = n_local > 1;
    const int64_t cnt = 2 * nn * depth;
    std::vector<P2pRankArgs> ra(static_cast<size_t>(n_local));
    for (int k = 0; k < n_local; ++k) {
      const int g = rank0 + k;
      Local& L = loc[k];
      const auto it = std::find(L.bufs.begin(), L.bufs.end(), v[k]);
      if (it == L.bufs.end()) throw std::runtime_error("p2p exchange: unregistered vector");
      const size_t j = static_cast<size_t>(it - L.bufs.begin());
      u64 *ls, *rs;
      slots(k, &ls, &rs);
      ra[k] = {reinterpret_cast<u64*>(L.flags), ls, rs, v[k], g > 0 ? L.left[j] : nullptr,
               g < world - 1 ? L.right[j] : nullptr, b[g], b[g + 1]};
    }
    if (loopback && n_local <= kP2pMaxLocal && !legacy_loopback) {
      // one cooperative grid over all ranks (see k_p2p_pull_multi)
      P2pMultiArgs ma{};
      for (int k = 0; k < n_local; ++k) ma.r[k] = ra[k];
      int bpr = static_cast<int>(std::min<int64_t>((cnt + 255) / 256, std::max(1, 148 / n_local)));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(bpr * n_local));
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      launch_check(static_cast<int>(cudaLaunchKernelEx(&cfg, k_p2p_pull_multi, ma, bpr, static_cast<int64_t>(depth), nn)),
                   "p2p pull (cooperative, all ranks)");
      return;
    }
    if (loopback) {  // every rank posts, then every rank pulls (waits already satisfied)
      for (int k = 0; k < n_local; ++k) {
        k_p2p_signal<<<1, 32, 0, s>>>(ra[k].mine, ra[k].left_slot, ra[k].right_slot);
        launch_check(static_cast<int>(cudaGetLastError()), "p2p signal");
      }
    }
    for (int k = 0; k < n_local; ++k) {
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>((cnt + 255) / 256, 148));
      const P2pRankArgs& r = ra[k];
      if (loopback)
        k_p2p_pull<false><<<grid, 256, 0, s>>>(r.mine, r.left_slot, r.right_slot, r.x, r.left, r.right, r.lo, r.hi,
                                               depth, nn);
      else
        k_p2p_pull<true><<<grid, 256, 0, s>>>(r.mine, r.left_slot, r.right_slot, r.x, r.left, r.right, r.lo, r.hi,
                                              depth, nn);
      launch_check(static_cast<int>(cudaGetLastError()), "p2p pull");
    }
  }
  void allreduce_sum(const std::vector<double*>& in, const std::vector<double*>& out,
                     cudaStream_t s) override {
    base->allreduce_sum(in, out, s);
  }
  void gather_rows(const std::vector<double*>& src, double* dst,
                   const std::vector<std::pair<int64_t, int64_t>>& rows, int64_t nn,
                   cudaStream_t s) override {
    base->gather_rows(src, dst, rows, nn, s);
  }
  void broadcast(const double* root, const std::vector<double*>& dst, int64_t count,
                 cudaStream_t s) override {
    base->broadcast(root, dst, count, s);
  }
};

// ---------------------------------------------------------------------------
// Distributed hierarchy
// ---------------------------------------------------------------------------
// Slab-local level vector: only rows [lo, hi) = the rank's slab plus kSlabMargin
// levels on each side are allocated; `p` is the globally indexed base
// (p + n * nn + i addresses level n), so the kernels and transports index
// exactly as on a full-size vector.
constexpr int64_t kSlabMargin = 4;  // >= the deepest ghost any slab kernel reads (2)
struct SlabBuf {
  std::unique_ptr<DeviceBuf> mem;
  double* p = nullptr;
  int64_t lo = 0, hi = 0, nn = 0;  // allocated rows [lo, hi), nn doubles per row
  SlabBuf(int64_t n_lo, int64_t n_hi, int64_t n_t, int64_t nodes)
      : lo(std::max<int64_t>(0, n_lo - kSlabMargin)), hi(std::min<int64_t>(n_t + 1, n_hi + kSlabMargin)),
        nn(nodes) {
    mem = std::make_unique<DeviceBuf>((hi - lo) * nn + kVecPad);
    p = mem->p - lo * nn;
    cuda_check(cudaMemset(mem->p, 0, sizeof(double) * static_cast<size_t>((hi - lo) * nn + kVecPad)),
               "memset");
  }
  int64_t count() const { return (hi - lo) * nn; }
  double* first() const { return p + lo * nn; }
};

struct RankState {
  // levels [0, Lg): slab-local, globally indexed (device memory per rank ~ 1/W of a level)
  std::vector<std::unique_ptr<SlabBuf>> f, xa, xb;
  std::unique_ptr<DeviceBuf> fg, xg;                   // first gathered level: f rows out, x in
  std::unique_ptr<DeviceBuf> partials, scalars;
  std::vector<LevelView> views;  // levels [0, Lg) with this rank's slab row range
};

}  // namespace
}  // namespace stmgb

struct stmg_dist {
  int device = 0;
  bool adjoint = false;
  std::vector<stmgb::HostLevel> host;
  std::vector<int32_t> dirs;
  stmgb::SlabPlan plan;
  std::unique_ptr<stmgb::Comm> comm;
  std::vector<std::unique_ptr<stmgb::DeviceBuf>> coef;
  std::vector<stmgb::LevelView> full_views;
  std::vector<stmgb::RankState> ranks;  // local ranks
  stmg_hierarchy* tail = nullptr;       // root process: levels [Lg, L)
  cudaStream_t stream = nullptr, cap_stream = nullptr;
  double* pinned = nullptr;
  std::map<stmgb::GraphKey, stmgb::GraphEntry> graphs;
  int64_t device_bytes = 0;
  // device-side cycle loop (dist_loop): SolveLoopCtl + history on the device, pinned mirror
  std::unique_ptr<stmgb::DeviceBuf> loop;
  double* loop_host = nullptr;
  bool device_loop = false;
  bool last_on_device = false;  // the last solve's cycle loop ran as the device graph
  // Ghost exchanges overlapped with interior rows (STMG_DIST_OVERLAP = minimum slab DOFs
  // of a level to split its passes; 0 = off): side stream and fork / join events
  int64_t overlap_dofs = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t split_passes = 0;  // passes emitted in split form (tests)

  ~stmg_dist() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& kv : graphs) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
      if (kv.second.loop_exec) cudaGraphExecDestroy(kv.second.loop_exec);
      if (kv.second.loop_graph) cudaGraphDestroy(kv.second.loop_graph);
    }
    if (loop_host) cudaFreeHost(loop_host);
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    // Peer-memory transport: no rank may free slab buffers a neighbour can still
    // read.  Every rank first closes its mappings of the neighbours' buffers,
    // then all ranks meet (a one-double all-reduce on the base communicator),
    // and only then are the exported buffers freed.
    if (auto* pc = dynamic_cast<stmgb::P2pComm*>(comm.get())) {
      pc->close_peers();
      if (!ranks.empty() && ranks.front().scalars) {
        try {
          std::vector<double*> v{ranks.front().scalars->p + 5};
          pc->base->allreduce_sum(v, v, stream);
          cudaStreamSynchronize(stream);
        } catch (...) {
        }
      }
    }
    delete tail;
    ranks.clear();
    coef.clear();
    comm.reset();
    if (pinned) cudaFreeHost(pinned);
    if (stream) cudaStreamDestroy(stream);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    cudaSetDevice(prev);
  }
  int L() const { return static_cast<int>(host.size()); }
  int Lg() const { return plan.Lg; }
  int64_t nn(int l) const { return host[l].g.n_el + 1; }
  int64_t ndofs(int l) const { return nn(l) * (host[l].g.n_t + 1); }
};

namespace stmgb {
namespace {

struct DistEmitter {
  stmg_dist* d;
  int nu;
  double omega;
  cudaStream_t s;
  int64_t kernels = 0;

  int W() const { return static_cast<int>(d->ranks.size()); }
  double* buf(int k, int l, int which) {
    return which == 0 ? d->ranks[k].xa[l]->p : d->ranks[k].xb[l]->p;
  }
  std::vector<double*> bufs(int l, int which) {
    std::vector<double*> v;
    for (int k = 0; k < W(); ++k) v.push_back(buf(k, l, which));
    return v;
  }
  void exchange(int l, int which, int depth = 1, cudaStream_t on = nullptr) {
    d->comm->exchange(bufs(l, which), d->plan.bounds[l], d->nn(l), depth, on ? on : s);
  }

  // One pass over level l on every local rank, fed by a ghost exchange.  Plain form:
  // exchange, then each rank's kernel on its slab rows.  Split form (STMG_DIST_OVERLAP,
  // levels whose slabs are large enough): the exchange runs on a forked side stream while
  // each rank's kernel runs on the INTERIOR rows, whose tiles read no ghost level; after
  // the join the first and last kEdge rows of each slab follow.  kEdge is a multiple of
  // every tile depth and even, so the tiles and the t-restriction pairs are those of the
  // unsplit launch; the kernels are pointwise in the rows, so the values are identical.
  static constexpr int64_t kEdge = 16;
  bool splits(int l) const {
    if (d->overlap_dofs <= 0 || d->comm->world == 1) return false;
    for (const RankState& R : d->ranks) {
      const LevelView& V = R.views[l];
      if (V.n_hi - V.n_lo < 4 * kEdge || (V.n_hi - V.n_lo) * V.nn < d->overlap_dofs) return false;
    }
    return true;
  }
  template <class Exch, class Launch>
  void pass(int l, Exch&& exch, Launch&& launch) {
    if (!splits(l)) {
      exch(s);
      for (int k = 0; k < W(); ++k) launch(k, d->ranks[k].views[l]);
      return;
    }
    ++d->split_passes;
    cuda_check(cudaEventRecord(d->ev_fork, s), "fork");
    cuda_check(cudaStreamWaitEvent(d->side, d->ev_fork, 0), "fork wait");
    exch(d->side);
    cuda_check(cudaEventRecord(d->ev_join, d->side), "join");
    std::vector<std::pair<int64_t, int64_t>> inner(static_cast<size_t>(W()));
    for (int k = 0; k < W(); ++k) {
      LevelView V = d->ranks[k].views[l];
      const int64_t lo = V.n_lo + kEdge, hi = (V.n_hi - kEdge) & ~int64_t{1};
      inner[k] = {lo, hi};
      V.n_lo = lo;
      V.n_hi = hi;
      launch(k, V);
    }
    cuda_check(cudaStreamWaitEvent(s, d->ev_join, 0), "join wait");
    for (int k = 0; k < W(); ++k) {
      LevelView V = d->ranks[k].views[l];
      LevelView A = V, B = V;
      A.n_hi = inner[k].first;
      B.n_lo = inner[k].second;
      launch(k, A);
      launch(k, B);
    }
  }

  void sweep_all(int l, int cur) {
    pass(
        l, [&](cudaStream_t on) { exchange(l, cur, 1, on); },
        [&](int k, const LevelView& V) {
          launch_check(launch_sweep(d->adjoint, V, d->ranks[k].f[l]->p, buf(k, l, cur), buf(k, l, 1 - cur), omega,
                                    nullptr, nullptr, s),
                       "dist sweep");
          ++kernels;
        });
  }

  // Returns the buffer index holding the level-l result on every rank (2 = the
  // broadcast gathered-level buffer xg, only for l == Lg).
  int level(int l, int start, int pre_done, bool from_zero) {
    const int Lg = d->Lg();
    if (l == Lg) {
      std::vector<double*> src;
      std::vector<std::pair<int64_t, int64_t>> rows;
      for (int k = 0; k < W(); ++k) src.push_back(d->ranks[k].fg->p);
      for (int g = 0; g < d->plan.world; ++g)
        rows.push_back(gathered_rows(d->plan, d->dirs[Lg - 1], g, d->host[Lg].g.n_t));
      double* tail_f = d->comm->is_root() ? d->tail->ws->f[0]->p : nullptr;
      d->comm->gather_rows(src, tail_f, rows, d->nn(Lg), s);
      const double* root = nullptr;
      if (d->comm->is_root()) {
        Emitter em{d->tail, nu, omega, s};
        const int fin = em.level(0, 0, 0, true);
        kernels += em.kernels;
        root = fin == 0 ? d->tail->ws->xa[0]->p : d->tail->ws->xb[0]->p;
      }
      std::vector<double*> dst;
      for (int k = 0; k < W(); ++k) dst.push_back(d->ranks[k].xg->p);
      d->comm->broadcast(root, dst, d->ndofs(Lg), s);
      return 2;
    }
    int cur = start;
    int pre = nu - pre_done;
    if (from_zero) {
      cur = 0;
      for (int k = 0; k < W(); ++k) {
        if (nu >= 1) {
          launch_check(launch_sweep_from_zero(d->ranks[k].views[l], d->ranks[k].f[l]->p, buf(k, l, 0),
                                              omega, s),
                       "dist sweep0");
          ++kernels;
        } else {
          const LevelView& V = d->ranks[k].views[l];
          cuda_check(cudaMemsetAsync(buf(k, l, 0) + V.n_lo * V.nn, 0,
                                     sizeof(double) * static_cast<size_t>((V.n_hi - V.n_lo) * V.nn), s),
                     "memset");
        }
      }
      pre = nu >= 1 ? nu - 1 : 0;
    }
    if (from_zero && l > 0 && pre >= 2) {
      // the fused pair's first sweep also runs on the ghost level next to the slab,
      // which needs that level's right-hand side from the neighbour
      std::vector<double*> fv;
      for (int k = 0; k < W(); ++k) fv.push_back(d->ranks[k].f[l]->p);
      d->comm->exchange(fv, d->plan.bounds[l], d->nn(l), 1, s);
    }
    smooth_all(l, cur, pre);
    // residual + restriction into level l+1 (slab rows of l+1, or the rows this
    // rank contributes to the first gathered level)
    pass(
        l, [&](cudaStream_t on) { exchange(l, cur, 1, on); },
        [&](int k, const LevelView& V) {
          const LevelView C = l + 1 < Lg ? d->ranks[k].views[l + 1] : d->full_views[l + 1];
          double* fc = l + 1 < Lg ? d->ranks[k].f[l + 1]->p : d->ranks[k].fg->p;
          launch_check(launch_restrict_residual(d->adjoint, V, C, d->dirs[l], d->ranks[k].f[l]->p, buf(k, l, cur), fc,
                                                s),
                       "dist restrict");
          ++kernels;
        });
    const int child = level(l + 1, 0, 0, true);
    if (child != 2) exchange(l + 1, child);  // coarse ghosts for the prolongation of ghost rows
    std::vector<const double*> xc;
    for (int k = 0; k < W(); ++k) xc.push_back(child == 2 ? d->ranks[k].xg->p : buf(k, l + 1, child));
    int post = nu;
    if (nu >= 1) {
      for (int k = 0; k < W(); ++k) {
        const LevelView C = l + 1 < Lg ? d->ranks[k].views[l + 1] : d->full_views[l + 1];
        launch_check(launch_sweep_prolong(d->adjoint, d->ranks[k].views[l], C, d->dirs[l],
                                          d->ranks[k].f[l]->p, buf(k, l, cur), xc[k],
                                          buf(k, l, 1 - cur), omega, s),
                     "dist sweep_prolong");
        ++kernels;
      }
      cur = 1 - cur;
      post = nu - 1;
    } else {
      for (int k = 0; k < W(); ++k) {
        const LevelView C = l + 1 < Lg ? d->ranks[k].views[l + 1] : d->full_views[l + 1];
        launch_check(launch_prolong_add(d->ranks[k].views[l], C, d->dirs[l], xc[k], buf(k, l, cur), s),
                     "dist prolong");
        ++kernels;
      }
    }
    smooth_all(l, cur, post);
    return cur;
  }

  // `count` sweeps on every rank's slab: fused pairs after a two-level ghost
  // exchange (one exchange per two sweeps), then a single sweep if count is odd.
  void smooth_all(int l, int& cur, int count) {
    for (; count >= 2; count -= 2) {
      pass(
          l, [&](cudaStream_t on) { exchange(l, cur, 2, on); },
          [&](int k, const LevelView& V) {
            launch_check(launch_sweep2(d->adjoint, V, d->ranks[k].f[l]->p, buf(k, l, cur), buf(k, l, 1 - cur), omega,
                                       s),
                         "dist sweep2");
            ++kernels;
          });
      cur = 1 - cur;
    }
    if (count == 1) {
      sweep_all(l, cur);
      cur = 1 - cur;
    }
  }
};

// Switch the ghost exchange to peer-memory pulls (P2pComm): register every
// distributed level vector of every local rank (f, xa, xb per level) and map the
// neighbours' copies -- local pointers in loopback, CUDA IPC mappings of the
// neighbour processes' allocations (handles all-gathered over NCCL) otherwise.
void enable_p2p(stmg_dist* d) {
  const int Lg = d->plan.Lg, W = d->plan.world;
  auto pc = std::make_unique<P2pComm>(std::move(d->comm));
  const int nl = pc->n_local;
  auto slabs = [&](int k) {
    std::vector<const SlabBuf*> v;
    for (int l = 0; l < Lg; ++l) {
      v.push_back(d->ranks[k].f[l].get());
      v.push_back(d->ranks[k].xa[l].get());
      v.push_back(d->ranks[k].xb[l].get());
    }
    return v;
  };
  for (int k = 0; k < nl; ++k)
    for (const SlabBuf* sb : slabs(k)) pc->loc[k].bufs.push_back(sb->p);
  auto* nc = dynamic_cast<NcclComm*>(pc->base.get());
  if (!nc) {  // loopback: every rank is local
    for (int k = 0; k < nl; ++k) {
      P2pComm::Local& L = pc->loc[k];
      if (k > 0) {
        L.left = pc->loc[k - 1].bufs;
        L.left_flags = pc->loc[k - 1].flags;
      }
      if (k < W - 1) {
        L.right = pc->loc[k + 1].bufs;
        L.right_flags = pc->loc[k + 1].flags;
      }
    }
  } else {
    // one NCCL rank per process (a world of one still gathers its handles)
    const int g = pc->rank0;
    const std::vector<const SlabBuf*> mine = slabs(0);
    const size_t n = mine.size() + 1, hb = sizeof(cudaIpcMemHandle_t);
    std::vector<cudaIpcMemHandle_t> hs(n), all(n * static_cast<size_t>(W));
    for (size_t j = 0; j < mine.size(); ++j) cuda_check(cudaIpcGetMemHandle(&hs[j], mine[j]->mem->p), "ipc handle");
    cuda_check(cudaIpcGetMemHandle(&hs[n - 1], pc->loc[0].flags), "ipc handle");
    DeviceBuf send(static_cast<int64_t>((n * hb + 7) / 8)), recv(static_cast<int64_t>((n * hb * W + 7) / 8));
    cuda_check(cudaMemcpy(send.p, hs.data(), n * hb, cudaMemcpyHostToDevice), "ipc handles h2d");
    nccl_check(nccl().AllGather(send.p, recv.p, n * hb, ncclChar, nc->comm, d->stream), "allgather handles");
    cuda_check(cudaStreamSynchronize(d->stream), "sync");
    cuda_check(cudaMemcpy(all.data(), recv.p, n * hb * W, cudaMemcpyDeviceToHost), "ipc handles d2h");
    P2pComm::Local& L = pc->loc[0];
    for (int r : {g - 1, g + 1}) {
      if (r < 0 || r >= W) continue;
      std::vector<double*>& dst = r < g ? L.left : L.right;
      for (size_t j = 0; j < n; ++j) {
        void* ptr = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&ptr, all[static_cast<size_t>(r) * n + j], cudaIpcMemLazyEnablePeerAccess),
                   "ipc open");
        pc->opened.push_back(ptr);
        if (j + 1 == n) {
          (r < g ? L.left_flags : L.right_flags) = static_cast<double*>(ptr);
          continue;
        }
        // globally indexed base of rank r's slab vector of level l = j / 3
        const int l = static_cast<int>(j / 3);
        const int64_t lo = std::max<int64_t>(0, d->plan.bounds[l][r] - kSlabMargin);
        dst.push_back(static_cast<double*>(ptr) - lo * d->nn(l));
      }
    }
  }
  d->comm = std::move(pc);
}

void dist_build(stmg_dist* d, int world, int rank, const void* nccl_id, int64_t min_slab) {
  DeviceGuard dg(d->device);
  launch_check(kernels_init(), "kernels_init");
  std::vector<int64_t> nts;
  for (const HostLevel& h : d->host) nts.push_back(h.g.n_t);
  d->plan = plan_slabs(nts, d->dirs, world, min_slab);
  if (d->plan.Lg < 1)
    throw std::invalid_argument("dist: the finest level cannot be split into time slabs for this world size");
  if (nccl_id) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    d->comm = std::make_unique<NcclComm>(world, rank, id);
  } else {
    d->comm = std::make_unique<LoopbackComm>(world);
  }
  for (const HostLevel& hl : d->host) {
    const std::vector<double> t = hl.table(d->adjoint);
    auto buf = std::make_unique<DeviceBuf>(static_cast<int64_t>(t.size()));
    cuda_check(cudaMemcpy(buf->p, t.data(), t.size() * 8, cudaMemcpyHostToDevice), "coef upload");
    LevelView v{hl.g.n_el, hl.g.n_t, hl.g.n_el + 1, hl.w, hl.inv_w, buf->p, 0, hl.g.n_t + 1};
    v.tile_nt = tile_nt_for(v.nn * (v.n_t + 1));
    d->full_views.push_back(v);
    d->device_bytes += static_cast<int64_t>(t.size() * 8);
    d->coef.push_back(std::move(buf));
  }
  const int Lg = d->plan.Lg;
  d->ranks.resize(static_cast<size_t>(d->comm->n_local));
  for (int k = 0; k < d->comm->n_local; ++k) {
    const int g = d->comm->rank0 + k;
    RankState& R = d->ranks[k];
    int64_t max_partials = sumsq_partials_needed(0);
    for (int l = 0; l < Lg; ++l) {
      LevelView v = d->full_views[l];
      v.n_lo = d->plan.bounds[l][g];
      v.n_hi = d->plan.bounds[l][g + 1];
      R.f.push_back(std::make_unique<SlabBuf>(v.n_lo, v.n_hi, v.n_t, v.nn));
      R.xa.push_back(std::make_unique<SlabBuf>(v.n_lo, v.n_hi, v.n_t, v.nn));
      R.xb.push_back(std::make_unique<SlabBuf>(v.n_lo, v.n_hi, v.n_t, v.nn));
      d->device_bytes += 3 * 8 * (R.f.back()->count() + kVecPad);
      R.views.push_back(v);
      max_partials = std::max(max_partials, sweep_partials_needed(v));
    }
    R.fg = std::make_unique<DeviceBuf>(d->ndofs(Lg));
    R.xg = std::make_unique<DeviceBuf>(d->ndofs(Lg));
    R.partials = std::make_unique<DeviceBuf>(max_partials + kPartialsScratch);
    R.scalars = std::make_unique<DeviceBuf>(8);
    d->device_bytes += 8 * (2 * d->ndofs(Lg) + max_partials + 8);
  }
  if (d->comm->is_root()) {
    auto t = std::make_unique<stmg_hierarchy>();
    t->device = d->device;
    t->adjoint = d->adjoint;
    t->dirs.assign(d->dirs.begin() + Lg, d->dirs.end());
    t->host.assign(d->host.begin() + Lg, d->host.end());
    finish_create(t.get(), false, nullptr);
    d->device_bytes += t->device_bytes;
    d->tail = t.release();
  }
  cuda_check(cudaStreamCreateWithFlags(&d->stream, cudaStreamDefault), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&d->cap_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaMallocHost(&d->pinned, 8 * sizeof(double)), "cudaMallocHost");
  d->loop = std::make_unique<DeviceBuf>(kLoopCtlDoubles + kLoopHistory + 1);
  cuda_check(cudaMallocHost(&d->loop_host, sizeof(double) * (kLoopCtlDoubles + kLoopHistory + 1)), "cudaMallocHost");
  // The cycle loop runs on the device (one conditional WHILE graph, dist_loop) when
  // every rank is in this process (loopback).  Across processes the body holds NCCL
  // calls; that form is opt-in (STMG_DIST_DEVICE_LOOP=1) until it has run at world > 1.
  d->device_loop = nccl_id == nullptr;
  if (const char* e = std::getenv("STMG_DIST_DEVICE_LOOP")) d->device_loop = std::atoi(e) != 0;
  if (const char* e = std::getenv("STMG_DIST_OVERLAP")) d->overlap_dofs = std::atoll(e);
  if (d->overlap_dofs > 0) {
    cuda_check(cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming), "cudaEventCreate");
  }
  if (const char* e = std::getenv("STMG_DIST_P2P"); e && std::atoi(e) != 0) {
    enable_p2p(d);
    if (std::atoi(e) == 2) static_cast<P2pComm*>(d->comm.get())->legacy_loopback = true;
  }
  cuda_check(cudaDeviceSynchronize(), "sync");
}

GraphEntry& dist_graph(stmg_dist* d, int nu, double omega) {
  const GraphKey key{nu, omega, 0};
  auto it = d->graphs.find(key);
  if (it != d->graphs.end()) return it->second;
  GraphEntry e;
  DistEmitter em{d, nu, omega, d->cap_stream};
  cuda_check(cudaStreamBeginCapture(d->cap_stream, cudaStreamCaptureModeThreadLocal), "capture");
  e.final_buf = em.level(0, nu >= 1 ? 1 : 0, nu >= 1 ? 1 : 0, false);
  cuda_check(cudaStreamEndCapture(d->cap_stream, &e.graph), "end capture");
  cuda_check(cudaGraphInstantiate(&e.exec, e.graph, 0), "graph instantiate");
  e.kernels = em.kernels;
  return d->graphs.emplace(key, e).first->second;
}

// residual-norm pass on level 0 of every local rank (optionally the speculative
// first sweep), all-reduced into scalars[slot] of every rank
void dist_norm(stmg_dist* d, bool spec, double omega, int slot, cudaStream_t s = nullptr) {
  if (s == nullptr) s = d->stream;
  std::vector<double*> X, in, out;
  for (auto& R : d->ranks) X.push_back(R.xa[0]->p);
  d->comm->exchange(X, d->plan.bounds[0], d->nn(0), 1, s);
  for (auto& R : d->ranks) {
    int64_t np = 0;
    launch_check(launch_sweep(d->adjoint, R.views[0], R.f[0]->p, R.xa[0]->p, spec ? R.xb[0]->p : nullptr,
                              omega, R.partials->p, &np, s),
                 "dist norm sweep");
    launch_check(launch_finalize_sum(R.partials->p, np, R.scalars->p + 4, s), "finalize");
    in.push_back(R.scalars->p + 4);
    out.push_back(R.scalars->p + slot);
  }
  d->comm->allreduce_sum(in, out, s);
}

// The whole cycle loop of the time-slab solve as one graph (as get_loop for one GPU):
// a conditional WHILE node whose body is the distributed V-cycle (ghost exchanges,
// the gathered tail), the all-reduced residual norm with the speculative first sweep,
// and the bookkeeping kernel (history, status, loop condition) on this process's
// first rank.  Every process sees the same all-reduced norm, so all of them leave the
// loop after the same cycle and their collectives stay matched.  Returns nullptr
// (host loop) when the graph cannot be built.
cudaGraphExec_t dist_loop(stmg_dist* d, int nu, double omega) {
  GraphEntry& e = dist_graph(d, nu, omega);
  if (e.loop_tried) return e.loop_exec;
  e.loop_tried = true;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  auto fail = [&] {
    cudaGetLastError();
    if (ex) cudaGraphExecDestroy(ex);
    if (g) cudaGraphDestroy(g);
    return static_cast<cudaGraphExec_t>(nullptr);
  };
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return fail();
  cudaGraphConditionalHandle handle;
  if (cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) return fail();
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) return fail();
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t cs = d->cap_stream;
  if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail();
  bool ok = true;
  try {
    DistEmitter em{d, nu, omega, cs};
    const bool spec = nu >= 1;
    if (em.level(0, spec ? 1 : 0, spec ? 1 : 0, false) != 0)
      throw std::logic_error("dist: level-0 iterate left the primary buffer");
    dist_norm(d, spec, omega, 1, cs);
    auto* ctl = reinterpret_cast<SolveLoopCtl*>(d->loop->p);
    launch_check(launch_cycle_check(d->ranks[0].scalars->p, ctl, d->loop->p + kLoopCtlDoubles, handle, cs),
                 "cycle check");
  } catch (...) {
    ok = false;
  }
  cudaGraph_t captured = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &captured);
  if (!ok || ec != cudaSuccess) return fail();
  if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) return fail();
  e.loop_graph = g;
  e.loop_exec = ex;
  return ex;
}

double dist_fetch(stmg_dist* d, int slot) {
  cuda_check(cudaMemcpyAsync(d->pinned, d->ranks[0].scalars->p + slot, sizeof(double),
                             cudaMemcpyDeviceToHost, d->stream), "scalar d2h");
  cuda_check(cudaStreamSynchronize(d->stream), "sync");
  return d->pinned[0];
}

// local = false: b and u are full-size global vectors (every process reads its
// slab rows and their margins from them); local = true: b and u hold only this
// process's rows [row_lo, row_hi) of level 0 (stmg_dist_info), so the caller's
// memory scales as 1/W too, and the ghost rows are exchanged instead.
void dist_solve(stmg_dist* d, const double* b, double* u, const stmg_solve_options& o,
                stmg_solve_report* rep, double* history, int32_t cap, bool local = false) {
  if (!b || !u) throw std::invalid_argument("mg_solve: vector size mismatch");
  if (o.nu < 0 || o.omega <= 0.0 || o.tol <= 0.0 || o.div_tol <= o.tol || o.max_cycles < 0)
    throw std::invalid_argument("mg_solve: invalid options");
  if (!history || cap < o.max_cycles + 1)
    throw std::invalid_argument("mg_solve: history buffer smaller than max_cycles + 1");
  DeviceGuard dg(d->device);
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t nn = d->nn(0);
  const bool b_dev = is_device_ptr(b), u_dev = is_device_ptr(u);
  const int64_t row0 = d->ranks.front().views[0].n_lo;  // first local row (local mode)
  for (auto& R : d->ranks) {
    if (local) {  // this rank's slab rows; ghosts follow by exchange
      const LevelView& V = R.views[0];
      const size_t src = static_cast<size_t>((V.n_lo - row0) * nn), dst = static_cast<size_t>(V.n_lo * nn);
      const size_t bytes = sizeof(double) * static_cast<size_t>((V.n_hi - V.n_lo) * nn);
      cuda_check(cudaMemcpyAsync(R.f[0]->p + dst, b + src, bytes,
                                 b_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, d->stream), "b copy");
      cuda_check(cudaMemcpyAsync(R.xa[0]->p + dst, u + src, bytes,
                                 u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, d->stream), "u copy");
      continue;
    }
    // the allocated rows (slab + margins) of the global b and u
    const SlabBuf& F = *R.f[0];
    const size_t off = static_cast<size_t>(F.lo * nn), bytes = sizeof(double) * static_cast<size_t>(F.count());
    cuda_check(cudaMemcpyAsync(F.first(), b + off, bytes,
                               b_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, d->stream), "b copy");
    cuda_check(cudaMemcpyAsync(R.xa[0]->first(), u + off, bytes,
                               u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, d->stream), "u copy");
  }
  if (local) {  // the right-hand side's ghost rows (the first norm pass exchanges u's)
    std::vector<double*> F0;
    for (auto& R : d->ranks) F0.push_back(R.f[0]->p);
    d->comm->exchange(F0, d->plan.bounds[0], nn, 1, d->stream);
  }
  std::vector<double*> in, out;
  for (auto& R : d->ranks) {
    const LevelView& V = R.views[0];
    int64_t np = 0;
    launch_check(launch_sumsq(R.f[0]->p + V.n_lo * nn, (V.n_hi - V.n_lo) * nn, R.partials->p, &np, d->stream),
                 "sumsq");
    launch_check(launch_finalize_sum(R.partials->p, np, R.scalars->p + 4, d->stream), "finalize");
    in.push_back(R.scalars->p + 4);
    out.push_back(R.scalars->p + 0);
  }
  d->comm->allreduce_sum(in, out, d->stream);
  const double norm_b = std::sqrt(dist_fetch(d, 0));
  rep->absolute_norms = norm_b == 0.0 ? 1 : 0;
  const double denom = rep->absolute_norms ? 1.0 : norm_b;
  const bool spec = o.nu >= 1;
  GraphEntry* g = o.max_cycles > 0 ? &dist_graph(d, o.nu, o.omega) : nullptr;
  dist_norm(d, spec && o.max_cycles > 0, o.omega, 1);
  const double r0 = std::sqrt(dist_fetch(d, 1)) / denom;
  int nh = 0;
  history[nh++] = r0;
  rep->cycles = 0;
  rep->factor = 1.0;
  rep->smoother_dof_updates = 0.0;
  rep->fine_sweeps = rep->fine_restricts = rep->fine_prolong_sweeps = rep->fine_sweep_pairs = 0;
  rep->fine_sweep_seconds = rep->fine_restrict_seconds = rep->fine_prolong_sweep_seconds = 0.0;
  rep->fine_sweep_pair_seconds = 0.0;
  // work of this process: its slab rows on distributed levels, the tail on the root
  double per_cycle = 0.0;
  for (const RankState& R : d->ranks)
    for (int l = 0; l < d->Lg(); ++l)
      per_cycle += 2.0 * o.nu * static_cast<double>((R.views[l].n_hi - R.views[l].n_lo) * R.views[l].nn);
  if (d->comm->is_root())
    for (int l = d->Lg(); l + 1 < d->L(); ++l) per_cycle += 2.0 * o.nu * static_cast<double>(d->ndofs(l));
  int64_t launches = 0;
  cudaGraphExec_t loop = nullptr;
  if (d->device_loop && r0 >= o.tol && o.max_cycles > 0 && o.max_cycles <= kLoopHistory)
    loop = dist_loop(d, o.nu, o.omega);
  d->last_on_device = loop != nullptr;
  if (r0 < o.tol) {
    rep->status = STMG_CONVERGED;
  } else if (loop) {
    // the whole cycle loop on the device: one launch, one read-back
    auto* ctl = reinterpret_cast<SolveLoopCtl*>(d->loop_host);
    *ctl = SolveLoopCtl{o.tol, o.div_tol, o.max_cycles, 0, STMG_MAX_CYCLES, 0};
    cuda_check(cudaMemcpyAsync(d->loop->p, d->loop_host, sizeof(SolveLoopCtl), cudaMemcpyHostToDevice, d->stream),
               "loop ctl");
    cuda_check(cudaGraphLaunch(loop, d->stream), "loop graph launch");
    cuda_check(cudaMemcpyAsync(d->loop_host, d->loop->p, sizeof(double) * (kLoopCtlDoubles + o.max_cycles + 1),
                               cudaMemcpyDeviceToHost, d->stream),
               "loop read-back");
    cuda_check(cudaStreamSynchronize(d->stream), "sync");
    const double* dh = d->loop_host + kLoopCtlDoubles;
    for (int c = 1; c <= ctl->cycles; ++c) history[nh++] = dh[c];
    rep->cycles = ctl->cycles;
    rep->status = ctl->status;
    rep->smoother_dof_updates = per_cycle * ctl->cycles;
    launches = static_cast<int64_t>(ctl->cycles) * (g->kernels + 3 * static_cast<int64_t>(d->ranks.size()));
  } else {
    rep->status = STMG_MAX_CYCLES;
    for (int cycle = 1; cycle <= o.max_cycles; ++cycle) {
      Nvtx cyc("stmg::dist_v_cycle");
      cuda_check(cudaGraphLaunch(g->exec, d->stream), "graph launch");
      launches += g->kernels;
      if (g->final_buf != 0) throw std::logic_error("dist: level-0 iterate left the primary buffer");
      dist_norm(d, spec && cycle < o.max_cycles, o.omega, 1);
      const double rn = std::sqrt(dist_fetch(d, 1)) / denom;
      history[nh++] = rn;
      rep->cycles = cycle;
      rep->smoother_dof_updates += per_cycle;
      if (rn < o.tol) {
        rep->status = STMG_CONVERGED;
        break;
      }
      if (!std::isfinite(rn) || rn > o.div_tol) {
        rep->status = STMG_DIVERGED;
        break;
      }
    }
  }
  if (rep->cycles > 0) rep->factor = std::pow(history[nh - 1] / r0, 1.0 / rep->cycles);
  if (auto* pc = dynamic_cast<P2pComm*>(d->comm.get()); pc && pc->timed_out(d->stream))
    throw std::runtime_error("p2p exchange: a neighbour's epoch wait timed out (rank skew above 20 s)");
  // this process's slab rows of u (loopback: every rank's rows -> the full vector)
  for (auto& R : d->ranks) {
    const LevelView& V = R.views[0];
    const size_t off = static_cast<size_t>(V.n_lo * nn);
    const size_t dst = local ? static_cast<size_t>((V.n_lo - row0) * nn) : off;
    cuda_check(cudaMemcpyAsync(u + dst, R.xa[0]->p + off, sizeof(double) * static_cast<size_t>((V.n_hi - V.n_lo) * nn),
                               u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, d->stream),
               "u copy back");
  }
  cuda_check(cudaStreamSynchronize(d->stream), "sync");
  rep->n_history = nh;
  rep->kernel_launches = launches;
  rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  rep->device_seconds = rep->seconds;
}

}  // namespace
}  // namespace stmgb
