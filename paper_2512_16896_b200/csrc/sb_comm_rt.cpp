// Native shard communicator (sb_comm_*, include/scenebatch_b200.h): the multi-GPU data
// plane of the engine without PyTorch.
//
//   * bootstrap + host exchange: a TCP star through rank 0 (host:port, e.g. MASTER_ADDR /
//     MASTER_PORT + 1 under torchrun); every rank sends its bytes to rank 0, which returns
//     the rank-major concatenation. Used once at creation (board handles) and for the
//     host-side sb_shard.allgather.
//   * device exchange (sb_shard.allgather_dev): per-rank count boards in HBM, mapped by every
//     peer through CUDA IPC (other GPUs over NVLink / NVSwitch, or the same GPU from another
//     process). A rank pushes its values into every board with remote stores + a
//     system-scope release of a per-(slot, rank) epoch flag (k_comm_push); the stream then
//     waits for the peers' flags with cuStreamWaitValue64 (GPU front end, no SM spinning
//     and no host round trip) and k_comm_collect copies the slot into the caller's buffer.
//     Without 64-bit stream memory operations (or SB_COMM_SPIN=1) k_comm_collect spins on
//     the flags itself.
#include <arpa/inet.h>
#include <cuda.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <thread>

#include "sb_comm.h"
#include "sb_rt.hpp"

namespace {

void send_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      throw std::runtime_error("sb_comm: send failed (peer gone?)");
    }
    c += k;
    n -= static_cast<size_t>(k);
  }
}

void recv_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    ssize_t k = ::recv(fd, c, n, 0);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      throw std::runtime_error("sb_comm: recv failed (peer gone?)");
    }
    c += k;
    n -= static_cast<size_t>(k);
  }
}

constexpr uint64_t kMagic = 0x73625f636f6d6d31ull;  // "sb_comm1"

struct PeerInfo {  // exchanged once at creation
  int32_t pid, device, has_board, pad;
  cudaIpcMemHandle_t handle;
};

typedef CUresult (*PFN_waitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_devAttr)(int*, CUdevice_attribute, CUdevice);

}  // namespace

struct sb_comm {
  int rank = 0, world = 1, device = -1;
  std::vector<int> fds;  // rank 0: fd per peer rank (index 0 unused); others: fds[0] = rank 0
  int listen_fd = -1;
  // device exchange
  DevArray<uint64_t> board;
  std::vector<uint64_t*> peer_ptr;  // as mapped here (own board for rank)
  std::vector<bool> opened;
  DevArray<uint64_t*> d_peers;
  uint64_t epoch = 0;
  bool spin = false;
  PFN_waitValue64 wait64 = nullptr;

  sb_comm(int rank_, int world_, int device_, const char* host, int port, double timeout_s)
      : rank(rank_), world(world_), device(device_) {
    if (world < 1 || world > sbk::kCommMaxRanks) throw std::invalid_argument("sb_comm: world_size outside [1, 64]");
    if (rank < 0 || rank >= world) throw std::invalid_argument("sb_comm: rank outside [0, world_size)");
    if (world > 1) connect_star(host ? host : "127.0.0.1", port, timeout_s);
    if (device >= 0) setup_boards();
  }

  ~sb_comm() {
    if (device >= 0) {
      cudaSetDevice(device);
      cudaDeviceSynchronize();
      for (int r = 0; r < static_cast<int>(peer_ptr.size()); ++r)
        if (opened[r]) cudaIpcCloseMemHandle(peer_ptr[r]);
    }
    for (int fd : fds)
      if (fd >= 0) ::close(fd);
    if (listen_fd >= 0) ::close(listen_fd);
  }

  void connect_star(const char* host, int port, double timeout_s) {
    if (port <= 0 || port > 65535) throw std::invalid_argument("sb_comm: port outside [1, 65535]");
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
    addrinfo hints{}, *res = nullptr;
    hints.ai_family = AF_INET;
    hints.ai_socktype = SOCK_STREAM;
    if (getaddrinfo(host, std::to_string(port).c_str(), &hints, &res) != 0 || !res)
      throw std::invalid_argument(std::string("sb_comm: cannot resolve ") + host);
    sockaddr_in addr;
    std::memcpy(&addr, res->ai_addr, sizeof addr);
    freeaddrinfo(res);
    const int one = 1;
    if (rank == 0) {
      listen_fd = ::socket(AF_INET, SOCK_STREAM, 0);
      if (listen_fd < 0) throw std::runtime_error("sb_comm: socket");
      setsockopt(listen_fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
      if (::bind(listen_fd, reinterpret_cast<sockaddr*>(&addr), sizeof addr) != 0)
        throw std::runtime_error("sb_comm: bind " + std::string(host) + ":" + std::to_string(port) + ": " + std::strerror(errno));
      if (::listen(listen_fd, world) != 0) throw std::runtime_error("sb_comm: listen");
      fds.assign(world, -1);
      for (int k = 1; k < world; ++k) {
        timeval tv{};
        tv.tv_sec = static_cast<long>(timeout_s);
        setsockopt(listen_fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
        int fd = ::accept(listen_fd, nullptr, nullptr);
        if (fd < 0) throw std::runtime_error("sb_comm: rank 0 timed out waiting for peers");
        setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
        uint64_t hello[3];
        recv_all(fd, hello, sizeof hello);
        if (hello[0] != kMagic || hello[1] != static_cast<uint64_t>(world) || hello[2] == 0 ||
            hello[2] >= static_cast<uint64_t>(world) || fds[hello[2]] >= 0) {
          ::close(fd);
          throw std::runtime_error("sb_comm: bad hello (world size / rank mismatch)");
        }
        fds[hello[2]] = fd;
      }
      for (int r = 1; r < world; ++r) send_all(fds[r], &kMagic, 8);  // release the peers
    } else {
      int fd = -1;
      for (;;) {
        fd = ::socket(AF_INET, SOCK_STREAM, 0);
        if (fd < 0) throw std::runtime_error("sb_comm: socket");
        if (::connect(fd, reinterpret_cast<sockaddr*>(&addr), sizeof addr) == 0) break;
        ::close(fd);
        fd = -1;
        if (std::chrono::steady_clock::now() > deadline)
          throw std::runtime_error("sb_comm: cannot reach rank 0 at " + std::string(host) + ":" + std::to_string(port));
        std::this_thread::sleep_for(std::chrono::milliseconds(20));
      }
      setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
      const uint64_t hello[3] = {kMagic, static_cast<uint64_t>(world), static_cast<uint64_t>(rank)};
      send_all(fd, hello, sizeof hello);
      uint64_t ack = 0;
      recv_all(fd, &ack, 8);
      if (ack != kMagic) throw std::runtime_error("sb_comm: bad ack from rank 0");
      fds.assign(1, fd);
    }
  }

  // every rank contributes len bytes; returns the rank-major concatenation (world * len)
  std::vector<uint8_t> allgather_bytes(const void* send, size_t len) {
    std::vector<uint8_t> out(len * world);
    std::memcpy(out.data() + len * rank, send, len);
    if (world == 1) return out;
    const uint64_t hdr = len;
    if (rank == 0) {
      for (int r = 1; r < world; ++r) {
        uint64_t h = 0;
        recv_all(fds[r], &h, 8);
        if (h != hdr) throw std::runtime_error("sb_comm: allgather size differs between ranks");
        recv_all(fds[r], out.data() + len * r, len);
      }
      for (int r = 1; r < world; ++r) send_all(fds[r], out.data(), out.size());
    } else {
      send_all(fds[0], &hdr, 8);
      send_all(fds[0], send, len);
      recv_all(fds[0], out.data(), out.size());
    }
    return out;
  }

  void setup_boards() {
    device = current_device_checked(device);
    const size_t words = static_cast<size_t>(sbk::kCommSlots) * world * sbk::kCommStride;
    board.alloc(words);
    cuda_check(cudaMemset(board.p, 0, words * 8), "memset board");
    cuda_check(cudaDeviceSynchronize(), "sync");
    PeerInfo me{};
    me.pid = static_cast<int32_t>(::getpid());
    me.device = device;
    me.has_board = 1;
    cuda_check(cudaIpcGetMemHandle(&me.handle, board.p), "cudaIpcGetMemHandle");
    std::vector<uint8_t> all = allgather_bytes(&me, sizeof me);
    peer_ptr.assign(world, nullptr);
    opened.assign(world, false);
    for (int r = 0; r < world; ++r) {
      PeerInfo pi;
      std::memcpy(&pi, all.data() + sizeof pi * r, sizeof pi);
      if (!pi.has_board) throw std::invalid_argument("sb_comm: every rank needs a device for the device exchange");
      if (r == rank) {
        peer_ptr[r] = board.p;
        continue;
      }
      if (pi.pid == me.pid)
        throw std::invalid_argument("sb_comm: ranks must be separate processes (one process per GPU)");
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, pi.handle, cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle (peer board; P2P between these GPUs?)");
      peer_ptr[r] = static_cast<uint64_t*>(p);
      opened[r] = true;
    }
    d_peers.alloc(world);
    cuda_check(cudaMemcpy(d_peers.p, peer_ptr.data(), world * sizeof(uint64_t*), cudaMemcpyHostToDevice), "H2D peers");
    const char* sp = std::getenv("SB_COMM_SPIN");
    spin = sp && std::atoi(sp) != 0;
    if (!spin) {
      void* fa = nullptr;
      void* fw = nullptr;
      cudaDriverEntryPointQueryResult qa, qw;
      int ok = 0;
      if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fa, cudaEnableDefault, &qa) == cudaSuccess &&
          qa == cudaDriverEntryPointSuccess && fa &&
          reinterpret_cast<PFN_devAttr>(fa)(&ok, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, device) == CUDA_SUCCESS &&
          ok && cudaGetDriverEntryPoint("cuStreamWaitValue64", &fw, cudaEnableDefault, &qw) == cudaSuccess &&
          qw == cudaDriverEntryPointSuccess && fw)
        wait64 = reinterpret_cast<PFN_waitValue64>(fw);
      cudaGetLastError();
      spin = wait64 == nullptr;
    }
  }

  void allgather_dev(const uint64_t* d_send, uint32_t n, uint64_t* d_recv, cudaStream_t st) {
    if (device < 0) throw std::logic_error("sb_comm: created without a device (host exchange only)");
    if (n > static_cast<uint32_t>(sbk::kCommMaxValues)) throw std::invalid_argument("sb_comm: more than 31 values per device exchange");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    const uint64_t e = ++epoch;
    const int slot = static_cast<int>(e % sbk::kCommSlots);
    sb_stream_t s = reinterpret_cast<sb_stream_t>(st);
    sbk::comm_push(d_peers.p, world, rank, slot, e, d_send, n, s);
    if (!spin) {
      for (int r = 0; r < world; ++r) {
        const uint64_t* flag = board.p + (static_cast<size_t>(slot) * world + r) * sbk::kCommStride;
        if (wait64(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), e,
                   CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
          throw std::runtime_error("sb_comm: cuStreamWaitValue64 failed");
      }
    }
    sbk::comm_collect(board.p, world, slot, e, n, d_recv, spin ? 1 : 0, s);
  }

  void allgather(const uint64_t* send, uint32_t n, uint64_t* recv) {
    std::vector<uint8_t> all = allgather_bytes(send, n * 8ull);
    std::memcpy(recv, all.data(), all.size());
  }
};

namespace {
int cb_allgather(void* ctx, const uint64_t* send, uint32_t n, uint64_t* recv) {
  try {
    static_cast<sb_comm*>(ctx)->allgather(send, n, recv);
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}
int cb_allgather_dev(void* ctx, const uint64_t* d_send, uint32_t n, uint64_t* d_recv, void* st) {
  try {
    static_cast<sb_comm*>(ctx)->allgather_dev(d_send, n, d_recv, static_cast<cudaStream_t>(st));
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

sb_status sb_comm_create(int32_t rank, int32_t world_size, int device, const char* host, int32_t port,
                         double timeout_s, sb_comm** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    *out = new sb_comm(rank, world_size, device, host, port, timeout_s > 0 ? timeout_s : 300.0);
  });
}

void sb_comm_destroy(sb_comm* c) { delete c; }

sb_status sb_comm_shard(sb_comm* c, uint64_t n_total, sb_shard* out) {
  return guard([&] {
    if (!c || !out) throw std::invalid_argument("NULL argument");
    out->begin = n_total * static_cast<uint64_t>(c->rank) / static_cast<uint64_t>(c->world);
    out->end = n_total * static_cast<uint64_t>(c->rank + 1) / static_cast<uint64_t>(c->world);
    out->rank = c->rank;
    out->world_size = c->world;
    out->allgather = cb_allgather;
    out->ctx = c;
    out->allgather_dev = c->device >= 0 ? cb_allgather_dev : nullptr;
    out->ctx_dev = c->device >= 0 ? c : nullptr;
  });
}

sb_status sb_comm_allgather(sb_comm* c, const uint64_t* send, uint32_t n, uint64_t* recv) {
  return guard([&] {
    if (!c || (n && (!send || !recv))) throw std::invalid_argument("NULL argument");
    c->allgather(send, n, recv);
  });
}

sb_status sb_comm_allgather_dev(sb_comm* c, const uint64_t* d_send, uint32_t n, uint64_t* d_recv,
                                void* cuda_stream) {
  return guard([&] {
    if (!c || !d_send || !d_recv) throw std::invalid_argument("NULL argument");
    c->allgather_dev(d_send, n, d_recv, static_cast<cudaStream_t>(cuda_stream));
  });
}

sb_status sb_comm_barrier(sb_comm* c) {
  return guard([&] {
    if (!c) throw std::invalid_argument("NULL argument");
    const uint8_t b = 1;
    c->allgather_bytes(&b, 1);
  });
}

int32_t sb_comm_uses_stream_waits(const sb_comm* c) { return c && c->device >= 0 && !c->spin ? 1 : 0; }

}  // extern "C"
