// the NCCL world of the GPU row-block path bootstrapped
// over the reference's OWN control plane -- its launcher
// (launch_with_master / connect_from_env, launch.hpp:247-360) and its TCP
// Communicator (comm.hpp) -- via mmws::gpu::share_unique_id.  Built against
// the unmodified reference headers by tests/test_abi.py.
//
//   ref_control_plane master <world>   rank 0: spawns ranks 1.. (this binary,
//                                       mode "worker"), ships the 128-byte
//                                       NCCL id, checks every rank got it
//   ref_control_plane worker           ranks >= 1 (spawned by the launcher)
//   ref_control_plane gpu              1-rank world + NCCL communicator from it,
//                                       then master_run through the GPU path
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "mmws/comm.hpp"
#include "mmws/launch.hpp"
#include "mmws/matrix.hpp"
#include "mmws_gpu.hpp"

namespace {

std::int64_t digest(const std::vector<std::uint8_t>& id) {
  std::uint64_t h = 1469598103934665603ULL;  // FNV-1a
  for (std::uint8_t b : id) h = (h ^ b) * 1099511628211ULL;
  return static_cast<std::int64_t>(h >> 1);
}

constexpr std::uint32_t kDigestTag = 99;

int master(int world) {
  mmws::MsgWorld w = mmws::launch_with_master("/proc/self/exe", {"worker"}, world);
  const std::vector<std::uint8_t> id = mmws::gpu::share_unique_id(w.comm);
  if (id.size() != 128) return std::fprintf(stderr, "bad id size\n"), 1;
  const std::int64_t mine = digest(id);
  for (int r = 1; r < world; ++r) {
    const std::int64_t got = w.comm.recv_i64(r, kDigestTag);
    if (got != mine) return std::fprintf(stderr, "rank %d holds a different id\n", r), 1;
  }
  std::printf("ok: %d ranks share one NCCL id over the reference control plane\n", world);
  return 0;
}

int worker() {
  mmws::Communicator comm = mmws::connect_from_env();
  const std::vector<std::uint8_t> id = mmws::gpu::share_unique_id(comm);
  comm.send_i64(0, kDigestTag, digest(id));
  return 0;
}

int gpu() {
  mmws::MsgWorld w = mmws::launch_with_master("/proc/self/exe", {"worker"}, 1);
  mmws::gpu::Context ctx(0);
  mmws::gpu::comm_init_from(ctx, w.comm);
  const mmws::Matrix a = mmws::random_matrix(300, 200, 1), b = mmws::random_matrix(200, 100, 2);
  auto [c, elapsed] = mmws::gpu::master_run(ctx, a, b, mmws::gpu::Mode::exact);
  if (!mmws::bitwise_equal(c, mmws::matmul_seq(a, b)) || !(elapsed > 0.0))
    return std::fprintf(stderr, "master_run over the bootstrapped communicator differs\n"), 1;
  std::printf("ok: master_run over an NCCL world bootstrapped by the reference launcher\n");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "";
  try {
    if (mode == "master") return master(argc > 2 ? std::stoi(argv[2]) : 3);
    if (mode == "worker") return worker();
    if (mode == "gpu") return gpu();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_control_plane %s: %s\n", mode.c_str(), e.what());
    return 2;
  }
  std::fprintf(stderr, "usage: ref_control_plane master <world> | worker | gpu\n");
  return 2;
}
