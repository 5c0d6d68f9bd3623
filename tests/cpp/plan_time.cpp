// plan_time — times the planner/simulator entry points BASELINE.md §2-3
// lists, through the public `shardplan` API only:
//   solve                            (reference proj/src/planner.cpp:144-166)
//   build_schedule + simulate_step   (reference proj/src/overlap_sim.cpp:442-517)
// It is compiled twice, like plan_dump.cpp: against the compiled reference
// (oracle/build_ref.sh -> oracle/_ref/plan_time_ref, the reference arm's CPU
// path) and against this repo's libamsp.so (build.py -> _build/plan_time).
// Output: one JSON object per line {"entry", "workload", "best_us",
// "median_us", "runs", "result"}; `result` (the solver pick / simulated
// step) lets the caller check both builds agree.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

#include "shardplan/comm_model.hpp"
#include "shardplan/cost_model.hpp"
#include "shardplan/domain.hpp"
#include "shardplan/overlap_sim.hpp"
#include "shardplan/planner.hpp"

using namespace shardplan;

namespace {

// LLaMA-7B (H=4096, L=32, F=11008, V=32000): the bench workload's model.
ModelSpec llama7b(int micro_batches) {
  ModelSpec m;
  const std::uint64_t h = 4096, f = 11008, v = 32000;
  m.module_params = {h * h, h * h, h * h, h * h, f * h, f * h, h * f, h, h};
  m.modules_per_layer = 9;
  m.layer_count = 32;
  std::uint64_t layer = 0;
  for (auto x : m.module_params) layer += x;
  m.total_params = 32 * layer + 2 * v * h + h;
  m.hidden = 4096;
  m.seq_len = 4096;
  m.micro_batch = 1;
  m.micro_batch_count = micro_batches;
  m.vocab = 32000;
  return m;
}

ClusterSpec cluster(int R, int N) {
  ClusterSpec c;
  c.gpus_per_node = R;
  c.node_count = N;
  c.gpu_memory_capacity = 180'000'000'000ull;  // B200
  c.dp_mesh = DeviceMesh{R, N};
  c.topology.leaf_count = N;
  c.topology.nodes_per_leaf = 1;
  return c;
}

template <class F>
void timed(const char* entry, const std::string& workload, int runs, F&& f) {
  std::vector<double> us;
  std::string result;
  for (int i = 0; i < runs; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    result = f();
    const auto t1 = std::chrono::steady_clock::now();
    us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(us.begin(), us.end());
  std::printf(
      "{\"entry\": \"%s\", \"workload\": \"%s\", \"best_us\": %.3f, \"median_us\": %.3f, "
      "\"runs\": %d, \"result\": \"%s\"}\n",
      entry, workload.c_str(), us.front(), us[us.size() / 2], runs, result.c_str());
}

}  // namespace

int main(int argc, char** argv) {
  const int scale = argc > 1 ? std::max(1, std::atoi(argv[1])) : 1;
  std::vector<DeviceMesh> meshes;
  for (int a = 1; a <= 8; ++a)
    for (int b : {1, 2, 4, 8, 16, 32, 64, 128}) meshes.push_back({a, b});
  std::vector<std::uint64_t> sizes;
  for (std::uint64_t s = 1024; s <= (1ull << 34); s *= 4) sizes.push_back(s);
  // B200 NVLink 5 intra-node, 400 Gb/s NIC inter-node alpha-beta rings.
  const BandwidthProfile prof = synthetic_profile({5e-6, 680e9}, {10e-6, 50e9}, meshes, sizes);
  const CostConfig cfg;
  SolveOptions serial;
  serial.policy = ExecPolicy::Serial;
  for (auto rn : std::vector<std::pair<int, int>>{{8, 1}, {8, 8}, {8, 128}}) {
    const ModelSpec m = llama7b(1);
    const ClusterSpec c = cluster(rn.first, rn.second);
    timed("solve", "llama-7b R=" + std::to_string(rn.first) + " N=" + std::to_string(rn.second) +
                       " serial",
          20 * scale, [&] {
            const SearchReport r = solve(m, c, prof, cfg, serial);
            return to_string(r.best.plan);
          });
  }
  for (int M : {1, 128}) {
    const ModelSpec m = llama7b(M);
    const ClusterSpec c = cluster(8, 1);
    const ShardingPlan plan{DeviceMesh{1, 1}, DeviceMesh{8, 1}, DeviceMesh{8, 1}};
    SimConfig sim;
    sim.peak_flops_per_gpu = 1413.6e12;
    timed("build_schedule+simulate_step", "llama-7b 8x1 p=1x1,g=os=8x1 M=" + std::to_string(M),
          (M == 1 ? 20 : 3) * scale, [&] {
            const EventGraph g = build_schedule(m, c, plan, prof, cfg, sim);
            const Timeline t = simulate_step(g);
            char buf[96];
            std::snprintf(buf, sizeof buf, "events=%zu step=%a", g.events.size(), t.step_time);
            return std::string(buf);
          });
  }
  return 0;
}
