// plan_dump — golden-vector driver for the planner/simulator API surface.
//
// Uses ONLY the public `shardplan` API (the reference's headers:
// proj/include/shardplan/{domain,comm_model,cost_model,planner,overlap_sim,
// placement}.hpp). It is compiled twice:
//   * against the compiled reference (oracle/build_ref.sh -> oracle/_ref/
//     plan_dump_ref) to produce tests/golden/plan_dump.txt.gz, and
//   * against this repo's drop-in library (include/shardplan/*.hpp ->
//     libamsp.so) by tests/test_plan_golden.py,
// and the two outputs must be byte-identical. Doubles print as C99 hex
// floats (%a) so "identical" means bit-exact.
//
// Sections cover every reference entry point of SURVEY.md §8(a) rows a1-a16
// plus placement (the §2 row 6 module).
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

#include "shardplan/comm_model.hpp"
#include "shardplan/cost_model.hpp"
#include "shardplan/domain.hpp"
#include "shardplan/overlap_sim.hpp"
#include "shardplan/placement.hpp"
#include "shardplan/planner.hpp"

using namespace shardplan;

namespace {

std::string hx(double d) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", d);
  return buf;
}

std::uint64_t fnv(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

void out(const std::string& s) { std::fputs(s.c_str(), stdout); std::fputc('\n', stdout); }

std::string ms(const DeviceMesh& m) { return to_string(m); }

std::string plan_s(const ShardingPlan& p) { return to_string(p); }

// Error tag: most-derived known type.
template <class F>
std::string attempt(F&& f) {
  try {
    return f();
  } catch (const NoFeasiblePlanError& e) {
    return std::string("ERR NoFeasible ") + e.what() + " closest=" +
           plan_s(e.closest().plan) + " d_total=" + hx(e.closest().memory.d_total);
  } catch (const InfeasibleError& e) {
    return std::string("ERR Infeasible ") + e.what();
  } catch (const Error& e) {
    return std::string("ERR Error ") + e.what();
  } catch (const std::exception& e) {
    return std::string("ERR std ") + e.what();
  }
}

// LLaMA-shaped model: per-layer modules q,k,v,o,gate,up,down,attn_norm,mlp_norm.
ModelSpec llama(int H, int L, int F, int V, int M = 1, int B = 1, int S = 2048) {
  ModelSpec m;
  const std::uint64_t h = H, f = F, v = V;
  m.module_params = {h * h, h * h, h * h, h * h, f * h, f * h, h * f, h, h};
  m.modules_per_layer = 9;
  m.layer_count = L;
  std::uint64_t layer = 0;
  for (auto x : m.module_params) layer += x;
  m.total_params = static_cast<std::uint64_t>(L) * layer + 2 * v * h + h;
  m.hidden = H;
  m.seq_len = S;
  m.micro_batch = B;
  m.micro_batch_count = M;
  m.vocab = V;
  return m;
}

std::vector<std::uint64_t> llama_tensors(const ModelSpec& m) {
  std::vector<std::uint64_t> t;
  const std::uint64_t head = static_cast<std::uint64_t>(m.vocab) * m.hidden;
  t.push_back(head);
  for (int l = 0; l < m.layer_count; ++l)
    for (auto x : m.module_params) t.push_back(x);
  t.push_back(static_cast<std::uint64_t>(m.hidden));
  t.push_back(head);
  return t;
}

ModelSpec toy(std::uint64_t total, int L, std::vector<std::uint64_t> mods, int M) {
  ModelSpec m;
  m.total_params = total;
  m.layer_count = L;
  m.modules_per_layer = static_cast<int>(mods.size());
  m.module_params = std::move(mods);
  m.hidden = 64;
  m.seq_len = 128;
  m.micro_batch = 2;
  m.micro_batch_count = M;
  m.vocab = 100;
  return m;
}

ClusterSpec cluster(int R, int N, std::uint64_t cap, DeviceMesh dp) {
  ClusterSpec c;
  c.gpus_per_node = R;
  c.node_count = N;
  c.gpu_memory_capacity = cap;
  c.dp_mesh = dp;
  c.topology.leaf_count = N;
  c.topology.nodes_per_leaf = 1;
  return c;
}

ClusterSpec cluster(int R, int N, std::uint64_t cap = 80'000'000'000ull) {
  return cluster(R, N, cap, DeviceMesh{R, N});
}

std::vector<DeviceMesh> all_meshes(int maxa, int maxb) {
  std::vector<DeviceMesh> v;
  for (int a = 1; a <= maxa; ++a)
    for (int b = 1; b <= maxb; ++b) v.push_back({a, b});
  return v;
}

std::vector<std::uint64_t> geo(std::uint64_t lo, std::uint64_t hi, int mul) {
  std::vector<std::uint64_t> v;
  for (std::uint64_t x = lo; x <= hi; x *= mul) v.push_back(x);
  return v;
}

const CollectiveKind kKinds[] = {CollectiveKind::AllGather,
                                 CollectiveKind::ReduceScatter,
                                 CollectiveKind::AllReduce,
                                 CollectiveKind::Broadcast};

std::string tb(const TimeBreakdown& t) {
  return "t_p=" + hx(t.t_p) + " t_g=" + hx(t.t_g) + " t_os0=" +
         hx(t.t_os_allreduce) + " t_os1=" + hx(t.t_os_broadcast) +
         " total=" + hx(t.total);
}

std::string mb(const MemoryBreakdown& m) {
  return "dp=" + hx(m.d_params) + " dg=" + hx(m.d_grads) + " dos=" +
         hx(m.d_os) + " dms=" + hx(m.d_modelstate) + " dact=" +
         hx(m.d_activation) + " dtmp=" + hx(m.d_tmp) + " dtot=" +
         hx(m.d_total);
}

std::string pr(const PlanResult& r) {
  return plan_s(r.plan) + " " + tb(r.time) + " " + mb(r.memory) +
         " feasible=" + std::to_string(r.feasible) + " rank=" +
         std::to_string(r.rank);
}

// ---------------------------------------------------------------- comm model
void section_comm(const BandwidthProfile& p1) {
  out("## comm");
  for (auto k : kKinds) {
    out(std::string("kind ") + to_string(k) + " rt=" +
        to_string(collective_from_string(to_string(k))));
  }
  out("from_string bogus " + attempt([] {
        return std::string(to_string(collective_from_string("alltoall")));
      }));
  const AlphaBetaParams abs[] = {{0.0, 1e9}, {5e-6, 1.5e11}, {2e-5, 3.3e10}};
  const double sizes[] = {0.0, 1.0, 1024.0, 1e6, 134217728.0, 3.7e9};
  const int parts[] = {1, 2, 3, 4, 8, 16, 64, 1024};
  for (auto k : kKinds)
    for (const auto& ab : abs)
      for (double v : sizes)
        for (int p : parts)
          out(std::string("ring ") + to_string(k) + " " + hx(ab.alpha) + " " +
              hx(ab.link_bandwidth) + " " + hx(v) + " " + std::to_string(p) +
              " = " + hx(ring_time(k, v, p, ab)));
  out("ring p0 " + attempt([] {
        return hx(ring_time(CollectiveKind::AllReduce, 1.0, 0, {}));
      }));
  out("ring neg " + attempt([] {
        return hx(ring_time(CollectiveKind::AllReduce, -1.0, 2, {}));
      }));

  // Interpolation, clamping, exact hits, fallback, missing series.
  BandwidthProfile q;
  q.add_series(CollectiveKind::AllReduce, {8, 2},
               {{4u << 20, 80e9}, {1u << 20, 50e9}, {64u << 20, 120e9}});
  q.add_series(CollectiveKind::AllGather, {2, 2}, {{4096, 1e9}});
  q.add_series(CollectiveKind::AllGather, {4, 1}, {{4096, 3e9}, {8192, 4e9}});
  const std::uint64_t qs[] = {0,        1,        1u << 19, 1u << 20,
                              (1u << 20) + 1, 2u << 20, 3u << 20, 4u << 20,
                              5u << 20, 63u << 20, 64u << 20, 1ull << 40};
  for (auto s : qs) {
    out("eff ar 8x2 " + std::to_string(s) + " " + attempt([&] {
          return hx(q.effective_bandwidth(CollectiveKind::AllReduce, s, {8, 2})) +
                 " t=" + hx(q.collective_time(CollectiveKind::AllReduce, s, {8, 2}));
        }));
  }
  const DeviceMesh fb[] = {{2, 2}, {4, 1}, {1, 4}, {16, 1}, {1, 1}, {8, 2}, {2, 8}};
  for (auto m : fb)
    for (auto k : kKinds)
      out(std::string("fallback ") + to_string(k) + " " + ms(m) + " " +
          attempt([&] {
            return hx(q.collective_time(k, 6000, m)) + " has=" +
                   std::to_string(q.has_series(k, m));
          }));
  out("add empty " + attempt([&] {
        BandwidthProfile b;
        b.add_series(CollectiveKind::Broadcast, {2, 1}, {});
        return std::string("ok");
      }));
  out("add dup " + attempt([&] {
        BandwidthProfile b;
        b.add_series(CollectiveKind::Broadcast, {2, 1}, {{10, 1.0}, {10, 2.0}});
        return std::string("ok");
      }));
  out("add nonpos " + attempt([&] {
        BandwidthProfile b;
        b.add_series(CollectiveKind::Broadcast, {2, 1}, {{10, 1.0}, {20, 0.0}});
        return std::string("ok");
      }));
  out("add twice " + attempt([&] {
        BandwidthProfile b;
        b.add_series(CollectiveKind::Broadcast, {2, 1}, {{10, 1.0}});
        b.add_series(CollectiveKind::Broadcast, {2, 1}, {{20, 1.0}});
        return std::string("ok");
      }));
  out("empty profile " + std::to_string(BandwidthProfile{}.empty()) + " " +
      std::to_string(q.empty()));

  // Synthetic profile + canonical JSON.
  const std::string j1 = profile_to_canonical_json(p1);
  out("synthetic p1 json_len=" + std::to_string(j1.size()) + " fnv=" +
      std::to_string(fnv(j1)));
  {
    out("synthetic dupmesh " + attempt([] {
          return profile_to_canonical_json(synthetic_profile(
              {1e-6, 1e11}, {5e-6, 2e10}, {{2, 1}, {4, 2}, {2, 1}}, {4096}));
        }));
    auto small = synthetic_profile({1e-6, 1e11}, {5e-6, 2e10},
                                   {{1, 1}, {2, 1}, {4, 2}},
                                   {4096, 1024, 4096, 1u << 20});
    out("synthetic small " + profile_to_canonical_json(small));
    const std::string rt =
        profile_to_canonical_json(profile_from_json(profile_to_canonical_json(small)));
    out("roundtrip small " + std::to_string(rt == profile_to_canonical_json(small)));
  }
  out("synthetic empty " + attempt([] {
        return profile_to_canonical_json(synthetic_profile({}, {}, {}, {1}));
      }));
  out("synthetic zero " + attempt([] {
        return profile_to_canonical_json(synthetic_profile({}, {}, {{2, 1}}, {0, 5}));
      }));
  out("json p1 roundtrip " +
      std::to_string(profile_to_canonical_json(profile_from_json(j1)) == j1));

  // CSV import.
  const char* hdr = "op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s\n";
  const std::string csvs[] = {
      std::string(hdr) + "allreduce,4096,8,1,1e9\nallreduce,1024,8,1,5e8\n"
                         "allgather,1024,2,2,2.5e8\r\n\nbroadcast,65536,4,1,7e9\n",
      std::string(hdr) + "allreduce,4096,8,1,1e9\nallreduce,4096,8,1,2e9\n",
      std::string(hdr) + "allreduce,4096,8,1\n",
      std::string(hdr) + "alltoall,4096,8,1,1e9\n",
      std::string(hdr) + "allreduce,4096,0,1,1e9\n",
      std::string(hdr) + "allreduce,4096,8,1,-3\n",
      std::string(hdr) + "allreduce,abc,8,1,1e9\n",
      std::string(hdr) + "allreduce,4096,8,1,xyz\n",
      std::string("op,size,gpus_per_node,nodes,bw\nallreduce,1,1,1,1\n"),
      std::string(""),
      std::string(hdr),
      std::string("op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s\r\n"
                  "reducescatter,8,2,1,3.25\n"),
  };
  int i = 0;
  for (const auto& c : csvs) {
    out("csv " + std::to_string(i++) + " " +
        attempt([&] { return profile_to_canonical_json(profile_from_csv(c)); }));
  }
  const std::string jsons[] = {
      "{\"allreduce/8 x 1\":[[1024,500000000.0],[4096,1000000000.0]]}",
      "{\"allreduce/8 x 1\":[[4096,1e9],[1024,5e8]],\"broadcast/2 x 2\":[[1,1]]}",
      "[1,2]",
      "{\"allreduce-8 x 1\":[[1,1]]}",
      "{\"allreduce/8x1\":[[1,1]]}",
      "{\"allreduce/8 x 1\":{}}",
      "{\"allreduce/8 x 1\":[[1,2,3]]}",
      "{\"allreduce/8 x 1\":[[1,1],[1,2]]}",
      "{\"gather/8 x 1\":[[1,1]]}",
      "{not json",
      "{}",
  };
  i = 0;
  for (const auto& j : jsons) {
    out("json " + std::to_string(i++) + " " +
        attempt([&] { return profile_to_canonical_json(profile_from_json(j)); }));
  }
  out("load bad ext " + attempt([] {
        return profile_to_canonical_json(load_profile("/nonexistent/profile.txt"));
      }));
  out("load missing csv " + attempt([] {
        return profile_to_canonical_json(load_profile("/nonexistent/x.csv"));
      }));
  out("load missing json " + attempt([] {
        return profile_to_canonical_json(load_profile("/nonexistent/x.json"));
      }));
}

// -------------------------------------------------------------------- domain
void section_domain() {
  out("## domain");
  out("mesh " + ms({3, 5}) + " size=" + std::to_string(DeviceMesh{3, 5}.size()));
  ShardingPlan zpp{{8, 1}, {8, 1}, {8, 1}, DeviceMesh{8, 1}};
  out("plan " + plan_s(zpp) + " sp=" + std::to_string(zpp.sp()) + " sg=" +
      std::to_string(zpp.sg()) + " sos=" + std::to_string(zpp.sos()));
  out("mesh cmp " + std::to_string(DeviceMesh{1, 2} < DeviceMesh{2, 1}) +
      std::to_string(DeviceMesh{2, 1} == DeviceMesh{2, 1}));

  // Cluster checks.
  std::vector<ClusterSpec> bad;
  {
    auto c = cluster(8, 1); c.gpus_per_node = 0; bad.push_back(c);
    c = cluster(8, 1); c.gpu_memory_capacity = 0; bad.push_back(c);
    c = cluster(8, 1); c.dp_mesh = {0, 1}; bad.push_back(c);
    c = cluster(8, 1); c.dp_mesh = {16, 1}; bad.push_back(c);
    c = cluster(8, 2); c.dp_mesh = {8, 4}; bad.push_back(c);
    c = cluster(8, 1); c.topology.leaf_count = 0; bad.push_back(c);
    c = cluster(8, 4); c.topology = {1, 2, 1.0}; bad.push_back(c);
    c = cluster(8, 4); c.topology = {2, 2, 0.5}; bad.push_back(c);
    c = cluster(8, 4); c.topology = {2, 2, 1.5}; bad.push_back(c);
  }
  int i = 0;
  for (const auto& c : bad) {
    out("cluster_check " + std::to_string(i++) + " " + attempt([&] {
          c.check();
          return std::string("ok gpus=") + std::to_string(c.gpu_count());
        }));
  }
  // Model checks.
  std::vector<ModelSpec> mods;
  {
    auto m = llama(384, 6, 1024, 8192); mods.push_back(m);
    m.total_params = 0; mods.push_back(m);
    m = llama(384, 6, 1024, 8192); m.micro_batch_count = 0; mods.push_back(m);
    m = llama(384, 6, 1024, 8192); m.module_params.pop_back(); mods.push_back(m);
    m = llama(384, 6, 1024, 8192); m.module_params[2] = 0; mods.push_back(m);
    m = llama(384, 6, 1024, 8192); m.total_params = 10; mods.push_back(m);
    m = llama(384, 6, 1024, 8192); m.bytes_per_grad = 0; mods.push_back(m);
    m = llama(384, 6, 1024, 8192); m.vocab = 0; mods.push_back(m);
  }
  i = 0;
  for (const auto& m : mods) {
    out("model_check " + std::to_string(i++) + " " + attempt([&] {
          m.check();
          return "ok layer=" + std::to_string(m.layer_template_params());
        }));
  }

  // validate_plan over raw grids (extended by 0 and cap+1 on small clusters).
  struct CaseV { int R, N; DeviceMesh dp; int lo; int ext; };
  const CaseV cases[] = {{2, 2, {2, 2}, 0, 1}, {3, 1, {3, 1}, 0, 1},
                         {4, 2, {4, 2}, 1, 0}, {8, 1, {8, 1}, 1, 0},
                         {4, 4, {2, 2}, 1, 0}, {6, 1, {6, 1}, 1, 0},
                         {2, 4, {2, 4}, 1, 0}};
  for (const auto& cv : cases) {
    auto c = cluster(cv.R, cv.N, 1ull << 40, cv.dp);
    c.topology = {cv.N, 1, 1.0};
    out("validate cluster " + std::to_string(cv.R) + "x" + std::to_string(cv.N) +
        " dp=" + ms(cv.dp));
    const int ha = cv.R + cv.ext, hb = cv.N + cv.ext;
    for (int p0 = cv.lo; p0 <= ha; ++p0)
      for (int p1 = cv.lo; p1 <= hb; ++p1)
        for (int g0 = cv.lo; g0 <= ha; ++g0)
          for (int g1 = cv.lo; g1 <= hb; ++g1)
            for (int o0 = cv.lo; o0 <= ha; ++o0)
              for (int o1 = cv.lo; o1 <= hb; ++o1) {
                ShardingPlan p{{p0, p1}, {g0, g1}, {o0, o1}, std::nullopt};
                auto v = validate_plan(p, c);
                std::string line = "v " + plan_s(p) + (v.ok() ? " OK" : " |");
                for (const auto& x : v.violations)
                  line += " " + x.constraint + ":" + x.detail + ";";
                out(line);
              }
  }

  // Presets on many clusters.
  std::vector<ClusterSpec> pcs;
  for (int R : {1, 2, 4, 8})
    for (int N : {1, 2, 4, 128}) pcs.push_back(cluster(R, N));
  pcs.push_back(cluster(8, 4, 80'000'000'000ull, {8, 2}));
  pcs.push_back(cluster(8, 4, 80'000'000'000ull, {4, 1}));
  {
    auto c = cluster(8, 1); c.gpu_memory_capacity = 0; pcs.push_back(c);
  }
  for (const auto& c : pcs) {
    for (const auto& name : preset_names()) {
      out("preset " + name + " R=" + std::to_string(c.gpus_per_node) + " N=" +
          std::to_string(c.node_count) + " dp=" + ms(c.dp_mesh) + " " +
          attempt([&] { return plan_s(preset(name, c)); }));
    }
    out("preset bogus " + attempt([&] { return plan_s(preset("ZeRO-2", c)); }));
  }
}

// ---------------------------------------------------------------- cost model
struct NamedModel { std::string name; ModelSpec m; };

std::vector<NamedModel> models() {
  std::vector<NamedModel> v;
  v.push_back({"tiny", llama(384, 6, 1024, 8192)});
  v.push_back({"1B", llama(2048, 18, 5632, 32000)});
  v.push_back({"7B", llama(4096, 32, 11008, 32000)});
  v.push_back({"13B", llama(5120, 40, 13824, 32000)});
  v.push_back({"7B_M4", llama(4096, 32, 11008, 32000, 4, 2, 4096)});
  v.push_back({"paper7e9", toy(7'000'000'000ull, 32, {200'000'000ull}, 1)});
  v.push_back({"toyM3", toy(1'000'000ull, 2, {100'000ull, 250'000ull, 3ull}, 3)});
  return v;
}

std::vector<CostConfig> cost_configs() {
  std::vector<CostConfig> v;
  v.push_back(CostConfig{});
  CostConfig c;
  c.exact_residual_buckets = true;
  c.activation_mode = ActivationMode::FullRecompute;
  v.push_back(c);
  c = CostConfig{};
  c.bucket_size = 25'000'000;
  c.tmp_include_gather_buffer = false;
  c.tmp_in_flight_buckets = 3;
  c.exact_residual_buckets = true;
  v.push_back(c);
  return v;
}

void section_cost(const std::vector<BandwidthProfile>& profiles) {
  out("## cost");
  const auto ms_ = models();
  const auto cfgs = cost_configs();
  std::vector<ClusterSpec> cls = {cluster(8, 1), cluster(4, 1), cluster(2, 1),
                                  cluster(8, 4), cluster(2, 4), cluster(4, 2),
                                  cluster(8, 128)};
  for (const auto& nm : ms_) {
    for (std::size_t ci = 0; ci < cfgs.size(); ++ci) {
      const auto& cfg = cfgs[ci];
      out("flops " + nm.name + " cfg" + std::to_string(ci) + " " +
          hx(flops_per_step(nm.m, cfg)) + " mfu=" +
          hx(mfu(nm.m, 0.25, 1.4136e15, 8, cfg)));
      for (const auto& c : cls) {
        std::vector<ShardingPlan> plans = enumerate_candidates(c);
        for (const auto& name : preset_names()) {
          try {
            plans.push_back(preset(name, c));
          } catch (const Error&) {
          }
        }
        for (std::size_t pi = 0; pi < profiles.size(); ++pi) {
          for (const auto& p : plans) {
            const auto& prof = profiles[pi];
            std::string line = "cost " + nm.name + " cfg" + std::to_string(ci) +
                               " prof" + std::to_string(pi) + " R" +
                               std::to_string(c.gpus_per_node) + "N" +
                               std::to_string(c.node_count) + " " + plan_s(p);
            line += " tp=" + attempt([&] { return hx(time_params_sharding(nm.m, p, prof)); });
            line += " nb=" + std::to_string(grad_bucket_count(nm.m, p, cfg));
            line += " tos0=" + attempt([&] { return hx(time_os_allreduce(nm.m, c, p, prof, cfg)); });
            line += " tos1=" + attempt([&] { return hx(time_os_broadcast(nm.m, p, prof)); });
            line += " tg=" + attempt([&] { return hx(time_grads_sharding(nm.m, p, prof, cfg)); });
            line += " T{" + attempt([&] { return tb(total_comm_time(nm.m, c, p, prof, cfg)); }) + "}";
            line += " M{" + mb(memory_breakdown(nm.m, p, cfg)) + "}";
            out(line);
          }
          // Only sweep both profiles on the first cfg to bound output.
          if (ci != 0) break;
        }
      }
    }
  }
  out("mfu zero " + attempt([] {
        return hx(mfu(llama(384, 6, 1024, 8192), 0.0, 1e15, 1, CostConfig{}));
      }));
  // Non-nesting ratio mesh error path (invalid plan through the cost model).
  out("ratio bad " + attempt([&] {
        ShardingPlan p{{3, 1}, {3, 1}, {8, 1}, std::nullopt};
        return hx(time_os_broadcast(llama(384, 6, 1024, 8192), p, profiles[0]));
      }));
  out("ratio bad2 " + attempt([&] {
        ShardingPlan p{{3, 1}, {3, 1}, {3, 1}, std::nullopt};
        return hx(time_os_allreduce(llama(384, 6, 1024, 8192), cluster(8, 1), p,
                                    profiles[0], CostConfig{}));
      }));
  // Literal BASELINE config 3 (invalid, still costed).
  {
    ShardingPlan p{{1, 1}, {4, 1}, {8, 1}, std::nullopt};
    auto m = llama(4096, 32, 11008, 32000, 2);
    out("literal cfg3 " + attempt([&] {
          return tb(total_comm_time(m, cluster(8, 1), p, profiles[0], CostConfig{})) +
                 " " + mb(memory_breakdown(m, p, CostConfig{}));
        }));
  }

  // Greedy partitioner.
  for (const auto& nm : ms_) {
    if (nm.name.rfind("toy", 0) == 0 || nm.name == "paper7e9") continue;
    const auto t = llama_tensors(nm.m);
    for (int k : {1, 2, 3, 4, 8, 16}) {
      auto part = partition_tensors_greedy(t, k);
      std::string line = "greedy " + nm.name + " k=" + std::to_string(k) +
                         " n=" + std::to_string(t.size()) + " sizes";
      for (auto s : part.shard_sizes) line += " " + std::to_string(s);
      line += " assign";
      for (auto a : part.assignment) line += " " + std::to_string(a);
      out(line);
    }
  }
  {
    std::uint64_t x = 12345;
    for (int trial = 0; trial < 60; ++trial) {
      std::vector<std::uint64_t> t;
      x = x * 6364136223846793005ull + 1442695040888963407ull;
      const int n = static_cast<int>((x >> 33) % 12);
      for (int j = 0; j < n; ++j) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        t.push_back(1 + (x >> 33) % (trial % 3 == 0 ? 5 : 1000));
      }
      const int k = 1 + trial % 5;
      auto part = partition_tensors_greedy(t, k);
      std::string line = "greedy rnd" + std::to_string(trial) + " k=" + std::to_string(k);
      for (auto s : part.shard_sizes) line += " " + std::to_string(s);
      line += " |";
      for (auto a : part.assignment) line += " " + std::to_string(a);
      out(line);
    }
  }
  out("greedy k0 " + attempt([] {
        partition_tensors_greedy({1, 2}, 0);
        return std::string("ok");
      }));
  out("greedy zero " + attempt([] {
        partition_tensors_greedy({1, 0}, 2);
        return std::string("ok");
      }));
  out("greedy spec [7,5,4,3,1] k=2 " + [] {
    auto p = partition_tensors_greedy({7, 5, 4, 3, 1}, 2);
    std::string s;
    for (auto a : p.assignment) s += std::to_string(a) + ",";
    for (auto z : p.shard_sizes) s += " " + std::to_string(z);
    return s;
  }());
}

// ------------------------------------------------------------------- planner
void section_planner(const std::vector<BandwidthProfile>& profiles) {
  out("## planner");
  for (int R = 1; R <= 8; ++R)
    for (int N = 1; N <= 8; ++N) {
      auto c = cluster(R, N);
      c.topology = {N, 1, 1.0};
      auto cands = enumerate_candidates(c);
      std::string line = "enum " + std::to_string(R) + "x" + std::to_string(N) +
                         " n=" + std::to_string(cands.size());
      for (const auto& p : cands) line += " [" + plan_s(p) + "]";
      out(line);
    }
  {
    auto c = cluster(8, 4, 1ull << 40, {4, 2});
    auto cands = enumerate_candidates(c);
    std::string line = "enum partial dp 4x2 on 8x4 n=" + std::to_string(cands.size());
    for (const auto& p : cands) line += " [" + plan_s(p) + "]";
    out(line);
  }
  out("enum bad " + attempt([] {
        auto c = cluster(8, 1);
        c.gpu_memory_capacity = 0;
        return std::to_string(enumerate_candidates(c).size());
      }));

  const auto ms_ = models();
  const std::uint64_t caps[] = {1'000'000'000'000ull, 80'000'000'000ull,
                                40'000'000'000ull, 180'000'000'000ull,
                                1'000'000ull};
  const std::pair<int, int> full_clusters[] = {{1, 1}, {2, 1}, {4, 1}, {8, 1},
                                               {2, 2}, {4, 2}, {2, 4}, {8, 2},
                                               {1, 8}, {8, 4}};
  for (const auto& nm : ms_) {
    for (std::size_t pi = 0; pi < profiles.size(); ++pi) {
      for (auto cap : caps) {
        for (int R = 1; R <= 8; ++R)
          for (int N : {1, 2, 4, 8, 128}) {
            auto c = cluster(R, N, cap);
            c.topology = {N, 1, 1.0};
            bool full = false;
            for (auto fc : full_clusters) full |= (fc.first == R && fc.second == N);
            const std::string head = "solve " + nm.name + " prof" +
                                     std::to_string(pi) + " cap=" +
                                     std::to_string(cap) + " " +
                                     std::to_string(R) + "x" + std::to_string(N);
            std::string res = attempt([&] {
              SolveOptions o;
              o.keep_all_results = full;
              o.policy = (R + N) % 2 ? ExecPolicy::Serial : ExecPolicy::Parallel;
              auto rep = solve(nm.m, c, profiles[pi], CostConfig{}, o);
              std::string s = "best " + pr(rep.best) + " eval=" +
                              std::to_string(rep.candidates_evaluated) +
                              " filt=" + std::to_string(rep.candidates_filtered) +
                              " all=" + std::to_string(rep.all_results.has_value());
              if (rep.all_results) {
                for (const auto& r : *rep.all_results) s += "\n  " + pr(r);
              }
              return s;
            });
            out(head + " " + res);
          }
      }
      if (nm.name == "toyM3" || nm.name == "paper7e9") continue;
    }
  }
  // Brute-force oracle on small clusters.
  for (const auto& nm : ms_) {
    if (nm.name != "7B" && nm.name != "toyM3" && nm.name != "13B") continue;
    for (std::size_t pi = 0; pi < profiles.size(); ++pi)
      for (auto rn : {std::pair{1, 1}, std::pair{2, 2}, std::pair{4, 2},
                      std::pair{8, 1}, std::pair{3, 3}, std::pair{2, 8},
                      std::pair{8, 4}})
        for (auto cap : {80'000'000'000ull, 40'000'000'000ull}) {
          auto c = cluster(rn.first, rn.second, cap);
          c.topology = {rn.second, 1, 1.0};
          out("oracle " + nm.name + " prof" + std::to_string(pi) + " " +
              std::to_string(rn.first) + "x" + std::to_string(rn.second) +
              " cap=" + std::to_string(cap) + " " + attempt([&] {
                auto rep = brute_force_oracle(nm.m, c, profiles[pi], CostConfig{});
                return "best " + pr(rep.best) + " eval=" +
                       std::to_string(rep.candidates_evaluated) + " filt=" +
                       std::to_string(rep.candidates_filtered);
              }));
        }
  }
  out("oracle guard " + attempt([&] {
        auto c = cluster(8, 16);
        c.topology = {16, 1, 1.0};
        return pr(brute_force_oracle(ms_[0].m, c, profiles[0], CostConfig{}).best);
      }));
  // compare_presets.
  for (const auto& nm : ms_) {
    for (std::size_t pi = 0; pi < profiles.size(); ++pi)
      for (auto rn : {std::pair{8, 1}, std::pair{8, 128}, std::pair{4, 1},
                      std::pair{1, 1}, std::pair{8, 4}})
        for (auto cap : {80'000'000'000ull, 1'000'000ull}) {
          auto c = cluster(rn.first, rn.second, cap);
          c.topology = {rn.second, 1, 1.0};
          std::string line = "compare " + nm.name + " prof" + std::to_string(pi) +
                             " " + std::to_string(rn.first) + "x" +
                             std::to_string(rn.second) + " cap=" + std::to_string(cap);
          line += attempt([&] {
            std::string s;
            for (const auto& row : compare_presets(nm.m, c, profiles[pi], CostConfig{})) {
              s += "\n  " + row.name + " has=" + std::to_string(row.result.has_value());
              if (row.result) s += " " + pr(*row.result);
              s += " err=" + row.error;
            }
            return s;
          });
          out(line);
        }
  }
}

// --------------------------------------------------------------- overlap sim
std::string dump_graph(const EventGraph& g) {
  std::string s = "streams=" + std::to_string(g.stream_count) + " n=" +
                  std::to_string(g.events.size());
  for (const auto& e : g.events) {
    s += "\n  e" + std::to_string(e.id) + " " + to_string(e.kind) + " L" +
         std::to_string(e.layer) + " M" + std::to_string(e.module) + " s" +
         std::to_string(e.stream) + " d=" + hx(e.duration) + " deps";
    for (int d : e.depends_on) s += " " + std::to_string(d);
  }
  return s;
}

std::string dump_timeline(const Timeline& t, bool full) {
  std::string s = "step=" + hx(t.step_time);
  for (std::size_t i = 0; i < t.busy.size(); ++i)
    s += " busy" + std::to_string(i) + "=" + hx(t.busy[i]) + " idle" +
         std::to_string(i) + "=" + hx(t.idle[i]);
  auto br = bubble_report(t);
  s += " cidle=" + hx(br.compute_idle_total) + " nint=" +
       std::to_string(br.compute_intervals.size());
  const std::string trace = render_trace(t);
  s += " trace_fnv=" + std::to_string(fnv(trace)) + " trace_len=" +
       std::to_string(trace.size());
  if (full) {
    for (std::size_t i = 0; i < t.streams.size(); ++i) {
      s += "\n  stream" + std::to_string(i) + ":";
      for (const auto& se : t.streams[i])
        s += " " + std::to_string(se.event_id) + "@" + hx(se.start) + "-" + hx(se.end);
    }
    s += "\n  bubbles:";
    for (const auto& iv : br.compute_intervals) s += " " + hx(iv.start) + ":" + hx(iv.end);
    s += "\n  sidle:";
    for (double x : br.stream_idle) s += " " + hx(x);
    s += "\n" + trace;
  }
  return s;
}

void section_sim(const std::vector<BandwidthProfile>& profiles) {
  out("## sim");
  for (auto t : {OverlapTier::None, OverlapTier::AgRs, OverlapTier::AgRsAr,
                 OverlapTier::AgRsArBc})
    out(std::string("tier ") + to_string(t) + " " +
        to_string(tier_from_string(to_string(t))));
  out("tier bogus " + attempt([] { return std::string(to_string(tier_from_string("all"))); }));
  for (int k = 0; k <= 7; ++k)
    out(std::string("kind ") + to_string(static_cast<EventKind>(k)));

  struct SimModel { std::string name; ModelSpec m; bool full; };
  std::vector<SimModel> sms;
  sms.push_back({"s2x1", toy(2'000'000ull, 2, {1'000'000ull}, 1), true});
  sms.push_back({"s3x3h", toy(3'000'000ull, 3, {100'000ull, 250'000ull, 3'000ull}, 1), true});
  sms.push_back({"s2x2M2h", toy(900'000ull, 2, {200'000ull, 150'000ull}, 2), true});
  sms.push_back({"s3x2M3", toy(1'800'000ull, 3, {250'000ull, 350'000ull}, 3), false});
  sms.push_back({"tiny", llama(384, 6, 1024, 8192), false});
  sms.push_back({"tinyM2", llama(384, 6, 1024, 8192, 2), false});

  std::vector<ClusterSpec> cls = {cluster(2, 1), cluster(4, 1), cluster(2, 2),
                                  cluster(4, 2), cluster(8, 1)};
  std::vector<SimConfig> scs;
  for (auto tier : {OverlapTier::None, OverlapTier::AgRs, OverlapTier::AgRsAr,
                    OverlapTier::AgRsArBc})
    for (bool rc : {false, true})
      for (int cs : {1, 2})
        for (int src : {0, 1}) {
          SimConfig s;
          s.overlap_tier = tier;
          s.recompute = rc;
          s.comm_streams = cs;
          s.peak_flops_per_gpu = 1e12;
          s.compute_efficiency = 0.5;
          if (src == 1) s.compute_time_source = ComputeTimeSource::Table;
          scs.push_back(s);
        }
  for (auto& sm : sms) {
    for (auto& c : cls) {
      std::vector<ShardingPlan> plans = enumerate_candidates(c);
      for (const auto& name : preset_names()) {
        try {
          plans.push_back(preset(name, c));
        } catch (const Error&) {
        }
      }
      for (const auto& p : plans) {
        for (std::size_t si = 0; si < scs.size(); ++si) {
          SimConfig s = scs[si];
          const int K = sm.m.modules_per_layer;
          if (s.compute_time_source == ComputeTimeSource::Table) {
            for (int k = 0; k < K; ++k) {
              s.fwd_times.push_back(1e-3 * (k + 1));
              s.bwd_grad_weight_times.push_back(1.5e-3 * (k + 1));
              s.bwd_grad_input_times.push_back(0.7e-3 * (k + 2));
            }
            s.head_fwd_time = 2e-3;
            s.head_bwd_time = 3e-3;
          }
          CostConfig cfg;
          cfg.bucket_size = 300'000;
          cfg.exact_residual_buckets = (si % 3 == 0);
          const std::string head = "sim " + sm.name + " R" +
                                   std::to_string(c.gpus_per_node) + "N" +
                                   std::to_string(c.node_count) + " " + plan_s(p) +
                                   " sc" + std::to_string(si);
          const std::size_t pidx = si % profiles.size();
          out(head + " " + attempt([&] {
                auto g = build_schedule(sm.m, c, p, profiles[pidx], cfg, s);
                auto t = simulate_step(g);
                const bool full = sm.full && c.node_count * c.gpus_per_node <= 4 &&
                                  (si % 8 == 0 || si == scs.size() - 1);
                return (full ? dump_graph(g) + "\n  " : std::string("n=") +
                               std::to_string(g.events.size()) + " ") +
                       dump_timeline(t, full);
              }));
        }
      }
    }
  }
  // Large models: summary only.
  for (auto nm : {std::pair<std::string, ModelSpec>{"7B", llama(4096, 32, 11008, 32000)},
                  {"13B", llama(5120, 40, 13824, 32000)},
                  {"7B_M8", llama(4096, 32, 11008, 32000, 8)}}) {
    auto c = cluster(8, 1);
    auto plans = enumerate_candidates(c);
    for (const auto& p : plans) {
      for (auto tier : {OverlapTier::None, OverlapTier::AgRsArBc}) {
        for (bool rc : {false, true}) {
          SimConfig s;
          s.overlap_tier = tier;
          s.recompute = rc;
          s.peak_flops_per_gpu = 1.4136e15;
          out("simL " + nm.first + " " + plan_s(p) + " " + to_string(tier) +
              " rc=" + std::to_string(rc) + " " + attempt([&] {
                auto g = build_schedule(nm.second, c, p, profiles[0], CostConfig{}, s);
                auto t = simulate_step(g);
                return "n=" + std::to_string(g.events.size()) + " " + dump_timeline(t, false);
              }));
        }
      }
    }
  }
  // Errors and hand-built graphs.
  auto m = toy(2'000'000ull, 2, {1'000'000ull}, 1);
  out("sim invalid " + attempt([&] {
        ShardingPlan p{{1, 1}, {4, 1}, {8, 1}, std::nullopt};
        return dump_graph(build_schedule(m, cluster(8, 1), p, profiles[0], CostConfig{}, SimConfig{}));
      }));
  out("sim streams3 " + attempt([&] {
        SimConfig s;
        s.comm_streams = 3;
        return dump_graph(build_schedule(m, cluster(8, 1), ShardingPlan{}, profiles[0], CostConfig{}, s));
      }));
  out("sim streams0 " + attempt([&] {
        SimConfig s;
        s.comm_streams = 0;
        return dump_graph(build_schedule(m, cluster(8, 1), ShardingPlan{}, profiles[0], CostConfig{}, s));
      }));
  out("sim table bad " + attempt([&] {
        SimConfig s;
        s.compute_time_source = ComputeTimeSource::Table;
        s.fwd_times = {1.0};
        s.bwd_grad_weight_times = {1.0};
        s.bwd_grad_input_times = {0.0};
        return dump_graph(build_schedule(m, cluster(8, 1), ShardingPlan{}, profiles[0], CostConfig{}, s));
      }));
  out("sim table size " + attempt([&] {
        SimConfig s;
        s.compute_time_source = ComputeTimeSource::Table;
        return dump_graph(build_schedule(m, cluster(8, 1), ShardingPlan{}, profiles[0], CostConfig{}, s));
      }));
  out("sim zero peak " + attempt([&] {
        SimConfig s;
        s.compute_efficiency = 0.0;
        return dump_graph(build_schedule(m, cluster(8, 1), ShardingPlan{}, profiles[0], CostConfig{}, s));
      }));
  out("sim bad model " + attempt([&] {
        auto mm = m;
        mm.total_params = 0;
        return dump_graph(build_schedule(mm, cluster(8, 1), ShardingPlan{}, profiles[0], CostConfig{}, SimConfig{}));
      }));
  {
    EventGraph g;
    g.stream_count = 2;
    out("simulate empty " + dump_timeline(simulate_step(g), true));
    Event a; a.id = 0; a.duration = 1e-3; a.stream = 0;
    Event b; b.id = 1; b.duration = 2.5e-3; b.stream = 1;
    Event c; c.id = 2; c.duration = 0.5e-3; c.stream = 0; c.depends_on = {0, 1};
    Event d; d.id = 3; d.duration = 0.25e-3; d.stream = 1; d.kind = EventKind::AllReduceBucket; d.module = 4;
    g.events = {a, b, c, d};
    out("simulate hand " + dump_timeline(simulate_step(g), true));
    g.events[0].depends_on = {2};
    out("simulate cycle " + attempt([&] { return dump_timeline(simulate_step(g), true); }));
    g.events[0].depends_on = {9};
    out("simulate dangling " + attempt([&] { return dump_timeline(simulate_step(g), true); }));
    g.events[0].depends_on = {};
    g.events[3].stream = 5;
    out("simulate badstream " + attempt([&] { return dump_timeline(simulate_step(g), true); }));
    EventGraph one;
    one.stream_count = 1;
    Event f; f.id = 0; f.duration = 1e-3; f.stream = 0;
    one.events = {f};
    out("trace one " + render_trace(simulate_step(one)));
  }
  out("export bad path " + attempt([&] {
        EventGraph g;
        export_trace(simulate_step(g), "/nonexistent_dir/trace.json");
        return std::string("ok");
      }));
}

// ----------------------------------------------------------------- placement
void section_placement(const BandwidthProfile& p1) {
  out("## placement");
  for (int N = 1; N <= 8; ++N)
    for (int F = 1; F <= 4; ++F)
      for (int s1 = 1; s1 <= N + 1; ++s1) {
        Topology topo{(N + F - 1) / F, F, 1.5};
        auto c = cluster(8, N, 1ull << 40, {8, N});
        c.topology = topo;
        ShardingPlan p{{1, 1}, {1, 1}, {8, s1}, std::nullopt};
        out("assign N=" + std::to_string(N) + " F=" + std::to_string(F) + " s1=" +
            std::to_string(s1) + " " + attempt([&] {
              auto a = assign_nodes(topo, c, p);
              std::string s = "gs=" + std::to_string(a.group_size) + " cross=" +
                              std::to_string(a.cross_leaf_groups) + " groups";
              for (int g : a.group_of) s += " " + std::to_string(g);
              s += " leaves";
              for (int l : a.leaf_of) s += " " + std::to_string(l);
              for (auto mesh : {DeviceMesh{8, 1}, DeviceMesh{8, 2}, DeviceMesh{4, 1}}) {
                s += " t" + ms(mesh) + "=" + attempt([&] {
                  return hx(placed_collective_time(topo, a, p1, CollectiveKind::AllReduce,
                                                   1u << 24, mesh));
                });
              }
              return s;
            }));
      }
  out("cross interleaved " +
      std::to_string(count_cross_leaf_groups({0, 1, 0, 1}, 2, {0, 0, 1, 1})) +
      " contiguous " +
      std::to_string(count_cross_leaf_groups({0, 0, 1, 1}, 2, {0, 0, 1, 1})));
}

}  // namespace

int main(int argc, char** argv) {
  const std::string only = argc > 1 ? argv[1] : "";
  std::vector<DeviceMesh> meshes = all_meshes(8, 8);
  for (int a = 1; a <= 8; ++a)
    for (int b : {16, 32, 64, 128}) meshes.push_back({a, b});
  std::vector<BandwidthProfile> profiles;
  profiles.push_back(synthetic_profile({5e-6, 150e9}, {10e-6, 50e9}, meshes,
                                       geo(1024, 1ull << 34, 4)));
  profiles.push_back(synthetic_profile({2e-6, 300e9}, {20e-6, 25e9}, meshes,
                                       geo(4096, 1ull << 32, 2)));
  if (only.empty() || only == "comm") section_comm(profiles[0]);
  if (only.empty() || only == "domain") section_domain();
  if (only.empty() || only == "cost") section_cost(profiles);
  if (only.empty() || only == "planner") section_planner(profiles);
  if (only.empty() || only == "sim") section_sim(profiles);
  if (only.empty() || only == "placement") section_placement(profiles[0]);
  return 0;
}
