// Shard layouts and process groups (see layout.h).
#include "layout.h"

#include <algorithm>
#include <string>

namespace amsp {

using shardplan::DeviceMesh;
using shardplan::Error;

PShardMap pshard_map(const std::vector<std::uint64_t>& tensor_sizes, int sp) {
  if (sp < 1) throw Error("layout: s_p must be >= 1");
  PShardMap m;
  std::uint64_t flat = 0;
  for (std::size_t t = 0; t < tensor_sizes.size(); ++t) {
    const std::uint64_t n = tensor_sizes[t];
    if (n == 0) throw Error("layout: tensor sizes must be positive");
    if (n % static_cast<std::uint64_t>(sp) != 0)
      throw Error("layout: tensor " + std::to_string(t) + " (" + std::to_string(n) +
                  " elements) is not divisible by s_p=" + std::to_string(sp));
    m.tensor_offset.push_back(flat);
    m.pshard_offset.push_back(m.pshard_elems);
    m.slice_len.push_back(n / sp);
    m.pshard_elems += n / sp;
    flat += n;
  }
  return m;
}

ShardLayout pshard_layout(const std::vector<std::uint64_t>& tensor_sizes, int sp,
                          int p_pos, int k, int os_pos, int kind) {
  if (k < 1 || os_pos < 0 || os_pos >= k)
    throw Error("layout: shard " + std::to_string(os_pos) + " out of range for " +
                std::to_string(k) + " shards");
  if (p_pos < 0 || p_pos >= sp) throw Error("layout: P position out of range");
  const PShardMap map = pshard_map(tensor_sizes, sp);
  ShardLayout out;
  auto append = [&out](std::uint64_t flat, std::uint64_t dst, std::uint64_t len) {
    if (len == 0) return;
    if (!out.segs.empty()) {
      Segment& last = out.segs.back();
      if (last.flat + last.len == flat && last.dst + last.len == dst) {
        last.len += len;
        out.owned += len;
        return;
      }
    }
    out.segs.push_back({flat, out.owned, dst, len});
    out.owned += len;
  };
  const std::size_t n = tensor_sizes.size();
  auto slice_flat = [&](std::size_t t) {
    return map.tensor_offset[t] + static_cast<std::uint64_t>(p_pos) * map.slice_len[t];
  };
  if (kind == kLayoutGreedy) {
    const shardplan::TensorPartition part =
        shardplan::partition_tensors_greedy(map.slice_len, k);
    for (std::size_t t = 0; t < n; ++t)
      if (part.assignment[t] == os_pos)
        append(slice_flat(t), map.pshard_offset[t], map.slice_len[t]);
  } else if (kind == kLayoutContiguous) {
    const std::uint64_t total = map.pshard_elems;
    auto cut = [&](int j) -> std::uint64_t {
      if (j >= k) return total;
      const unsigned __int128 x = static_cast<unsigned __int128>(total) *
                                  static_cast<unsigned>(j) / static_cast<unsigned>(k);
      return static_cast<std::uint64_t>(x) & ~std::uint64_t{7};
    };
    const std::uint64_t lo = cut(os_pos), hi = cut(os_pos + 1);
    for (std::size_t t = 0; t < n; ++t) {
      const std::uint64_t a = std::max(lo, map.pshard_offset[t]);
      const std::uint64_t b = std::min(hi, map.pshard_offset[t] + map.slice_len[t]);
      if (a < b) append(slice_flat(t) + (a - map.pshard_offset[t]), a, b - a);
    }
  } else {
    throw Error("layout: unknown layout kind " + std::to_string(kind));
  }
  return out;
}

ShardLayout shard_layout(const std::vector<std::uint64_t>& tensor_sizes, int shards,
                         int shard, int kind) {
  return pshard_layout(tensor_sizes, 1, 0, shards, shard, kind);
}

MeshGroup mesh_group(DeviceMesh dp, DeviceMesh mesh, int rank) {
  if (dp.per_node < 1 || dp.nodes < 1 || mesh.per_node < 1 || mesh.nodes < 1 ||
      dp.per_node % mesh.per_node || dp.nodes % mesh.nodes)
    throw Error("group: mesh " + shardplan::to_string(mesh) +
                " does not tile dp mesh " + shardplan::to_string(dp));
  if (rank < 0 || rank >= dp.size())
    throw Error("group: rank " + std::to_string(rank) + " outside dp mesh " +
                shardplan::to_string(dp));
  const int local = rank % dp.per_node, node = rank / dp.per_node;
  const int bl = local / mesh.per_node, bn = node / mesh.nodes;
  MeshGroup g;
  g.block = bn * (dp.per_node / mesh.per_node) + bl;
  g.position = (node % mesh.nodes) * mesh.per_node + (local % mesh.per_node);
  for (int pos = 0; pos < mesh.size(); ++pos) {
    const int n = bn * mesh.nodes + pos / mesh.per_node;
    const int l = bl * mesh.per_node + pos % mesh.per_node;
    g.members.push_back(n * dp.per_node + l);
  }
  return g;
}

}  // namespace amsp
