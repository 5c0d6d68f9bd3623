// Shard layouts and process groups (see layout.h).
#include "layout.h"

#include <string>

namespace amsp {

using shardplan::DeviceMesh;
using shardplan::Error;

ShardLayout shard_layout(const std::vector<std::uint64_t>& tensor_sizes,
                         int shards, int shard, int kind) {
  if (shards < 1 || shard < 0 || shard >= shards)
    throw Error("layout: shard " + std::to_string(shard) + " out of range for " +
                std::to_string(shards) + " shards");
  std::uint64_t phi = 0;
  for (auto s : tensor_sizes) phi += s;
  ShardLayout out;
  auto append = [&out](std::uint64_t flat, std::uint64_t len) {
    if (len == 0) return;
    if (!out.segs.empty()) {
      Segment& last = out.segs.back();
      if (last.flat + last.len == flat) {
        last.len += len;
        out.owned += len;
        return;
      }
    }
    out.segs.push_back({flat, out.owned, len});
    out.owned += len;
  };
  if (kind == kLayoutGreedy) {
    const shardplan::TensorPartition part =
        shardplan::partition_tensors_greedy(tensor_sizes, shards);
    std::uint64_t flat = 0;
    for (std::size_t t = 0; t < tensor_sizes.size(); ++t) {
      if (part.assignment[t] == shard) append(flat, tensor_sizes[t]);
      flat += tensor_sizes[t];
    }
  } else if (kind == kLayoutContiguous) {
    auto cut = [&](int j) -> std::uint64_t {
      if (j >= shards) return phi;
      const unsigned __int128 x =
          static_cast<unsigned __int128>(phi) * static_cast<unsigned>(j) /
          static_cast<unsigned>(shards);
      return static_cast<std::uint64_t>(x) & ~std::uint64_t{7};
    };
    append(cut(shard), cut(shard + 1) - cut(shard));
  } else {
    throw Error("layout: unknown layout kind " + std::to_string(kind));
  }
  return out;
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
