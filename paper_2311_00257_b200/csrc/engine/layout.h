// Shard layouts and process groups of the AMSP data plane (host only).
#pragma once

#include <cstdint>
#include <vector>

#include "amsp/plan.hpp"

namespace amsp {

// A contiguous run of flat parameter elements [flat, flat+len) stored at
// [os, os+len) of a rank's fp32 optimizer-state shard.
struct Segment {
  std::uint64_t flat = 0, os = 0, len = 0;
};

struct ShardLayout {
  std::vector<Segment> segs;  // ascending flat order
  std::uint64_t owned = 0;    // elements in the shard
};

enum LayoutKind { kLayoutGreedy = 0, kLayoutContiguous = 1 };

// Shard `shard` of `shards` over the concatenated tensors.
//  greedy:     the reference's inter-tensor LPT map
//              (shardplan::partition_tensors_greedy, cost_model.cpp:189-219);
//              a shard owns whole tensors; adjacent owned tensors merge.
//  contiguous: [floor8(j*Phi/k), floor8((j+1)*Phi/k)), last shard to Phi.
ShardLayout shard_layout(const std::vector<std::uint64_t>& tensor_sizes,
                         int shards, int shard, int kind);

// The block of ranks forming `mesh`'s group around `rank` in the DP mesh
// (ranks node-major: rank = node * dp.per_node + local). Position is
// (node % mesh.nodes) * mesh.per_node + (local % mesh.per_node).
struct MeshGroup {
  int block = 0;
  int position = 0;
  std::vector<int> members;  // by position
};

MeshGroup mesh_group(shardplan::DeviceMesh dp, shardplan::DeviceMesh mesh, int rank);

}  // namespace amsp
