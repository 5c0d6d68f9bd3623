// Shard layouts and process groups of the AMSP data plane (host only).
#pragma once

#include <cstdint>
#include <vector>

#include "amsp/plan.hpp"

namespace amsp {

// A contiguous run of elements of one rank's optimizer-state shard:
// flat parameter elements [flat, flat+len) (the index space of gradients and
// of the synthetic data), stored at [os, os+len) of the rank's fp32 shard,
// whose updated bf16 values go to [dst, dst+len) of the parameter buffer
// (the full parameter vector when s_p = 1, the P shard when s_p > 1).
struct Segment {
  std::uint64_t flat = 0, os = 0, dst = 0, len = 0;
};

struct ShardLayout {
  std::vector<Segment> segs;  // ascending os order
  std::uint64_t owned = 0;    // elements in the shard
};

enum LayoutKind { kLayoutGreedy = 0, kLayoutContiguous = 1 };

// Optimizer-state shard `shard` of `shards` when parameters are NOT
// sharded (s_p = 1): the flat vector is split over the OS group.
//  greedy:     the reference's inter-tensor LPT map
//              (shardplan::partition_tensors_greedy, cost_model.cpp:189-219);
//              a shard owns whole tensors; adjacent owned tensors merge.
//  contiguous: [floor8(j*Phi/k), floor8((j+1)*Phi/k)), last shard to Phi.
ShardLayout shard_layout(const std::vector<std::uint64_t>& tensor_sizes,
                         int shards, int shard, int kind);

// Parameter sharding (s_p > 1, ZeRO-3 style intra-tensor split): P-group
// position `p_pos` holds slice p_pos of every tensor (each tensor must be a
// multiple of s_p elements). Its P shard is those slices concatenated in
// tensor order. The P shard's slices are then split over the k = s_os/s_p
// ranks sharing that P position inside the OS group (greedy over slice
// sizes, or contiguous over the P shard). dst offsets are P-shard offsets.
ShardLayout pshard_layout(const std::vector<std::uint64_t>& tensor_sizes, int sp,
                          int p_pos, int k, int os_pos, int kind);

// Per-tensor view of a P shard: tensor t's slice p_pos lives at
// pshard_offset[t] and has slice_len[t] elements.
struct PShardMap {
  std::vector<std::uint64_t> tensor_offset;  // flat start of each tensor
  std::vector<std::uint64_t> pshard_offset;
  std::vector<std::uint64_t> slice_len;
  std::uint64_t pshard_elems = 0;
};
PShardMap pshard_map(const std::vector<std::uint64_t>& tensor_sizes, int sp);

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
