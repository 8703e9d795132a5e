// Stage graph: nodes are stage engines, edges are transfer functions
// (reference graph.hpp:15-242; SPEC.md core_model).
#pragma once
#include <string>
#include <vector>

#include "omni/context.hpp"
#include "omni/errors.hpp"

namespace omni {

enum class StageKind { AR, DIFFUSION };
enum class EdgeMode { FULL, STREAMING };
// INPROC/SHM/TCP as in the reference; DEVICE is the B200 transport (payload
// blobs stay in HBM, only locators cross the control plane).
enum class TransportKind { INPROC, SHM, TCP, DEVICE };

struct StageNode {
  StageId id;
  StageKind kind = StageKind::AR;
  std::string engine_config_ref;
  std::string preprocess_ref;
  std::string forward_ref;
};

struct TransferEdge {
  StageId from;
  StageId to;
  std::string transfer_ref;
  EdgeMode mode = EdgeMode::FULL;
  TransportKind transport = TransportKind::INPROC;
  uint32_t streaming_chunk_size = 0;
  std::string key() const { return from + "->" + to; }
};

struct StageGraph {
  std::vector<StageNode> nodes;
  std::vector<TransferEdge> edges;
  StageId entry;
  std::vector<StageId> exits;

  const StageNode* find_node(const StageId& id) const;
  std::vector<const TransferEdge*> edges_from(const StageId& id) const;
  std::vector<const TransferEdge*> edges_to(const StageId& id) const;
};

struct Violation {
  enum class Kind {
    CycleDetected,
    Unreachable,
    DanglingRef,
    BadEntry,
    BadExit,
    DuplicateEdge,
    DuplicateNode,
    BadEdgeEndpoint,
    SelfEdge,
    BadChunkSize,
    PreprocessOnDiffusion,
  };
  Kind kind;
  std::string subject;
  bool operator==(const Violation&) const = default;
  bool operator<(const Violation& o) const {
    return kind != o.kind ? kind < o.kind : subject < o.subject;
  }
};

const char* violation_kind_name(Violation::Kind k);
std::string violation_to_string(const Violation& v);

struct FunctionResolver {
  virtual ~FunctionResolver() = default;
  virtual bool has_forward(const std::string& name) const = 0;
  virtual bool has_preprocess(const std::string& name) const = 0;
  virtual bool has_transfer(const std::string& name) const = 0;
};

struct AcceptAllResolver final : FunctionResolver {
  bool has_forward(const std::string&) const override { return true; }
  bool has_preprocess(const std::string&) const override { return true; }
  bool has_transfer(const std::string&) const override { return true; }
};

// Every violation, sorted by (kind, subject); empty = valid.
std::vector<Violation> validate_graph(const StageGraph& g,
                                      const FunctionResolver& r = AcceptAllResolver{});
// Kahn's algorithm, lexicographically smallest ready node first.
std::vector<StageId> topo_order(const StageGraph& g);

}  // namespace omni
