// polegrad/proto_node.hpp — one field of a protobuf-text document.
//
// Mirrors the reference ProtoNode (proto_node.hpp:8-26): a scalar (`key: v`)
// or a block (`key { ... }`), children in source order, scalar tokens kept
// verbatim (strings unescaped) so unknown fields round-trip unchanged.  Layer
// parameter blocks this library understands beyond the reference's
// (convolution_param, pooling_param, loss_param, ...) are read from these
// nodes at layer construction, so parse/print stays byte-identical.
#pragma once

#include <string>
#include <vector>

namespace polegrad {

struct ProtoNode {
  enum class Kind { kString, kNumber, kIdentifier, kBlock };

  std::string key;
  Kind kind = Kind::kIdentifier;
  std::string value;               // scalars only
  std::vector<ProtoNode> children; // blocks only
  int line = 0;                    // 1-based source line; 0 when synthesized

  // Structure only: the source line does not take part.
  bool operator==(const ProtoNode& o) const {
    return key == o.key && kind == o.kind && value == o.value && children == o.children;
  }
};

}  // namespace polegrad
