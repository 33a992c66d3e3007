// polegrad/prototxt.hpp — the model-definition boundary (reference
// prototxt.hpp:10-25): protobuf-text <-> NetDef.
//
// Recognised: top-level `name` and `layer`; per layer name, type, repeated
// bottom/top, inner_product_param.num_output, memory_data_param's four
// extents.  Everything else (convolution_param, weight_filler, include, ...)
// is preserved as opaque nodes.  `#` comments are dropped; a repeated
// recognised scalar keeps the last value and records a warning (stderr when
// `warnings` is null); malformed text throws ParseError(line).
#pragma once

#include <string>
#include <string_view>
#include <vector>

#include "polegrad/net.hpp"

namespace polegrad::prototxt {

NetDef parse(std::string_view text, std::vector<std::string>* warnings = nullptr);

// Canonical text: two-space indentation, one field per line, quoted strings.
// Idempotent: print(parse(print(parse(t)))) == print(parse(t)).
std::string print(const NetDef& def);

}  // namespace polegrad::prototxt
