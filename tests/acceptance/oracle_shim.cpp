// See oracle_shim.hpp: the out-of-scope test oracle, unimplemented on purpose.
#include "oracle_shim.hpp"

#include <stdexcept>

namespace seqpipe {
Rational oracle_min_makespan(const ScenarioConfig&, const SequencePartition&) {
  throw std::logic_error("oracle_min_makespan is a test-only search outside this repository's scope");
}
}  // namespace seqpipe
