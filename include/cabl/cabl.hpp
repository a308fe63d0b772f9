// cabl/cabl.hpp — umbrella header of the B200 drop-in for the reference's
// hot path (reference proj/include/cabl/cabl.hpp).  The reference's
// analysis/bench modules (io_bounds, cache_sim, bench, descriptor_json) are
// out of scope for this build and not provided.
#pragma once

#include "dense.hpp"
#include "kernels.hpp"
#include "machine.hpp"
