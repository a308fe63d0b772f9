// cabl/cabl.hpp — umbrella header of the B200 drop-in for the reference's
// hot path (reference proj/include/cabl/cabl.hpp).  The reference's
// analysis modules (io_bounds, cache_sim, the CPU bench) are out of scope for
// this build and not provided; the descriptor loader is
// (descriptor_json.hpp), for the GPU bench CLI's --machine documents.
#pragma once

#include "dense.hpp"
#include "descriptor_json.hpp"
#include "kernels.hpp"
#include "machine.hpp"
