// hgr_b200/hgr/hgr.hpp -- drop-in for the reference's umbrella header
// (hgr.hpp:7-15): the public API of hgr on the B200 library. The analytical
// launch cost model (perf_model.hpp) is outside the GPU path; the CLI
// (hgr-b200 rank-configs) carries its restatement.
#pragma once

#include "correction.hpp"
#include "error.hpp"
#include "grid_hierarchy.hpp"
#include "ndarray.hpp"
#include "parallel.hpp"
#include "refactor.hpp"
#include "storage.hpp"
#include "transforms.hpp"
