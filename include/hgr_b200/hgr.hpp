// hgr_b200/hgr.hpp -- single-include form of the C++ drop-in (include/hgr_b200/hgr/).
// `#include <hgr_b200/hgr.hpp>` with -I include, or put include/hgr_b200 on the
// include path and keep the reference's own `#include "hgr/hgr.hpp"` lines.
#pragma once

#include "hgr/hgr.hpp"
