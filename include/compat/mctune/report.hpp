// Drop-in for the reference's <mctune/report.hpp> as far as the tuning path
// reaches: trace_to_text (report.hpp:33-38) from include/mctune_b200.hpp.  The
// file-format helpers (config/input readers, CSV/JSON writers) are host I/O off
// the data-parallel path and stay with the reference.
#pragma once
#include "mctune_b200.hpp"
namespace mctune = mctune_b200;
