// Drop-in for the reference's <mctune/search.hpp>: the same names in namespace
// mctune, served by the B200 engine (include/mctune_b200.hpp).
#pragma once
#include "mctune_b200.hpp"
namespace mctune = mctune_b200;
