// Drop-in for the reference's <mctune/kernel.hpp>: the cost-and-effect programs
// the engine runs (build_abstract_kernel / build_minimum_kernel), in namespace mctune.
#pragma once
#include "mctune_b200.hpp"
namespace mctune = mctune_b200;
