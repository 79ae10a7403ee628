// Drop-in for the reference's <mctune/report.hpp>: the same names in namespace
// mctune, served by include/mctune_b200_report.hpp over the B200 engine.
#pragma once
#include "mctune_b200_report.hpp"
namespace mctune = mctune_b200;
