// Drop-in for the reference's <mctune/machine.hpp>: Machine, MachineState,
// Transition and run over the B200 engine, in namespace mctune.
#pragma once
#include "mctune_b200.hpp"
namespace mctune = mctune_b200;
