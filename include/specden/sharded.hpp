// Drop-in forward for the reference module header specden/sharded.hpp
// (proj/include/specden/sharded.hpp): the whole API lives in specden_b200.hpp.
#pragma once
#include "specden/specden_b200.hpp"
