// Drop-in forward for the reference module header specden/pool.hpp
// (proj/include/specden/pool.hpp): the whole API lives in specden_b200.hpp.
#pragma once
#include "specden/specden_b200.hpp"
