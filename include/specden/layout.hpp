// Drop-in forward for the reference module header specden/layout.hpp
// (proj/include/specden/layout.hpp): the whole API lives in specden_b200.hpp.
#pragma once
#include "specden/specden_b200.hpp"
