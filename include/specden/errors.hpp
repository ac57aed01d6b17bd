// Drop-in forward for the reference module header specden/errors.hpp
// (proj/include/specden/errors.hpp): the whole API lives in specden_b200.hpp.
#pragma once
#include "specden/specden_b200.hpp"
