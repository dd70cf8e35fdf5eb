// TEST INFRASTRUCTURE ONLY: forwards to the oracle Boost.Geometry stand-in.
#pragma once
#include <boost/geometry.hpp>
