// loadflow/runtime.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/runtime.hpp).
#pragma once
#include "loadflow/api.hpp"
