// loadflow/time.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/time.hpp).
#pragma once
#include "loadflow/api.hpp"
