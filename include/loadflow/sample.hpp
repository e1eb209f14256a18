// loadflow/sample.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/sample.hpp).
#pragma once
#include "loadflow/api.hpp"
