// loadflow/batcher.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/batcher.hpp).
#pragma once
#include "loadflow/api.hpp"
