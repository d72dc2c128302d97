// shim: the reference header reuse_graph.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
