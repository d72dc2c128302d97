// shim: the reference header cost_model.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
