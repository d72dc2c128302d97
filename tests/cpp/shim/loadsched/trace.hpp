// shim: the reference header trace.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
