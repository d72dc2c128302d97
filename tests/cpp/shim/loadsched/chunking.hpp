// shim: the reference header chunking.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
