// shim: the reference header epoch_order.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
