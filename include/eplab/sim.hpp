// eplab/sim.hpp -- the reference header's name (/root/reference/proj/src/eplab/sim.hpp:16-85) for the task-list
// part of it (Role, role_name, TaskQueueInfo, build_task_list); the discrete-event simulator it also declares
// is replaced by the MegaKernels themselves. Every declaration lives in eplab.hpp.
#pragma once
#include "eplab/eplab.hpp"
