// rankweave/simulate.hpp -- forwards to the consolidated drop-in API header.
#pragma once
#include "rankweave/rankweave.hpp"
