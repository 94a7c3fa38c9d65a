// Forwarding header: the B200 blockpipe API lives in one header.
#pragma once
#include "blockpipe/blockpipe_b200.hpp"
