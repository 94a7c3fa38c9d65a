// Forwarding header: the operator surface lives in operator.hpp.
#pragma once
#include "blockpipe/operator.hpp"
