// Drop-in forwarder: the reference header name, resolved to the B200 API.
#pragma once
#include "../dfakit_b200.hpp"
