// SPDX-License-Identifier: Apache-2.0
// Compatibility include: the whole API is declared in seqbal/seqbal.hpp.
#pragma once
#include "seqbal/seqbal.hpp"
