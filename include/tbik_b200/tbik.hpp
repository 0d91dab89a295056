// tbik_b200/tbik.hpp -- everything of the B200 TBIK C++ API in one include:
// the drop-in reference headers (include/tbik/{errors,numerics,rng,matrix,
// matmul,collective,layers,demo}.hpp -- a caller of the reference keeps its
// `#include "tbik/layers.hpp"` and links libtbik_b200 instead), the C ABI
// (tbik_b200.h) and the one-process-per-GPU PeerGroup (peer_group.hpp).
#pragma once

#include "tbik/collective.hpp"
#include "tbik/demo.hpp"
#include "tbik/errors.hpp"
#include "tbik/layers.hpp"
#include "tbik/matmul.hpp"
#include "tbik/matrix.hpp"
#include "tbik/numerics.hpp"
#include "tbik/rng.hpp"
#include "tbik_b200.h"
#include "tbik_b200/peer_group.hpp"
