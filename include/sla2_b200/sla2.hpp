// sla2_b200/sla2.hpp -- the C++ drop-in for the reference's SLA2 forward hot path.
//
// Two modes, one call syntax (the reference's names, signatures, argument meaning, value
// semantics and exception classes):
//
//  * The reference headers are on the include path (`#include "sla2/attention.hpp"` resolves):
//    reference_dropin.hpp. It includes the reference's own sla2/common.hpp, matrix.hpp,
//    router.hpp, quant.hpp and attention.hpp and explicitly specializes smooth_k, block_scores,
//    hard_topk and sla2_forward_blockwise for float and double, so the reference's own callers
//    (Tape::sla2_attention, tape.hpp:263-286; model_forward, model.hpp:265-268) run on the B200.
//    Include this header BEFORE sla2/tape.hpp / sla2/model.hpp.
//
//  * They are not (e.g. on the GPU box, or a consumer that only has this repository):
//    standalone.hpp mirrors the reference's types and entry points (float) on the C ABI.
//
// Define SLA2_B200_STANDALONE to force the second mode. Both map to include/sla2_capi.h and
// link libsla2_b200.so (+ libcudart).
#pragma once

#if !defined(SLA2_B200_STANDALONE) && defined(__has_include)
#if __has_include("sla2/attention.hpp")
#include "reference_dropin.hpp"
#define SLA2_B200_MODE_REFERENCE 1
#endif
#endif

#ifndef SLA2_B200_MODE_REFERENCE
#include "standalone.hpp"
#endif
