// crpq_eval: placeholder until the CRPQ join lands.
#include "internal.h"

extern "C" rpq_status crpq_eval(const rpq_graph *g, const crpq_query *q, const rpq_eval_opts *opts,
                                rpq_result **out) {
    (void)g; (void)q; (void)opts;
    if (out) *out = nullptr;
    return rpq_fail(RPQ_EUNSUPPORTED, "crpq_eval: not built yet");
}
