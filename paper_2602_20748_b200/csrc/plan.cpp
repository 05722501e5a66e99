// Source-batch plan and shard ownership (host logic, no GPU).
//
// The productive sources P (candidate indices, ascending) are cut into
// batches of B consecutive entries; batch b owns the candidate interval
// [jstart(b), jstart(b+1)) with jstart(0) = 0, jstart(b) = P[b*B] and
// jstart(nbatches) = nsrc, so the non-productive candidates between two
// batches (which only contribute their epsilon pair, reading R1) belong to
// the batch before them.  Batch b is evaluated by shard b % shard_count
// (round-robin, since source ranges are skewed).  With no
// productive source there is one virtual batch 0 (shard 0).
#include "internal.h"

void batch_plan(const uint32_t *bfirst, uint64_t nbatches, uint64_t nsrc, std::vector<uint64_t> &jstart) {
    const uint64_t nb_eff = nbatches ? nbatches : 1;
    jstart.assign(nb_eff + 1, 0);
    for (uint64_t b = 1; b < nb_eff; ++b) jstart[b] = bfirst[b];
    jstart[nb_eff] = nsrc;
}

extern "C" rpq_status rpq_shard_plan(const uint32_t *pidx, uint64_t np, uint64_t nsrc, uint64_t batch_sources,
                                     uint32_t shard_count, uint32_t *owner) {
    if ((np && !pidx) || (nsrc && !owner) || batch_sources == 0 || shard_count == 0)
        return rpq_fail(RPQ_EINVAL, "rpq_shard_plan: bad argument");
    for (uint64_t i = 1; i < np; ++i)
        if (pidx[i] <= pidx[i - 1] || pidx[i] >= nsrc) return rpq_fail(RPQ_EINVAL, "rpq_shard_plan: unsorted");
    const uint64_t nb = np ? (np + batch_sources - 1) / batch_sources : 0;
    std::vector<uint32_t> bfirst(nb);
    for (uint64_t b = 0; b < nb; ++b) bfirst[b] = pidx[b * batch_sources];
    std::vector<uint64_t> js;
    batch_plan(bfirst.data(), nb, nsrc, js);
    for (uint64_t b = 0; b + 1 < js.size(); ++b)
        for (uint64_t j = js[b]; j < js[b + 1]; ++j) owner[j] = (uint32_t)(b % shard_count);
    return RPQ_OK;
}
