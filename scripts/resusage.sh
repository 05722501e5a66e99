#!/bin/bash
# Registers / stack of the level kernels in a built library (development aid)
cuobjdump -res-usage "$1" 2>/dev/null | awk '/Function/ {name=$2} /REG:/ {print name, $1, $2}' | grep -E "k_level|k_seed_expand|k_sparse" | sed -E 's/_ZN[0-9]+_GLOBAL__N__[0-9a-f_]+eval_cu_[0-9a-f]+//'
