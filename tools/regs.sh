#!/bin/bash
# registers / shared memory per kernel of libmpcore.so (filter by pattern)
cuobjdump --dump-resource-usage ${2:-paper_2107_12550_b200/libmpcore.so} 2>&1 | awk '/Function/ {f=$2} /REG:/ {print f, $0}' | grep -E "${1:-.}" | sed -E 's/_ZN3mpk[0-9]+_GLOBAL__N__[0-9a-f]+_[0-9]+_[a-z]+_cu_[0-9a-f]+//; s/Resource usage://; s/TEXTURE:0 SURFACE:0 SAMPLER:0//'
