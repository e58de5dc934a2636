"""B200-native BatMap all-pairs support counting (Amossen & Pagh, arXiv 1102.1003).

The product is the C-ABI library ``libbatmap.so`` (include/batmap.h); this package is
its thin binding (``batmap``), the multi-GPU gather (``dist``) and the build script.
"""
from .batmap import (  # noqa: F401
    BatMapError,
    Collection,
    Collection3,
    candidate_triples,
    dense_pair_supports,
    load_library,
    FimiDB,
    frequent_items,
    merge_pair_supports,
    mine_fimi,
    parse_fimi,
    mine_host,
    mine_triples,
    plan_groups,
    plan_tile,
    plan_work,
    select_csr,
    sort_triples,
    swar_device,
    version,
)
