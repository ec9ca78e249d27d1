"""B200-native SO / l0 descriptor search (drop-in for descsearch.search).

    from paper_2502_20072_b200 import l0_search, L0Config
    models = l0_search(values, y, task_slices, L0Config(dimension=3))

or, inside an existing descsearch pipeline::

    import paper_2502_20072_b200 as l0
    l0.install()          # descsearch.pipeline.l0_search now runs on the GPU
"""

from .search import (  # noqa: F401
    CapacityError,
    DescsearchError,
    L0Config,
    Model,
    RankDeficient,
    RankOutOfRange,
    SearchStats,
    count_models,
    fit_tuple,
    fit_tuples,
    install,
    l0_search,
    rank_tuple,
    residuals,
    unrank_tuple,
)

__version__ = "0.1.0"
