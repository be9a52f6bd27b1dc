"""The BASELINE.json workload shapes as concrete synthetic configurations.

Shapes follow SURVEY.md §8.d.1 (node counts and stored-entry counts of the
paper's dataset table, and BASELINE.json `configs`).
Feature dims are padded to a multiple of 4 floats (16-byte rows); output classes
are padded to C_pad (zero weight columns, masked out of the softmax).
"""
from dataclasses import dataclass, field, replace


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


@dataclass(frozen=True)
class GraphConfig:
    name: str
    num_nodes: int
    nnz: int                 # stored entries of the symmetric adjacency (both directions)
    d0: int                  # raw feature width
    hidden: tuple            # hidden widths d_1..d_{L-1}
    num_classes: int         # C
    c_pad: int               # C padded (output width d_L)
    parts: tuple             # partition counts M the config is run at
    sync_interval: int       # N_sync (the paper's N, north_star's I)
    train_frac: float
    seed: int
    mu: float = 0.05         # cross-block edge fraction of the planted generator
    sigma: float = 1.0       # log-normal degree spread
    blocks: int = 8          # planted blocks K

    @property
    def d0_pad(self) -> int:
        return round_up(self.d0, 4)

    @property
    def num_layers(self) -> int:
        return len(self.hidden) + 1

    @property
    def dims(self) -> tuple:
        """Layer widths d_0..d_L as the kernels see them (padded)."""
        return (self.d0_pad, *self.hidden, self.c_pad)

    @property
    def raw_dims(self) -> tuple:
        return (self.d0, *self.hidden, self.num_classes)


CONFIGS = {
    # Cora is not in the paper; BASELINE.json configs[0] ("CPU oracle in seconds").
    "cora": GraphConfig("cora", 2708, 10556, 1433, (16,), 7, 8, (2,), 1,
                        140 / 2708, 101),
    "flickr": GraphConfig("flickr", 89250, 899756, 500, (256,), 7, 8, (2, 4), 10,
                          0.50, 102),
    "arxiv": GraphConfig("arxiv", 169343, 2315598, 128, (256, 256), 40, 48, (4, 8), 10,
                         0.537, 103),
    "reddit": GraphConfig("reddit", 232965, 114615892, 602, (256,), 41, 48, (1, 2, 4, 8), 10,
                          0.66, 104),
    # mu calibrated so the halo/local ratio at M=8 is ~0.58 (58.43%).
    "products": GraphConfig("products", 2449029, 123718280, 100, (256, 256), 47, 48,
                            (1, 2, 4, 8), 10, 0.08, 105, mu=0.0129),
}


def get_config(name: str) -> GraphConfig:
    return CONFIGS[name]


def small_config(name="tiny", num_nodes=48, nnz=200, d0=6, hidden=(5,), num_classes=3,
                 c_pad=8, seed=7, **kw) -> GraphConfig:
    """A small graph for oracle pins and quick GPU parity cases."""
    base = dict(name=name, num_nodes=num_nodes, nnz=nnz, d0=d0, hidden=tuple(hidden),
                num_classes=num_classes, c_pad=c_pad, parts=(2,), sync_interval=1,
                train_frac=0.5, seed=seed)
    base.update(kw)
    return GraphConfig(**base)


def scaled(cfg: GraphConfig, factor: float, name=None) -> GraphConfig:
    """Same shape family with node and edge counts scaled down (parity sizes)."""
    n = max(16, int(cfg.num_nodes * factor))
    nnz = max(32, int(cfg.nnz * factor)) // 2 * 2
    nnz = min(nnz, n * (n - 1) // 2)
    return replace(cfg, name=name or f"{cfg.name}x{factor:g}", num_nodes=n, nnz=nnz)
