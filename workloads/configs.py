"""The five workload configurations of BASELINE.json `configs` (shapes per SURVEY.md §8(d),
unstated fields per SURVEY.md §8(c) reading S20)."""
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Config:
    name: str
    hq: int           # query heads
    hkv: int          # kv heads
    d: int            # head dim
    page: int         # page size (tokens)
    n_queries: int    # concurrent queries (whole job)
    dag: str          # DAG family name in workloads.dags.DAGS
    lp: int           # shared prefix tokens per query
    t: int            # tokens per point (|S_k| = content + output) in the snapshot
    lc: int           # content tokens per point
    layers: int
    seed: int

    @property
    def g(self):
        return self.hq // self.hkv

    def with_(self, **kw):
        return replace(self, **kw)


CONFIGS = {
    # configs[0]: 1 query, diamond, prefix 128, 32 tok/point, 1 layer, 4q/2kv heads, d=64
    "c1": Config("c1", 4, 2, 64, 64, 1, "diamond", 128, 32, 8, 1, 1001),
    # configs[1]: Llama-3-8B attention shape, 1 query x mixed8, prefix 2K, 256 tok/point
    "c2": Config("c2", 32, 8, 128, 64, 1, "mixed8", 2048, 256, 32, 32, 1002),
    # configs[2]: Qwen2.5-7B attention shape, 16 queries x mixed8, prefix 4K, page 64
    "c3": Config("c3", 28, 4, 128, 64, 16, "mixed8", 4096, 256, 32, 28, 1003),
    # configs[3]: Llama-3-8B shape, 64 queries x mixed16, prefix 4K, 512 tok/point
    "c4": Config("c4", 32, 8, 128, 64, 64, "mixed16", 4096, 512, 32, 32, 1004),
    # configs[4]: stress, wide-64 vs chain-64, prefix 8K, 32 layers (64 queries = 8 per GPU at 8 GPUs)
    "c5w": Config("c5w", 32, 8, 128, 64, 64, "wide64", 8192, 256, 32, 32, 1005),
    "c5c": Config("c5c", 32, 8, 128, 64, 64, "chain64", 8192, 256, 32, 32, 1005),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]
