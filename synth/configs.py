"""Workload shapes from BASELINE.json ``configs``.

Each config fixes T (horizon), B (env columns; multi-agent envs fold agents into columns,
column = env * agents + agent), the observation width, the tanh trunk widths and the
categorical head sizes.  ``ld_obs`` is the fp16 row stride of the observation matrix,
rounded up to a multiple of 8 elements so every row starts 16-byte aligned (TMA rule).
"""
from dataclasses import dataclass, field
from typing import Tuple


@dataclass(frozen=True)
class Config:
    name: str
    T: int
    B: int
    obs_dim: int
    hidden: Tuple[int, ...]
    heads: Tuple[int, ...]
    agents: int = 1            # agent columns per env (columns of one env are contiguous)
    frame_skip: int = 1        # frames per sample (Atari/DMLab 4-frameskip)
    gamma: float = 0.99
    lam: float = 0.95
    clip_eps: float = 0.2
    value_coef: float = 0.5
    entropy_coef: float = 0.01
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    recipe: str = "tiny"       # reward / done process, SURVEY.md §8(d) D-1
    separate_critic: bool = False   # NEXT-3: separate actor and critic trunks (reading R-AC)
    notes: str = field(default="", compare=False)

    @property
    def ld_obs(self) -> int:
        return (self.obs_dim + 7) // 8 * 8

    @property
    def n_actions(self) -> int:
        return sum(self.heads)

    @property
    def N(self) -> int:
        return self.T * self.B

    @property
    def dims(self) -> Tuple[int, ...]:
        return (self.obs_dim,) + tuple(self.hidden) + (self.n_actions + 1,)

    @property
    def layer_shapes(self):
        """(out, in) of every weight matrix in flat-layout order (C-A10; R-AC with
        separate_critic: actor trunk, policy head [A], critic trunk, value head [1])."""
        d = self.dims
        if not self.separate_critic:
            return [(d[i + 1], d[i]) for i in range(len(d) - 1)]
        trunk = [(d[i + 1], d[i]) for i in range(len(d) - 2)]
        return trunk + [(self.n_actions, d[-2])] + trunk + [(1, d[-2])]

    @property
    def head_layers(self):
        """indices into layer_shapes of the linear head layers"""
        L = len(self.hidden)
        return (L, 2 * L + 1) if self.separate_critic else (L,)

    @property
    def n_params(self) -> int:
        return sum(o * i + o for o, i in self.layer_shapes)

    def with_(self, **kw) -> "Config":
        from dataclasses import replace
        return replace(self, **kw)


CONFIGS = {
    # configs[0]: CartPole-shaped, oracle in seconds
    "tiny": Config("tiny", T=8, B=4, obs_dim=4, hidden=(64, 64), heads=(2,), recipe="tiny"),
    # configs[1]: Atari-shaped, the N=1 bench workload
    "atari": Config("atari", T=128, B=1024, obs_dim=512, hidden=(512, 512), heads=(18,),
                    frame_skip=4, recipe="atari"),
    # configs[2]
    "gfootball": Config("gfootball", T=200, B=4096, obs_dim=115, hidden=(256, 256, 256),
                        heads=(19,), recipe="gfootball"),
    # configs[3]: 2048 envs x 10 agents
    "smac": Config("smac", T=400, B=20480, obs_dim=300, hidden=(512, 512), heads=(16,),
                   agents=10, recipe="smac"),
    # configs[4]: 8192 envs x 4 agents, multi-head actions (SURVEY C-A8 reading)
    "hns": Config("hns", T=160, B=32768, obs_dim=512, hidden=(1024, 1024, 1024, 1024),
                  heads=(11, 11, 11, 2, 2), agents=4, recipe="hns"),
}


def get_config(name: str) -> Config:
    try:
        return CONFIGS[name]
    except KeyError:
        raise KeyError(f"unknown config {name!r}; known: {sorted(CONFIGS)}") from None
