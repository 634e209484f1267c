"""CPU oracle for the Checkmate two-phase-rounding hot path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
(paper_1910_02653_b200).  Shares no code with the CUDA path."""
from .checkmate_oracle import (Instance, best_per_budget, evaluate, evaluate_S, free_matrix,  # noqa: F401
                               masks_u64, memory_U, round_S, two_phase_R)
from .randomized import (evaluate_randomized, philox4x32_10, round_S_randomized,  # noqa: F401
                         uniforms)
from .max_batch import B_CAP, b_max, max_batch_per_budget  # noqa: F401
from .plan_sim import generate_plan, hoisted_plan, simulate_plan, spurious_checkpoints  # noqa: F401
from .policies import (S_from_K, articulation_points, evaluate_policy, policy_K)  # noqa: F401
