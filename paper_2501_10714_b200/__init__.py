"""B200-native FSMoE MoE-layer hot path (gate -> order -> expert FFN -> I-order,
forward and backward, expert-parallel over NCCL) behind the reference's C++
operator API. Native code lives in lib/ (built by __graft_entry__.build())."""

__all__ = ["ops"]
