"""CPU oracle for the SortedRL rollout hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct reference implementations written from
PAPER.md (arXiv 2603.23414) and the readings recorded in DESIGN.md.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything from here.  The product path
(`paper_2603_23414_b200`, `libsrl.so`) never imports, links or executes this
package, and this package never imports the product path: the two share only
the seeded input generators in `workload/`.

Modules
  philox   Philox4x32-10 counter-based RNG (Salmon et al. 2011), SURVEY §8(c) O-S
  logf     FreeBSD-msun e_logf.c transcribed op by op in fp32 (IEEE RN, no FMA)
  sampler  Gumbel-max sampling + chosen-token log-probability ("exact log
           probability value that was used to generate each token")
  model    naive fp64 LLaMA/Qwen-style decode with a per-trajectory KV list
  attention  brute-force softmax attention over a paged KV cache
  sched    the SortedRL controller / rollout buffer state machine
  metrics  bubble ratio Eq. (bubble), throughput, staleness, curriculum
  learner  the update group's consumer: Eq. (1) clipped objective, Eq. (2) GAE,
           Eq. (3) Reinforce++ advantages, token staleness
"""
