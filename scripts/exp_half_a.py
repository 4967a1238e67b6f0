"""Experiment (timing only, wrong results): emulate halving K3's A-operand L2
feed -- what a cluster of two pairs sharing each A block by TMA multicast would
save -- by skipping the A load on every second tile of a unit. Patches a COPY
of csrc/lmhead.cu in place:

    cp -r . /tmp/exp && python scripts/exp_half_a.py /tmp/exp/paper_2601_06562_b200/csrc/lmhead.cu
"""
import sys

p = sys.argv[1]
s = open(p).read()
old = """            if (rank == 0) mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES * CG);
            if constexpr (CG == 1)
              tma_load_2d(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);
            else
              tma_load_2d_cg2(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);"""
new = """            const bool skip_a = ((t - t0) & 1) != 0;  // EXPERIMENT: A feed halved
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], (skip_a ? C::B_BYTES : C::STAGE_BYTES) * CG);
            if constexpr (CG == 1)
              tma_load_2d(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);
            else
              tma_load_2d_cg2(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);
            if (skip_a) {
              if (++stage == C::STAGES) {
                stage = 0;
                phase ^= 1;
              }
              continue;
            }"""
assert old in s, "pattern"
s = s.replace(old, new)
open(p, "w").write(s)
print("patched", p)
