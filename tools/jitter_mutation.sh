#!/bin/bash
# Does the schedule-jitter build catch a missing barrier?  Mutant: the per-level named barrier of
# k_eik2 removed (a real inter-warp race: thread 32 reads the node thread 31 wrote one level
# earlier).  The eikonal parity tests run on the normal and on the jitter build of the mutant.
set -u
OUT=gpurun_out/jmut; mkdir -p $OUT
cp paper_1008_3699_b200/csrc/eik2.cuh /tmp/eik2.orig
sed -i 's|        asm volatile("bar.sync 1, %0;" ::"r"(ek::LT) : "memory");   // the level threads only|        /* MUTANT: barrier removed */|' paper_1008_3699_b200/csrc/eik2.cuh
grep -c MUTANT paper_1008_3699_b200/csrc/eik2.cuh > $OUT/mutant_applied.txt
python -c "from paper_1008_3699_b200 import build; build.build(force=True)" > $OUT/build.log 2>&1
python -m pytest tests/test_gpu_eikonal.py -m gpu -q -p no:cacheprovider > $OUT/normal.log 2>&1; echo "normal build exit $?" >> $OUT/summary.txt
for seed in 1 7 12345; do
  SW_LIBRARY=libsweep_jitter.so SW_JITTER_SEED=$seed python -m pytest tests/test_gpu_eikonal.py -m gpu -q -p no:cacheprovider > $OUT/jitter_$seed.log 2>&1; echo "jitter seed $seed exit $?" >> $OUT/summary.txt
done
tail -1 $OUT/normal.log >> $OUT/summary.txt
for seed in 1 7 12345; do tail -1 $OUT/jitter_$seed.log >> $OUT/summary.txt; done
cp /tmp/eik2.orig paper_1008_3699_b200/csrc/eik2.cuh
cat $OUT/summary.txt
