# SASS evidence of the headline sweep kernel (sweep_ws_kernel<5,4,64>) from the built library:
# mnemonic counts (TMA tensor loads, bulk copies, mbarrier ops, FP64) and the TMA issue excerpt.
K='_ZN6strait15sweep_ws_kernelILi5ELi4ELi64EEEv15StraitSweepArgs15StraitRefitArgsiiii14CUtensorMap_stS3_i'
cuobjdump -sass -fun "$K" paper_2604_28175_b200/_strait.so > /tmp/sweep.sass
echo "# cuobjdump -sass -fun $K paper_2604_28175_b200/_strait.so"
echo "# $(grep -c '/\*[0-9a-f]*\*/' /tmp/sweep.sass) SASS instructions; sha256 of the SASS: $(sha256sum /tmp/sweep.sass | cut -c1-16)"
echo "## mnemonic counts"
grep -o "UTMALDG[.A-Z0-9]*\|UBLKCP[.A-Z0-9]*\|SYNCS[.A-Z0-9_]*\|DFMA\|DMUL\|DADD\|MUFU.RCP64H\|LDGSTS\|BAR.SYNC[.A-Z]*\|BAR.ARV\|SHFL.BFLY\|STL\|LDL\|HMMA\|UTC[A-Z]*MMA" /tmp/sweep.sass | sort | uniq -c | sort -rn
echo "## TMA tensor-copy issue (producer warp)"
grep -n -B3 -A3 "UTMALDG" /tmp/sweep.sass | head -40
echo "## mbarrier wait (consumers)"
grep -n -B2 -A2 "SYNCS.PHASECHK.TRANS64.TRYWAIT" /tmp/sweep.sass | head -20
