# A/B of library builds (development): HEAD lib vs working tree, gap probe (no profile buffer)
python -m paper_2604_26039_b200._build > /dev/null
for r in 1 2; do
for L in scripts/_ab/lib_head.so paper_2604_26039_b200/libramp_b200.so; do
RAMP_B200_LIB=$L python scripts/gap_probe.py --points 1:0.2,8:0.5,16:1.0,128:0.2,512:0.2 | sed "s#^#$L #"
RAMP_B200_LIB=$L python scripts/gap_probe.py --fp8 --points 8:0.5,128:0.5 | sed "s#^#$L #"
done
done
