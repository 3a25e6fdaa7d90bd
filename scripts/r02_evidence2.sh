O=gpurun_out/r02e; mkdir -p $O
timeout 1200 python scripts/ag_sweep.py --worlds 2,4,8 --max-log2 31 --steps 5 --out $O/ag_sweep.json > $O/ag_sweep.txt 2>&1
echo "sweep rc=$?" >> $O/ag_sweep.txt
for c in 64 296; do
  DC_AG_MAX_CTAS=$c timeout 900 ncu --set full --import-source on --clock-control none -k regex:ag_push -c 4 -o $O/ag_push_n8_ctas$c \
    python scripts/ag_sweep.py --ncu-push 8 --max-log2 30 > $O/ncu_ag_$c.txt 2>&1
  echo "ncu ag rc=$?" >> $O/ncu_ag_$c.txt
  DC_AG_MAX_CTAS=$c timeout 900 ncu --set full --import-source on --clock-control none -k regex:ag_push -c 4 -o $O/ag_push_n2_ctas$c \
    python scripts/ag_sweep.py --ncu-push 2 --max-log2 30 > $O/ncu_ag2_$c.txt 2>&1
done
