# collective / kernel evidence on one GPU: T_c sweep (virtual ranks), ncu of ag_push / rs_adam, sanitizer
O=gpurun_out/r02d; mkdir -p $O
timeout 1200 python scripts/ag_sweep.py --worlds 2,4,8 --max-log2 31 --steps 5 --out $O/ag_sweep.json > $O/ag_sweep.txt 2>&1
echo "sweep rc=$?" >> $O/ag_sweep.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ag_push -c 6 -o $O/ag_push_n8 \
  python scripts/ag_sweep.py --ncu-push 8 --max-log2 30 > $O/ncu_ag.txt 2>&1
echo "ncu ag rc=$?" >> $O/ncu_ag.txt
for b in 0 1; do
  RS_SERIAL=1 DC_RS_BULK=$b timeout 900 ncu --set full --import-source on --clock-control none -k regex:rs_adam -c 3 \
    -o $O/rs_adam_n8_bulk$b python scripts/rs_bench.py 8 > $O/ncu_rs8_$b.txt 2>&1
  echo "ncu rs8 bulk$b rc=$?" >> $O/ncu_rs8_$b.txt
done
RS_SERIAL=1 DC_RS_BULK=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:rs_adam -c 2 \
  -o $O/rs_adam_n1_bulk1 python scripts/rs_bench.py 1 > $O/ncu_rs1.txt 2>&1
echo "ncu rs1 rc=$?" >> $O/ncu_rs1.txt
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.txt 2>&1
echo "memcheck rc=$?" >> $O/memcheck_smoke.txt
timeout 1500 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $O/synccheck_smoke.txt 2>&1
echo "synccheck rc=$?" >> $O/synccheck_smoke.txt
