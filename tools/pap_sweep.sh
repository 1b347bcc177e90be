for ty in 4 8 16 32; do for bps in 4 8 16; do
SSCG_PAP_TY=$ty SSCG_PAP_BPS=$bps ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pap --csv --log-file gpurun_out/pap_$ty_$bps.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "ty $ty bps $bps $(grep gpu__time_duration gpurun_out/pap_$ty_$bps.csv | awk -F'","' '{print $NF}' | tr -d '"' | head -3 | tr '\n' ' ')"
done; done
