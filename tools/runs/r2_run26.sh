# mass / stiffness tables on every shape (P=2..8)
timeout 1200 python bench.py --sweep on --sweep-tables mass_deformed,stiff_deformed --steps 5 > gpurun_out/r2run26_sweep.json 2> gpurun_out/r2run26_sweep.err; echo "sweep rc=$?"
tail -c 300 gpurun_out/r2run26_sweep.err
