# A/B of library builds under ab/ on the persistent lockstep rollout (diagnostic)
for v in ab/*.so; do echo "$v"; GFNX_LIB=$PWD/$v python profiles/persist_phases.py ${1:-ising_tb_b32768} 2>&1 | tail -4; done
