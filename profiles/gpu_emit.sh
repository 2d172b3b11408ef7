for m in 0 1; do echo "mode $m"; GFNX_EMIT_MODE=$m python profiles/rollout_phases.py | tr -d '\n '; echo; done
