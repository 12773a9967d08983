for i in 1 2; do
 for g in operator none none operator; do echo -n "$g "; timeout -s KILL 300 python tools/step_time.py --granularity $g | grep STEP_MS; done
done
