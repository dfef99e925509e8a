#!/bin/bash
# Rebuild the git-ignored .cache/ (bases + oracle fixtures) from precompute/ and oracle/ only.
# usage: tools/rebuild_cache.sh [stage...]   stages: bases newton c5basis traj c5fix
cd "$(dirname "$0")/.."
export PYTHONUNBUFFERED=1
stages=${@:-bases newton c5basis traj c5fix}
for st in $stages; do
  case $st in
    bases)   for c in 1 2 3 4; do python -c "
import time; from precompute.mesh import make_scene; from precompute.basis import cached_basis
t=time.time(); s=make_scene($c); b=cached_basis(s); print('C$c basis', b.m, round(time.time()-t,1),'s', flush=True)"; done ;;
    newton)  for c in 1 2 3 4; do python tools/oracle_fixtures.py newton $c; done ;;
    c5basis) python -c "
import time; from precompute.mesh import make_scene; from precompute.basis import cached_basis
t=time.time(); s=make_scene(5); b=cached_basis(s, verbose=True); print('C5 basis', b.m, round(time.time()-t,1),'s', flush=True)" ;;
    traj)    python tools/oracle_fixtures.py traj 4 20; python tools/oracle_fixtures.py traj 3 30; python tools/oracle_fixtures.py traj 2 20 ;;
    c5fix)   python tools/oracle_fixtures.py newton 5; python tools/oracle_fixtures.py traj 5 1 ;;
  esac
done
echo ALL DONE
