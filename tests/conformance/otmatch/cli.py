from . import _out_of_scope

main = _out_of_scope("otmatch.cli.main")
