from paper_2111_05366_b200 import cli as _cli

from . import _out_of_scope


def main(argv=None):
    if argv and argv[0] == "qaplib":
        _out_of_scope("otmatch.cli qaplib")()
    return _cli.main(argv)
