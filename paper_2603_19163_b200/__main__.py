"""Entry point of `python -m paper_2603_19163_b200 <command>` (see cli.py)."""

if __name__ == "__main__":
    from .cli import main as _cli_main

    raise SystemExit(_cli_main())
